#!/bin/bash
# build scratch/trace_prune (prune.cu with PRUNE_TRACE) and run it on the GPU box for the given K/b pairs
set -e
cd /root/repo/scratch && nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I ../include -o trace_prune trace_prune.cu
timeout 900 /usr/local/graft/bin/gpurun --timeout 300 -- "cd scratch; for kb in $*; do ./trace_prune \${kb%/*} \${kb#*/}; done" 2>&1 | grep -v "^\[gpurun\] send" | grep "rep 3\|max over\|keys"
