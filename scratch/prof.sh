# usage: prof.sh <kernel regex> <outname> [bench args...]
K=$1; O=$2; shift 2
ncu --set full --clock-control none --import-source on -k regex:$K -s 8 -c 1 -o gpurun_out/$O python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 "$@" > gpurun_out/$O.log 2>&1; tail -2 gpurun_out/$O.log
