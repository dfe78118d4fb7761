set -x
timeout 1500 python -m pytest tests -q -m gpu 2>&1 | tail -3 > gpurun_out/gpu_tests.txt; cat gpurun_out/gpu_tests.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.txt 2>&1; tail -2 gpurun_out/smoke.txt
python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; tail -1 gpurun_out/bench_default.json | head -c 300; echo
python bench.py --dtype bf16 --no-cpu-baseline > gpurun_out/bench_bf16.json 2>/dev/null
python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/bench_reference.json 2>/dev/null
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 2 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:prune_kernel -s 3 -c 1 -o gpurun_out/prof_prune_kernel python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ncu_prune.log 2>&1; tail -1 gpurun_out/ncu_prune.log
ls gpurun_out
