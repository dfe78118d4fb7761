set -x
python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; tail -3 gpurun_out/bench_default.err
cat gpurun_out/bench_default.json
python bench.py --dtype bf16 --no-cpu-baseline > gpurun_out/bench_bf16.json 2>&1; cat gpurun_out/bench_bf16.json | tail -2
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 2 > /dev/null 2>&1
wc -l gpurun_out/launches.csv
ncu --set full --clock-control none --import-source on -k regex:wgrad_tc -s 6 -c 1 -o gpurun_out/prof_wgrad python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ncu_wgrad.log 2>&1; tail -3 gpurun_out/ncu_wgrad.log
ncu --set full --clock-control none --import-source on -k regex:prune_kernel -s 6 -c 1 -o gpurun_out/prof_prune python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ncu_prune.log 2>&1; tail -3 gpurun_out/ncu_prune.log
ncu --set full --clock-control none --import-source on -k regex:decompress -s 6 -c 1 -o gpurun_out/prof_dec python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ncu_dec.log 2>&1; tail -3 gpurun_out/ncu_dec.log
ls -la gpurun_out
