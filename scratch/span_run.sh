# span kernel: parity, then C2 bench lines for span (CG=2, CG=1) vs runs
timeout 600 python -m pytest tests/test_wgrad_tc_parity.py -q -x 2>&1 | tail -2
for dt in f32 bf16; do for v in span2 span1 runs; do
case $v in span2) E="BSRP_WGRAD=span BSRP_WGRAD_CG=2";; span1) E="BSRP_WGRAD=span BSRP_WGRAD_CG=1";; runs) E="BSRP_WGRAD=runs";; esac
env $E timeout 300 python bench.py --no-cpu-baseline --steps 500 --e2e-steps 5 --dtype $dt > gpurun_out/b_${dt}_$v.json 2>gpurun_out/b_${dt}_$v.err; python -c "
import json
d=json.loads(open('gpurun_out/b_${dt}_$v.json').read().strip().splitlines()[-1])
print('$dt $v', round(d['value']), 'us/step', round(d['ms_per_step']*1e3,1), {k:(round(v['ms']*1e3,1), round(v.get('GB/s',0)), round(v.get('TFLOP/s',0))) for k,v in d['kernels'].items()})
" || tail -3 gpurun_out/b_${dt}_$v.err; done; done
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_span.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 2 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:wgrad_span -s 3 -c 1 -o gpurun_out/prof_wgrad_span python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ncu_span.log 2>&1; tail -1 gpurun_out/ncu_span.log
