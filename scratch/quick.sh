# quick: TC parity + bench lines
timeout 600 python -m pytest tests/test_wgrad_tc_parity.py tests/test_wgrad_parity.py tests/test_bench.py -q -x 2>&1 | tail -2
for dt in f32 bf16; do python bench.py --no-cpu-baseline --steps 500 --dtype $dt > gpurun_out/b_$dt.json 2>gpurun_out/b_$dt.err; python -c "
import json
d=json.loads(open('gpurun_out/b_$dt.json').read().strip().splitlines()[-1])
print('$dt', round(d['value']), 'us/step', round(d['ms_per_step']*1e3,1), {k:(round(v['ms']*1e3,1), round(v.get('GB/s',0))) for k,v in d['kernels'].items()}, d['clocks']['sm_mhz'], d['gpu_launches_per_step'])
"; done
