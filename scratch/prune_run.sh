timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -3
for sm in 1 0; do for dt in f32 bf16; do
BSRP_PRUNE_SMALL=$sm timeout 300 python bench.py --no-cpu-baseline --steps 500 --e2e-steps 5 --dtype $dt > gpurun_out/bp_${dt}_$sm.json 2>gpurun_out/bp_${dt}_$sm.err; python -c "
import json
d=json.loads(open('gpurun_out/bp_${dt}_$sm.json').read().strip().splitlines()[-1])
print('small=$sm $dt', round(d['value']), 'us/step', round(d['ms_per_step']*1e3,1), {k:(round(v['ms']*1e3,1), round(v.get('GB/s',0))) for k,v in d['kernels'].items()})
" || tail -3 gpurun_out/bp_${dt}_$sm.err; done; done
