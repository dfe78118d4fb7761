# PDL flag sweep on the C2 step (BSRP_PDL bit mask, launch.h)
for dt in f32 bf16; do for pdl in 0 123 112 113 116 117 120 48 80 96; do
BSRP_PDL=$pdl timeout 300 python bench.py --no-cpu-baseline --steps 1000 --dtype $dt --e2e-steps 3 > gpurun_out/pdl_${dt}_$pdl.json 2>gpurun_out/pdl_${dt}_$pdl.err
python -c "
import json
d=json.loads(open('gpurun_out/pdl_${dt}_$pdl.json').read().strip().splitlines()[-1])
print('$dt pdl=$pdl', round(d['value']), 'us/step', round(d['ms_per_step']*1e3,2), {k:(round(v['ms']*1e3,1), round(v.get('GB/s',0))) for k,v in d['kernels'].items()}, d['clocks']['sm_mhz'])
" || tail -5 gpurun_out/pdl_${dt}_$pdl.err
done; done
