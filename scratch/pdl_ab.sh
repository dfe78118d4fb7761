# PDL A/B: parity of the touched kernels, then C2 bench with and without PDL
timeout 900 python -m pytest tests/test_wgrad_tc_parity.py tests/test_prune_parity.py tests/test_fusion_gpu.py -q -x -m gpu 2>&1 | tail -3
for dt in f32 bf16; do for pdl in 1 0; do
BSRP_PDL=$pdl timeout 300 python bench.py --no-cpu-baseline --steps 1000 --dtype $dt --e2e-steps 5 > gpurun_out/pdl_${dt}_$pdl.json 2>gpurun_out/pdl_${dt}_$pdl.err
python -c "
import json
d=json.loads(open('gpurun_out/pdl_${dt}_$pdl.json').read().strip().splitlines()[-1])
print('$dt pdl=$pdl', round(d['value']), 'us/step', round(d['ms_per_step']*1e3,2), {k:(round(v['ms']*1e3,1), round(v.get('GB/s',0))) for k,v in d['kernels'].items()}, d['clocks']['sm_mhz'])
" || tail -5 gpurun_out/pdl_${dt}_$pdl.err
done; done
