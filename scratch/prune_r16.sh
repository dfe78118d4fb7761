# prune: 16 rows in flight per lane, 1 CTA/SM bound; parity then C2 + B24 benches
timeout 900 python -m pytest tests/test_prune_parity.py tests/test_global_select_gpu.py tests/test_fusion_gpu.py -q -x -m gpu 2>&1 | tail -2
for a in "--dtype f32" "--dtype bf16" "--config C4_fc1" "--config C4_fc2" "--config C3_fc2"; do
timeout 300 python bench.py --no-cpu-baseline --steps 300 $a --e2e-steps 2 > gpurun_out/r16.json 2>gpurun_out/r16.err
python -c "
import json
d=json.loads(open('gpurun_out/r16.json').read().strip().splitlines()[-1])
print('$a', round(d['value']), 'us/step', round(d['ms_per_step']*1e3,2), {k:(round(v['ms']*1e3,1), round(v.get('GB/s',0))) for k,v in d['kernels'].items()})
" || tail -5 gpurun_out/r16.err
done
