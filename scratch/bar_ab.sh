# release/acquire grid barrier: parity of every cooperative kernel, then C2 bench
timeout 900 python -m pytest tests/test_prune_parity.py tests/test_global_select_gpu.py tests/test_rows_gpu.py tests/test_fusion_gpu.py tests/test_pdl_gpu.py -q -x -m gpu 2>&1 | tail -3
for dt in f32 bf16; do
timeout 300 python bench.py --no-cpu-baseline --steps 1000 --dtype $dt --e2e-steps 3 > gpurun_out/bar_${dt}.json 2>gpurun_out/bar_${dt}.err
python -c "
import json
d=json.loads(open('gpurun_out/bar_${dt}.json').read().strip().splitlines()[-1])
print('$dt', round(d['value']), 'us/step', round(d['ms_per_step']*1e3,2), {k:(round(v['ms']*1e3,1), round(v.get('GB/s',0))) for k,v in d['kernels'].items()}, d['clocks']['sm_mhz'])
" || tail -5 gpurun_out/bar_${dt}.err
done
