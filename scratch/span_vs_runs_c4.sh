for k in runs span; do for dt in f32 bf16; do BSRP_WGRAD=$k timeout 600 python bench.py --config C4_fc2 --dtype $dt --steps 50 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/c4_$k_$dt.json 2>/dev/null; python -c "
import json
d=json.loads(open('gpurun_out/c4_$k_$dt.json').read().strip().splitlines()[-1])
print('$k $dt', 'wgrad', round(d['kernels']['wgrad']['ms']*1e3,1))
"; done; done
