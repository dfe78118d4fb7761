for o in pwd pdw pwd pdw; do for dt in f32 bf16; do
timeout 300 python bench.py --no-cpu-baseline --steps 1000 --dtype $dt --order $o --e2e-steps 2 > gpurun_out/ord.json 2>gpurun_out/ord.err
python -c "
import json
d=json.loads(open('gpurun_out/ord.json').read().strip().splitlines()[-1])
print('$o $dt', round(d['value']), 'us/step', round(d['ms_per_step']*1e3,2), {k:(round(v['ms']*1e3,1)) for k,v in d['kernels'].items()})
" || tail -5 gpurun_out/ord.err
done; done
