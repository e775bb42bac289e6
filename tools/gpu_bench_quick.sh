timeout 600 python -m pytest tests/test_gpu_kernels.py -q -x -k "gram" --timeout 120 2>&1 | tail -1
timeout 300 python tools/iter_profile.py 2 2>&1 | grep -E "^rep"
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -2 gpurun_out/bench.err
python -c "
import json; d=json.load(open('gpurun_out/bench.json')); r=d['roofline']
print('value', round(d['value'],1), 'ms/step', round(d['ms_per_step'],1), 'e2e', d['e2e'] and round(d['e2e']['value'],1))
print('roofline', r['kernel'], round(r['achieved']), round(r['frac'],3), {k:round(v['GBs']) for k,v in r['per_kernel'].items()}, 'step_frac', round(r['step_model_frac'],3), 'clocks', d['clocks'])
"
