mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kernels.py -q -x 2>&1 | tail -3
timeout 300 python tools/kernel_times.py 2>&1 | tail -6
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -2 gpurun_out/bench.err
python -c "
import json; d=json.load(open('gpurun_out/bench.json')); r=d['roofline']
print('value', round(d['value'],1), 'ms/step', round(d['ms_per_step'],1), 'e2e', d['e2e'] and round(d['e2e']['value'],1))
print('roofline', r['kernel'], round(r['achieved']), round(r['frac'],3), r['per_kernel'], 'step_frac', round(r['step_model_frac'],3), 'clocks', d['clocks'])
"
timeout 1200 python tools/run_configs.py --configs 3,4 2>&1 | cut -c1-300
