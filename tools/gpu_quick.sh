# quick GPU check: all gpu tests + a bench line
python -m pytest tests -q -m gpu -x 2>&1 | tail -4
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -3 gpurun_out/bench.err
python -c "
import json; d=json.load(open('gpurun_out/bench.json')); r=d['roofline']
print('value', round(d['value'],1), 'ms/step', round(d['ms_per_step'],1), 'e2e', d['e2e'] and round(d['e2e']['value'],1))
print('roofline', r['kernel'], round(r['achieved']), round(r['frac'],3), r['per_kernel'], 'step_frac', round(r['step_model_frac'],3), 'clocks', d['clocks'])
"
