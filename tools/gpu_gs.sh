timeout 600 python -m pytest tests/test_gpu_kernels.py -q -x 2>&1 | tail -3
timeout 300 python tools/kernel_times.py 2>&1 | tail -6 | python -c "
import sys,json
for line in sys.stdin:
    if '{' not in line: print(line.strip()); continue
    k,j=line.split(' ',1); d=json.loads(j)
    print(k, {kk: round(v['GBs']) for kk,v in d.items()})
"
