mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kernels.py -q -x -k "wide or gram or update" 2>&1 | tail -2
timeout 600 python tools/kernel_times.py --wide 2>&1 | tail -8 | python -c "
import sys,json
for line in sys.stdin:
    k,_,rest=line.partition(' ')
    try: d=json.loads(rest)
    except Exception: print(line.strip()); continue
    print(k, {kk:(round(v.get('TF',0),1), round(v['GBs'])) for kk,v in d.items()})
"
