# per-tag breakdowns and full-size runs of configs 3-5
mkdir -p gpurun_out
timeout 600 python tools/breakdown.py --config 3 --kmax 200 2>&1 | tail -1
timeout 600 python tools/breakdown.py --config 4 --kmax 40 2>&1 | tail -1
timeout 900 python tools/breakdown.py --config 5 --kmax 8 2>&1 | tail -1
timeout 1500 python tools/run_configs.py --configs 1,2,3,4,5 > gpurun_out/configs.jsonl 2>gpurun_out/configs.err; cut -c1-400 gpurun_out/configs.jsonl
