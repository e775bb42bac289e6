mkdir -p gpurun_out
timeout 1200 python -m pytest tests -q -m gpu -x 2>&1 | tail -2
timeout 600 python tools/breakdown.py --config 3 --kmax 200 2>&1 | tail -1
timeout 900 python tools/run_configs.py --configs 3 --repeats 1 2>&1 | tail -1 | cut -c1-330
