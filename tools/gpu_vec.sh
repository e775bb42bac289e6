timeout 1500 python -m pytest tests -q -m gpu -x --timeout 300 2>&1 | tail -1
timeout 600 python tools/breakdown.py --config 4 --kmax 60 2>&1 | tail -1
timeout 1200 python tools/run_configs.py --configs 3,4,5 2>&1 | cut -c1-220
