timeout 600 python -m pytest tests -q -m gpu -x 2>&1 | tail -1
timeout 600 python tools/breakdown.py --config 4 --kmax 40 2>&1 | tail -1
