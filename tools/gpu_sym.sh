timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -1
timeout 900 python tools/breakdown.py --config 4 --kmax 30 2>&1 | tail -1 | cut -c1-400
