timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -1
timeout 600 python tools/stencil_bw.py --configs 3,5 2>&1 | tail -4
