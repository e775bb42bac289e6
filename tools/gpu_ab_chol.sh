timeout 600 python -m pytest tests -q -m gpu -x 2>&1 | tail -1
timeout 600 python tools/ab_lib.py build/lib_ctachol.so build/lib_warpchol.so 1 4 2>&1 | tail -3
timeout 900 python tools/ab_lib.py build/lib_ctachol.so build/lib_warpchol.so 2 3 2>&1 | tail -3
