timeout 600 python tools/probe_stencil.py 2>&1 | tail -12
timeout 1200 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_rings.py -q -x -p no:cacheprovider 2>&1 | tail -4
timeout 900 python tools/breakdown.py --config 3 --kmax 40 2>&1 | tail -1
timeout 900 python tools/breakdown.py --config 5 --kmax 8 2>&1 | tail -1
