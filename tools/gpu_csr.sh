timeout 900 python -m pytest tests/test_gpu_kernels.py -q -x -k "csr" 2>&1 | tail -1
timeout 600 python tools/stencil_bw.py --configs 2,3 --csr 2>&1 | grep csr
