timeout 600 python -m pytest tests/test_gpu_kernels.py -q -x -k "stencil" --timeout 120 2>&1 | tail -2
timeout 300 python tools/kernel_times.py --stencil 2>&1 | tail -8
timeout 600 python tools/breakdown.py --config 3 --kmax 300 2>&1 | tail -1
