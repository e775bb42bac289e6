timeout 300 python tools/kernel_times.py --fused 1 2>&1 | tail -3
timeout 300 python tools/kernel_times.py --fused 0 2>&1 | tail -3
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_solver.py -q -x --timeout 120 2>&1 | tail -5
timeout 600 python tools/ab_solve.py 2 2>&1 | tail -5
