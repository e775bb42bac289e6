timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_solver.py -q -x --timeout 120 2>&1 | tail -3
timeout 120 python tools/short_solve.py 2 4 && timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv --log-file gpurun_out/short_launches.csv python tools/short_solve.py 2 4 > gpurun_out/ncu_s.log 2>&1
timeout 300 python tools/iter_profile.py 2 2>&1 | grep -E "^rep|sum iters"
