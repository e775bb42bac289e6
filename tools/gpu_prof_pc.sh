timeout 300 ncu --set full --import-source on --clock-control none -k regex:prechol -s 3 -c 1 -o gpurun_out/prechol -f python tools/short_solve.py 2 4 > gpurun_out/ncu_pc.log 2>&1; tail -1 gpurun_out/ncu_pc.log
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_solver.py -q -x --timeout 120 2>&1 | tail -2
