timeout 1200 python -m pytest tests/test_gpu_multirank.py -x -q -s > gpurun_out/multirank.log 2>&1; tail -30 gpurun_out/multirank.log
