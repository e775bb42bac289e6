# full GPU test suite + smoke; logs to gpurun_out/
timeout 2400 python -m pytest tests/ -q -m gpu -x -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo "pytest rc $?"
tail -25 gpurun_out/gpu_tests.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc $?"; tail -3 gpurun_out/smoke.log
