timeout 1500 python -m pytest tests -q -m gpu -x --timeout 300 2>&1 | tail -1
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err; grep "step ms" gpurun_out/bench.err; cut -c1-200 gpurun_out/bench.json
timeout 600 python tools/run_configs.py --configs 2 2>&1 | cut -c1-200
