# round snapshot: gpu tests, smoke, default bench, all five configs at full size
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -q -m gpu -x 2>&1 | tail -1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -1 gpurun_out/bench.err; cut -c1-300 gpurun_out/bench.json
timeout 2400 python tools/run_configs.py --configs 1,2,3,4,5 > gpurun_out/configs.jsonl 2>gpurun_out/configs.err; cut -c1-250 gpurun_out/configs.jsonl
