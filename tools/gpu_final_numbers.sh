# all five configs at full size + the default bench + the config-1 / config-3 bench lines
timeout 1500 python tools/run_configs.py --configs 1,2,3,4,5 > gpurun_out/r02_configs_full_size.jsonl 2> gpurun_out/r02_configs.err; echo "configs rc $?"
timeout 1200 python bench.py --steps 5 --warmup 3 > gpurun_out/r02_bench_cfg5.json 2> gpurun_out/r02_bench_cfg5.err; echo "bench rc $?"
tail -2 gpurun_out/r02_bench_cfg5.err
