# full-size configs 1-5 -> gpurun_out/configs.jsonl, then the bench line
mkdir -p gpurun_out
timeout 1500 python tools/run_configs.py --configs 1,2,3,4,5 > gpurun_out/configs.jsonl 2> gpurun_out/configs.err; tail -2 gpurun_out/configs.err
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_r01.json 2> gpurun_out/bench_r01.err; tail -3 gpurun_out/bench_r01.err
cut -c1-250 gpurun_out/configs.jsonl
