# ncu launch list of one config-5 bench step on the current build (after the plain run exited 0)
NCU=/usr/local/cuda/bin/ncu
timeout 900 python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/r02_bench_plain.json 2>&1 || exit 1
timeout 1500 $NCU --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_launches_cfg5.csv \
  python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --no-kernel-timer > gpurun_out/r02_launches.log 2>&1
echo "launch list rc $?"
