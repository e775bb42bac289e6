# ncu captures of the plane-march stencils after the tile-layer hoisting (each after the plain run exited 0)
NCU=/usr/local/cuda/bin/ncu
timeout 300 python tools/prof_stencil_cfg.py 5 8192 64 > gpurun_out/r02_e0.log 2>&1; echo "plain rc $?"
timeout 900 $NCU --set full --import-source on --clock-control none -k regex:stencil_march_kernel --launch-skip 2 --launch-count 1 \
  -f -o gpurun_out/r02_cfg5full_stencil_hoisted python tools/prof_stencil_cfg.py 5 8192 64 > gpurun_out/r02_e1.log 2>&1; echo "cfg5 stencil rc $?"
timeout 900 $NCU --set full --import-source on --clock-control none -k regex:stencil_march_kernel --launch-skip 2 --launch-count 1 \
  -f -o gpurun_out/r02_cfg3_stencil_hoisted python tools/prof_stencil_cfg.py 3 128 32 > gpurun_out/r02_e2.log 2>&1; echo "cfg3 stencil rc $?"
timeout 900 python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/r02_bench_plain.json 2>&1 || exit 1
timeout 1500 $NCU --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_launches_cfg5.csv \
  python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --no-kernel-timer > gpurun_out/r02_launches.log 2>&1
echo "launch list rc $?"
