# ncu evidence for the one-kernel cluster solve (config 1) and the plane-march stencils after the wave-aware
# chunking; each capture only after the plain command has exited 0
NCU=/usr/local/cuda/bin/ncu
timeout 300 python tools/cluster_time.py --edges 100 --repeats 1 > gpurun_out/r02_cluster_plain.log 2>&1; echo "plain rc $?"
timeout 900 $NCU --set full --import-source on --clock-control none -k regex:cluster_solve_kernel --launch-count 1 \
  -f -o gpurun_out/r02_cfg1_cluster_solve python tools/cluster_time.py --edges 100 --repeats 1 > gpurun_out/r02_d1.log 2>&1; echo "cluster rc $?"
timeout 600 $NCU --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/r02_launches_cfg1.csv \
  python tools/run_configs.py --configs 1 --repeats 1 > gpurun_out/r02_d2.log 2>&1; echo "launch list rc $?"
timeout 300 python tools/prof_stencil_cfg.py 5 8192 64 > gpurun_out/r02_d3.log 2>&1; echo "plain rc $?"
timeout 900 $NCU --set full --import-source on --clock-control none -k regex:stencil_march_kernel --launch-skip 2 --launch-count 1 \
  -f -o gpurun_out/r02_cfg5full_stencil_waves python tools/prof_stencil_cfg.py 5 8192 64 > gpurun_out/r02_d4.log 2>&1; echo "cfg5 stencil rc $?"
timeout 900 $NCU --set full --import-source on --clock-control none -k regex:stencil_march_kernel --launch-skip 2 --launch-count 1 \
  -f -o gpurun_out/r02_cfg3_stencil_waves python tools/prof_stencil_cfg.py 3 128 32 > gpurun_out/r02_d5.log 2>&1; echo "cfg3 stencil rc $?"
