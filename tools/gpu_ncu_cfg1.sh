NCU=/usr/local/cuda/bin/ncu
timeout 600 $NCU --set full --import-source on --clock-control none -k regex:update_epi_kernel --launch-skip 40 --launch-count 1 \
  -f -o gpurun_out/r02_cfg1_update_epi python tools/ab_graphs.py --config 1 --reps 1 > /dev/null 2>&1; echo rc $?
timeout 600 $NCU --set full --import-source on --clock-control none -k regex:stencil_cholinv --launch-skip 20 --launch-count 1 \
  -f -o gpurun_out/r02_cfg1_stencil_cholinv python tools/ab_graphs.py --config 1 --reps 1 > /dev/null 2>&1; echo rc $?
