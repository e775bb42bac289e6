NCU=/usr/local/cuda/bin/ncu
set -x
timeout 300 python tools/prof_stencil_cfg.py 5 8192 64 > gpurun_out/r02_cfg5full_stencil.log 2>&1 || exit 1
timeout 900 $NCU --set full --import-source on --clock-control none -k regex:stencil_march --launch-skip 2 --launch-count 1 \
  -f -o gpurun_out/r02_cfg5full_stencil python tools/prof_stencil_cfg.py 5 8192 64 >> gpurun_out/r02_cfg5full_stencil.log 2>&1
echo "stencil rc $?"
timeout 900 $NCU --set full --import-source on --clock-control none -k regex:update_smem_kernel --launch-skip 10 --launch-count 1 \
  -f -o gpurun_out/r02_cfg5full_hist_update python tools/breakdown.py --config 5 --kmax 5 --once > gpurun_out/r02_cfg5full_update.log 2>&1
echo "update rc $?"
tail -3 gpurun_out/r02_cfg5full_update.log
