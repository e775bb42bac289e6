NCU=/usr/local/cuda/bin/ncu
timeout 900 $NCU --set full --import-source on --clock-control none -k regex:update_smem_kernel --launch-skip 10 --launch-count 1 \
  -f -o gpurun_out/r02_cfg5full_hist_update python tools/breakdown.py --config 5 --kmax 5 --once > gpurun_out/r02_c1.log 2>&1; echo "upd rc $?"
timeout 900 $NCU --set full --import-source on --clock-control none -k regex:gram_dmma_kernel --launch-skip 10 --launch-count 1 \
  -f -o gpurun_out/r02_cfg5full_hist_gram python tools/breakdown.py --config 5 --kmax 5 --once > gpurun_out/r02_c2.log 2>&1; echo "gram rc $?"
timeout 900 $NCU --set full --import-source on --clock-control none -k regex:update_smem_kernel --launch-skip 12 --launch-count 1 \
  -f -o gpurun_out/r02_cfg5full_tri_apply python tools/breakdown.py --config 5 --kmax 5 --once > gpurun_out/r02_c3.log 2>&1; echo "tri rc $?"
timeout 900 $NCU --set full --import-source on --clock-control none -k regex:update_wide_stream_kernel --launch-skip 14 --launch-count 1 \
  -f -o gpurun_out/r02_cfg3_hist_update python tools/breakdown.py --config 3 --edge 128 --kmax 6 --once > gpurun_out/r02_c4.log 2>&1; echo "cfg3 upd rc $?"
timeout 900 $NCU --set full --import-source on --clock-control none -k regex:stencil_march_kernel --launch-skip 8 --launch-count 1 \
  -f -o gpurun_out/r02_cfg3_stencil python tools/breakdown.py --config 3 --edge 128 --kmax 6 --once > gpurun_out/r02_c5.log 2>&1; echo "cfg3 stencil rc $?"
timeout 900 $NCU --set full --import-source on --clock-control none -k regex:update_smem_kernel --launch-skip 6 --launch-count 1 \
  -f -o gpurun_out/r02_cfg4_hist_update python tools/breakdown.py --config 4 --edge 256 --kmax 4 --once > gpurun_out/r02_c6.log 2>&1; echo "cfg4 upd rc $?"
