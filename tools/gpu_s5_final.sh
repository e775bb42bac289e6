# end-of-round evidence on the final build: ncu capture of the tile-symmetric W^T W, then all configs, the GPU
# suite, smoke, the default bench and the reference arm (tools/gpu_final_numbers.sh)
NCU=/usr/local/cuda/bin/ncu
timeout 300 python tools/kbench_gram_self.py paper_2305_19013_b200/libekcg_b200.so 16777216 64 > gpurun_out/r02_gram_self_plain.log 2>&1; echo "plain rc $?"
timeout 900 $NCU --set full --import-source on --clock-control none -k regex:gram_dmma_kernel --launch-skip 2 --launch-count 1 \
  -f -o gpurun_out/r02_cfg5_gram_self_sym python tools/kbench_gram_self.py paper_2305_19013_b200/libekcg_b200.so 16777216 64 \
  > gpurun_out/r02_gram_self_ncu.log 2>&1; echo "ncu rc $?"
bash tools/gpu_final_numbers.sh
