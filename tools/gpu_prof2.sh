# ncu full captures of the streamed CGS2 kernels at d = 100 (config-2 bench) + e2e host profile
mkdir -p gpurun_out
timeout 300 python tools/e2e_profile.py 2>&1 | head -60
CMD="python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gram16_stream -s 298 -c 1 -o gpurun_out/prof_hist_gram -f $CMD > gpurun_out/ncu_g.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:update16_stream -s 298 -c 1 -o gpurun_out/prof_hist_update -f $CMD > gpurun_out/ncu_u.log 2>&1
tail -2 gpurun_out/ncu_g.log gpurun_out/ncu_u.log
