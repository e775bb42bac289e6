mkdir -p gpurun_out
python tools/prof_march.py 32 128 128 128 0 && \
ncu --set full --import-source on --clock-control none -k regex:stencil_march -s 2 -c 1 -o gpurun_out/march_const32 -f python tools/prof_march.py 32 128 128 128 0 > gpurun_out/ncu_march.log 2>&1
python tools/prof_march.py 32 128 128 128 0 tile && \
ncu --set full --import-source on --clock-control none -k regex:stencil_march -s 2 -c 1 -o gpurun_out/march_tile32 -f python tools/prof_march.py 32 128 128 128 0 tile >> gpurun_out/ncu_march.log 2>&1
tail -3 gpurun_out/ncu_march.log
