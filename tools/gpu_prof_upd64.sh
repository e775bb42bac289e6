mkdir -p gpurun_out
python tools/prof_update.py 2 2 64 4194304 && ncu --set full --import-source on --clock-control none -k regex:update_smem -s 2 -c 1 -o gpurun_out/upd64 -f python tools/prof_update.py 2 2 64 4194304 > gpurun_out/ncu_upd64.log 2>&1; tail -1 gpurun_out/ncu_upd64.log
