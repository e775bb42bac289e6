mkdir -p gpurun_out
python tools/prof_update.py 2 110 && ncu --set full --import-source on --clock-control none -k regex:update16 -s 2 -c 1 -o gpurun_out/upd_s2 -f python tools/prof_update.py 2 110 > gpurun_out/ncu_upd.log 2>&1; tail -2 gpurun_out/ncu_upd.log
