timeout 600 /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_launches_cfg1.csv python tools/ab_graphs.py --config 1 --reps 1 --prechol > /dev/null 2>&1
echo rc $?
