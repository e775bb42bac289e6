mkdir -p gpurun_out
python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b_launch.json 2>gpurun_out/b_launch.err && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 2500 --csv --log-file gpurun_out/launches_cur.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_l.log 2>&1
tail -2 gpurun_out/ncu_l.log
