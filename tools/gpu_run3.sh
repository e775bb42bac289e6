set -x
python -m pytest tests -q -m gpu 2>&1 | tail -4
timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/bench3.json 2> gpurun_out/bench3.err; tail -3 gpurun_out/bench3.err; cat gpurun_out/bench3.json
CMD="python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e"
$CMD > gpurun_out/plain.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu1.log 2>&1
$CMD > gpurun_out/plain2.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:gram_dmma -s 400 -c 1 -o gpurun_out/prof_gram $CMD > gpurun_out/ncu2.log 2>&1
$CMD > gpurun_out/plain3.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:update_dmma -s 200 -c 1 -o gpurun_out/prof_update $CMD > gpurun_out/ncu3.log 2>&1
ls -la gpurun_out
