# ncu evidence for the bench workload (config 2): launch list + full captures of the CGS2 kernels at d = 100
mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e"
$CMD > gpurun_out/prof_plain.log 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches_r01.csv $CMD > gpurun_out/ncu_list.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:gram16_stream -s 298 -c 1 -o gpurun_out/prof_hist_gram -f $CMD > gpurun_out/ncu_g.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:update16_stream -s 298 -c 1 -o gpurun_out/prof_hist_update -f $CMD > gpurun_out/ncu_u.log 2>&1
ls -la gpurun_out/*.ncu-rep gpurun_out/launches_r01.csv
