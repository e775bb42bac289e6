# ncu evidence for configs 3-5 (round 2): the bench launch list (config 5, full size) and one --set full
# capture per hot kernel at steady-state history depth.  Each capture runs only after the plain command
# exited 0.  Outputs: gpurun_out/r02_*.ncu-rep, gpurun_out/r02_launches_cfg5.csv
NCU=/usr/local/cuda/bin/ncu
set -x
timeout 900 python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/r02_bench_plain.json 2>&1 || exit 1
timeout 1500 $NCU --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_launches_cfg5.csv \
  python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --no-kernel-timer > gpurun_out/r02_launches.log 2>&1
cap() {  # name config edge kmax regex skip
  timeout 900 $NCU --set full --import-source on --clock-control none -k regex:$5 --launch-skip $6 --launch-count 1 \
    -f -o gpurun_out/r02_$1 python tools/breakdown.py --config $2 --edge $3 --kmax $4 --once > gpurun_out/r02_$1.log 2>&1
  echo "$1 rc $?"
}
timeout 600 python tools/breakdown.py --config 5 --edge 4096 --kmax 5 --once > gpurun_out/r02_bd5.json 2>&1 || exit 1
cap cfg5_hist_update 5 4096 5 update_smem_kernel 10
cap cfg5_hist_gram 5 4096 5 gram_dmma_kernel 10
cap cfg5_tri_apply 5 4096 5 update_smem_kernel 12
cap cfg5_stencil 5 4096 5 stencil_march_kernel 10
cap cfg5_xr 5 4096 5 xr_update4_kernel 3
timeout 600 python tools/breakdown.py --config 3 --edge 128 --kmax 6 --once > gpurun_out/r02_bd3.json 2>&1 || exit 1
cap cfg3_hist_update 3 128 6 update_wide_stream_kernel 14
cap cfg3_hist_gram 3 128 6 gram_wide_stream_kernel 14
cap cfg3_stencil 3 128 6 stencil_march_kernel 8
timeout 600 python tools/breakdown.py --config 4 --edge 256 --kmax 4 --once > gpurun_out/r02_bd4.json 2>&1 || exit 1
cap cfg4_hist_update 4 256 4 update_smem_kernel 6
cap cfg4_hist_gram 4 256 4 gram_dmma_kernel 6
cap cfg4_stencil 4 256 4 stencil_march_kernel 13
timeout 600 python tools/prof_csr.py 5 2048 64 > gpurun_out/r02_csr.log 2>&1 || exit 1
timeout 900 $NCU --set full --import-source on --clock-control none -k regex:csr_spmm --launch-skip 2 --launch-count 1 \
  -f -o gpurun_out/r02_csr_m64 python tools/prof_csr.py 5 2048 64 >> gpurun_out/r02_csr.log 2>&1
echo "csr rc $?"
ls -la gpurun_out/
