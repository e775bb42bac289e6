mkdir -p gpurun_out
python tools/prof_csr.py 3 32 && ncu --set full --import-source on --clock-control none -k regex:csr_spmm -s 2 -c 1 -o gpurun_out/csr32 -f python tools/prof_csr.py 3 32 > gpurun_out/ncu_csr.log 2>&1; tail -1 gpurun_out/ncu_csr.log
