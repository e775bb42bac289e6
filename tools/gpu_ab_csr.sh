# A/B of two library builds on the CSR SpMM (configs 2, 3, 5-class), bitwise checksum
for lib in paper_2305_19013_b200/libekcg_old.so paper_2305_19013_b200/libekcg_b200.so; do
  timeout 200 python tools/kbench_csr.py $lib 3 128 32 2>&1 | tail -1
  timeout 200 python tools/kbench_csr.py $lib 2 64 16 2>&1 | tail -1
  timeout 200 python tools/kbench_csr.py $lib 5 2048 64 2>&1 | tail -1
  timeout 200 python tools/kbench_csr.py $lib 4 128 64 2>&1 | tail -1
  timeout 200 python tools/kbench_csr.py $lib 1 100 8 2>&1 | tail -1
done
