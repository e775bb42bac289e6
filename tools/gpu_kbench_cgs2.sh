for rep in 1 2; do
for lib in tools/lib_base.so tools/lib_swap.so; do
  timeout 120 python tools/kbench_cgs2.py $lib 262144 16 100 inplace 2>&1 | tail -1
  timeout 120 python tools/kbench_cgs2.py $lib 262144 16 8 inplace 2>&1 | tail -1
  timeout 120 python tools/kbench_cgs2.py $lib 2097152 32 4 inplace 2>&1 | tail -1
  timeout 120 python tools/kbench_cgs2.py $lib 16777216 64 3 inplace 2>&1 | tail -1
done; done
