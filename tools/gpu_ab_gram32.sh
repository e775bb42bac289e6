# A/B of the m = 32 streamed Gram (padded slab rows) against the previous build, then the kernel tests
for rep in 1 2; do
for lib in paper_2305_19013_b200/libekcg_old.so paper_2305_19013_b200/libekcg_b200.so; do
  timeout 120 python tools/kbench_cgs2.py $lib 2097152 32 4 inplace 2>&1 | tail -1
  timeout 120 python tools/kbench_cgs2.py $lib 2097152 32 1 inplace 2>&1 | tail -1
done; done
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_rings.py -q -x -p no:cacheprovider 2>&1 | tail -4
