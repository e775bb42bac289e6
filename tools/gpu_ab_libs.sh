# Event-timed CGS2 Gram / update at the config-3 shape for several builds of the library:
#   gpurun -- 'bash tools/gpu_ab_libs.sh libA.so libB.so ...'   (paths under paper_2305_19013_b200/)
for rep in 1 2; do
for lib in "$@"; do
  timeout 120 python tools/kbench_cgs2.py paper_2305_19013_b200/$lib 2097152 32 4 inplace 2>&1 | tail -1
  timeout 120 python tools/kbench_cgs2.py paper_2305_19013_b200/$lib 2097152 32 1 inplace 2>&1 | tail -1
done; done
