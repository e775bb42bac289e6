timeout 900 python -m pytest tests/test_gpu_kernels.py -q -x -k "csr or stencil_equals" 2>&1 | tail -2
timeout 600 python tools/stencil_bw.py --configs 2,3 --csr 2>&1 | grep csr
timeout 600 python bench.py --form csr --steps 2 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | cut -c1-300
