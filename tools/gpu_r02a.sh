set -x
./tools/fp64_peak > gpurun_out/fp64_peak.txt 2>&1
cat gpurun_out/fp64_peak.txt
timeout 900 python -m pytest tests/test_gpu_full_parity.py -x -q -s > gpurun_out/full_parity.log 2>&1; tail -15 gpurun_out/full_parity.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench5.json 2> gpurun_out/bench5.err; tail -3 gpurun_out/bench5.err; cat gpurun_out/bench5.json
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench5_ref.json 2> gpurun_out/bench5_ref.err; tail -3 gpurun_out/bench5_ref.err; cat gpurun_out/bench5_ref.json
