set -x
free -g; nproc; nvidia-smi --query-gpu=name,memory.total,clocks.max.sm --format=csv
python -c "import torch; print('meminfo', torch.cuda.mem_get_info())"
python paper_2305_19013_b200/build.py > gpurun_out/build.log 2>&1; echo build rc $?
timeout 600 python tools/breakdown.py --config 5 --kmax 8 > gpurun_out/bd5.json 2> gpurun_out/bd5.err
timeout 300 python tools/breakdown.py --config 3 --kmax 40 > gpurun_out/bd3.json 2> gpurun_out/bd3.err
timeout 300 python tools/breakdown.py --config 4 --kmax 12 > gpurun_out/bd4.json 2> gpurun_out/bd4.err
cat gpurun_out/bd*.json
