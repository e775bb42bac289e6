mkdir -p gpurun_out
for c in "2" "3 --kmax 300" "4 --kmax 60" "5 --kmax 6"; do timeout 900 python tools/breakdown.py --config $c 2>&1 | tail -2; done
