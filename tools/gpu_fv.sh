for v in 2 5 6; do echo "variant $v"; timeout 300 python tools/kernel_times.py --fused $v 2>&1 | tail -3; done
