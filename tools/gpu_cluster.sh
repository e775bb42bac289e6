# cluster-solve tests + config-1 timing (launch-per-phase vs one-kernel cluster solve)
timeout 600 python -m pytest tests/test_gpu_cluster.py -q -x -p no:cacheprovider 2>&1 | tail -25
timeout 300 python tools/run_configs.py --configs 1 --repeats 5 2>&1 | tail -8
