timeout 1500 python -m pytest tests/test_gpu_full_parity.py -q -s -p no:cacheprovider 2>&1 | tail -15
