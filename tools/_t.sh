timeout 600 python -m pytest tests/test_gpu_parity.py -q -k "gae" -p no:cacheprovider 2>&1 | tail -15
