timeout 600 python -m pytest tests/test_wire.py -q -x -p no:cacheprovider 2>&1 | tail -2
timeout 600 python tools/measure_configs.py 2>&1 | grep wire
