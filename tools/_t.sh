timeout 600 python -m pytest tests -m gpu -q -x -p no:cacheprovider 2>&1 | tail -2
timeout 300 python bench.py --no-cpu-baseline --no-e2e --steps 100 2>&1 | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());print('c2', d['value'], d['ms_per_step'], d['roofline']['frac'], d['roofline']['kernel_ms'])"
timeout 300 python tools/measure_configs.py --out gpurun_out/configs_s2e.json 2>&1 | python -c "
import sys, json
for l in sys.stdin:
    l = l.strip()
    if l.startswith('{'):
        d = json.loads(l); print({k: (round(v, 4) if isinstance(v, float) else v) for k, v in d.items() if k != 'placements'})"
