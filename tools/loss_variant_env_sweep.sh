# the loss kernel's instantiated variants (DFX_LOSS_VARIANT: unroll x CTAs/SM) on the C2 bench line and the C5 share
for v in u2b3 u3b2 u4b2 u2b2 u1b4; do
  DFX_LOSS_VARIANT=$v timeout 120 python bench.py --steps 100 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());print('$v C2', d['ms_per_step'], d['roofline']['frac'], d['roofline']['kernel_ms'])"
  DFX_LOSS_VARIANT=$v timeout 300 python tools/measure_configs.py --only C5 2>/dev/null | grep C5 | python -c "import json,sys;d=json.loads(sys.stdin.read());print('$v C5', round(d['kernel_ms'],5), round(d['kernel_frac_of_hbm'],4), round(d['step_graph_ms'],5))"
done
