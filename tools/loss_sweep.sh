#!/bin/bash
# Loss-kernel tuning sweep (on the box): DFX_LOSS_VARIANT (unroll x CTAs/SM) on the C2 bench, DFX_SLOT_SHIFT
# (slot window 2^s tokens) on the C2 bench and on measure_configs C3 / C5-share. Knobs are benchmarking-only.
python paper_2507_13833_b200/build.py > /dev/null
mkdir -p gpurun_out
for v in u2b3 u3b2 u4b2 u2b2 u1b4 u2b4; do
  DFX_LOSS_VARIANT=$v timeout 120 python bench.py --steps 50 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());print('variant $v', d['ms_per_step'], d['roofline']['frac'], d['roofline']['kernel_ms'])"
done
for s in 9 10 11 12; do
  DFX_SLOT_SHIFT=$s timeout 120 python bench.py --steps 50 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());print('shift $s C2', d['ms_per_step'], d['roofline']['frac'], d['roofline']['kernel_ms'])"
  DFX_SLOT_SHIFT=$s timeout 200 python tools/measure_configs.py --out gpurun_out/cfg_shift$s.json 2>/dev/null | grep '"C3"\|C5/8' | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print('shift $s', d['config'], d.get('loss_kernel_ms', d.get('kernel_ms')))"
done
