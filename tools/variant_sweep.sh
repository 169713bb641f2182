#!/bin/bash
# Kernel-variant sweep on the box (benchmarking only): for every variants/*/libdfx.so (tools/build_variant.py),
# the C2 bench line (loss kernel ms, HBM fraction) and measure_configs' C3 / C5-share loss timings.
mkdir -p gpurun_out
for lib in variants/*/libdfx.so; do
  v=$(basename $(dirname $lib))
  for rep in 1 2; do
    DFX_LIB_PATH=$PWD/$lib timeout 120 python bench.py --steps 100 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());print('$v C2 rep $rep', d['ms_per_step'], d['roofline']['frac'], d['roofline']['kernel_ms'])"
  done
  DFX_LIB_PATH=$PWD/$lib timeout 200 python tools/measure_configs.py --out gpurun_out/cfg_$v.json 2>/dev/null | grep '"C3"\|C5/8' | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print('$v', d['config'][:12], 'loss', d.get('loss_kernel_ms', d.get('kernel_ms')), 'gae', d.get('gae_graph_ms'), 'step', d.get('step_graph_ms'))"
done
# C3 with the round-1 fixed 2048-token windows (runtime knob) on the default build
for s in 11 10; do
DFX_SLOT_SHIFT=$s timeout 200 python tools/measure_configs.py --out gpurun_out/cfg_shift$s.json 2>/dev/null | grep '"C3"' | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print('default+shift$s', d['config'][:12], 'loss', d.get('loss_kernel_ms'), 'gae', d.get('gae_graph_ms'), 'step', d.get('step_graph_ms'))"
done
