#!/bin/bash
# Kernel-variant sweep on the box (benchmarking only): the default build against every variants/*/libdfx.so
# (tools/build_variant.py) on the C2 bench line (loss kernel ms, HBM fraction).
mkdir -p gpurun_out
for lib in paper_2507_13833_b200/lib/libdfx.so variants/*/libdfx.so; do
  v=$(basename $(dirname $(dirname $lib)))/$(basename $(dirname $lib))
  for rep in 1 2; do
    DFX_LIB_PATH=$PWD/$lib timeout 120 python bench.py --steps 100 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());print('$v C2 rep $rep', d['ms_per_step'], d['roofline']['frac'], d['roofline']['kernel_ms'])"
  done
done
