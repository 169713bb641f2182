#!/bin/bash
# Kernel-variant sweep on the box (benchmarking only): the default build against every variants/*/libdfx.so
# (tools/build_variant.py) on the C2 bench line (ms/step, loss kernel fraction of HBM, kernel ms) and the C5 share.
mkdir -p gpurun_out
for lib in paper_2507_13833_b200/lib/libdfx.so $(ls variants/*/libdfx.so 2>/dev/null); do
  v=$(basename $(dirname $lib))
  for rep in 1 2; do
    DFX_LIB_PATH=$PWD/$lib timeout 120 python bench.py --steps 100 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());print('$v C2 rep $rep', d['ms_per_step'], d['roofline']['frac'], d['roofline']['kernel_ms'])"
    DFX_LIB_PATH=$PWD/$lib timeout 300 python tools/measure_configs.py --only C5 2>/dev/null | grep C5 | python -c "import json,sys;d=json.loads(sys.stdin.read());print('$v C5 rep $rep', round(d['kernel_ms'],5), round(d['kernel_frac_of_hbm'],4))"
  done
done
