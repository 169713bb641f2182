# C3 two-pass: loss kernel variants of the per-token-advantage path (unroll x CTAs/SM) and slot windows
for lib in variants/*/libdfx.so; do
  v=$(basename $(dirname $lib))
  for sh in 11 10; do
  echo "[$v sh$sh] $(DFX_SLOT_SHIFT=$sh DFX_LIB_PATH=$PWD/$lib timeout 300 python tools/measure_configs.py --out /tmp/x.json 2>&1 | grep '"C3"' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('step', round(d['step_graph_ms'],5), 'loss', round(d['loss_kernel_ms'],5), 'gae', round(d['gae_graph_ms'],5), 'frac', round(d['step_frac_of_hbm'],3))")"
  done
done
