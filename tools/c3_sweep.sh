# C3 two-launch step under loss-kernel variants of the per-token-advantage path (variants/*/libdfx.so) and slot
# windows (DFX_SLOT_SHIFT)
for lib in paper_2507_13833_b200/lib/libdfx.so $(ls variants/*/libdfx.so 2>/dev/null); do
  v=$(basename $(dirname $lib))
  for sh in ${SHIFTS:-11 10}; do
  echo "[$v sh$sh] $(DFX_SLOT_SHIFT=$sh DFX_LIB_PATH=$PWD/$lib timeout 300 python tools/measure_configs.py --only C3 --out /tmp/x.json 2>&1 | grep '"C3"' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('step', round(d['step_graph_ms'],5), 'loss', round(d['loss_kernel_ms'],5), 'gae', round(d['gae_graph_ms'],5), 'frac', round(d['step_frac_of_hbm'],3))")"
  done
done
