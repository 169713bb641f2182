# GAE variants (DFX_GAE_VARIANT): parity of the GAE tests, then the C3 microbenchmark (plain / whitened / a large
# ragged batch) and the C3 rows of measure_configs (two-launch step and fused GAE + loss)
mkdir -p gpurun_out
for v in ${GAE_VARIANTS:-seg lb lb64}; do
  echo "== $v"
  DFX_GAE_VARIANT=$v timeout 300 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_sweep.py -q -x -k "gae or c3" -p no:cacheprovider 2>&1 | grep -E "FAILED|passed|failed|Error|assert" | head -8
  DFX_GAE_VARIANT=$v timeout 60 python tools/gae_bench.py
  DFX_GAE_VARIANT=$v timeout 60 python tools/gae_bench.py --whiten
  DFX_GAE_VARIANT=$v timeout 60 python tools/gae_bench.py --records 4096 --n 16 --len 4096 --dist uniform
  DFX_GAE_VARIANT=$v timeout 300 python tools/measure_configs.py --only C3 --out /tmp/x.json 2>&1 | grep C3 | cut -c 1-400
done
