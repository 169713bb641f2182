# GAE under each library build (default + variants/*): GAE parity tests, C3 microbenchmark, C3 rows
for lib in paper_2507_13833_b200/lib/libdfx.so $(ls variants/*/libdfx.so 2>/dev/null); do
  v=$(basename $(dirname $lib)); export DFX_LIB_PATH=$PWD/$lib
  for gv in ${GAE_VARIANTS:-seg}; do
    export DFX_GAE_VARIANT=$gv
    echo "== $v $gv"
    timeout 300 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_sweep.py -q -x -k "gae or c3" -p no:cacheprovider 2>&1 | grep -E "FAILED|passed|failed|Error|assert" | head -6
    timeout 60 python tools/gae_bench.py
    timeout 60 python tools/gae_bench.py --records 4096 --n 16 --len 4096 --dist uniform
    timeout 300 python tools/measure_configs.py --only C3 --out /tmp/x.json 2>&1 | grep C3 | cut -c 1-330
  done
done
