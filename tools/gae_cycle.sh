mkdir -p gpurun_out
for v in default s128b4 s256 s64; do
  DFX_GAE_VARIANT=$v timeout 120 python -m pytest tests/test_gpu_parity.py -q -x -k gae -p no:cacheprovider 2>&1 | tail -1
  DFX_GAE_VARIANT=$v timeout 60 python tools/gae_bench.py
  DFX_GAE_VARIANT=$v timeout 60 python tools/gae_bench.py --whiten
  DFX_GAE_VARIANT=$v timeout 60 python tools/gae_bench.py --records 4096 --n 16 --len 4096 --dist uniform
done
