# C4 round trip at N=2/4 with constant (aligned) and ragged (misaligned runs) lengths, per library build
for lib in paper_2507_13833_b200/lib/libdfx.so $(ls variants/*/libdfx.so 2>/dev/null); do
  for rg in 0 1; do for n in 2 4; do
    DFX_C4_RAGGED=$rg DFX_LIB_PATH=$PWD/$lib timeout 200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2958$n bench.py --workload c4 --gpus $n --transport pull --steps 30 --warmup 5 2>/dev/null | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());print('$lib ragged=$rg N=$n', d['ms_per_step'], d['roofline']['frac'])"
  done; done
done
