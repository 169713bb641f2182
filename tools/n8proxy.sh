# the N=8 path previewed on 4 GPUs (--workers 4: TP partners on different GPUs, multi-source NVLink loss)
for lib in paper_2507_13833_b200/lib/libdfx.so $(ls variants/*/libdfx.so 2>/dev/null); do
  DFX_LIB_PATH=$PWD/$lib timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29532 bench.py --gpus 4 --workers 4 --steps 20 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());print('$lib', d['ms_per_step'], d['roofline']['kernel_ms'], d['roofline']['frac'])"
done
