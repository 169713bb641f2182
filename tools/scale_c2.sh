# C2 bench.py at N = 1, 2, 4 (weak scaling, box placement; one JSON line each)
for n in ${NS:-1 2 4}; do
  if [ $n = 1 ]; then timeout 300 python bench.py --steps 50 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 > /tmp/s$n.json
  else timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2952$n bench.py --gpus $n --steps 50 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 > /tmp/s$n.json; fi
  python -c "import json; d=json.load(open('/tmp/s$n.json')); print('N=$n', d['value'], d['ms_per_step'], d['roofline']['frac'])"
done
