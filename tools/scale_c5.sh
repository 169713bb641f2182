# C5 (BASELINE config 5: 4096 prompts x 16 x skewed <=16k tokens split over the GPUs; strong scaling) at N = 1, 2, 4
for n in ${NS:-1 2 4}; do
  if [ $n = 1 ]; then timeout 300 python bench.py --workload c5 --steps 30 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 > /tmp/c5_$n.json
  else timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2954$n bench.py --workload c5 --gpus $n --steps 30 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 > /tmp/c5_$n.json; fi
  python -c "import json; d=json.load(open('/tmp/c5_$n.json')); print('C5 N=$n', d['value'], d['ms_per_step'], d['roofline']['frac'], d['config'].get('parallelism'))"
done
