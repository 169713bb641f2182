# C4 (bench.py --workload c4, pull transport) at N GPUs under pull-kernel CTA counts (DFX_PULL_CTAS_PER_SM)
N=${N:-4}
for cps in ${CPS:-1 2 3 4}; do
  for rep in 1 2; do
    DFX_PULL_CTAS_PER_SM=$cps timeout 200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29512 bench.py --workload c4 --gpus $N --transport pull --steps 50 --warmup 5 2>/dev/null | tail -1 > /tmp/c4.json
    python -c "import json; d=json.load(open('/tmp/c4.json')); print('N=$N cps=$cps rep $rep', d['ms_per_step'], d['roofline']['achieved'], d['roofline']['frac'])"
  done
done
