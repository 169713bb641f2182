# C4 through the C++ host (cpp/bench_dstore) with the per-phase device trace
N=${N:-2}
for v in "DFX_PULL_CTAS_PER_SM=2" "DFX_PULL_CTAS_PER_SM=1" "DFX_PULL_CTAS_PER_SM=3"; do
  echo "[$v] $(env $v DFX_DSTORE_TRACE=1 timeout 120 ./cpp/_build/bench_dstore $N 50 5 pull 2>/tmp/tr.txt | cut -c1-260)"
  grep "rank 0" /tmp/tr.txt
done
for tr in pull nccl; do
timeout 200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29511 bench.py --workload c4 --gpus $N --transport $tr --steps 50 --warmup 5 2>/dev/null | tail -1 | cut -c 1-400
done
