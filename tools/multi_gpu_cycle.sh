#!/bin/bash
# Multi-GPU measurement pass (run on a box with >= 4 GPUs): 2-GPU parity tests, then bench.py at N = 1, 2, 4 with
# the default box placement, the N = 8 layout previewed on 4 GPUs (--workers 4: one logical worker per GPU, TP
# partners on different GPUs), and the store-per-GPU placement. JSON lines -> gpurun_out/multi_<tag>_*.json
TAG=${1:-run}
mkdir -p gpurun_out
python paper_2507_13833_b200/build.py > /dev/null || exit 1  # never measure a stale libdfx.so
timeout 600 python -m pytest tests/test_reshard.py -q -x -m gpu -p no:cacheprovider 2>&1 | tail -2
run() {  # name N extra...
  local name=$1 n=$2; shift 2
  if [ "$n" = 1 ]; then
    timeout 300 python bench.py --steps 50 "$@" > gpurun_out/multi_${TAG}_${name}.log 2>&1
  else
    timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
      --master-port $((29500 + RANDOM % 400)) bench.py --gpus $n --steps 50 "$@" > gpurun_out/multi_${TAG}_${name}.log 2>&1
  fi
  grep '^{' gpurun_out/multi_${TAG}_${name}.log | tail -1 > gpurun_out/multi_${TAG}_${name}.json
  python - "$name" gpurun_out/multi_${TAG}_${name}.json <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[2]).read())
    r = d.get("roofline") or {}
    e = d.get("e2e") or {}
    print(sys.argv[1], "value %.4g" % d["value"], "ms %.4f" % d["ms_per_step"], "roof", r.get("bound"), r.get("frac"),
          r.get("kernel_ms"), "e2e %.4g" % (e.get("value") or 0))
except Exception as ex:
    print(sys.argv[1], "FAILED", ex)
PY
}
run n1 1 --no-cpu-baseline
run n2 2
run n4 4
run n4_w4 4 --workers 4
run n2_w2 2 --workers 2
run n4_w4_read 4 --workers 4 --tp-read
run n4_store 4 --placement store
run c4_n1 1 --workload c4 --steps 20
run c4_n2 2 --workload c4 --steps 20
run c4_n4 4 --workload c4 --steps 20
run c5_n4 4 --workload c5 --steps 20
