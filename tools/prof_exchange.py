"""Phase timing of the dense DataBuffer exchange (store-per-GPU placement) under torchrun.

usage: torchrun --nproc-per-node N tools/prof_exchange.py [--records 1024] [--iters 5]
Prints per-rank wall time of put / ensure_ready (split into plan, sizes, alloc+local copies, NCCL, unpack, host
metadata) for the bench's C2 batch.
"""
import argparse

import numpy as np
import os
import sys
import time

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2507_13833_b200 as dfx  # noqa: E402
from paper_2507_13833_b200 import reshard as R  # noqa: E402
from paper_2507_13833_b200.store import DeviceBufferStore, StoreStagePlan  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--records", type=int, default=1024)
ap.add_argument("--iters", type=int, default=5)
ap.add_argument("--transport", default="pull")
ap.add_argument("--placement", default="store")
ap.add_argument("--workers", type=int, default=8)
a = ap.parse_args()
rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(rank)
dev = torch.device("cuda", rank)
dist.init_process_group("nccl", device_id=dev)
meta = dist.new_group(backend="gloo")
b = dfx.PackedBatch.synthetic(1, a.records, 16, dfx.TokenDist("uniform", 0, 1, 4096), device=dev,
                              first_id=rank * a.records)
ctx = dfx.StageContext()
dfx.fn_group_advantage(dfx.NodeSpec("a"), b, ctx)
if a.placement == "box":
    topo = R.Topology.box(a.workers, world)
    prod, cons = R.Layout(a.workers, 1), R.Layout(a.workers // 2, 2)
else:
    wpg = max(2, 8 // world)
    topo = R.Topology.store_per_gpu(world, wpg)
    prod, cons = R.Layout(world * wpg, 1), R.Layout(world * wpg // 2, 2)
st = DeviceBufferStore(topo, rank, {"s": StoreStagePlan(prod, cons)}, meta_group=meta, transport=a.transport)
local_p = [p for p in range(prod.dp) if topo.gpu_of_worker[p] == rank]
per = a.records // len(local_p)

# wrap the phases
orig_p2p, orig_unpack = R._p2p, R._abi.lib().dfx_reshard_unpack
T = {}


def timed(name, fn):
    def w(*args, **kw):
        torch.cuda.synchronize()
        t = time.perf_counter()
        r = fn(*args, **kw)
        torch.cuda.synchronize()
        T[name] = T.get(name, 0) + time.perf_counter() - t
        return r
    return w


R.Plan.__init__ = timed("plan", R.Plan.__init__)
R.PROFILE = T
allocs = []
for it in range(a.iters + 1):
    allocs.append(torch.cuda.memory_stats(dev).get("num_device_alloc", 0))
    if it == 1:
        T.clear()
    torch.cuda.synchronize()
    dist.barrier()
    t0 = time.perf_counter()
    for j, p in enumerate(local_p):
        st.put("s", it, p, 0, b.view_records(j * per, (j + 1) * per))
    cb = st.ensure_ready("s", it, cons)
    torch.cuda.synchronize()
    T["total ensure_ready"] = T.get("total ensure_ready", 0) + time.perf_counter() - t0
    for _ in st.local_workers:
        st.worker_done(it)
print(f"rank {rank} [{a.transport}]: " + ", ".join(f"{k} {1e3 * v / a.iters:.3f} ms" for k, v in T.items()) +
      f" | sent {cb.bytes_sent / 1e6:.1f} MB zero_copy {cb.zero_copy} | cudaMalloc per iter {list(np.diff(allocs))}",
      flush=True)
dist.destroy_process_group()
