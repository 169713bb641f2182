"""Per-verb host timing of the native C4 round trip (torchrun, N GPUs): put / ensure_ready / get / worker_done
with a device synchronize after each verb, plus the raw NCCL p2p rate of the same bytes (torch.distributed)."""
import os
import sys
import time

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2507_13833_b200 as dfx  # noqa: E402
from paper_2507_13833_b200.dstore import Comm, NativeBufferStore  # noqa: E402
from paper_2507_13833_b200.reshard import Layout, Topology  # noqa: E402
from paper_2507_13833_b200.store import StoreStagePlan  # noqa: E402

rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(rank)
dev = torch.device("cuda", rank)
dist.init_process_group("gloo")
comm = Comm.create(world, rank)
W = 8 // world
topo = Topology.store_per_gpu(world, W)
to_s, to_t = Layout(4, 2), Layout(8, 1)
stages = {"s": StoreStagePlan(Layout(8, 1), to_s), "t": StoreStagePlan(to_s, to_t)}
R = 1024 // world
batch = dfx.PackedBatch.synthetic(11, R, 16, dfx.TokenDist("constant", 1024), device=dev, first_id=rank * R,
                                  streams=("token_id", "lp", "old_lp", "ref_lp"))
dfx.fn_group_advantage(dfx.NodeSpec("a"), batch, dfx.StageContext())
local_p = [p for p in range(8) if topo.gpu_of_worker[p] == rank]
per = R // len(local_p)
views = [batch.view_records(j * per, (j + 1) * per) for j in range(len(local_p))]
mine_s = [d for d in range(4) if any(topo.gpu_of_worker[d * 2 + t] == rank for t in range(2))]
store = NativeBufferStore(topo, comm, stages, [("token_id", torch.int32), ("lp", torch.float32),
                                               ("old_lp", torch.float32), ("ref_lp", torch.float32)],
                          ["advantage", "reward"])
acc = {}


def T(name, fn):
    torch.cuda.synchronize()
    t = time.perf_counter()
    r = fn()
    torch.cuda.synchronize()
    acc[name] = acc.get(name, 0.0) + time.perf_counter() - t
    return r


for i in range(25):
    if i == 5:
        acc.clear()
    for j, p in enumerate(local_p):
        T("put s", lambda: store.put("s", i, p, 0, views[j]))
    T("ensure s", lambda: store.ensure_ready("s", i, to_s))
    for d in mine_s:
        b = T("get s", lambda: store.get("s", i, d, to_s))
        for t in range(2):
            if topo.gpu_of_worker[d * 2 + t] == rank:
                T("put t", lambda: store.put("t", i, d, t, b))
    T("ensure t", lambda: store.ensure_ready("t", i, to_t))
    for _ in store.local_workers:
        T("done", lambda: store.worker_done(i))
# sizes all-reduce alone
for i in range(25):
    if i == 5:
        acc["allreduce x20"] = 0.0
    T("allreduce x20" if i >= 5 else "warm", lambda: comm.allreduce_i64([1] * 24))
if rank == 0:
    print({k: round(v / 20 * 1e3, 4) for k, v in acc.items()}, "ms per step", flush=True)
    print(store.stats(), flush=True)
# raw NCCL p2p of one stage's bytes (torch's NCCL)
g = dist.new_group(backend="nccl")
n = 67 * 1024 * 1024
sb = torch.empty(n, dtype=torch.uint8, device=dev)
rb = torch.empty(n, dtype=torch.uint8, device=dev)
peer = rank ^ 1
for it in range(6):
    if it == 1:
        torch.cuda.synchronize()
        t = time.perf_counter()
    ops = [dist.P2POp(dist.isend, sb, peer, g), dist.P2POp(dist.irecv, rb, peer, g)]
    for w in dist.batch_isend_irecv(ops):
        w.wait()
torch.cuda.synchronize()
dt = (time.perf_counter() - t) / 5
if rank == 0:
    print(f"torch NCCL p2p 67 MB each way: {dt * 1e3:.3f} ms -> {n / dt / 1e9:.0f} GB/s per direction", flush=True)
store.close()
comm.close()
dist.destroy_process_group()
