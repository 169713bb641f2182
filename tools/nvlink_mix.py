"""NVLink microbenchmark for the lazy reshard (2 ranks, both reading their partner at once): the multi-source loss
kernel reading the partner's producer group in place vs copy-engine pulls of the same bytes, alone and together.

usage: torchrun --nproc-per-node 2 tools/nvlink_mix.py
"""
import ctypes as C
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2507_13833_b200 as dfx  # noqa: E402
from paper_2507_13833_b200 import _abi  # noqa: E402
from paper_2507_13833_b200.reshard import Layout, RemoteSource, Topology  # noqa: E402
from paper_2507_13833_b200.store import DeviceBufferStore, StoreStagePlan  # noqa: E402

rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(rank)
dev = torch.device("cuda", rank)
dist.init_process_group("nccl", device_id=dev)
meta = dist.new_group(backend="gloo")
b = dfx.PackedBatch.synthetic(1, 1024, 16, dfx.TokenDist("uniform", 0, 1, 4096), device=dev, first_id=rank * 1024)
ctx = dfx.StageContext()
dfx.fn_group_advantage(dfx.NodeSpec("a"), b, ctx)
store = DeviceBufferStore(Topology.box(2, 2), rank, {"s": StoreStagePlan(Layout(2, 1), Layout(1, 2))}, meta_group=meta)
store.put("s", 0, rank, 0, b)
cb = store.ensure_ready("s", 0, Layout(1, 2), lazy=True)
srcs = cb.sources[0]
remote = [x for x in srcs if isinstance(x, RemoteSource)][0]
local = [x for x in srcs if not isinstance(x, RemoteSource)][0]
L = _abi.lib()
names = ("lp", "old_lp", "ref_lp", "mask")
bufs = {k: torch.empty(remote.token_span + 16, dtype=b.streams[k].dtype, device=dev) for k in names}
side = torch.cuda.Stream(dev)
nbytes = sum(remote.token_span * bufs[k].element_size() for k in names)


def pull(st):
    for k in names:
        esz = bufs[k].element_size()
        _abi.check(L.dfx_copy_async(C.c_void_p(bufs[k].data_ptr()), C.c_void_p(remote.addr["s:" + k] + remote.token_base * esz),
                                    remote.token_span * esz, C.c_void_p(st.cuda_stream)))


def timeit(fn, iters=10):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / iters


def both():
    side.wait_stream(torch.cuda.current_stream())
    pull(side)
    dfx.ppo_loss_sources([local], ctx, device=dev)
    torch.cuda.current_stream().wait_stream(side)


def sm_and_ce():
    """the loss kernel reads the remote run over NVLink while the copy engines pull the same bytes again"""
    side.wait_stream(torch.cuda.current_stream())
    pull(side)
    dfx.ppo_loss_sources([remote], ctx, device=dev)
    torch.cuda.current_stream().wait_stream(side)


res = {
    "sm_read_plus_ce_pull_ms": timeit(sm_and_ce),
    "loss_local+remote_ms": timeit(lambda: dfx.ppo_loss_sources(srcs, ctx, device=dev)),
    "loss_remote_only_ms": timeit(lambda: dfx.ppo_loss_sources([remote], ctx, device=dev)),
    "loss_local_only_ms": timeit(lambda: dfx.ppo_loss_sources([local], ctx, device=dev)),
    "ce_pull_ms": timeit(lambda: pull(torch.cuda.current_stream())),
    "ce_pull_with_local_loss_ms": timeit(both),
}
res["remote_MB"] = nbytes / 1e6
res["sm_read_GBs"] = nbytes / res["loss_remote_only_ms"] / 1e6
res["ce_GBs"] = nbytes / res["ce_pull_ms"] / 1e6
res["sm_plus_ce_GBs"] = 2 * nbytes / res["sm_read_plus_ce_pull_ms"] / 1e6
print(rank, {k: round(v, 4) for k, v in res.items()}, flush=True)
store.worker_done(0)
dist.barrier()
dist.destroy_process_group()
