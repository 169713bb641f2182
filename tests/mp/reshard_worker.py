"""torchrun worker (2 GPUs): device reshard over NCCL P2P == the reference BufferStore, byte for byte.

Each rank holds the producer groups its logical workers own (store per GPU: B = 2 nodes x W = 2 workers for the
"dense" fixture; B = 2 x W = 4 for "cross"), runs the DeviceBufferStore put -> ensure_ready -> get, serializes its
destination groups in the reference blob format and compares them with tests/golden/blobs.npz.
"""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import paper_2507_13833_b200 as dfx  # noqa: E402
from oracle import oracle as O  # noqa: E402
from paper_2507_13833_b200.reshard import Layout, Topology  # noqa: E402
from paper_2507_13833_b200.store import DeviceBufferStore, StoreStagePlan  # noqa: E402
from tests.test_reshard import _blob_of  # noqa: E402

rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(rank)
dev = torch.device("cuda", rank)
dist.init_process_group("nccl", device_id=dev)
meta = dist.new_group(backend="gloo")
g = np.load(os.path.join(ROOT, "tests", "golden", "blobs.npz"))
sb = O.SynthBatch(7, 16, 2, O.token_dist("uniform", 0, 16, 48), streams=("token_id", "lp", "old_lp", "ref_lp", "mask"))
T = sb.n_tokens
full = dfx.PackedBatch.from_host(sb.ids, sb.group_off, sb.cu_seqlens, {"reward": sb.reward},
                                 {k: getattr(sb, k)[:T] for k in ("token_id", "lp", "old_lp", "ref_lp", "mask")},
                                 device=dev)
dfx.fn_group_advantage(dfx.NodeSpec("adv"), full, dfx.StageContext())
for name, transport in (("dense", "pull"), ("cross", "pull"), ("dense", "nccl"), ("cross", "nccl")):
    B, W, dp_p, tp_p, dp_c, tp_c = (int(x) for x in g[f"{name}_cfg"])
    topo = Topology.store_per_gpu(world, W) if B == world else Topology(B, W, tuple(w * world // (B * W)
                                                                                   for w in range(B * W)))
    store = DeviceBufferStore(topo, rank, {"s": StoreStagePlan(Layout(dp_p, tp_p), Layout(dp_c, tp_c))},
                              meta_group=meta, transport=transport)
    per = 16 // dp_p
    for it in range(2):  # iteration 1 reuses the exchange template of iteration 0 (same producer batches)
        for p in range(dp_p):
            for t in range(tp_p):
                w = p * tp_p + t
                if topo.gpu_of_worker[w] == rank:
                    store.put("s", it, p, t, full.view_records(p * per, (p + 1) * per))
        cb = store.ensure_ready("s", it, Layout(dp_c, tp_c))
        torch.cuda.synchronize()
        for i, d in enumerate(cb.groups):
            got = store.get("s", it, d, Layout(dp_c, tp_c))
            blob = _blob_of(O, cb.batch, cb.rec_off[i], cb.rec_off[i + 1])
            assert blob.tobytes() == g[f"{name}_blob_{d}"].tobytes(), (name, rank, d, it)
            assert got.n_records == int(g[f"{name}_counts"][d])
            assert got.host_cu is None or list(got.host_cu) == list(got.cu_seqlens.cpu().numpy())
        for w in range(topo.world):
            if topo.gpu_of_worker[w] == rank:
                store.worker_done(it)
    if transport == "pull" and cb.groups and not cb.zero_copy:
        assert sum(t.get("hits", 0) for t in store._mat_templates.values()) == 1, name
    assert store.bytes_sent > 0 or not cb.groups, name
    print(f"rank {rank} {name}/{transport}: dests {cb.groups} sent {store.bytes_sent} recv {store.bytes_recv} zero_copy "
          f"{cb.zero_copy}", flush=True)
dist.barrier()
print("RESHARD_OK", flush=True)
dist.destroy_process_group()
