"""torchrun worker (1, 2 or 4 GPUs): the NATIVE distributed DataBuffer (libdfx dfx_dstore_*, one process per GPU;
both transports: CUDA-IPC pulls by the copy engines, and NCCL send/recv) == the reference BufferStore, byte for byte.

For the golden configurations of tests/golden/blobs.npz (made by the compiled reference, tests/golden/make_golden.py)
every rank puts the producer groups its logical workers own, runs ensure_ready / get through the C ABI and
serializes each destination group in the reference blob format; three iterations over the same producer batches
(the plan cache path) and one with different producer batches. Then the round trip of a second stage (the consumer
groups put back, consumed at the producer layout) must give the original records.
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
from paper_2507_13833_b200.dstore import Comm, NativeBufferStore  # noqa: E402
from paper_2507_13833_b200.reshard import Layout, Topology  # noqa: E402
from paper_2507_13833_b200.store import StoreStagePlan  # noqa: E402
from tests.test_reshard import _blob_of  # noqa: E402

rank, world = int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1"))
torch.cuda.set_device(rank)
dev = torch.device("cuda", rank)
if world > 1:
    dist.init_process_group("gloo")  # setup only: carries the NCCL id bytes
comm = Comm.create(world, rank)
g = np.load(os.path.join(ROOT, "tests", "golden", "blobs.npz"))
STREAMS = [("token_id", torch.int32), ("lp", torch.float32), ("old_lp", torch.float32), ("ref_lp", torch.float32),
           ("mask", torch.uint8)]
sb = O.SynthBatch(7, 16, 2, O.token_dist("uniform", 0, 16, 48), streams=("token_id", "lp", "old_lp", "ref_lp", "mask"))
T = sb.n_tokens
full = dfx.PackedBatch.from_host(sb.ids, sb.group_off, sb.cu_seqlens, {"reward": sb.reward},
                                 {k: getattr(sb, k)[:T] for k, _ in STREAMS}, device=dev)
dfx.fn_group_advantage(dfx.NodeSpec("adv"), full, dfx.StageContext())
names = ["small", "cross", "dense"]
for transport, name in [(tr, nm) for tr in ("pull", "nccl") for nm in names]:
    B, W, dp_p, tp_p, dp_c, tp_c = (int(x) for x in g[f"{name}_cfg"])
    if (B * W) % world:
        continue
    topo = Topology(B, W, tuple(w * world // (B * W) for w in range(B * W)))
    stages = {"s": StoreStagePlan(Layout(dp_p, tp_p), Layout(dp_c, tp_c)),
              "t": StoreStagePlan(Layout(dp_c, tp_c), Layout(dp_p, tp_p))}
    store = NativeBufferStore(topo, comm, stages, STREAMS, ["advantage", "reward"], transport=transport)
    per = 16 // dp_p
    views = [full.view_records(p * per, (p + 1) * per) for p in range(dp_p)]
    for it in range(4):
        src = views if it < 3 else [full.view_records(p * per, (p + 1) * per) for p in range(dp_p)]  # new batches
        for p in range(dp_p):
            for t in range(tp_p):
                w = p * tp_p + t
                if topo.gpu_of_worker[w] == rank:
                    store.put("s", it, p, t, src[p])
        store.ensure_ready("s", it, Layout(dp_c, tp_c))
        mine = [d for d in range(dp_c) if any(topo.gpu_of_worker[d * tp_c + t] == rank for t in range(tp_c))]
        got = {}
        for d in mine:
            b = store.get("s", it, d, Layout(dp_c, tp_c))
            got[d] = b
            blob = _blob_of(O, b, 0, b.n_records)
            assert blob.tobytes() == g[f"{name}_blob_{d}"].tobytes(), (name, rank, d, it)
            assert b.n_records == int(g[f"{name}_counts"][d])
            assert list(b.host_cu) == list(b.cu_seqlens.cpu().numpy())
            # the group's records feed the loss kernels directly
            ctx = dfx.StageContext()
            out = dfx.ppo_loss(b, ctx, adv_source="rollout")["out"].cpu().numpy()[0]
            assert out[6] == b.n_rollouts or out[6] <= b.n_rollouts
        # round trip: every consumer group's TP-0 worker puts it back, consumed at the producer layout
        for d in mine:
            for t in range(tp_c):
                w = d * tp_c + t
                if topo.gpu_of_worker[w] == rank:
                    store.put("t", it, d, t, got[d])
        store.ensure_ready("t", it, Layout(dp_p, tp_p))
        for p in range(dp_p):
            if any(topo.gpu_of_worker[p * tp_p + t] == rank for t in range(tp_p)):
                back = store.get("t", it, p, Layout(dp_p, tp_p))
                want = _blob_of(O, full, p * per, (p + 1) * per)
                assert _blob_of(O, back, 0, back.n_records).tobytes() == want.tobytes(), (name, rank, p, it)
        torch.cuda.synchronize()
        for w in range(topo.world):
            if topo.gpu_of_worker[w] == rank:
                store.worker_done(it)
    st = store.stats()
    assert st["plan_hits"] >= 4, st  # iterations 1..3 reuse the plans of both stages
    print(f"rank {rank} {name}/{transport}: {st}", flush=True)
    store.close()
comm.close()
if world > 1:
    dist.barrier()
    dist.destroy_process_group()
print("DSTORE_OK", flush=True)
