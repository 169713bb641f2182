"""torchrun worker (2 or 4 GPUs): a lazy reshard where some GPUs are zero-copy and the others read a peer.

Box placement, one logical worker per GPU: producer dp N/2 (tp 2) -> consumer dp N (tp 1). Producer group p lives
on GPU 2p; consumer group d on GPU d takes half of a producer group's records: even GPUs find theirs in their
own producer batch (zero-copy view), odd GPUs map their partner's batch (CUDA IPC) and the loss kernel reads it
over NVLink. Several iterations run over the SAME producer batches, so the store's template path is taken -- by
every rank alike (a rank that took the zero-copy path used to re-enter the table all-gather while the
others only issued barriers, and deadlocked) -- with an unrelated collective between ensure_ready and
worker_done (it used to be misordered against the zero-copy ranks' early second barrier). Every consumer group's
loss is checked against the CPU ORACLE on its records (plain 1e-5 relative), and the peer mappings are closed
when the store retires them.
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
from paper_2507_13833_b200.reshard import Layout, RemoteSource, Topology, _declare  # noqa: E402
from paper_2507_13833_b200.store import DeviceBufferStore, StoreStagePlan  # noqa: E402
from tests.helpers import assert_rel  # noqa: E402

rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(rank)
dev = torch.device("cuda", rank)
dist.init_process_group("nccl", device_id=dev)
meta = dist.new_group(backend="gloo")
R, n, seed = 64, 4, 21
dp_p, dp_c = world // 2, world
topo = Topology.box(world, world)
schema = ({"lp": torch.float32, "old_lp": torch.float32, "ref_lp": torch.float32, "mask": torch.uint8},
          ["reward", "value", "advantage"])  # odd GPUs hold no producer group
store = DeviceBufferStore(topo, rank, {"s": StoreStagePlan(Layout(dp_p, 2), Layout(dp_c, 1))}, meta_group=meta,
                          schema=schema)
p_mine = rank // 2 if rank % 2 == 0 else None  # producer group led by this GPU's worker (tp 0), if any
b = None
if p_mine is not None:
    b = dfx.PackedBatch.synthetic(seed, R, n, dfx.TokenDist("skewed", 0, 1, 3000), device=dev, first_id=p_mine * R)
ctx = dfx.StageContext()
# the oracle: every record of the global batch, in producer order; consumer d gets records [d*R/2, (d+1)*R/2)
sb = O.SynthBatch(seed, R * dp_p, n, O.token_dist("skewed", 0, 1, 3000))
adv = O.grpo_advantage(sb.group_off, sb.reward, 1e-6)
adv_tok = O.broadcast_advantage(sb.cu_seqlens, adv, sb.mask)
d = rank
s0, s1 = d * (R // 2) * n, (d + 1) * (R // 2) * n
want, _ = O.ppo_loss(np.ascontiguousarray(sb.cu_seqlens[s0:s1 + 1]), sb.lp, sb.old_lp, sb.ref_lp, adv_tok, sb.mask,
                     O.loss_cfg())
L = _declare()
results = []
for it in range(4):
    if b is not None:
        dfx.fn_group_advantage(dfx.NodeSpec("adv"), b, ctx)
        store.put("s", it, p_mine, 0, b)  # the TP-0 worker puts (tp 1 lives on the odd GPU and would be suppressed)
    cb = store.ensure_ready("s", it, Layout(dp_c, 1), lazy=True)
    assert cb.groups == [d]
    if rank % 2 == 0:
        assert cb.zero_copy and cb.sources is None
        out = dfx.ppo_loss(cb.batch, ctx, adv_source="rollout", loss_group_off=cb.roll_off)["out"]
    else:
        assert cb.sources is not None and all(isinstance(x, RemoteSource) for x in cb.sources[0])
        out = dfx.ppo_loss_sources(cb.sources[0], ctx, loss_group_off=cb.roll_off, device=dev)["out"]
    # an unrelated collective on the default group between the exchange and worker_done
    tot = out[:, 5].clone()
    dist.all_reduce(tot)
    store.worker_done(it)
    got = out.cpu().numpy()[0]
    assert got[5] == want["n_tokens"] and got[6] == want["n_seqs"], (rank, it, got, want)
    for k, j in (("loss", 0), ("pg_loss", 1), ("kl", 2), ("clipfrac", 3), ("approx_kl", 4)):
        assert_rel(got[j], want[k], f"{k} rank {rank} it {it}")
    assert tot.item() == float(sb.mask[:sb.n_tokens].sum()), (tot.item(), rank)
    results.append(got.tobytes())
assert all(r == results[0] for r in results), "iterations over the same producer batches must give the same bits"
assert store.template_hits == 3, store.template_hits
torch.cuda.synchronize()
opened = L.dfx_ipc_open_count()
assert (opened > 0) == (rank % 2 == 1), (rank, opened)  # only the odd GPUs map a peer
# new producer batches (fresh memory; the old ones are kept alive so the allocations differ): each replaces the
# stage's template, and the replaced template's mappings close at worker_done -- the count does not grow
keep = []
for it in range(10, 13):
    if b is not None:
        keep.append(b)
        b = dfx.PackedBatch.synthetic(seed, R, n, dfx.TokenDist("skewed", 0, 1, 3000), device=dev,
                                      first_id=p_mine * R)
        dfx.fn_group_advantage(dfx.NodeSpec("adv"), b, ctx)
        store.put("s", it, p_mine, 0, b)
    cb = store.ensure_ready("s", it, Layout(dp_c, 1), lazy=True)
    store.worker_done(it)
    torch.cuda.synchronize()
    live = set(store._templates["s"][1].ipc_bases or [])  # the mappings the current template may replay
    assert L.dfx_ipc_open_count() == len(live), (rank, it, L.dfx_ipc_open_count(), len(live))
dist.barrier()
print(f"rank {rank}: loss {results and np.frombuffer(results[0])[0]:.9f} == oracle {want['loss']:.9f}; "
      f"mappings {opened} -> {L.dfx_ipc_open_count()}", flush=True)
print("MIXED_OK", flush=True)
dist.destroy_process_group()
