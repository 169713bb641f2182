"""torchrun worker (2 GPUs): the lazy reshard + fused multi-source loss == materialize-then-loss.

Box placement with W = 2 logical workers on 2 GPUs: producer dp 2 (tp 1), consumer dp 1 (tp 2), so the one
consumer group's TP workers sit on different GPUs and each GPU needs its partner's producer group. The lazy path
maps the partner's batch (CUDA IPC) and the loss kernel reads it over NVLink in place; the reference path pulls it
into a local consumer batch first; the TP-split path streams only the local group and folds the two loss rows
(all-gather + dfx_loss_combine). Losses must agree to f32 partial-sum rounding (the slot windows differ), per-token
advantages bit-exactly.
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
from tests.helpers import assert_rel  # noqa: E402
from paper_2507_13833_b200.reshard import Layout, RemoteSource, Topology  # noqa: E402
from paper_2507_13833_b200.store import DeviceBufferStore, StoreStagePlan  # noqa: E402

rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(rank)
dev = torch.device("cuda", rank)
dist.init_process_group("nccl", device_id=dev)
meta = dist.new_group(backend="gloo")
R = 48
for it, (dist_kind, hi) in enumerate((("uniform", 700), ("skewed", 3000), ("uniform", 37))):
    b = dfx.PackedBatch.synthetic(5 + it, R, 4, dfx.TokenDist(dist_kind, 0, 1, hi), device=dev, first_id=rank * R)
    ctx = dfx.StageContext()
    dfx.fn_group_advantage(dfx.NodeSpec("adv"), b, ctx)
    topo = Topology.box(2, world)
    plan = {"s": StoreStagePlan(Layout(2, 1), Layout(1, 2))}
    lazy_store = DeviceBufferStore(topo, rank, plan, meta_group=meta)
    ref_store = DeviceBufferStore(topo, rank, plan, meta_group=meta)
    lazy_store.put("s", it, rank, 0, b)
    ref_store.put("s", it, rank, 0, b)
    cb = lazy_store.ensure_ready("s", it, Layout(1, 2), lazy=True)
    assert cb.sources is not None and len(cb.sources) == 1
    srcs = cb.sources[0]
    assert [isinstance(x, RemoteSource) for x in srcs] == [rank == 1, rank == 0], srcs
    res = dfx.ppo_loss_sources(srcs, ctx, loss_group_off=cb.roll_off, adv_tok_out=True, device=dev)
    got = res["out"].cpu().numpy()[0]
    # TP-split: each GPU streams only its own producer group, the pair folds the loss rows (all-gather + combine)
    mine = [x for x in srcs if isinstance(x, dfx.PackedBatch)]
    part = dfx.ppo_loss(mine[0], ctx, adv_source="rollout")["out"]
    split = dfx.tp_combine_loss(part, ctx, None)
    both = [torch.empty_like(split) for _ in range(world)]
    dist.all_gather(both, split)
    assert all(b_.cpu().numpy().tobytes() == split.cpu().numpy().tobytes() for b_ in both)  # same bits everywhere
    split = split.cpu().numpy()[0]
    lazy_store.worker_done(it)
    rb = ref_store.ensure_ready("s", it, Layout(1, 2))
    ref = dfx.ppo_loss(rb.batch, dfx.StageContext(), adv_source="rollout", adv_tok_out=True)
    want = ref["out"].cpu().numpy()[0]
    assert got[5] == want[5] and got[6] == want[6], (got, want)  # token / sequence counts exact
    # f32 partial sums over different slot windows (each source keeps its own token coordinates): f32 rounding
    np.testing.assert_allclose(got[:5], want[:5], rtol=2e-6, atol=1e-9)
    assert split[5] == want[5] and split[6] == want[6], (split, want)
    np.testing.assert_allclose(split[:5], want[:5], rtol=2e-6, atol=1e-9)
    # and all three against the CPU ORACLE on the consumer group's records (both producer groups, in order)
    sb = O.SynthBatch(5 + it, world * R, 4, O.token_dist(dist_kind, 0, 1, hi))
    adv_o = O.grpo_advantage(sb.group_off, sb.reward, 1e-6)
    ref_o, _ = O.ppo_loss(sb.cu_seqlens, sb.lp, sb.old_lp, sb.ref_lp,
                          O.broadcast_advantage(sb.cu_seqlens, adv_o, sb.mask), sb.mask, O.loss_cfg())
    for name, row in (("lazy multi-source", got), ("tp-split fold", split), ("materialized", want)):
        assert row[5] == ref_o["n_tokens"] and row[6] == ref_o["n_seqs"], (name, row, ref_o)
        for k, j in (("loss", 0), ("pg_loss", 1), ("kl", 2), ("clipfrac", 3), ("approx_kl", 4)):
            assert_rel(row[j], ref_o[k], f"{k} {name} case {it} rank {rank}")
    # per-token advantages: source k's tokens land at the consumer's cumulative token offset
    want_tok = ref["adv_tok"].cpu().numpy()
    off = 0
    for x, buf in zip(srcs, res["adv_tok"]):
        a0 = x.token_base & ~3
        gt = buf.cpu().numpy()[x.token_base - a0: x.token_base - a0 + x.token_span]
        assert gt.tobytes() == want_tok[off: off + x.token_span].tobytes(), (it, rank)
        off += x.token_span
    # the next iteration over the same producer batches reuses the mapping (no table exchange): same result
    dfx.fn_group_advantage(dfx.NodeSpec("adv"), b, ctx)
    lazy_store.put("s", it + 100, rank, 0, b)
    cb2 = lazy_store.ensure_ready("s", it + 100, Layout(1, 2), lazy=True)
    assert lazy_store.template_hits == 1 and cb2.sources is cb.sources
    again = dfx.ppo_loss_sources(cb2.sources[0], ctx, loss_group_off=cb2.roll_off, device=dev)["out"]
    assert again.cpu().numpy().tobytes() == res["out"].cpu().numpy().tobytes()
    lazy_store.worker_done(it + 100)
    print(f"rank {rank} case {it}: loss {got[0]:.9f} == {want[0]:.9f}, {int(got[5])} tokens", flush=True)
# performance guard: the multi-source loss reading the partner's group over NVLink must run at NVLink speed (a
# per-lane L2 prefetch of peer-mapped memory once slowed it 50x while every numeric check above still passed)
big = dfx.PackedBatch.synthetic(9, 256, 16, dfx.TokenDist("uniform", 0, 1, 4096), device=dev, first_id=rank * 256)
ctx = dfx.StageContext()
dfx.fn_group_advantage(dfx.NodeSpec("adv"), big, ctx)
store = DeviceBufferStore(Topology.box(2, world), rank, {"s": StoreStagePlan(Layout(2, 1), Layout(1, 2))},
                          meta_group=meta)
store.put("s", 500, rank, 0, big)
cb = store.ensure_ready("s", 500, Layout(1, 2), lazy=True)
srcs = cb.sources[0]
remote = [x for x in srcs if isinstance(x, RemoteSource)][0]
run = lambda: dfx.ppo_loss_sources(srcs, ctx, loss_group_off=cb.roll_off, device=dev)  # noqa: E731
run()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(5):
    run()
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 5
gbs = remote.token_span * 13 / (ms / 1e3) / 1e9  # lp, old, ref (f32) + mask (u8) of the partner's tokens
print(f"rank {rank}: multi-source loss {ms:.3f} ms, partner tokens read at {gbs:.0f} GB/s over NVLink", flush=True)
assert gbs > 100, f"multi-source NVLink loss too slow: {gbs:.1f} GB/s"
store.worker_done(500)
dist.barrier()
print("LAZY_OK", flush=True)
dist.destroy_process_group()
