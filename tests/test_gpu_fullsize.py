"""Parity at BASELINE.json's full sizes: the CUDA path against the CPU oracle on the configurations the bench and the
measurements run (not scaled-down shapes).

- C2 (1024 prompts x 16 x UNIFORM[1,4096], ~33.5M tokens) along the bench's exact path: fn_group_advantage ->
  DeviceBufferStore put / ensure_ready (dp8 -> dp4 tp2, box placement) -> ppo_loss with adv_source="rollout",
  the 4 consumer groups as loss groups and adv_tok_out;
- C3 (512 x 8192 PPO): GAE (gamma 1, lambda 0.95) with whitening, then the whitened clipped loss on the per-token
  advantages; GAE outputs bit-identical run to run;
- C5's per-GPU share (4096 x 16 x skewed[1,16384] over 8 GPUs -> 512 prompts per GPU), first and last rank;
- the multi-source loss and the TP-split fold of record pieces, against the oracle on the whole batch.

Loss scalars: plain relative error <= 1e-5 (tests/helpers.assert_rel; achieved errors printed at session end).
Advantages, broadcasts, counts: bit-exact. GAE per-token outputs: the per-token tolerance of tests/helpers.py.
"""
from __future__ import annotations

import ctypes as C

import numpy as np
import pytest
import torch

from tests.helpers import assert_close_vec, assert_rel

pytestmark = pytest.mark.gpu

SCALARS = ("loss", "pg_loss", "kl", "clipfrac", "approx_kl")


def _check_loss(got_row, ref: dict, what: str):
    got = dict(zip(("loss", "pg_loss", "kl", "clipfrac", "approx_kl", "n_tokens", "n_seqs"),
                   np.asarray(got_row, np.float64).tolist()))
    assert got["n_tokens"] == ref["n_tokens"] and got["n_seqs"] == ref["n_seqs"], (what, got, ref)
    for k in SCALARS:
        assert_rel(got[k], ref[k], f"{k} {what}")


def _device_equals_host(db, sb, names):
    T = sb.n_tokens
    assert db.host_cu.tolist() == sb.cu_seqlens.tolist()
    for k in names:
        assert db.streams[k][:T].cpu().numpy().tobytes() == getattr(sb, k)[:T].tobytes(), k


def test_c2_bench_path_full_size(O, dfx):
    """C2 at full size through bench.py's own step (DagSlice at N=1): bit-exact advantages and broadcast, every
    consumer group's loss scalars within 1e-5 relative of the f64 oracle."""
    import bench
    from paper_2507_13833_b200.reshard import Layout, Topology
    from paper_2507_13833_b200.store import DeviceBufferStore, StoreStagePlan

    c2 = bench.C2
    R, n = c2["records"], c2["n_roll"]
    sb = O.SynthBatch(c2["seed"], R, n, O.token_dist(*c2["dist"]))
    dev = torch.device("cuda", 0)
    db = dfx.PackedBatch.synthetic(c2["seed"], R, n, dfx.TokenDist(*c2["dist"]), device=dev)
    _device_equals_host(db, sb, ("lp", "old_lp", "ref_lp", "mask"))
    ctx = dfx.StageContext()
    ctx.loss = dfx.LossConfig(kl="k3", agg="token-mean")
    resh = bench.DagSlice(dfx, 1, 0, R, ctx, Layout, Topology, DeviceBufferStore, StoreStagePlan, "box", 8,
                          lazy=True, dev=dev, tp_split=True)
    res, consumer = resh.step(db)
    torch.cuda.synchronize()
    lgo = resh.last.roll_off
    assert len(lgo) == 5, lgo  # dp8 -> dp4: 4 consumer groups on this GPU, one loss group each

    adv = O.grpo_advantage(sb.group_off, sb.reward, 1e-6)
    assert db.channels["advantage"].cpu().numpy().tobytes() == adv.tobytes()
    adv_tok = O.broadcast_advantage(sb.cu_seqlens, adv, sb.mask)
    T = sb.n_tokens
    assert res["adv_tok"][:T].cpu().numpy().tobytes() == adv_tok[:T].tobytes()
    out = res["out"].cpu().numpy()
    cfg = O.loss_cfg(kl="k3", agg="token-mean")
    for g in range(4):
        cu = np.ascontiguousarray(sb.cu_seqlens[lgo[g]:lgo[g + 1] + 1])
        ref, _ = O.ppo_loss(cu, sb.lp, sb.old_lp, sb.ref_lp, adv_tok, sb.mask, cfg)
        _check_loss(out[g], ref, f"C2 group {g}")
    # and the whole batch as one loss group, every aggregation
    for agg in ("token-mean", "seq-mean-token-mean", "seq-mean-token-sum"):
        ctx.loss = dfx.LossConfig(kl="k3", agg=agg)
        whole = dfx.ppo_loss(db, ctx, adv_source="rollout")["out"].cpu().numpy()[0]
        ref, _ = O.ppo_loss(sb.cu_seqlens, sb.lp, sb.old_lp, sb.ref_lp, adv_tok, sb.mask,
                            O.loss_cfg(kl="k3", agg=agg))
        _check_loss(whole, ref, f"C2 whole {agg}")


def test_c3_gae_whitened_loss_full_size(O, dfx):
    """C3 (512 x 8192): GAE + whitening sums vs the f64 oracle, bit-identical on a second run, then the whitened
    clipped loss + k3 KL on the per-token advantages."""
    R, L = 512, 8192
    streams = ("lp", "old_lp", "ref_lp", "mask", "value_tok", "token_reward")
    sb = O.SynthBatch(1, R, 1, O.token_dist("constant", L, L, L), streams=streams)
    db = dfx.PackedBatch.synthetic(1, R, 1, dfx.TokenDist("constant", L, L, L), streams=streams)
    _device_equals_host(db, sb, streams)
    ctx = dfx.StageContext(gae_gamma=1.0, gae_lambda=0.95)
    ctx.loss = dfx.LossConfig(kl="k3", agg="token-mean", whiten=True)
    dfx.fn_gae_advantage(dfx.NodeSpec("advantage_compute"), db, ctx)
    a1 = db.streams["advantage"].clone()
    r1 = db.streams["returns"].clone()
    w1 = db.channels["_whiten_sums"].clone()
    dfx.fn_gae_advantage(dfx.NodeSpec("advantage_compute"), db, ctx)
    T = sb.n_tokens
    assert torch.equal(a1[:T], db.streams["advantage"][:T]) and torch.equal(r1[:T], db.streams["returns"][:T])
    assert torch.equal(w1, db.channels["_whiten_sums"])
    A, Rt, ws = O.gae(sb.cu_seqlens, sb.token_reward, sb.value_tok, sb.mask, 1.0, 0.95)
    got_a = a1[:T].cpu().numpy()
    assert_close_vec(got_a, A[:T], "C3 gae adv")
    assert_close_vec(r1[:T].cpu().numpy(), Rt[:T], "C3 gae ret")
    wsg = w1.cpu().numpy()
    assert wsg[2] == ws[2]
    assert_rel(wsg[0], ws[0], "whiten_sum_A C3")
    assert_rel(wsg[1], ws[1], "whiten_sum_A2 C3")
    res = dfx.ppo_loss(db, ctx, adv_source="token")
    out = res["out"].cpu().numpy()[0]
    cfg = O.loss_cfg(kl="k3", agg="token-mean", whiten=True)
    # the loss consumes the stored f32 advantages; check against the oracle on those, and on the oracle's own
    # f64 GAE rounded to f32 once (the whole chain)
    ref, _ = O.ppo_loss(sb.cu_seqlens, sb.lp, sb.old_lp, sb.ref_lp, np.ascontiguousarray(got_a), sb.mask, cfg)
    _check_loss(out, ref, "C3 whitened loss")
    ref2, _ = O.ppo_loss(sb.cu_seqlens, sb.lp, sb.old_lp, sb.ref_lp, A[:T].astype(np.float32), sb.mask, cfg)
    _check_loss(out, ref2, "C3 whitened loss (oracle GAE)")


@pytest.mark.parametrize("rank", [0, 7])
def test_c5_share_full_size(O, dfx, rank):
    """C5's per-GPU share (512 prompts x 16 x skewed[1,16384], ids rank*512..): fused GRPO advantage + loss."""
    R = 4096 // 8
    sb = O.SynthBatch(11, R, 16, O.token_dist("skewed", 0, 1, 16384), first_id=rank * R)
    db = dfx.PackedBatch.synthetic(11, R, 16, dfx.TokenDist("skewed", 0, 1, 16384), first_id=rank * R)
    _device_equals_host(db, sb, ("lp", "old_lp", "ref_lp", "mask"))
    ctx = dfx.StageContext()
    res = dfx.ppo_loss(db, ctx, adv_source="group", adv_tok_out=True)
    adv = O.grpo_advantage(sb.group_off, sb.reward, 1e-6)
    assert db.channels["advantage"].cpu().numpy().tobytes() == adv.tobytes()
    adv_tok = O.broadcast_advantage(sb.cu_seqlens, adv, sb.mask)
    T = sb.n_tokens
    assert res["adv_tok"][:T].cpu().numpy().tobytes() == adv_tok[:T].tobytes()
    ref, _ = O.ppo_loss(sb.cu_seqlens, sb.lp, sb.old_lp, sb.ref_lp, adv_tok, sb.mask, O.loss_cfg())
    _check_loss(res["out"].cpu().numpy()[0], ref, f"C5 share rank {rank}")


@pytest.mark.parametrize("agg", ["token-mean", "seq-mean-token-mean", "seq-mean-token-sum"])
def test_multi_source_and_fold_vs_oracle(O, dfx, agg):
    """The N>1 loss paths against the ORACLE: a C2-sized batch cut into record pieces, (a) the multi-source loss
    over the pieces (the consumer side of the lazy reshard), (b) the TP-split fold of the pieces' separate losses
    (dfx_loss_combine) -- both within 1e-5 relative of the f64 oracle on the whole batch."""
    from paper_2507_13833_b200 import _abi
    from paper_2507_13833_b200.packed import _ptr
    R, n = 1024, 16
    sb = O.SynthBatch(1, R, n, O.token_dist("uniform", 0, 1, 4096))
    b = dfx.PackedBatch.synthetic(1, R, n, dfx.TokenDist("uniform", 0, 1, 4096))
    ctx = dfx.StageContext()
    ctx.loss = dfx.LossConfig(kl="k3", agg=agg)
    dfx.fn_group_advantage(dfx.NodeSpec("a"), b, ctx)
    adv = O.grpo_advantage(sb.group_off, sb.reward, 1e-6)
    adv_tok = O.broadcast_advantage(sb.cu_seqlens, adv, sb.mask)
    ref, _ = O.ppo_loss(sb.cu_seqlens, sb.lp, sb.old_lp, sb.ref_lp, adv_tok, sb.mask, O.loss_cfg(agg=agg))
    cuts = [0, 128, 512, 513, 1024]  # the N=8 TP pair halves are [0, 512) / [512, 1024); plus ragged pieces
    views = [b.view_records(cuts[i], cuts[i + 1]) for i in range(len(cuts) - 1)]
    multi = dfx.ppo_loss_sources(views, ctx, loss_group_off=[0, R * n])["out"].cpu().numpy()[0]
    _check_loss(multi, ref, f"multi-source {agg}")
    parts = torch.cat([dfx.ppo_loss(v, ctx, adv_source="rollout")["out"] for v in views]).reshape(-1)
    out = torch.empty(7, dtype=torch.float64, device="cuda")
    c = _abi.LossCfg(ctx.loss.clip_low, ctx.loss.clip_high, ctx.loss.beta, float(ctx.advantage_eps), _abi.KL["k3"],
                     _abi.AGG[agg], _abi.ADV["rollout"], 0)
    _abi.check(_abi.lib().dfx_loss_combine(_ptr(parts), len(views), 1, C.byref(c), _ptr(out),
                                           torch.cuda.current_stream().cuda_stream))
    _check_loss(out.cpu().numpy(), ref, f"tp-split fold {agg}")


def test_gae_long_rollouts_deterministic(O, dfx):
    """Rollouts far longer than 32 tiles (checkpoint chains across tiles without a rollout end): bit-identical
    outputs on repeated runs and agreement with the oracle."""
    streams = ("mask", "value_tok", "token_reward")
    L = 400_000
    sb = O.SynthBatch(5, 3, 1, O.token_dist("constant", L, L, L), streams=streams)
    db = dfx.PackedBatch.synthetic(5, 3, 1, dfx.TokenDist("constant", L, L, L), streams=streams)
    ctx = dfx.StageContext(gae_gamma=0.999, gae_lambda=0.99)
    outs = []
    T = sb.n_tokens
    for _ in range(3):  # (the streams' padding past T is never written: compare the tokens)
        dfx.fn_gae_advantage(dfx.NodeSpec("g"), db, ctx)
        outs.append((db.streams["advantage"][:T].clone(), db.streams["returns"][:T].clone(),
                     db.channels["_whiten_sums"].clone()))
    for o in outs[1:]:
        assert all(torch.equal(x, y) for x, y in zip(o, outs[0]))
    A, Rt, _ = O.gae(sb.cu_seqlens, sb.token_reward, sb.value_tok, sb.mask, 0.999, 0.99)
    assert_close_vec(outs[0][0][:T].cpu().numpy(), A[:T], "long gae adv")
    assert_close_vec(outs[0][1][:T].cpu().numpy(), Rt[:T], "long gae ret")


def test_gae_segment_cuts(O, dfx):
    """The segment scan around its cut rule: rollouts of 60k-140k tokens (some above the 64k no-cut limit, so their
    segments chain through published carries, some below), through a view of records 1..5 (its first token at an
    arbitrary offset); bit-identical on a second run and within tolerance of the oracle."""
    streams = ("mask", "value_tok", "token_reward")
    sb = O.SynthBatch(17, 7, 2, O.token_dist("uniform", 60000, 60000, 140000), streams=streams)
    db = dfx.PackedBatch.synthetic(17, 7, 2, dfx.TokenDist("uniform", 60000, 60000, 140000), streams=streams)
    r0, r1 = 1, 6
    v = db.view_records(r0, r1)
    s0, s1 = int(sb.group_off[r0]), int(sb.group_off[r1])
    cu = np.ascontiguousarray(sb.cu_seqlens[s0:s1 + 1])
    ctx = dfx.StageContext(gae_gamma=0.995, gae_lambda=0.97)
    dfx.fn_gae_advantage(dfx.NodeSpec("g"), v, ctx)
    a1 = v.streams["advantage"][cu[0]:cu[-1]].clone()
    r1_ = v.streams["returns"][cu[0]:cu[-1]].clone()
    dfx.fn_gae_advantage(dfx.NodeSpec("g"), v, ctx)
    assert torch.equal(a1, v.streams["advantage"][cu[0]:cu[-1]])
    assert torch.equal(r1_, v.streams["returns"][cu[0]:cu[-1]])
    A, Rt, _ = O.gae(cu, sb.token_reward, sb.value_tok, sb.mask, 0.995, 0.97)
    assert_close_vec(a1.cpu().numpy(), A[cu[0]:cu[-1]], "segment-cut gae adv")
    assert_close_vec(r1_.cpu().numpy(), Rt[cu[0]:cu[-1]], "segment-cut gae ret")


def test_workspace_reuse_across_sizes(O, dfx):
    """One workspace reused by calls of different sizes: GAE after a larger span, and the loss with a
    loss-group count crossing a multiple of 32 and back, all still equal to the oracle."""
    streams = ("lp", "old_lp", "ref_lp", "mask", "value_tok", "token_reward")
    ctx = dfx.StageContext(gae_gamma=0.99, gae_lambda=0.95)
    big = dfx.PackedBatch.synthetic(3, 64, 8, dfx.TokenDist("uniform", 0, 1, 4000), streams=streams)
    dfx.fn_gae_advantage(dfx.NodeSpec("g"), big, ctx)
    for seed, R in ((4, 6), (6, 20)):  # smaller spans, same (cached) workspace
        sb = O.SynthBatch(seed, R, 4, O.token_dist("uniform", 0, 1, 3000), streams=streams)
        db = dfx.PackedBatch.synthetic(seed, R, 4, dfx.TokenDist("uniform", 0, 1, 3000), streams=streams)
        dfx.fn_gae_advantage(dfx.NodeSpec("g"), db, ctx)
        A, Rt, ws = O.gae(sb.cu_seqlens, sb.token_reward, sb.value_tok, sb.mask, 0.99, 0.95)
        T = sb.n_tokens
        assert_close_vec(db.streams["advantage"][:T].cpu().numpy(), A[:T], f"gae adv after shrink R={R}")
        assert db.channels["_whiten_sums"].cpu().numpy()[2] == ws[2]
    sb = O.SynthBatch(8, 96, 4, O.token_dist("uniform", 0, 1, 700))
    db = dfx.PackedBatch.synthetic(8, 96, 4, dfx.TokenDist("uniform", 0, 1, 700))
    adv = O.grpo_advantage(sb.group_off, sb.reward, 1e-6)
    adv_tok = O.broadcast_advantage(sb.cu_seqlens, adv, sb.mask)
    cfg = O.loss_cfg()
    for ng in (1, 40, 3, 64, 2):
        lgo = np.linspace(0, 384, ng + 1).astype(np.int64).tolist()
        out = dfx.ppo_loss(db, ctx, adv_source="group", loss_group_off=lgo)["out"].cpu().numpy()
        for g in range(ng):
            cu = np.ascontiguousarray(sb.cu_seqlens[lgo[g]:lgo[g + 1] + 1])
            ref, _ = O.ppo_loss(cu, sb.lp, sb.old_lp, sb.ref_lp, adv_tok, sb.mask, cfg)
            assert out[g][5] == ref["n_tokens"], (ng, g)
            if ref["n_tokens"] > 0:
                assert_rel(out[g][0], ref["loss"], f"loss ng={ng} group {g}")


def test_multi_source_with_empty_source(dfx):
    """A source with no rollouts owns no slot and is never read (its cu_seqlens may be NULL)."""
    b = dfx.PackedBatch.synthetic(9, 32, 4, dfx.TokenDist("uniform", 0, 1, 900))
    ctx = dfx.StageContext()
    dfx.fn_group_advantage(dfx.NodeSpec("a"), b, ctx)
    whole = dfx.ppo_loss(b, ctx, adv_source="rollout")["out"].cpu().numpy()[0]
    empty = b.view_records(16, 16)
    assert empty.n_rollouts == 0
    got = dfx.ppo_loss_sources([b.view_records(0, 16), empty, b.view_records(16, 32)], ctx,
                               loss_group_off=[0, 128])["out"].cpu().numpy()[0]
    assert got[5] == whole[5] and got[6] == whole[6]
    np.testing.assert_allclose(got[:5], whole[:5], rtol=2e-6, atol=1e-9)


def test_multi_source_api_with_one_source(O, dfx):
    """dfx_ppo_loss_multi with a single source runs the multi-source kernel (its sources may be peer memory: no
    L2 prefetch there): same counts as, and the oracle's loss within 1e-5 like, the single-batch kernel."""
    sb = O.SynthBatch(12, 64, 8, O.token_dist("uniform", 0, 1, 3000))
    b = dfx.PackedBatch.synthetic(12, 64, 8, dfx.TokenDist("uniform", 0, 1, 3000))
    ctx = dfx.StageContext()
    dfx.fn_group_advantage(dfx.NodeSpec("a"), b, ctx)
    single = dfx.ppo_loss(b, ctx, adv_source="rollout")["out"].cpu().numpy()[0]
    multi = dfx.ppo_loss_sources([b], ctx, loss_group_off=[0, b.n_rollouts])["out"].cpu().numpy()[0]
    assert multi[5] == single[5] and multi[6] == single[6]
    adv = O.grpo_advantage(sb.group_off, sb.reward, 1e-6)
    ref, _ = O.ppo_loss(sb.cu_seqlens, sb.lp, sb.old_lp, sb.ref_lp, O.broadcast_advantage(sb.cu_seqlens, adv, sb.mask),
                        sb.mask, O.loss_cfg())
    _check_loss(single, ref, "single-batch kernel")
    _check_loss(multi, ref, "multi-source kernel, one source")


@pytest.mark.parametrize("kl", ["k3", "k1", "none"])
def test_c3_fused_gae_loss_full_size(O, dfx, kl):
    """C3 (512 x 8192) through the fused GAE + loss pass (dfx_gae_ppo_loss): two runs give the same bits; returns and
    the (optional) advantage match the standalone GAE (a different scan kernel: segments instead of look-back tiles)
    and the f64 oracle within tolerance; the loss scalars match the oracle on the oracle's own GAE within 1e-5."""
    R, L = 512, 8192
    streams = ("lp", "old_lp", "ref_lp", "mask", "value_tok", "token_reward")
    sb = O.SynthBatch(1, R, 1, O.token_dist("constant", L, L, L), streams=streams)
    db = dfx.PackedBatch.synthetic(1, R, 1, dfx.TokenDist("constant", L, L, L), streams=streams)
    ctx = dfx.StageContext(gae_gamma=1.0, gae_lambda=0.95)
    ctx.loss = dfx.LossConfig(kl=kl, agg="token-mean")
    T = sb.n_tokens
    r1 = dfx.gae_ppo_loss(db, ctx, want_adv=True)
    a1, ret1, o1 = r1["adv"][:T].clone(), db.streams["returns"][:T].clone(), r1["out"].clone()
    r2 = dfx.gae_ppo_loss(db, ctx)
    assert torch.equal(o1, r2["out"]) and torch.equal(ret1, db.streams["returns"][:T])
    dfx.fn_gae_advantage(dfx.NodeSpec("g"), db, ctx)  # the two-launch path: same advantages and returns
    A, Rt, _ = O.gae(sb.cu_seqlens, sb.token_reward, sb.value_tok, sb.mask, 1.0, 0.95)
    assert_close_vec(a1.cpu().numpy(), A[:T], "C3 fused adv")
    assert_close_vec(ret1.cpu().numpy(), Rt[:T], "C3 fused ret")
    assert_close_vec(db.streams["advantage"][:T].cpu().numpy(), a1.cpu().numpy(), "C3 fused vs two-launch adv")
    two = dfx.ppo_loss(db, ctx, adv_source="token")["out"].cpu().numpy()[0]
    ref, _ = O.ppo_loss(sb.cu_seqlens, sb.lp, sb.old_lp, sb.ref_lp, A[:T].astype(np.float32), sb.mask,
                        O.loss_cfg(kl=kl))
    _check_loss(o1.cpu().numpy()[0], ref, f"C3 fused {kl}")
    _check_loss(two, ref, f"C3 two-pass {kl}")


def test_fused_gae_loss_ragged(O, dfx):
    """The fused pass on ragged, skewed and empty rollouts and a view (token_base not tile-aligned)."""
    streams = ("lp", "old_lp", "ref_lp", "mask", "value_tok", "token_reward")
    sb = O.SynthBatch(13, 40, 6, O.token_dist("skewed", 0, 0, 9000), streams=streams)
    db = dfx.PackedBatch.synthetic(13, 40, 6, dfx.TokenDist("skewed", 0, 0, 9000), streams=streams)
    ctx = dfx.StageContext(gae_gamma=0.99, gae_lambda=0.95)
    v = db.view_records(3, 37)
    s0, s1 = int(sb.group_off[3]), int(sb.group_off[37])
    cu = np.ascontiguousarray(sb.cu_seqlens[s0:s1 + 1])
    out = dfx.gae_ppo_loss(v, ctx)["out"].cpu().numpy()[0]
    A, _, _ = O.gae(cu, sb.token_reward, sb.value_tok, sb.mask, 0.99, 0.95)
    ref, _ = O.ppo_loss(cu, sb.lp, sb.old_lp, sb.ref_lp, A.astype(np.float32), sb.mask, O.loss_cfg())
    _check_loss(out, ref, "fused ragged view")
