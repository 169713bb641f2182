"""GPU parity: the CUDA path (through libdfx's C ABI) against the CPU oracle on identical seeded inputs.

Bit-exact: synthetic token streams, GRPO group advantage (f64) and its per-token broadcast.
Within the tolerance in tests/helpers.py: GAE, PPO clipped surrogate + KL + aggregation, dlogp.
"""
from __future__ import annotations

import ctypes as C

import numpy as np
import pytest
import torch

from tests.helpers import assert_close_scalar, assert_close_vec, loss_term_scales

pytestmark = pytest.mark.gpu

STREAMS = ("lp", "old_lp", "ref_lp", "mask", "value_tok", "token_reward")


def device_batch(dfx, sb, streams=STREAMS):
    """Upload an oracle SynthBatch (host) to a device PackedBatch."""
    st = {k: getattr(sb, k)[: sb.n_tokens] for k in streams if getattr(sb, k) is not None}
    return dfx.PackedBatch.from_host(sb.ids, sb.group_off, sb.cu_seqlens, {"reward": sb.reward, "value": sb.value}, st)


def make(O, seed, R, n, kind, lo, hi, streams=STREAMS):
    return O.SynthBatch(seed, R, n, O.token_dist(kind, lo, lo, hi), streams=streams)


CASES = [
    # seed, records, rollouts, dist, min, max
    (1, 64, 8, "constant", 1024, 1024),      # C1 shape
    (7, 16, 2, "uniform", 16, 48),           # configs/grpo_small.json generation
    (3, 37, 5, "uniform", 1, 300),           # ragged, many window crossings
    (5, 8, 4, "uniform", 1, 3),              # tiny rollouts, many per window
    (11, 20, 16, "skewed", 1, 16384),        # C5-like skewed lengths
]


@pytest.mark.parametrize("case", CASES)
def test_device_synth_bit_exact(O, dfx, case):
    seed, R, n, kind, lo, hi = case
    sb = make(O, seed, R, n, kind, lo, hi, streams=STREAMS + ("token_id",))
    dist = dfx.TokenDist(kind, lo, lo, hi)
    db = dfx.PackedBatch.synthetic(seed, R, n, dist, streams=STREAMS + ("token_id",))
    torch.cuda.synchronize()
    assert db.host_cu.tolist() == sb.cu_seqlens.tolist()
    T = sb.n_tokens
    for k in STREAMS + ("token_id",):
        got = db.streams[k][:T].cpu().numpy()
        ref = getattr(sb, k)[:T]
        assert got.tobytes() == ref.tobytes(), k
    assert db.channels["reward"].cpu().numpy().tobytes() == sb.reward.tobytes()


@pytest.mark.parametrize("case", CASES)
def test_grpo_advantage_bit_exact(O, dfx, case):
    seed, R, n, kind, lo, hi = case
    sb = make(O, seed, R, n, kind, lo, hi)
    db = device_batch(dfx, sb)
    ctx = dfx.StageContext()
    dfx.fn_group_advantage(dfx.NodeSpec("adv"), db, ctx)
    got = db.channels["advantage"].cpu().numpy()
    ref = O.grpo_advantage(sb.group_off, sb.reward, 1e-6)
    assert got.tobytes() == ref.tobytes()
    if O.ref_available():  # the reference itself, compiled from /root/reference
        R_ = O.ref()
        out = np.zeros_like(ref)
        assert R_.ref_advantage(0, sb.n_records, O.ptr(sb.group_off), O.ptr(sb.reward), None, 1e-6, O.ptr(out)) == 0
        assert got.tobytes() == out.tobytes()
    from paper_2507_13833_b200.functions import broadcast_advantage
    tok = broadcast_advantage(db, ctx)[: sb.n_tokens].cpu().numpy()
    assert tok.tobytes() == O.broadcast_advantage(sb.cu_seqlens, ref, sb.mask)[: sb.n_tokens].tobytes()


def test_grpo_advantage_kats(dfx):
    """tests/test_functions.cpp:134-168 through the GPU path."""
    def adv(rewards, eps):
        S = len(rewards)
        b = dfx.PackedBatch.from_host([0], [0, S], np.zeros(S + 1, np.int64), {"reward": np.array(rewards)})
        ctx = dfx.StageContext(advantage_eps=eps)
        dfx.fn_group_advantage(dfx.NodeSpec("a"), b, ctx)
        return b.channels["advantage"].cpu().numpy()
    assert adv([1.0, 0.0, 1.0, 0.0], 0.0).tolist() == [1.0, -1.0, 1.0, -1.0]
    z = adv([0.75, 0.75, 0.75], 0.0)
    assert z.tolist() == [0.0, 0.0, 0.0] and np.isfinite(z).all()
    assert adv([1.0, 0.0], 0.0)[0] > adv([1.0, 0.0], 0.5)[0]


def test_ppo_advantage_and_errors(dfx):
    """tests/test_functions.cpp:170-192 through the GPU path."""
    b = dfx.PackedBatch.from_host([0], [0, 2], np.zeros(3, np.int64), {"reward": np.array([0.9, 0.2]),
                                                                         "value": np.array([0.4, -0.1])})
    dfx.fn_ppo_advantage(dfx.NodeSpec("a"), b, dfx.StageContext())
    assert b.channels["advantage"].cpu().numpy().tolist() == [0.9 - 0.4, 0.2 - (-0.1)]
    missing = dfx.PackedBatch.from_host([0], [0, 1], np.zeros(2, np.int64), {"reward": np.array([0.9])})
    with pytest.raises(dfx.errors.MissingChannelError):
        dfx.fn_ppo_advantage(dfx.NodeSpec("a"), missing, dfx.StageContext())
    empty = dfx.PackedBatch.from_host([0, 1], [0, 1, 1], np.zeros(2, np.int64), {"reward": np.array([0.5])})
    with pytest.raises(dfx.errors.MissingRolloutsError):
        dfx.fn_group_advantage(dfx.NodeSpec("a"), empty, dfx.StageContext())


LOSS_CFGS = [
    dict(kl="k3", agg="token-mean"),
    dict(kl="k1", agg="seq-mean-token-mean"),
    dict(kl="k2", agg="seq-mean-token-sum"),
    dict(kl="none", agg="token-mean", clip_low=0.1, clip_high=0.28),
]


@pytest.mark.parametrize("case", CASES)
@pytest.mark.parametrize("lc", LOSS_CFGS)
@pytest.mark.parametrize("src", ["group", "rollout"])
def test_fused_grpo_loss(O, dfx, case, lc, src):
    seed, R, n, kind, lo, hi = case
    sb = make(O, seed, R, n, kind, lo, hi)
    db = device_batch(dfx, sb)
    ctx = dfx.StageContext()
    ctx.loss = dfx.LossConfig(want_grad=True, **lc)
    adv = O.grpo_advantage(sb.group_off, sb.reward, 1e-6)
    if src == "rollout":
        dfx.fn_group_advantage(dfx.NodeSpec("a"), db, ctx)
    res = dfx.ppo_loss(db, ctx, adv_source=src, adv_tok_out=True)
    got = dfx.loss_dict(res["out"][0])
    adv_tok = O.broadcast_advantage(sb.cu_seqlens, adv, sb.mask)
    cfg = O.loss_cfg(kl=lc["kl"], agg=lc["agg"], clip_low=lc.get("clip_low", 0.2), clip_high=lc.get("clip_high", 0.2))
    ref, g = O.ppo_loss(sb.cu_seqlens, sb.lp, sb.old_lp, sb.ref_lp, adv_tok, sb.mask, cfg, want_grad=True)
    T = sb.n_tokens
    assert res["adv_tok"][:T].cpu().numpy().tobytes() == adv_tok[:T].tobytes()
    if src == "group":
        assert db.channels["advantage"].cpu().numpy().tobytes() == adv.tobytes()
    sc = loss_term_scales(sb, adv_tok, cfg)
    assert got["n_tokens"] == ref["n_tokens"] and got["n_seqs"] == ref["n_seqs"]
    for k in ("loss", "pg_loss", "kl", "approx_kl", "clipfrac"):
        assert_close_scalar(got[k], ref[k], sc[k] if lc["agg"] == "token-mean" else max(sc[k], abs(ref[k])), k)
    assert_close_vec(res["dlogp"][:T].cpu().numpy(), g[:T], "dlogp")


@pytest.mark.parametrize("whiten", [False, True])
def test_gae_and_ppo_loss(O, dfx, whiten):
    """C3-like (scaled down): GAE reverse scan + whitening + clipped surrogate with per-token advantages."""
    sb = make(O, 2, 24, 1, "uniform", 1, 5000)
    db = device_batch(dfx, sb)
    ctx = dfx.StageContext(gae_gamma=1.0, gae_lambda=0.95)
    ctx.loss = dfx.LossConfig(whiten=whiten)
    dfx.fn_gae_advantage(dfx.NodeSpec("gae"), db, ctx)
    A, Rt, ws = O.gae(sb.cu_seqlens, sb.token_reward, sb.value_tok, sb.mask, 1.0, 0.95)
    T = sb.n_tokens
    assert_close_vec(db.streams["advantage"][:T].cpu().numpy(), A[:T], "gae adv")
    assert_close_vec(db.streams["returns"][:T].cpu().numpy(), Rt[:T], "gae ret")
    wsg = db.channels["_whiten_sums"].cpu().numpy()
    assert wsg[2] == ws[2]
    assert_close_vec(wsg[:2], ws[:2], "whiten sums")
    res = dfx.ppo_loss(db, ctx, adv_source="token")
    got = dfx.loss_dict(res["out"][0])
    adv_f32 = db.streams["advantage"].cpu().numpy()  # the loss consumes the stored f32 advantages
    cfg = O.loss_cfg(whiten=whiten)
    ref, _ = O.ppo_loss(sb.cu_seqlens, sb.lp, sb.old_lp, sb.ref_lp, adv_f32, sb.mask, cfg)
    sc = loss_term_scales(sb, adv_f32, cfg)
    for k in ("loss", "pg_loss", "kl", "approx_kl", "clipfrac"):
        assert_close_scalar(got[k], ref[k], sc[k] * (3.0 if whiten else 1.0), k)


def test_gae_kat(dfx):
    """Hand-computed: one rollout r=[0,0,1], V=[0.5,0.5,0.5], mask=1, gamma=1, lam=0.5."""
    cu = np.array([0, 3], np.int64)
    streams = {"token_reward": np.array([0, 0, 1], np.float32), "value_tok": np.full(3, 0.5, np.float32),
               "mask": np.ones(3, np.uint8)}
    b = dfx.PackedBatch.from_host([0], [0, 1], cu, {}, streams)
    dfx.fn_gae_advantage(dfx.NodeSpec("g"), b, dfx.StageContext(gae_gamma=1.0, gae_lambda=0.5))
    # delta = [0+.5-.5, 0+.5-.5, 1-.5] = [0, 0, .5]; A2=.5, A1=0+.5*.5=.25, A0=.125
    assert b.streams["advantage"][:3].cpu().numpy().tolist() == [0.125, 0.25, 0.5]
    assert b.streams["returns"][:3].cpu().numpy().tolist() == [0.625, 0.75, 1.0]


def test_loss_groups_match_slices(O, dfx):
    """Per-loss-group outputs equal the oracle run on each group's rollout slice."""
    sb = make(O, 9, 32, 4, "uniform", 1, 700)
    db = device_batch(dfx, sb)
    ctx = dfx.StageContext()
    lgo = [0, 40, 41, 100, 128]
    res = dfx.ppo_loss(db, ctx, adv_source="group", loss_group_off=lgo)
    out = res["out"].cpu().numpy()
    adv = O.grpo_advantage(sb.group_off, sb.reward, 1e-6)
    adv_tok = O.broadcast_advantage(sb.cu_seqlens, adv, sb.mask)
    cfg = O.loss_cfg()
    for g in range(len(lgo) - 1):
        cu = np.ascontiguousarray(sb.cu_seqlens[lgo[g]:lgo[g + 1] + 1])
        ref, _ = O.ppo_loss(cu, sb.lp, sb.old_lp, sb.ref_lp, adv_tok, sb.mask, cfg)
        assert out[g][5] == ref["n_tokens"]
        assert_close_scalar(out[g][0], ref["loss"], 1.0, f"loss group {g}")


def test_empty_and_degenerate(O, dfx):
    ctx = dfx.StageContext()
    # zero-length rollouts mixed in, and a fully masked rollout
    cu = np.array([0, 0, 5, 5, 9], np.int64)
    T = 9
    rng = np.random.default_rng(0)
    streams = {"lp": -rng.random(T).astype(np.float32), "old_lp": -rng.random(T).astype(np.float32),
               "ref_lp": -rng.random(T).astype(np.float32), "mask": np.array([1, 1, 0, 1, 1, 0, 0, 0, 0], np.uint8)}
    b = dfx.PackedBatch.from_host([3, 4], [0, 2, 4], cu, {"reward": np.array([0.1, 0.9, 0.5, 0.5])}, streams)
    res = dfx.ppo_loss(b, ctx, adv_source="group")
    got = dfx.loss_dict(res["out"][0])
    adv = O.grpo_advantage(np.array([0, 2, 4], np.int32), np.array([0.1, 0.9, 0.5, 0.5]), 1e-6)
    assert b.channels["advantage"].cpu().numpy().tobytes() == adv.tobytes()
    adv_tok = O.broadcast_advantage(cu, adv, streams["mask"])
    ref, _ = O.ppo_loss(cu, streams["lp"], streams["old_lp"], streams["ref_lp"], adv_tok, streams["mask"],
                        O.loss_cfg())
    assert got["n_tokens"] == ref["n_tokens"] == 4
    assert got["n_seqs"] == ref["n_seqs"] == 1
    assert_close_scalar(got["loss"], ref["loss"], 1.0, "loss")
    # empty batch
    e = dfx.PackedBatch.from_host(np.zeros(0, np.uint64), [0], np.zeros(1, np.int64), {"reward": np.zeros(0)},
                                  {k: np.zeros(0, np.float32) for k in ("lp", "old_lp", "ref_lp")} |
                                  {"mask": np.zeros(0, np.uint8)})
    r = dfx.ppo_loss(e, ctx, adv_source="group")
    assert dfx.loss_dict(r["out"][0])["n_tokens"] == 0.0


def test_c2_scale_properties(dfx):
    """Full C2 size (1024 x 16 x U[1,4096], ~33.6M tokens): properties that need no CPU oracle pass.

    - the fused path's per-rollout advantage equals the standalone GRPO kernel's bit for bit
    - per-group advantage sums are ~0 (population-normalised), token count equals the mask sum
    - the run is deterministic: a second call gives bit-identical loss scalars
    """
    db = dfx.PackedBatch.synthetic(1, 1024, 16, dfx.TokenDist("uniform", 0, 1, 4096))
    ctx = dfx.StageContext()
    r1 = dfx.ppo_loss(db, ctx, adv_source="group")["out"].clone()
    fused_adv = db.channels["advantage"].clone()
    r2 = dfx.ppo_loss(db, ctx, adv_source="group")["out"]
    assert r1.cpu().numpy().tobytes() == r2.cpu().numpy().tobytes()
    dfx.fn_group_advantage(dfx.NodeSpec("a"), db, ctx)
    assert db.channels["advantage"].cpu().numpy().tobytes() == fused_adv.cpu().numpy().tobytes()
    a = fused_adv.cpu().numpy().reshape(1024, 16)
    assert np.abs(a.sum(1)).max() < 1e-9
    m = db.streams["mask"][: db.token_span].to(torch.float64).sum().item()
    assert r1[0, 5].item() == m


GAE_CASES = [
    # seed, records, rollouts, dist, min, max, view (records r0, r1 of the batch, or None)
    (3, 4, 1, "constant", 20000, 20000, None),   # rollouts spanning several 4096-token tiles with no end inside
    (5, 40, 8, "uniform", 0, 40, None),          # many empty and 1-token rollouts
    (11, 12, 16, "skewed", 1, 16384, None),      # C5-like skew
    (9, 16, 4, "uniform", 1, 3000, (3, 11)),     # a view: token_base not 4- or 16-aligned, neighbours untouched
    (2, 1, 1, "constant", 1, 1, None),           # a single token
]


@pytest.mark.parametrize("case", GAE_CASES)
def test_gae_shapes(O, dfx, case):
    """GAE over tile-spanning, empty, skewed and offset (view) rollouts: values within tolerance, whitening
    count exact, tokens outside the batch untouched."""
    seed, R, n, kind, lo, hi, view = case
    sb = make(O, seed, R, n, kind, lo, hi)
    db = device_batch(dfx, sb)
    cu = sb.cu_seqlens
    if view is not None:
        r0, r1 = view
        db = db.view_records(r0, r1)
        s0, s1 = int(sb.group_off[r0]), int(sb.group_off[r1])
        cu = np.ascontiguousarray(sb.cu_seqlens[s0:s1 + 1])
    ctx = dfx.StageContext(gae_gamma=0.99, gae_lambda=0.95)
    b0, b1 = int(cu[0]), int(cu[-1])
    # through the C ABI with sentinel-filled outputs: tokens outside [b0, b1) must stay untouched
    from paper_2507_13833_b200 import _abi
    L = _abi.lib()
    adv = torch.full_like(db.streams["lp"], 7.0)
    ret = torch.full_like(db.streams["lp"], 7.0)
    wsum = torch.zeros(3, dtype=torch.float64, device=adv.device)
    nb = L.dfx_gae_workspace_bytes(db.n_rollouts, db.token_span)
    ws = torch.zeros(max(nb, 256), dtype=torch.uint8, device=adv.device)
    st = db.struct()
    for _ in range(2):  # the workspace is reused: epoch tags and the self-clearing end bitmap
        _abi.check(L.dfx_gae(C.byref(st), db.token_base, db.token_span, 0.99, 0.95, adv.data_ptr(), ret.data_ptr(),
                             wsum.data_ptr(), ws.data_ptr(), ws.numel(), None))
    torch.cuda.synchronize()
    A, Rt, wref = O.gae(cu, sb.token_reward, sb.value_tok, sb.mask, 0.99, 0.95)
    got_a, got_r = adv.cpu().numpy(), ret.cpu().numpy()
    assert_close_vec(got_a[b0:b1], A[b0:b1], "gae adv")
    assert_close_vec(got_r[b0:b1], Rt[b0:b1], "gae ret")
    assert (got_a[:b0] == 7.0).all() and (got_a[b1:] == 7.0).all()
    assert (got_r[:b0] == 7.0).all() and (got_r[b1:] == 7.0).all()
    wsg = wsum.cpu().numpy()
    assert wsg[2] == wref[2]
    if wref[2] > 0:
        assert_close_vec(wsg[:2], wref[:2], "whiten sums")


@pytest.mark.parametrize("case", CASES[:3])
def test_reward_stats(O, dfx, case):
    """record_reward_stats (worker.hpp:177-190) on the device: count exact, sums to f64 reduction-order rounding."""
    seed, R, n, kind, lo, hi = case
    sb = make(O, seed, R, n, kind, lo, hi)
    db = device_batch(dfx, sb)
    got = dfx.reward_stats(db, dfx.StageContext()).cpu().numpy()
    s = q = 0.0
    for r in sb.reward.tolist():  # the reference's sequential accumulation
        s += r
        q += r * r
    assert got[0] == len(sb.reward)
    assert abs(got[1] - s) <= 1e-12 * abs(s) and abs(got[2] - q) <= 1e-12 * abs(q)


@pytest.mark.skipif(not torch.cuda.is_available() or torch.cuda.device_count() < 2, reason="needs 2 GPUs")
def test_batch_on_non_current_device(dfx):
    """The entry points launch on their stream's device: a batch on cuda:1 processed while cuda:0 is current gives
    the same bytes as the same batch on cuda:0 (one process driving several GPUs)."""
    torch.cuda.set_device(0)
    outs = []
    for dev in ("cuda:0", "cuda:1"):
        b = dfx.PackedBatch.synthetic(7, 64, 4, dfx.TokenDist("uniform", 0, 1, 900), device=dev,
                                      streams=("lp", "old_lp", "ref_lp", "mask", "token_reward", "value_tok"))
        ctx = dfx.StageContext()
        dfx.fn_group_advantage(dfx.NodeSpec("a"), b, ctx)
        dfx.fn_gae_advantage(dfx.NodeSpec("g"), b, ctx)
        res = dfx.ppo_loss(b, ctx, adv_source="token")
        assert torch.cuda.current_device() == 0
        outs.append((b.channels["advantage"].cpu().numpy(), b.streams["advantage"][:b.token_span].cpu().numpy(),
                     res["out"].cpu().numpy()))
    assert outs[0][0].tobytes() == outs[1][0].tobytes()  # group advantage: bit-exact
    # GAE's look-back composes a data-determined set of tile records: bit-exact across runs and devices, and so
    # is the loss that consumes it (fixed-order reductions)
    assert outs[0][1].tobytes() == outs[1][1].tobytes()
    assert outs[0][2].tobytes() == outs[1][2].tobytes()


@pytest.mark.parametrize("agg", ["token-mean", "seq-mean-token-sum", "seq-mean-token-mean"])
def test_loss_combine_parts(dfx, agg):
    """dfx_loss_combine (the TP-split loss): the loss rows of disjoint record ranges fold into the whole batch's."""
    from paper_2507_13833_b200 import _abi
    from paper_2507_13833_b200.packed import _ptr
    b = dfx.PackedBatch.synthetic(9, 96, 4, dfx.TokenDist("skewed", 0, 1, 3000), device="cuda")
    ctx = dfx.StageContext()
    ctx.loss = dfx.LossConfig(agg=agg)
    dfx.fn_group_advantage(dfx.NodeSpec("a"), b, ctx)
    whole = dfx.ppo_loss(b, ctx, adv_source="rollout")["out"].cpu().numpy()[0]
    cuts = [0, 17, 60, 96]
    parts = torch.cat([dfx.ppo_loss(b.view_records(cuts[i], cuts[i + 1]), ctx, adv_source="rollout")["out"]
                       for i in range(3)]).reshape(-1)
    out = torch.empty(7, dtype=torch.float64, device="cuda")
    c = _abi.LossCfg(ctx.loss.clip_low, ctx.loss.clip_high, ctx.loss.beta, float(ctx.advantage_eps), _abi.KL[ctx.loss.kl], _abi.AGG[agg],
                     _abi.ADV["rollout"], 0)
    _abi.check(_abi.lib().dfx_loss_combine(_ptr(parts), 3, 1, C.byref(c), _ptr(out),
                                           torch.cuda.current_stream().cuda_stream))
    got = out.cpu().numpy()
    assert got[5] == whole[5] and got[6] == whole[6]
    np.testing.assert_allclose(got[:5], whole[:5], rtol=2e-6, atol=1e-9)
