"""Seeded random sweep of the GPU path against the oracle (beyond the hand-picked shapes of test_gpu_parity):
random batch shapes and length distributions, loss configurations, advantage sources and GAE coefficients;
multi-source splits of a batch and the TP-split fold against the single-batch loss. Same tolerances as the
parity tests (bit-exact advantages / counts, tests/helpers.RTOL for the f32 loss sums and GAE)."""
from __future__ import annotations

import ctypes as C

import numpy as np
import pytest
import torch

from tests.helpers import assert_close_scalar, assert_close_vec, loss_term_scales
from tests.test_gpu_parity import device_batch, make

pytestmark = pytest.mark.gpu

KINDS = (("constant", 1, 2048), ("uniform", 1, 5000), ("uniform", 1, 40), ("skewed", 1, 16384))
KLS = ("k1", "k2", "k3", "none")
AGGS = ("token-mean", "seq-mean-token-mean", "seq-mean-token-sum")


def draw(seed):
    rng = np.random.default_rng(1000 + seed)
    kind, lo, hi = KINDS[rng.integers(len(KINDS))]
    if kind == "constant":
        lo = hi = int(rng.integers(1, hi))
    return dict(seed=int(rng.integers(1, 1 << 30)), R=int(rng.integers(1, 96)), n=int(rng.integers(1, 17)),
                kind=kind, lo=lo, hi=hi, kl=KLS[rng.integers(4)], agg=AGGS[rng.integers(3)],
                clip_low=float(rng.choice([0.1, 0.2, 0.3])), clip_high=float(rng.choice([0.2, 0.28])),
                src=("group", "rollout")[rng.integers(2)], gamma=float(rng.choice([1.0, 0.99, 0.9])),
                lam=float(rng.choice([1.0, 0.95, 0.5])))


@pytest.mark.parametrize("seed", range(24))
def test_random_loss_and_gae(O, dfx, seed):
    p = draw(seed)
    sb = make(O, p["seed"], p["R"], p["n"], p["kind"], p["lo"], p["hi"])
    db = device_batch(dfx, sb)
    T = sb.n_tokens
    # loss (fused group advantage or the rollout channel) vs the f64 oracle
    ctx = dfx.StageContext(gae_gamma=p["gamma"], gae_lambda=p["lam"])
    ctx.loss = dfx.LossConfig(kl=p["kl"], agg=p["agg"], clip_low=p["clip_low"], clip_high=p["clip_high"])
    adv = O.grpo_advantage(sb.group_off, sb.reward, 1e-6)
    if p["src"] == "rollout":
        dfx.fn_group_advantage(dfx.NodeSpec("a"), db, ctx)
        assert db.channels["advantage"].cpu().numpy().tobytes() == adv.tobytes()
    res = dfx.ppo_loss(db, ctx, adv_source=p["src"], adv_tok_out=True)
    got = dfx.loss_dict(res["out"][0])
    adv_tok = O.broadcast_advantage(sb.cu_seqlens, adv, sb.mask)
    cfg = O.loss_cfg(kl=p["kl"], agg=p["agg"], clip_low=p["clip_low"], clip_high=p["clip_high"])
    ref, _ = O.ppo_loss(sb.cu_seqlens, sb.lp, sb.old_lp, sb.ref_lp, adv_tok, sb.mask, cfg)
    assert res["adv_tok"][:T].cpu().numpy().tobytes() == adv_tok[:T].tobytes(), p
    assert got["n_tokens"] == ref["n_tokens"] and got["n_seqs"] == ref["n_seqs"], p
    sc = loss_term_scales(sb, adv_tok, cfg)
    for k in ("loss", "pg_loss", "kl", "approx_kl", "clipfrac"):
        assert_close_scalar(got[k], ref[k], sc[k] if p["agg"] == "token-mean" else max(sc[k], abs(ref[k])),
                            f"{k} {p}")
    # GAE with random coefficients
    dfx.fn_gae_advantage(dfx.NodeSpec("gae"), db, ctx)
    A, Rt, ws = O.gae(sb.cu_seqlens, sb.token_reward, sb.value_tok, sb.mask, p["gamma"], p["lam"])
    assert_close_vec(db.streams["advantage"][:T].cpu().numpy(), A[:T], f"gae adv {p}")
    assert_close_vec(db.streams["returns"][:T].cpu().numpy(), Rt[:T], f"gae ret {p}")
    assert db.channels["_whiten_sums"].cpu().numpy()[2] == ws[2]


@pytest.mark.parametrize("seed", range(12))
def test_random_multi_source_and_fold(O, dfx, seed):
    """A batch cut at random record boundaries: the multi-source loss over the pieces, and the TP-split fold of the
    pieces' separate losses, both equal the single-batch loss (counts exact, sums to f32 rounding)."""
    from paper_2507_13833_b200 import _abi
    from paper_2507_13833_b200.packed import _ptr
    p = draw(100 + seed)
    R = max(p["R"], 4)
    b = dfx.PackedBatch.synthetic(p["seed"] & 0xffff, R, p["n"], dfx.TokenDist(p["kind"], p["lo"], p["lo"], p["hi"]),
                                  device="cuda")
    ctx = dfx.StageContext()
    ctx.loss = dfx.LossConfig(kl=p["kl"], agg=p["agg"], clip_low=p["clip_low"], clip_high=p["clip_high"])
    dfx.fn_group_advantage(dfx.NodeSpec("a"), b, ctx)
    whole = dfx.ppo_loss(b, ctx, adv_source="rollout")["out"].cpu().numpy()[0]
    rng = np.random.default_rng(seed)
    k = int(rng.integers(2, 5))
    cuts = [0] + sorted(rng.choice(np.arange(1, R), size=k - 1, replace=False).tolist()) + [R]
    views = [b.view_records(cuts[i], cuts[i + 1]) for i in range(k)]
    go = b.group_off.cpu().numpy()
    multi = dfx.ppo_loss_sources(views, ctx, loss_group_off=[0, int(go[R]) - int(go[0])])["out"].cpu().numpy()[0]
    parts = torch.cat([dfx.ppo_loss(v, ctx, adv_source="rollout")["out"] for v in views]).reshape(-1)
    out = torch.empty(7, dtype=torch.float64, device="cuda")
    c = _abi.LossCfg(p["clip_low"], p["clip_high"], ctx.loss.beta, float(ctx.advantage_eps), _abi.KL[p["kl"]],
                     _abi.AGG[p["agg"]], _abi.ADV["rollout"], 0)
    _abi.check(_abi.lib().dfx_loss_combine(_ptr(parts), k, 1, C.byref(c), _ptr(out),
                                           torch.cuda.current_stream().cuda_stream))
    fold = out.cpu().numpy()
    for got in (multi, fold):
        assert got[5] == whole[5] and got[6] == whole[6], (p, got, whole)
        np.testing.assert_allclose(got[:5], whole[:5], rtol=2e-6, atol=1e-9, err_msg=str(p))
