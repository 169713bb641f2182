"""Shared test helpers: build matching host (oracle) and device batches, and the tolerance definition.

TOLERANCE (written once, used by every floating-point parity test):
  loss scalars (loss, pg_loss, kl, clipfrac, approx_kl):  |x - y| <= 1e-5 * |y|   (plain relative, north_star)
  per-token outputs (GAE advantages / returns, dlogp):   |x - y| <= 1e-5 * max(|y|, rms(y))
The norm floor is kept only for per-token values, which cross zero. Integer, index, byte
and f64 group-advantage results are compared bit-exactly. Every scalar check records its achieved relative
error; the session prints the maximum per quantity (tests/conftest.py).
"""
from __future__ import annotations

import numpy as np

RTOL = 1e-5


def assert_close_vec(x, y, what=""):
    x = np.asarray(x, np.float64)
    y = np.asarray(y, np.float64)
    assert x.shape == y.shape, (what, x.shape, y.shape)
    if y.size == 0:
        return
    rms = float(np.sqrt(np.mean(y * y)))
    tol = RTOL * np.maximum(np.abs(y), rms)
    bad = np.abs(x - y) > tol
    assert not bad.any(), (f"{what}: {int(bad.sum())} of {y.size} outside tolerance; worst at "
                           f"{int(np.argmax(np.abs(x - y) - tol))}: {x[np.argmax(np.abs(x - y) - tol)]} vs "
                           f"{y[np.argmax(np.abs(x - y) - tol)]}")


ACHIEVED: dict = {}   # quantity -> (max relative error, where)


def assert_rel(x, y, what=""):
    """Loss scalars: plain relative error <= RTOL (x == y exactly when y == 0); records the achieved error."""
    x, y = float(x), float(y)
    err = abs(x - y) / abs(y) if y != 0.0 else (0.0 if x == 0.0 else float("inf"))
    key = what.split(" ")[0]
    if err > ACHIEVED.get(key, (-1.0, ""))[0]:
        ACHIEVED[key] = (err, what)
    assert err <= RTOL, f"{what}: {x!r} vs {y!r} (relative error {err:.3e} > {RTOL:g})"


def assert_close_scalar(x, y, scale=None, what=""):
    """Kept for call sites that passed a scale: the scale is ignored, the check is plain relative."""
    assert_rel(x, y, what)


def loss_term_scales(sb, adv_tok, cfg):
    """mean |term| per loss scalar, computed in f64 from the same inputs (tolerance floor)."""
    T = sb.n_tokens
    m = sb.mask[:T].astype(np.float64)
    lp, old, ref = (a[:T].astype(np.float64) for a in (sb.lp, sb.old_lp, sb.ref_lp))
    A = np.abs(adv_tok[:T].astype(np.float64))
    rho = np.exp(lp - old)
    n = max(m.sum(), 1.0)
    pg = (m * A * np.maximum(rho, 1.2)).sum() / n
    x = ref - lp
    kl = (m * (np.abs(np.expm1(x) - x) + np.abs(x) + 0.5 * x * x)).sum() / n
    akl = (m * np.abs(old - lp)).sum() / n
    return {"pg_loss": pg, "kl": kl, "loss": pg + cfg.beta * kl, "approx_kl": akl, "clipfrac": 1.0}
