"""GAE scan and token-path loss time vs batch size (benchmarking only): R x 8192-token rollouts, per-token (GAE) vs
per-rollout advantages, to separate the kernel's fixed cost (ramp, tail) from its per-byte cost."""
from __future__ import annotations

import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2507_13833_b200 as dfx  # noqa: E402
from tools.measure_configs import graph_ms, kernel_ms  # noqa: E402

for R in (128, 256, 512, 1024, 2048, 4096):
    b = dfx.PackedBatch.synthetic(1, R, 1, dfx.TokenDist("constant", 8192),
                                  streams=("lp", "old_lp", "ref_lp", "mask", "value_tok", "token_reward"))
    ctx = dfx.StageContext(gae_gamma=1.0, gae_lambda=0.95)
    ctx.loss = dfx.LossConfig(whiten=True)
    dfx.fn_gae_advantage(dfx.NodeSpec("gae"), b, ctx)
    wsum = b.channels["_whiten_sums"]
    g_ms = graph_ms(lambda: dfx.fn_gae_advantage(dfx.NodeSpec("gae"), b, ctx))
    b.channels["_whiten_sums"] = wsum
    kt = kernel_ms(lambda ev: dfx.ppo_loss(b, ctx, adv_source="token", events=ev))
    dfx.fn_ppo_advantage(dfx.NodeSpec("adv"), b, ctx)
    ctx.loss = dfx.LossConfig()
    kr = kernel_ms(lambda ev: dfx.ppo_loss(b, ctx, adv_source="rollout", events=ev))
    T = b.token_span
    print(json.dumps({"R": R, "tokens": T, "token_ms": round(kt, 5), "token_frac": round(T * 17 / kt / 1e6 / 6531.9, 3),
                      "gae_graph_ms": round(g_ms, 5), "gae_frac": round(T * 17 / g_ms / 1e6 / 6531.9, 3),
                      "rollout_ms": round(kr, 5), "rollout_frac": round((T * 13 + R * 16) / kr / 1e6 / 6531.9, 3)}))
