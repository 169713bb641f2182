"""C3 (512 x 8192) driver for ncu: the fused GAE + loss pass (--fused) or the two-launch step (GAE with whitening,
then the loss), a few calls. usage: [DFX_GAE_VARIANT=...] python tools/c3_prof.py [--fused] [--calls N]"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2507_13833_b200 as dfx  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--fused", action="store_true")
ap.add_argument("--calls", type=int, default=4)
a = ap.parse_args()
b = dfx.PackedBatch.synthetic(1, 512, 1, dfx.TokenDist("constant", 8192),
                              streams=("lp", "old_lp", "ref_lp", "mask", "value_tok", "token_reward"))
ctx = dfx.StageContext(gae_gamma=1.0, gae_lambda=0.95)
if a.fused:
    ctx.loss = dfx.LossConfig(kl="k3", agg="token-mean")
else:
    ctx.loss = dfx.LossConfig(whiten=True)
for _ in range(a.calls):
    if a.fused:
        dfx.gae_ppo_loss(b, ctx)
    else:
        dfx.fn_gae_advantage(dfx.NodeSpec("gae"), b, ctx)
        dfx.ppo_loss(b, ctx, adv_source="token")
torch.cuda.synchronize()
print("ok")
