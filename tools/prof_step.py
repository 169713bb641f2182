"""Profiling driver: one C2 batch, W warm-up steps then N steps of the bench's GPU step (no graph), for ncu.

usage: python tools/prof_step.py [--steps N] [--warmup W] [--mode group|rollout|gae]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2507_13833_b200 as dfx  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--steps", type=int, default=3)
ap.add_argument("--warmup", type=int, default=3)
ap.add_argument("--mode", default="rollout")
a = ap.parse_args()
if a.mode == "gae":
    b = dfx.PackedBatch.synthetic(1, 512, 1, dfx.TokenDist("constant", 8192),
                                  streams=("lp", "old_lp", "ref_lp", "mask", "value_tok", "token_reward"))
else:
    b = dfx.PackedBatch.synthetic(1, 1024, 16, dfx.TokenDist("uniform", 0, 1, 4096))
ctx = dfx.StageContext()
if a.mode == "gae":
    ctx.loss = dfx.LossConfig(whiten=True)


def step():
    if a.mode == "gae":
        dfx.fn_gae_advantage(dfx.NodeSpec("gae"), b, ctx)
        dfx.ppo_loss(b, ctx, adv_source="token")
    elif a.mode == "group":
        dfx.ppo_loss(b, ctx, adv_source="group", adv_tok_out=True)
    else:
        dfx.fn_group_advantage(dfx.NodeSpec("adv"), b, ctx)
        dfx.ppo_loss(b, ctx, adv_source="rollout", loss_group_off=None, adv_tok_out=True)


for _ in range(a.warmup + a.steps):
    step()
torch.cuda.synchronize()
print("ok", b.token_span)
