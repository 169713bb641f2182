"""C3 (512 x 8192 tokens: every f32 token stream exactly 2^24 bytes) with the token streams re-homed into one
allocation at a per-stream byte skew (benchmarking only): tests whether the power-of-two distance between the
separately allocated streams costs DRAM throughput (channel / bank aliasing) in the loss and GAE kernels.

usage: python tools/c3_alias.py [--skews 0,4096,65536+256,...]  (0 = the streams as allocated)
"""
from __future__ import annotations

import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2507_13833_b200 as dfx  # noqa: E402
from tools.measure_configs import graph_ms, kernel_ms  # noqa: E402


def rehome(b, skew: int) -> list:
    """Copy every token stream into one buffer, stream k starting at k * (stream bytes + skew)."""
    names = sorted(b.streams)
    sizes = [b.streams[n].numel() * b.streams[n].element_size() for n in names]
    pitch = max(sizes) + skew
    buf = torch.empty(pitch * len(names) + 4096, dtype=torch.uint8, device=b.device)
    for k, n in enumerate(names):
        t = b.streams[n]
        nb = sizes[k]
        v = buf[k * pitch:k * pitch + nb].view(t.dtype)
        v.copy_(t)
        b.streams[n] = v
    return [buf]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--skews", default="0,256,4096,65536,2097152,1048576+384")
    a = ap.parse_args()
    for sk in a.skews.split(","):
        skew = eval(sk)  # noqa: S307  (e.g. "1048576+384")
        b = dfx.PackedBatch.synthetic(1, 512, 1, dfx.TokenDist("constant", 8192),
                                      streams=("lp", "old_lp", "ref_lp", "mask", "value_tok", "token_reward"))
        ctx = dfx.StageContext(gae_gamma=1.0, gae_lambda=0.95)
        ctx.loss = dfx.LossConfig(whiten=True)
        node = dfx.NodeSpec("gae")
        dfx.fn_gae_advantage(node, b, ctx)
        keep = rehome(b, skew) if sk != "0" else []
        wsum = b.channels["_whiten_sums"]
        ref = dfx.ppo_loss(b, ctx, adv_source="token")
        km = kernel_ms(lambda ev: dfx.ppo_loss(b, ctx, adv_source="token", events=ev))
        # the GAE inputs at the same skew (its outputs are fresh allocations each call)
        g_ms = graph_ms(lambda: dfx.fn_gae_advantage(node, b, ctx))
        b.channels["_whiten_sums"] = wsum
        T = b.token_span
        print(json.dumps({"skew": sk, "loss_kernel_ms": round(km, 5), "loss_frac": round(T * 17 / (km / 1e3) / 1e9
                          / 6531.9, 3), "gae_graph_ms": round(g_ms, 5),
                          "ptrs_mod_16M": [hex(b.streams[n].data_ptr() % (1 << 24)) for n in sorted(b.streams)]}))
        del keep, ref


if __name__ == "__main__":
    main()
