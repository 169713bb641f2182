"""Per-config kernel timings (CUDA events, warm, inputs resident in HBM) for BASELINE.json's configs.

usage: python tools/measure_configs.py [--out profiles/r01_configs.json]
C1 GRPO 64x8x1024 dense; C2 GRPO 1024x16xU[1,4096]; C3 PPO 512x8192 (GAE + whitening + clipped loss, timed as
CUDA-graph replays: the GAE call is three short launches);
C5 GRPO per-GPU share of 4096x16 skewed <=16k at 8 GPUs (512 prompts); C4 reshard 16.8M tokens dp8->dp4->dp8
on one GPU (logical workers; zero-copy) -- the multi-GPU reshard is measured by bench.py --gpus N.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2507_13833_b200 as dfx  # noqa: E402
from paper_2507_13833_b200 import _abi  # noqa: E402

PEAK = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                   "MEASURED_PEAKS.json")))["hbm_gbs"]


def timeit(fn, iters=30, warm=5):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(iters):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / iters


def graph_ms(fn, reps=20):
    """Device time per call of fn captured `reps` times in one CUDA graph (launch overhead of a real pipeline,
    no Python in the timed region)."""
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=side):
        for _ in range(reps):
            fn()
    g.replay()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(5):
        s.record()
        g.replay()
        e.record()
        torch.cuda.synchronize()
        ts.append(s.elapsed_time(e) / reps)
    return sorted(ts)[len(ts) // 2]


def kernel_ms(fn_with_events, iters=20):
    L = _abi.lib()
    e0, e1 = C.c_void_p(), C.c_void_p()
    L.dfx_event_create(C.byref(e0))
    L.dfx_event_create(C.byref(e1))
    out = []
    for i in range(iters + 3):
        fn_with_events((e0, e1))
        ms = C.c_float()
        L.dfx_event_elapsed_ms(e0, e1, C.byref(ms))
        if i >= 3:
            out.append(ms.value)
    out.sort()
    return out[len(out) // 2]


def grpo(name, R, n, dist, streams=("lp", "old_lp", "ref_lp", "mask")):
    b = dfx.PackedBatch.synthetic(1, R, n, dist, streams=streams)
    ctx = dfx.StageContext()
    T = b.token_span
    bytes_ = T * 17 + b.n_rollouts * 16
    step = lambda: dfx.ppo_loss(b, ctx, adv_source="group", adv_tok_out=True)  # noqa: E731
    ms = timeit(step)
    gms = graph_ms(step)
    km = kernel_ms(lambda ev: dfx.ppo_loss(b, ctx, adv_source="group", adv_tok_out=True, events=ev))
    return {"config": name, "tokens": T, "rollouts": b.n_rollouts, "step_ms": ms, "step_graph_ms": gms,
            "tokens_per_s_graph": T / (gms / 1e3), "kernel_ms": km,
            "tokens_per_s": T / (ms / 1e3), "kernel_gbs": bytes_ / (km / 1e3) / 1e9,
            "kernel_frac_of_hbm": bytes_ / (km / 1e3) / 1e9 / PEAK, "bytes_per_launch": bytes_,
            "step": "fused GRPO group stats + broadcast + clipped surrogate + k3 KL (+adv write)"}


def ppo_c3():
    b = dfx.PackedBatch.synthetic(1, 512, 1, dfx.TokenDist("constant", 8192),
                                  streams=("lp", "old_lp", "ref_lp", "mask", "value_tok", "token_reward"))
    ctx = dfx.StageContext(gae_gamma=1.0, gae_lambda=0.95)
    ctx.loss = dfx.LossConfig(whiten=True)
    T = b.token_span
    node = dfx.NodeSpec("gae")

    def step():
        dfx.fn_gae_advantage(node, b, ctx)
        dfx.ppo_loss(b, ctx, adv_source="token")

    ms = graph_ms(step)
    g_ms = graph_ms(lambda: dfx.fn_gae_advantage(node, b, ctx))
    km = kernel_ms(lambda ev: dfx.ppo_loss(b, ctx, adv_source="token", events=ev))
    gae_bytes = T * 17
    loss_bytes = T * 17
    return {"config": "C3", "tokens": T, "step_graph_ms": ms, "tokens_per_s": T / (ms / 1e3),
            "gae_graph_ms": g_ms, "gae_gbs": gae_bytes / (g_ms / 1e3) / 1e9,
            "gae_frac_of_hbm": gae_bytes / (g_ms / 1e3) / 1e9 / PEAK,
            "loss_kernel_ms": km, "loss_gbs": loss_bytes / (km / 1e3) / 1e9,
            "loss_frac_of_hbm": loss_bytes / (km / 1e3) / 1e9 / PEAK,
            "step_frac_of_hbm": (gae_bytes + loss_bytes) / (ms / 1e3) / 1e9 / PEAK,
            "step": "GAE reverse scan (+whitening sums) -> whitened clipped surrogate + k3 KL token-mean"}


def ppo_c3_fused():
    """C3 through the fused GAE + loss pass (dfx_gae_ppo_loss): read r, V, mask, lp, old, ref (21 B/token), write
    the returns (4 B/token); the advantage stays on chip. Token-mean, unwhitened (BASELINE config 3 names no
    whitening)."""
    b = dfx.PackedBatch.synthetic(1, 512, 1, dfx.TokenDist("constant", 8192),
                                  streams=("lp", "old_lp", "ref_lp", "mask", "value_tok", "token_reward"))
    ctx = dfx.StageContext(gae_gamma=1.0, gae_lambda=0.95)
    ctx.loss = dfx.LossConfig(kl="k3", agg="token-mean")
    T = b.token_span
    ms = graph_ms(lambda: dfx.gae_ppo_loss(b, ctx))
    bytes_ = T * 25
    return {"config": "C3 fused", "tokens": T, "step_graph_ms": ms, "tokens_per_s": T / (ms / 1e3),
            "bytes_per_step": bytes_, "step_gbs": bytes_ / (ms / 1e3) / 1e9,
            "step_frac_of_hbm": bytes_ / (ms / 1e3) / 1e9 / PEAK,
            "step": "fused GAE reverse scan + clipped surrogate + k3 KL token-mean (dfx_gae_ppo_loss: 25 B/token)"}


def reshard_c4():
    from paper_2507_13833_b200.reshard import Layout, Topology
    from paper_2507_13833_b200.store import DeviceBufferStore, StoreStagePlan
    b = dfx.PackedBatch.synthetic(11, 1024, 16, dfx.TokenDist("constant", 1024),
                                  streams=("token_id", "lp", "old_lp", "ref_lp"))
    ctx = dfx.StageContext()
    dfx.fn_group_advantage(dfx.NodeSpec("a"), b, ctx)
    res = {}
    for name, topo in {"box_B1_W8": Topology.box(8, 1), "store_B2_W4": Topology(2, 4, (0,) * 8),
                       "store_B4_W2": Topology(4, 2, (0,) * 8)}.items():
        st = DeviceBufferStore(topo, 0, {"s": StoreStagePlan(Layout(8, 1), Layout(4, 2)),
                                         "t": StoreStagePlan(Layout(4, 2), Layout(8, 1))})
        it = [0]

        def rt():
            i = it[0]
            for p in range(8):
                st.put("s", i, p, 0, b.view_records(128 * p, 128 * (p + 1)))
            cb = st.ensure_ready("s", i, Layout(4, 2))
            for d in range(4):
                st.put("t", i, d, 0, cb.group_view(d))
                st.put("t", i, d, 1, cb.group_view(d))
            st.ensure_ready("t", i, Layout(8, 1))
            for _ in range(8):
                st.worker_done(i)
            it[0] += 1
        ms = timeit(rt, iters=10, warm=2)
        res[name] = {"round_trip_ms": ms, "tokens_per_s": b.token_span / (ms / 1e3),
                     "moved_bytes_per_trip": 0 if name.startswith("box") else 2 * b.token_span * 16}
    return {"config": "C4 (1 GPU, 8 logical workers)", "tokens": b.token_span, "payload_bytes_per_token": 16,
            "placements": res}


def wire_c4():
    """Device serialize_records of a C4-size batch (16.8M tokens, 17 B/token payload + reward/advantage)."""
    from paper_2507_13833_b200 import wire
    b = dfx.PackedBatch.synthetic(11, 1024, 16, dfx.TokenDist("constant", 1024),
                                  streams=("token_id", "lp", "old_lp", "ref_lp", "mask"))
    dfx.fn_group_advantage(dfx.NodeSpec("a"), b, dfx.StageContext())
    out = wire.serialize(b, channels=("advantage", "reward"))
    n = out.numel()
    ms = timeit(lambda: wire.serialize(b, channels=("advantage", "reward")), iters=10, warm=2)
    run, dst = wire.serialize_prepared(b, channels=("advantage", "reward"))
    kms = timeit(lambda: run(dst), iters=20, warm=3)  # the device serializer alone (plan and H2D done once)
    return {"config": "C4 wire (device serialize_records)", "tokens": b.token_span, "blob_bytes": n, "ms": ms,
            "kernel_ms": kms, "gbs_rw": 2 * n / (kms / 1e3) / 1e9, "frac_of_hbm": 2 * n / (kms / 1e3) / 1e9 / PEAK,
            "call_frac_of_hbm": 2 * n / (ms / 1e3) / 1e9 / PEAK,
            "note": "ms: the Python call (host plan, pageable H2D of the record offsets, kernel); kernel_ms: kernel"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    ap.add_argument("--only", default=None, help="C1|C2|C3|C4|C5: that config's rows only")
    a = ap.parse_args()
    makers = [("C1", lambda: grpo("C1", 64, 8, dfx.TokenDist("constant", 1024))),
              ("C2", lambda: grpo("C2", 1024, 16, dfx.TokenDist("uniform", 0, 1, 4096))),
              ("C3", ppo_c3),
              ("C3", ppo_c3_fused),
              ("C5", lambda: grpo("C5/8 (one GPU's share: 512 prompts)", 512, 16,
                                  dfx.TokenDist("skewed", 0, 1, 16384))),
              ("C4", reshard_c4),
              ("C4", wire_c4)]
    rows = [mk() for tag, mk in makers if a.only in (None, tag)]
    for r in rows:
        print(json.dumps(r), flush=True)
    if a.out:
        json.dump({"peak_hbm_gbs": PEAK, "gpu": torch.cuda.get_device_name(), "rows": rows}, open(a.out, "w"),
                  indent=1)


if __name__ == "__main__":
    main()
