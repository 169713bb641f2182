"""GAE microbenchmark on C3 (512 x 8192 tokens): the GAE call captured 20x in a CUDA graph, replayed; per-call
device time, algorithmic GB/s (17 B/token) and fraction of the measured HBM peak.

usage: DFX_GAE_VARIANT=... python tools/gae_bench.py [--whiten] [--records R --len L --dist constant|uniform|skewed]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2507_13833_b200 as dfx  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--whiten", action="store_true")
ap.add_argument("--records", type=int, default=512)
ap.add_argument("--n", type=int, default=1)
ap.add_argument("--len", type=int, default=8192)
ap.add_argument("--dist", default="constant")
ap.add_argument("--reps", type=int, default=20)
a = ap.parse_args()
dist = dfx.TokenDist("constant", a.len) if a.dist == "constant" else dfx.TokenDist(a.dist, 0, 1, a.len)
b = dfx.PackedBatch.synthetic(1, a.records, a.n, dist, streams=("mask", "value_tok", "token_reward"))
ctx = dfx.StageContext(gae_gamma=1.0, gae_lambda=0.95)
ctx.loss = dfx.LossConfig(whiten=a.whiten)
node = dfx.NodeSpec("gae")
for _ in range(3):
    dfx.fn_gae_advantage(node, b, ctx)
torch.cuda.synchronize()
s = torch.cuda.Stream()
s.wait_stream(torch.cuda.current_stream())
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g, stream=s):
    for _ in range(a.reps):
        dfx.fn_gae_advantage(node, b, ctx)
g.replay()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
ts = []
for _ in range(10):
    e0.record()
    g.replay()
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1) / a.reps)
ts.sort()
ms = ts[len(ts) // 2]
T = b.token_span
peak = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")))["hbm_gbs"]
gbs = T * 17 / (ms / 1e3) / 1e9
print(json.dumps({"variant": os.environ.get("DFX_GAE_VARIANT", "default"), "whiten": a.whiten, "tokens": T,
                  "us": round(ms * 1e3, 2), "gbs": round(gbs, 1), "frac": round(gbs / peak, 4)}))
