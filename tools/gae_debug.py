"""Debug: GAE of small batches against the oracle; prints the mismatching token ranges (benchmarking aid)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2507_13833_b200 as dfx  # noqa: E402
from tests.test_gpu_parity import device_batch, make  # noqa: E402

from oracle import oracle as O  # noqa: E402

O.lib()

for case in [(3, 4, 1, "constant", 20000, 20000), (5, 40, 8, "uniform", 0, 40), (11, 12, 16, "skewed", 1, 16384),
             (1, 8, 4, "uniform", 1, 3000)]:
    seed, R, n, kind, lo, hi = case
    sb = make(O, seed, R, n, kind, lo, hi)
    db = device_batch(dfx, sb)
    ctx = dfx.StageContext(gae_gamma=0.99, gae_lambda=0.95)
    dfx.fn_gae_advantage(dfx.NodeSpec("g"), db, ctx)
    torch.cuda.synchronize()
    T = sb.n_tokens
    A, Rt, ws = O.gae(sb.cu_seqlens, sb.token_reward, sb.value_tok, sb.mask, 0.99, 0.95)
    got = db.streams["advantage"][:T].cpu().numpy().astype(np.float64)
    bad = np.abs(got - A[:T]) > 1e-5 * np.maximum(np.abs(A[:T]), 1.0)
    idx = np.nonzero(bad)[0]
    ranges = []
    for i in idx:
        if ranges and ranges[-1][1] == i - 1:
            ranges[-1][1] = i
        else:
            ranges.append([i, i])
    print(case, "T", T, "bad", len(idx), "ranges", ranges[:12], "cu", sb.cu_seqlens[:8].tolist(), flush=True)
    for r in ranges[:3]:
        print("   got", got[r[0]:r[0] + 4], "want", A[r[0]:r[0] + 4])
