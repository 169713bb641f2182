"""One process, two GPUs: the multi-source loss kernel on cuda:0 streaming a local C2 batch and a second C2 batch
that lives on cuda:1 (read over NVLink through peer access) -- the lazy reshard's N=8 step in a form ncu can
profile (a single process; ncu replays the kernel on cuda:0).
usage: python tools/prof_multi.py [--steps N]"""
import argparse
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2507_13833_b200 as dfx  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--steps", type=int, default=3)
a = ap.parse_args()
cudart = C.CDLL("/usr/local/cuda/lib64/libcudart.so.12")
torch.cuda.set_device(0)
loc = dfx.PackedBatch.synthetic(1, 1024, 16, dfx.TokenDist("uniform", 0, 1, 4096), device="cuda:0")
ctx = dfx.StageContext()
dfx.fn_group_advantage(dfx.NodeSpec("a"), loc, ctx)
rem = dfx.PackedBatch.synthetic(1, 1024, 16, dfx.TokenDist("uniform", 0, 1, 4096), device="cuda:1", first_id=1024)
dfx.fn_group_advantage(dfx.NodeSpec("a"), rem, dfx.StageContext())  # launches on cuda:1 (the stream's device)
torch.cuda.synchronize(1)
rc = cudart.cudaDeviceEnablePeerAccess(1, 0)  # from cuda:0 (current) to cuda:1
assert rc in (0, 704), rc                      # 704: already enabled
torch.cuda.synchronize(0)
lgo = [0, loc.n_rollouts, loc.n_rollouts + rem.n_rollouts]
for _ in range(a.steps):
    dfx.ppo_loss_sources([loc, rem], ctx, loss_group_off=lgo, adv_tok_out=True, device=torch.device("cuda", 0))
torch.cuda.synchronize(0)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10):
    dfx.ppo_loss_sources([loc, rem], ctx, loss_group_off=lgo, adv_tok_out=True, device=torch.device("cuda", 0))
e1.record()
torch.cuda.synchronize(0)
ms = e0.elapsed_time(e1) / 10
nv = rem.token_span * 13 + rem.n_rollouts * 16
print(f"multi-source loss: {ms:.4f} ms per call; {nv / 1e6:.1f} MB over NVLink -> {nv / ms / 1e6:.0f} GB/s "
      f"(one GPU reading, the other idle)", flush=True)
