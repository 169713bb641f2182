"""Host-side profile of the bench step (cProfile on rank 0) for the lazy reshard path.

usage: torchrun --nproc-per-node N tools/host_profile.py [--workers W] [--steps S]
"""
import argparse
import cProfile
import os
import pstats
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import bench  # noqa: E402
import paper_2507_13833_b200 as dfx  # noqa: E402
from paper_2507_13833_b200.reshard import Layout, Topology  # noqa: E402
from paper_2507_13833_b200.store import DeviceBufferStore, StoreStagePlan  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workers", type=int, default=8)
ap.add_argument("--steps", type=int, default=30)
a = ap.parse_args()
rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(rank)
dev = torch.device("cuda", rank)
dist.init_process_group("nccl", device_id=dev)
batch = dfx.PackedBatch.synthetic(1, 1024, 16, dfx.TokenDist("uniform", 0, 1, 4096), device=dev, first_id=rank * 1024)
ctx = dfx.StageContext()
resh = bench.DagSlice(dfx, world, rank, 1024, ctx, Layout, Topology, DeviceBufferStore, StoreStagePlan, "box",
                      a.workers, dev=dev)
for _ in range(5):
    resh.step(batch)
torch.cuda.synchronize()
dist.barrier()
prof = cProfile.Profile()
t0 = time.perf_counter()
prof.enable()
for _ in range(a.steps):
    resh.step(batch)
prof.disable()
host = (time.perf_counter() - t0) / a.steps
torch.cuda.synchronize()
dev_t = (time.perf_counter() - t0) / a.steps
if rank == 0:
    print(f"host {host * 1e3:.3f} ms/step, host+drain {dev_t * 1e3:.3f} ms/step", flush=True)
    pstats.Stats(prof).sort_stats("tottime").print_stats(18)
dist.barrier()
dist.destroy_process_group()
