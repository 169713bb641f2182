"""torch NCCL isend/irecv rate between a GPU pair (both directions at once), 67 MB messages."""
import os
import time

import torch
import torch.distributed as dist

rank = int(os.environ["RANK"])
torch.cuda.set_device(rank)
dev = torch.device("cuda", rank)
dist.init_process_group("nccl", device_id=dev)
n = 67 * 1024 * 1024
sb = torch.empty(n, dtype=torch.uint8, device=dev)
rb = torch.empty(n, dtype=torch.uint8, device=dev)
peer = rank ^ 1
for it in range(11):
    if it == 1:
        torch.cuda.synchronize()
        t = time.perf_counter()
    for w in dist.batch_isend_irecv([dist.P2POp(dist.isend, sb, peer), dist.P2POp(dist.irecv, rb, peer)]):
        w.wait()
torch.cuda.synchronize()
dt = (time.perf_counter() - t) / 10
if rank == 0:
    print(f"67 MB each way: {dt * 1e3:.3f} ms -> {n / dt / 1e9:.0f} GB/s per direction", flush=True)
dist.destroy_process_group()
