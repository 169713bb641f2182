"""NCCL P2P bandwidth between rank pairs: one big message vs several per-stream messages (torchrun, 2 GPUs)."""
import os
import time

import torch
import torch.distributed as dist

rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(rank)
dev = torch.device("cuda", rank)
dist.init_process_group("nccl", device_id=dev)
peer = rank ^ 1
for mb, parts, mis in [(220, 4, 0), (220, 4, 4), (220, 4, 1), (55, 1, 4)]:
    n = mb * 1024 * 1024 // parts
    sb = [torch.empty(n + 64, dtype=torch.uint8, device=dev)[mis:mis + n] for _ in range(parts)]
    rb = [torch.empty(n + 64, dtype=torch.uint8, device=dev)[2 * mis:2 * mis + n] for _ in range(parts)]
    for it in range(6):
        if it == 1:
            torch.cuda.synchronize()
            dist.barrier()
            t = time.perf_counter()
        ops = [dist.P2POp(dist.isend, s, peer) for s in sb] + [dist.P2POp(dist.irecv, r, peer) for r in rb]
        for w in dist.batch_isend_irecv(ops):
            w.wait()
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t) / 5
    if rank == 0:
        print(f"misalign {mis}: {mb} MB in {parts} msgs each way: {dt * 1e3:.3f} ms -> {mb * 1.048576e6 / dt / 1e9:.0f} GB/s per direction",
              flush=True)
dist.destroy_process_group()
