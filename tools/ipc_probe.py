import os, torch, torch.distributed as dist
rank = int(os.environ["RANK"]); torch.cuda.set_device(rank); dev = torch.device("cuda", rank)
dist.init_process_group("nccl", device_id=dev); meta = dist.new_group(backend="gloo")
t = torch.arange(1 << 20, dtype=torch.float32, device=dev) + 1000 * rank
view = t[12345:]
h = view.untyped_storage()._share_cuda_()
hs = [None, None]
dist.all_gather_object(hs, (h, view.storage_offset(), view.numel()), group=meta)
peer = rank ^ 1
ph, off, n = hs[peer]
st = torch.UntypedStorage._new_shared_cuda(*ph)
pt = torch.empty(0, dtype=torch.float32, device=st.device).set_(st, off, (n,), (1,))
print(rank, "peer tensor on", pt.device, pt[:3].tolist(), flush=True)
local = torch.empty(n, dtype=torch.float32, device=dev)
dist.barrier()
import time; torch.cuda.synchronize(); t0 = time.perf_counter()
for _ in range(10): local.copy_(pt, non_blocking=True)
torch.cuda.synchronize(); dt = (time.perf_counter() - t0) / 10
print(rank, "copy ok", bool((local[:5].cpu() == pt[:5].cpu()).all()), f"{n*4/dt/1e9:.0f} GB/s", flush=True)
big = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
hb = big.untyped_storage()._share_cuda_(); hbs = [None, None]
dist.all_gather_object(hbs, hb, group=meta)
pb = torch.UntypedStorage._new_shared_cuda(*hbs[peer]); pbt = torch.empty(0, dtype=torch.uint8, device=pb.device).set_(pb, 0, (256 << 20,), (1,))
lb = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
dist.barrier(); torch.cuda.synchronize(); t0 = time.perf_counter()
for _ in range(10): lb.copy_(pbt, non_blocking=True)
torch.cuda.synchronize(); dt = (time.perf_counter() - t0) / 10
print(rank, f"256MB pull {dt*1e3:.3f} ms {256*1.048576e6/dt/1e9:.0f} GB/s (both ranks pulling)", flush=True)
dist.barrier(); dist.destroy_process_group()
