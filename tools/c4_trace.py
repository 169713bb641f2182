"""Device-side breakdown (torch.profiler / CUPTI, rank 0) of bench.py --workload c4's round trip: per kernel /
memcpy / NCCL totals over the profiled steps, and the chrome trace in gpurun_out/.
usage: torchrun --nproc-per-node N tools/c4_trace.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import bench  # noqa: E402


class A:
    warmup, steps = 3, 10


prof = profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA])
orig = bench.ClockSampler.__enter__
orig_exit = bench.ClockSampler.__exit__


def enter(self):
    prof.__enter__()
    return orig(self)


def leave(self, *a):
    r = orig_exit(self, *a)
    prof.__exit__(None, None, None)
    return r


bench.ClockSampler.__enter__ = enter
bench.ClockSampler.__exit__ = leave
bench.run_c4(A())
if int(os.environ.get("RANK", "0")) == 0:
    print(prof.key_averages().table(sort_by="self_cuda_time_total", row_limit=18, max_name_column_width=70))
    os.makedirs("gpurun_out", exist_ok=True)
    prof.export_chrome_trace(f"gpurun_out/c4_trace_n{os.environ.get('WORLD_SIZE', '1')}.json")
