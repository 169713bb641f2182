"""Host profile (cProfile, rank 0) of bench.py --workload c4's round trip.
usage: torchrun --nproc-per-node N tools/c4_profile.py"""
import cProfile
import os
import pstats
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402


class A:
    warmup, steps = 3, 20


prof = cProfile.Profile()
orig = bench.ClockSampler.__enter__


def enter(self):
    prof.enable()
    return orig(self)


bench.ClockSampler.__enter__ = enter
bench.run_c4(A())
prof.disable()
if int(os.environ.get("RANK", "0")) == 0:
    pstats.Stats(prof).sort_stats("tottime").print_stats(22)
