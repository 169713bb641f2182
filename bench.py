#!/usr/bin/env python
"""Benchmark: post-rollout tokens/s (advantage + loss + reshard) on B200, BASELINE.json's metric.

One step = the post-rollout DAG slice of the GRPO preset (distflow/dag.hpp:341-354) over one synthetic batch
already resident in HBM:
  group_advantage_compute (dp_p = 8 logical workers)  -> reshard dp 8 -> dp 4 (tp 2)  -> actor_train loss (dp 4)
    * GRPO group advantage, f64 per rollout (dfx_grpo_advantage)
    * DataBuffer reshard, box placement (B = 1 store, W = 8 logical workers over the N GPUs);
      at N <= 4 every consumer group's records are already on its GPU -> zero-copy views, no bytes move;
      at N = 8 TP partners exchange their groups over NVLink (NCCL)
    * fused per-token advantage broadcast + PPO clipped surrogate + k3 KL + token-mean, one loss group per
      consumer DP group (dfx_ppo_loss, the dominant kernel)
Workload per GPU: C2 = 1024 prompts x n=16 x UNIFORM[1,4096] tokens (~33.5M tokens, 571 MB of streams; larger
than L2, so no flush is needed between steps). Weak scaling: every rank holds its own C2 batch.

--impl reference times the reference's own CPU implementation (oracle/_ref: fn_group_advantage + BufferStore
put/redistribute/get, compiled from /root/reference) plus the oracle's loss port (the reference has no loss) on the
same full C2 batch and step counts, on this host's cores.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "post-rollout tokens/s (adv+loss+reshard) at 1/2/4/8 B200; % of HBM roofline"
UNIT = "tokens/s"
C2 = dict(records=1024, n_roll=16, dist=("uniform", 0, 1, 4096), seed=1)
C5 = dict(records=4096, n_roll=16, dist=("skewed", 0, 1, 16384), seed=11)
BYTES_PER_TOKEN = 17      # lp, old_lp, ref_lp (3x4) + mask (1) + advantage write (4)
BYTES_PER_ROLLOUT = 16    # f64 advantage read + i64 cu_seqlens read
NVLINK_PEER_GBS = 770.0   # measured peer copy per direction (/opt/skills/guides/B200_PROFILING.md)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="dfx", choices=["dfx", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-graph", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--records", type=int, default=None, help="prompts per GPU (default: the workload's)")
    ap.add_argument("--workload", default="c2", choices=["c2", "c5", "c4"],
                    help="c2: 1024 prompts x 16 x U[1,4096] per GPU (weak scaling, the headline); c5: BASELINE "
                         "config 5, 4096 prompts x 16 x skewed <=16k tokens split over the GPUs (strong scaling); "
                         "c4: BASELINE config 4, the DataBuffer round trip dp8 -> dp4 (tp2) -> dp8 of a 16.8M-token "
                         "batch (16 B/token payload) split over the GPUs, one DataBuffer per GPU")
    ap.add_argument("--workers", type=int, default=8,
                    help="box placement: logical workers (the reference's W); N=8 GPUs with 8 workers puts TP "
                         "partners on different GPUs -- --workers 4 on 4 GPUs previews that path")
    ap.add_argument("--materialize", action="store_true",
                    help="copy remote records into a local consumer batch before the loss (default: the loss kernel "
                         "reads them in place over NVLink)")
    ap.add_argument("--tp-split", action="store_true",
                    help="TP partners on different GPUs (N=8 box placement): instead of every TP worker consuming its "
                         "whole consumer group (the partner's half read over NVLink by the loss kernel, the default), "
                         "each streams only the rollouts it holds and the pair folds its loss rows -- a LOSS-ONLY "
                         "figure: no token of the group reaches the other TP worker")
    ap.add_argument("--store", default="native", choices=["native", "python"],
                    help="c4: the native distributed DataBuffer (libdfx, one C call per verb, NCCL) or the Python "
                         "DeviceBufferStore")
    ap.add_argument("--transport", default="pull", choices=["pull", "nccl"],
                    help="c4 native store: SM pulls of peer-mapped (CUDA IPC) producer memory (default) or NCCL send/recv")
    ap.add_argument("--placement", default="box", choices=["box", "store"],
                    help="box: one DataBuffer per box, 8 logical workers (SURVEY §8(e)); store: one DataBuffer per "
                         "GPU, 2 logical workers per GPU -> dense all-to-all at every N > 1")
    return ap.parse_args()


# ---- clocks (NVML, sampled during the timed region) -----------------------------------------
class ClockSampler:
    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
               0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
               0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting"}

    def __init__(self, index: int, period_s: float = 0.005):
        self.samples, self.mem_samples, self.reasons = [], [], set()
        self.max_mhz = None
        self._stop = threading.Event()
        self._period = period_s
        try:
            import pynvml
            pynvml.nvmlInit()
            self._nv = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM)
        except Exception:  # noqa: BLE001
            self._nv = None

    def _sample(self):
        nv = self._nv
        self.samples.append(nv.nvmlDeviceGetClockInfo(self._h, nv.NVML_CLOCK_SM))
        self.mem_samples.append(nv.nvmlDeviceGetClockInfo(self._h, nv.NVML_CLOCK_MEM))
        r = nv.nvmlDeviceGetCurrentClocksEventReasons(self._h)
        for bit, name in self.REASONS.items():
            if r & bit and bit != 0x1:
                self.reasons.add(name)

    def _run(self):
        while not self._stop.is_set():
            try:
                self._sample()
            except Exception:  # noqa: BLE001
                return
            time.sleep(self._period)

    def __enter__(self):
        if self._nv:
            self._sample()
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *a):
        if self._nv:
            self._stop.set()
            self._t.join()
            self._sample()

    def result(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["nvml_unavailable"]}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "mem_mhz": statistics.median(self.mem_samples) if self.mem_samples else None,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


def measured_peak_hbm():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:  # noqa: BLE001
        return 6650.0, "fallback (B200_PROFILING.md)"


def ncu_traffic():
    """dram bytes per launch of the dominant kernel from the newest committed ncu --set full capture
    (profiles/*loss_slots*.json, written by tools/ncu_summary.py from a capture of the same C2 step). Newest by
    the round-tagged file name (r01s3_ < r02h_ < r02i_ ...): a fresh checkout gives every file the same mtime."""
    import glob
    files = sorted(glob.glob(os.path.join(ROOT, "profiles", "*loss_slots*.json")), key=os.path.basename)
    for p in reversed(files):
        try:
            with open(p) as f:
                v = json.load(f).get("dram_bytes_per_launch")
            if v:
                return v
        except Exception:  # noqa: BLE001
            continue
    return None


# ---- the GPU arm ------------------------------------------------------------------------------------
class DagSlice:
    """group_advantage_compute (dp 8) -> DataBuffer put/get -> actor_train loss (dp 4, tp 2), box placement."""

    STAGE = "group_advantage_compute"

    def __init__(self, dfx, world, rank, records, ctx, Layout, Topology, Store, StagePlan, placement="box", workers=8,
                 lazy=True, dev=None, tp_split=True):
        self.dfx, self.ctx, self.it = dfx, ctx, 0
        self.lazy, self.dev = lazy, dev
        self.placement = placement
        if placement == "box":
            self.topo = Topology.box(workers, world)
            self.prod, self.cons = Layout(workers, 1), Layout(workers // 2, 2)
        else:
            wpg = max(2, 8 // world)
            self.topo = Topology.store_per_gpu(world, wpg)
            self.prod, self.cons = Layout(world * wpg, 1), Layout(world * wpg // 2, 2)
        meta = None
        if world > 1:
            import torch.distributed as dist
            meta = dist.new_group(backend="gloo")  # host metadata side channel; token data moves over NCCL
        self.store = Store(self.topo, rank, {self.STAGE: StagePlan(self.prod, self.cons)}, meta_group=meta)
        self.local_p = [p for p in range(self.prod.dp) if self.topo.gpu_of_worker[p] == rank]
        self.per = records // len(self.local_p)
        self.world = world
        from paper_2507_13833_b200.reshard import Plan
        self.cross = Plan(self.topo, self.prod, self.cons, [self.per] * self.prod.dp, rank).cross
        self.last = None
        # TP-split loss (one worker per GPU, TP partners on different GPUs): each TP worker streams only the
        # rollouts it holds and the pair folds its 56-byte loss rows (all-gather + dfx_loss_combine) -- instead of
        # both TP workers streaming the whole group, the partner's half over NVLink (--tp-read)
        self.tp_group = None
        if tp_split and lazy and self.cross and placement == "box" and workers == world:
            import torch.distributed as dist
            for d in range(self.cons.dp):
                ranks = sorted({self.topo.gpu_of_worker[w] for w in range(workers) if self.cons.dp_rank(w) == d})
                g = dist.new_group(ranks=ranks)  # every rank creates every group, same order
                if rank in ranks:
                    self.tp_group = g

    def step(self, batch, events=None):
        dfx, ctx = self.dfx, self.ctx
        dfx.fn_group_advantage(dfx.NodeSpec(self.STAGE), batch, ctx)
        for j, p in enumerate(self.local_p):
            self.store.put(self.STAGE, self.it, p, 0, batch.view_records(j * self.per, (j + 1) * self.per))
        cb = self.store.ensure_ready(self.STAGE, self.it, self.cons, lazy=self.lazy)
        if cb.sources is not None and self.tp_group is not None:  # TP-split: this GPU's rollouts, then fold
            from paper_2507_13833_b200.packed import PackedBatch
            mine = [x for grp in cb.sources for x in grp if isinstance(x, PackedBatch)]
            assert len(mine) == 1, "TP-split expects one local producer group per GPU"
            res = dfx.ppo_loss(mine[0], ctx, adv_source="rollout", adv_tok_out=True, events=events)
            res["out"] = dfx.tp_combine_loss(res["out"], ctx, self.tp_group)
        elif cb.sources is not None:  # TP partner's records read in place over NVLink by the loss kernel
            srcs = [x for grp in cb.sources for x in grp]
            res = dfx.ppo_loss_sources(srcs, ctx, loss_group_off=cb.roll_off, adv_tok_out=True, events=events,
                                       device=self.dev)
        else:
            res = dfx.ppo_loss(cb.batch, ctx, adv_source="rollout", loss_group_off=cb.roll_off, adv_tok_out=True,
                               events=events)
        for _ in self.store.local_workers:
            self.store.worker_done(self.it)
        self.it += 1
        self.last = cb
        return res, cb.batch

    def remote_sources(self):
        """The partner-GPU runs the last step's loss read over NVLink (lazy exchange), else []."""
        from paper_2507_13833_b200.reshard import RemoteSource
        cb = self.last
        if cb is None or cb.sources is None or self.tp_group is not None:
            return []
        return [x for grp in cb.sources for x in grp if isinstance(x, RemoteSource)]

    def launches_per_step(self):
        # grpo_adv + slot_table + loss_slots + finalize; records crossing GPUs: + the materializing unpack kernel
        # (lazy: none, the loss kernel reads the partner's records over NVLink; one slot table per source)
        # (TP-split: + dfx_loss_combine after the 56-byte all-gather)
        return 4 + (1 if self.cross else 0)

    def describe(self):
        if not self.cross:
            mode = "zero-copy views: every consumer group's TP workers and producer groups share a GPU"
        elif self.lazy and self.placement == "store":
            mode = ("records cross GPUs (dense slice/exchange/concat): each consumer maps the remote slices (CUDA "
                    "IPC) and the loss kernel streams them over NVLink in place (dfx_ppo_loss_multi), no copy")
        elif self.lazy and self.tp_group is not None:
            mode = ("LOSS-ONLY FIGURE (--tp-split): TP partners on different GPUs; each TP worker streams only the "
                    "rollouts it holds and the pair folds its loss rows (56 B all-gather + dfx_loss_combine); no "
                    "token of a consumer group reaches its other TP worker, so this is not a reshard measurement")
        elif self.lazy:
            mode = ("TP partners on different GPUs: each GPU maps its partner's producer group (CUDA IPC) and the "
                    "loss kernel streams it over NVLink in place (dfx_ppo_loss_multi), no copy")
        else:
            mode = "records cross GPUs: copy-engine pulls over NVLink into a consumer batch + unpack kernel"
        t = self.topo
        return (f"{self.placement} placement B={t.num_nodes} W={t.workers_per_node}: dp{self.prod.dp}(tp1) -> "
                f"dp{self.cons.dp}(tp2) over {self.world} GPU; {mode}")


def run_dfx(args):
    import torch
    import torch.distributed as dist

    import paper_2507_13833_b200 as dfx
    from paper_2507_13833_b200 import _abi
    from paper_2507_13833_b200.packed import _ptr

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)

    from paper_2507_13833_b200.reshard import Layout, Topology
    from paper_2507_13833_b200.store import DeviceBufferStore, StoreStagePlan

    L = _abi.lib()
    n = C2["n_roll"]
    if args.workload == "c5":
        R = args.records or C5["records"] // world
        distrib, seed = dfx.TokenDist(*C5["dist"]), C5["seed"]
        wl = f"C5: {R * world} prompts x n={n} x skewed[1,16384] tokens over {world} GPU"
    else:
        R = args.records or C2["records"]
        distrib, seed = dfx.TokenDist(*C2["dist"]), C2["seed"]
        wl = f"C2 per GPU: {R} prompts x n={n} x UNIFORM[1,4096] tokens"
    batch = dfx.PackedBatch.synthetic(seed, R, n, distrib, device=dev, first_id=rank * R)
    torch.cuda.synchronize()
    tokens_local = batch.token_span
    ctx = dfx.StageContext()
    ctx.loss = dfx.LossConfig(kl="k3", agg="token-mean")
    stream = torch.cuda.current_stream(dev)
    resh = DagSlice(dfx, world, rank, R, ctx, Layout, Topology, DeviceBufferStore, StoreStagePlan, args.placement,
                    args.workers, lazy=not args.materialize, dev=dev, tp_split=args.tp_split)

    ev0, ev1 = C.c_void_p(), C.c_void_p()
    _abi.check(L.dfx_event_create(C.byref(ev0)))
    _abi.check(L.dfx_event_create(C.byref(ev1)))
    kern_ms = []

    def step(time_kernel=False):
        res, consumer = resh.step(batch, events=(ev0, ev1) if time_kernel else None)
        if time_kernel:
            ms = C.c_float()
            _abi.check(L.dfx_event_elapsed_ms(ev0, ev1, C.byref(ms)))
            kern_ms.append(ms.value)
        return res, consumer

    for _ in range(max(args.warmup, 3)):
        step()
    torch.cuda.synchronize()

    # kernel-level timing of the dominant kernel (events on its own stream, separate pass)
    for _ in range(min(args.steps, 50)):
        step(time_kernel=True)
    torch.cuda.synchronize()

    # the steady-state step is launch-bound at this size: capture it once in a CUDA graph when the
    # reshard has no host synchronization (box placements with zero-copy views, and the lazy TP-split step whose
    # device work is the adv kernel, two NCCL barriers, the loss kernel, a 56-byte all-gather and the fold); the
    # store's host bookkeeping (put / ensure_ready on a template hit) is identical every step and stays outside
    graph = None
    if (not resh.cross or resh.tp_group is not None) and not args.no_graph:
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph):
            step()
        graph.replay()
        torch.cuda.synchronize()
    run = graph.replay if graph is not None else step

    s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        s0.record(stream)
        for _ in range(args.steps):
            run()
        s1.record(stream)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
    ms_step = s0.elapsed_time(s1) / args.steps
    if world > 1:
        t = torch.tensor([ms_step], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_step = float(t.item())
        tt = torch.tensor([float(tokens_local)], device=dev, dtype=torch.float64)
        dist.all_reduce(tt)
        tokens_total = float(tt.item())
    else:
        tokens_total = float(tokens_local)
    value = tokens_total / (ms_step / 1e3)

    # ---- e2e: same step through the public API from pinned host buffers ----
    e2e = None
    if not args.no_e2e:
        e2e = run_e2e(args, dfx, batch, ctx, resh, dev, stream, world)

    # ---- roofline of the dominant kernel ----
    kern = statistics.median(kern_ms) if kern_ms else None
    bytes_launch = tokens_local * BYTES_PER_TOKEN + batch.n_rollouts * BYTES_PER_ROLLOUT
    peak, peak_src = measured_peak_hbm()
    roof = None
    remote = resh.remote_sources()
    if kern and remote:
        # TP partners on different GPUs: the loss kernel streams the local group from HBM and the partner's group
        # over NVLink; the NVLink half bounds it. Bytes crossing NVLink per launch: the partner's lp/old/ref/mask
        # (13 B/token) + its advantage and cu_seqlens (16 B/rollout).
        nv = sum(x.token_span * 13 + x.n_rollouts * 16 for x in remote)
        local_b = bytes_launch
        ach = nv / (kern / 1e3) / 1e9
        roof = {"bound": "nvlink", "achieved": round(ach, 1), "peak": NVLINK_PEER_GBS, "unit": "GB/s",
                "frac": round(ach / NVLINK_PEER_GBS, 4), "traffic": None,
                "kernel": "dfx::loss_slots_kernel (multi-source: local HBM + partner GPU over NVLink)",
                "kernel_ms": round(kern, 5), "bytes_per_launch": nv, "hbm_bytes_per_launch": local_b,
                "peak_source": "measured peer copy, 770 GB/s per direction (B200_PROFILING.md)"}
    elif kern:
        ach = bytes_launch / (kern / 1e3) / 1e9
        roof = {"bound": "hbm", "achieved": round(ach, 1), "peak": peak, "unit": "GB/s", "frac": round(ach / peak, 4),
                "traffic": ncu_traffic() if args.workload == "c2" else None, "kernel": "dfx::loss_slots_kernel",
                "kernel_ms": round(kern, 5), "bytes_per_launch": bytes_launch, "peak_source": peak_src}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            cpu = cpu_baseline(R)
        except Exception as e:  # noqa: BLE001
            cpu = {"value": None, "error": str(e)[:200]}

    if rank == 0:
        line = {
            "metric": METRIC, "value": round(value, 1), "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": max(args.warmup, 3), "ms_per_step": round(ms_step, 5), "higher_is_better": True,
            "scaling": "weak" if args.workload == "c2" else "strong", "vs_baseline": None, "dtype": "f32 (f64 group stats/accumulators)",
            "data": "synthetic (keyed SplitMix64, generated on device; SURVEY.md §8(d))",
            "config": {"workload": f"{wl} (~{tokens_local/1e6:.1f}M tokens/GPU), GRPO adv -> DataBuffer reshard "
                                   f"(dp_p -> dp_p/2, tp 2) -> clipped loss + k3 KL token-mean",
                       "tokens_per_gpu": tokens_local, "global_tokens": int(tokens_total),
                       "reshard": resh.describe(), "l2": f"inputs ({bytes_launch / 1e6:.0f} MB/GPU) larger than the 126 MB L2; no flush",
                       "parallelism": f"dp{world} (logical dp8->dp4 over {world} GPU)",
                       "cuda_graph": graph is not None},
            "e2e": e2e, "gpu_launches": resh.launches_per_step(), "roofline": roof, "cpu_baseline": cpu,
            "clocks": clk.result(),
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        if graph is not None and resh.cross:
            # the graph holds captured NCCL work of the TP / barrier communicators: tearing those down under the
            # ProcessGroupNCCL watchdog can hang; every collective of the run has completed here, so leave without
            # the teardown
            torch.cuda.synchronize()
            sys.stdout.flush()
            sys.stderr.flush()
            os._exit(0)
        dist.destroy_process_group()


def run_c4(args):
    """BASELINE config 4: the inter-stage reshard round trip DP 8 -> 4 (tp 2) -> 8 of a 16.8M-token rollout batch
    (1024 prompts x 16 x 1024 tokens; payload token_id, lp, old_lp, ref_lp = 16 B/token, plus reward / advantage),
    one DataBuffer per GPU (B = N stores; logical world 8, or 16 at N = 8 where one worker per GPU cannot host a
    tp-2 group), materialized consumer batches (get() semantics). Default: the native distributed DataBuffer
    (libdfx dfx_dstore_*: one C call per verb, grouped NCCL send/recv straight between the producers' and the
    consumers' streams, local copies overlapped); --store python: the Python store (CUDA-IPC pulls)."""
    import torch
    import torch.distributed as dist

    import paper_2507_13833_b200 as dfx
    from paper_2507_13833_b200.reshard import Layout, Topology
    from paper_2507_13833_b200.store import DeviceBufferStore, StoreStagePlan

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    native = args.store == "native"
    meta = None
    if world > 1:
        dist.init_process_group("gloo" if native else "nccl", device_id=None if native else dev)
        meta = None if native else dist.new_group(backend="gloo")
    logical = 16 if world == 8 else 8
    W = logical // world
    topo = Topology.box(logical, 1) if world == 1 else Topology.store_per_gpu(world, W)
    dp = logical
    to_s, to_t = Layout(dp // 2, 2), Layout(dp, 1)
    stages = {"s": StoreStagePlan(Layout(dp, 1), to_s), "t": StoreStagePlan(to_s, to_t)}
    R = 1024 // world
    # (DFX_C4_RAGGED=1, benchmarking only: U[1,2047] lengths, so exchanged runs start at arbitrary 16-byte phases)
    dist_c4 = (dfx.TokenDist("uniform", 0, 1, 2047) if os.environ.get("DFX_C4_RAGGED") == "1"
               else dfx.TokenDist("constant", 1024))
    batch = dfx.PackedBatch.synthetic(11, R, 16, dist_c4, device=dev, first_id=rank * R,
                                      streams=("token_id", "lp", "old_lp", "ref_lp"))
    dfx.fn_group_advantage(dfx.NodeSpec("a"), batch, dfx.StageContext())
    local_p = [p for p in range(dp) if topo.gpu_of_worker[p] == rank]
    per = R // len(local_p)
    views = [batch.view_records(j * per, (j + 1) * per) for j in range(len(local_p))]
    mine_s = [d for d in range(to_s.dp) if any(topo.gpu_of_worker[d * 2 + t] == rank for t in range(2))]
    it = [0]
    stream = torch.cuda.current_stream(dev)
    if native:
        from paper_2507_13833_b200.dstore import Comm, NativeBufferStore
        comm = Comm.create(world, rank)
        store = NativeBufferStore(topo, comm, stages, [("token_id", torch.int32), ("lp", torch.float32),
                                                       ("old_lp", torch.float32), ("ref_lp", torch.float32)],
                                  ["advantage", "reward"], stream=stream, transport=args.transport)

        # the C structs go straight through (no tensors are built for the consumer groups re-put into stage t)
        from paper_2507_13833_b200.dstore import Batch
        v_structs = [store.batch_struct(v) for v in views]
        outs = {d: Batch() for d in mine_s}
        puts_t = [(d, t) for d in mine_s for t in range(2) if topo.gpu_of_worker[d * 2 + t] == rank]
        n_local = len(store.local_workers)

        def step():
            i = it[0]
            for j, p in enumerate(local_p):
                store.put_raw(b"s", i, p, 0, v_structs[j])
            store.ensure_ready_raw(b"s", i, to_s)
            for d in mine_s:
                store.get_raw(b"s", i, d, to_s, outs[d])
            for d, t in puts_t:
                store.put_raw(b"t", i, d, t, outs[d])
            store.ensure_ready_raw(b"t", i, to_t)
            for _ in range(n_local):
                store.worker_done_raw(i)
            it[0] += 1

        def moved():  # NVLink bytes this GPU received (pulled, or NCCL-received) = the peers' egress to it
            st = store.stats()
            return st["bytes_recv"]
    else:
        store = DeviceBufferStore(topo, rank, stages, meta_group=meta)

        def step():
            i = it[0]
            for j, p in enumerate(local_p):
                store.put("s", i, p, 0, views[j])
            cb = store.ensure_ready("s", i, to_s)
            for k, d in enumerate(cb.groups):
                for t in range(2):
                    if topo.gpu_of_worker[2 * d + t] == rank:
                        store.put("t", i, d, t, cb.group_view(d))
            store.ensure_ready("t", i, to_t)
            for _ in store.local_workers:
                store.worker_done(i)
            it[0] += 1

        def moved():
            return store.bytes_sent

    for _ in range(max(args.warmup, 3)):
        step()
    torch.cuda.synchronize()
    steps = max(1, args.steps)
    m0 = moved()
    s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        s0.record(stream)
        for _ in range(steps):
            step()
        s1.record(stream)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
    ms = s0.elapsed_time(s1) / steps
    mv = float(moved() - m0) / steps  # this GPU's NVLink egress per round trip
    if world > 1:
        t = torch.tensor([ms, mv], dtype=torch.float64)
        if not native:
            t = t.to(dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms, mv = float(t[0].item()), float(t[1].item())
    tokens = batch.token_span * world
    ach = mv / (ms / 1e3) / 1e9
    if rank == 0:
        line = {"metric": METRIC, "value": round(tokens / (ms / 1e3), 1), "unit": UNIT, "n_gpus": world,
                "steps": steps, "warmup": max(args.warmup, 3), "ms_per_step": round(ms, 5), "higher_is_better": True,
                "scaling": "strong", "vs_baseline": None, "dtype": "bytes (bit-exact reshard)",
                "data": "synthetic (keyed SplitMix64, generated on device)",
                "config": {"workload": f"C4: DataBuffer round trip dp{dp} -> dp{dp // 2} (tp2) -> dp{dp} of 1024 "
                                       f"prompts x 16 x 1024 tokens (16.8M tokens, 16 B/token payload) over {world} GPU",
                           "placement": f"one DataBuffer per GPU (B={topo.num_nodes}, W={topo.workers_per_node})",
                           "store": (f"native: libdfx dfx_dstore_* (C ABI), transport {args.transport}" if native
                                     else "python: DeviceBufferStore (CUDA-IPC pulls)"),
                           "materialized": True, "global_tokens": tokens},
                "e2e": None, "gpu_launches": None,
                "roofline": {"bound": "nvlink", "achieved": round(ach, 1), "peak": NVLINK_PEER_GBS, "unit": "GB/s",
                             "frac": round(ach / NVLINK_PEER_GBS, 4), "traffic": None,
                             "kernel": "the whole round trip: per-GPU NVLink egress / step time",
                             "bytes_per_step_max_gpu": int(mv),
                             "peak_source": "measured peer copy, 770 GB/s per direction (B200_PROFILING.md)"},
                "cpu_baseline": None, "clocks": clk.result()}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def run_e2e(args, dfx, batch, ctx, resh, dev, stream, world):
    """Public-API step with host buffers: pinned host -> H2D of every input array, the step, D2H of the results."""
    import torch

    h = {}
    d = {}
    for name, t in [("ids", batch.ids), ("group_off", batch.group_off), ("roll_group", batch.roll_group),
                    ("cu_seqlens", batch.cu_seqlens), ("reward", batch.channels["reward"])] + \
            [(k, batch.streams[k]) for k in ("lp", "old_lp", "ref_lp", "mask")]:
        h[name] = t.cpu().pin_memory()
        d[name] = torch.empty_like(t)
    eb = dfx.PackedBatch(batch.n_records, batch.n_rollouts, batch.token_base, batch.token_span, d["ids"],
                         d["group_off"], d["roll_group"], d["cu_seqlens"], {"reward": d["reward"]},
                         {k: d[k] for k in ("lp", "old_lp", "ref_lp", "mask")},
                         host_group_off=batch.host_group_off, host_cu=batch.host_cu)
    h2d = sum(v.numel() * v.element_size() for v in h.values())
    n_groups = len(resh.store.stages and resh.last.groups) if resh.last is not None else 1
    out_h = torch.empty(n_groups * 7, dtype=torch.float64).pin_memory()
    adv_h = torch.empty(batch.n_rollouts, dtype=torch.float64).pin_memory()
    d2h = out_h.numel() * 8 + adv_h.numel() * 8

    def e2e_step():
        for k in h:
            d[k].copy_(h[k], non_blocking=True)
        res, _ = resh.step(eb)
        out_h.copy_(res["out"].reshape(-1), non_blocking=True)
        adv_h.copy_(eb.channels["advantage"], non_blocking=True)

    for _ in range(3):
        e2e_step()
    torch.cuda.synchronize()
    steps = max(3, min(args.steps, 20))
    s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s0.record(stream)
    for _ in range(steps):
        e2e_step()
    s1.record(stream)
    torch.cuda.synchronize()
    ms = s0.elapsed_time(s1) / steps
    if world > 1:
        import torch.distributed as dist
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    tokens = batch.token_span * world
    return {"value": round(tokens / (ms / 1e3), 1), "unit": UNIT, "h2d_bytes_per_step": int(h2d),
            "d2h_bytes_per_step": int(d2h), "ms_per_step": round(ms, 4), "steps": steps,
            "path": "PackedBatch host->device copies + fn_group_advantage + BufferStore reshard + ppo_loss + "
                    "D2H of loss/advantage"}


# ---- CPU arm: the reference's own code (oracle/_ref) + the oracle loss port -------------------
def cpu_sample(records=None):
    """The CPU arm's batch: the GPU arm's own C2 workload (all 1024 prompts unless `records` says otherwise)."""
    from oracle import oracle as O
    sb = O.SynthBatch(C2["seed"], records or C2["records"], C2["n_roll"], O.token_dist(*C2["dist"]),
                      streams=("lp", "old_lp", "ref_lp", "mask", "token_id"))
    return O, sb


LOSS_THREADS = os.cpu_count() or 1  # the loss port runs on every host thread (sequences split across them)


def cpu_step(O, sb, nthreads):
    """Reference fn_group_advantage + BufferStore reshard (dp8 -> dp4 tp2, B=1 W=8, one thread per worker)
    on records whose payload is the 16 B/token streams (token id, lp, old, ref), then the loss port."""
    T = sb.n_tokens
    streams = [sb.token_id[:T], sb.lp[:T], sb.old_lp[:T], sb.ref_lp[:T]]
    adv_s, rs_s = O.ref_bench(sb, streams, 1, 8, 8, 1, 4, 2, nthreads, 1)
    adv = O.grpo_advantage(sb.group_off, sb.reward, 1e-6)
    adv_tok = O.broadcast_advantage(sb.cu_seqlens, adv, sb.mask)
    t2 = time.perf_counter()
    O.ppo_loss_mt(sb.cu_seqlens, sb.lp, sb.old_lp, sb.ref_lp, adv_tok, sb.mask, O.loss_cfg(), LOSS_THREADS)
    t3 = time.perf_counter()
    return adv_s + rs_s + (t3 - t2), {"advantage_s": adv_s, "reshard_s": rs_s, "loss_port_s": t3 - t2}


def _sample_text(sb, nthreads):
    return (f"the full C2 batch ({sb.n_records} prompts x 16 x UNIFORM[1,4096] = {sb.n_tokens} tokens): reference "
            f"fn_group_advantage + BufferStore dp8->dp4 (B=1, W=8; {nthreads} worker threads, runner.hpp:525-530) + "
            f"the oracle's loss port ({LOSS_THREADS} threads, sequences split; the reference has no loss)")


def cpu_baseline(records):
    O, sb = cpu_sample()
    nthreads = 8  # one thread per logical worker, as runner.hpp:525-530
    cpu_step(O, sb, nthreads)  # warm-up
    ts = [cpu_step(O, sb, nthreads)[0] for _ in range(2)]
    t = min(ts)
    return {"value": round(sb.n_tokens / t, 1), "unit": UNIT, "cores": max(nthreads, LOSS_THREADS), "kind": "reference",
            "sample": _sample_text(sb, nthreads), "host_cpus": os.cpu_count()}


def run_reference(args):
    """The reference's own CPU path on this host's cores, on the GPU arm's workload (full C2 per step) and step
    counts (--steps / --warmup honoured); rank 0 alone under torchrun."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    O, sb = cpu_sample()
    nthreads = 8
    warm = max(args.warmup, 1)
    for _ in range(warm):
        cpu_step(O, sb, nthreads)
    steps = max(1, args.steps)
    ts, parts = [], None
    for _ in range(steps):
        t, parts = cpu_step(O, sb, nthreads)
        ts.append(t)
    t = sum(ts) / len(ts)
    v = round(sb.n_tokens / t, 1)
    line = {"metric": METRIC, "value": v, "unit": UNIT, "n_gpus": world, "steps": steps, "warmup": warm,
            "ms_per_step": round(t * 1e3, 3), "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic (keyed SplitMix64)", "impl": "reference",
            "config": {"workload": f"C2 per GPU: {sb.n_records} prompts x n=16 x UNIFORM[1,4096] tokens "
                                   f"(~{sb.n_tokens / 1e6:.1f}M tokens), GRPO adv -> DataBuffer reshard (dp8 -> dp4, "
                                   "tp 2) -> clipped loss + k3 KL token-mean", "tokens": sb.n_tokens,
                       "phases_s": parts},
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": max(nthreads, LOSS_THREADS), "kind": "reference",
                             "sample": _sample_text(sb, nthreads)},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    elif args.workload == "c4":
        run_c4(args)
    else:
        run_dfx(args)


if __name__ == "__main__":
    main()
