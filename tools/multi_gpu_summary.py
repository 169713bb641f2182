"""Summarise a tools/multi_gpu_cycle.sh run (gpurun_out/multi_<TAG>_*.json + bench_store_<TAG>_n*.json) into
profiles/r01s2_multi_gpu.{md,jsonl}.  usage: python tools/multi_gpu_summary.py TAG"""
import glob
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
tag = sys.argv[1]
rows, raw = [], []
for f in sorted(glob.glob(os.path.join(ROOT, "gpurun_out", f"multi_{tag}_*.json"))):
    name = os.path.basename(f)[len(f"multi_{tag}_"):-5]
    try:
        d = json.load(open(f))
    except Exception:  # noqa: BLE001
        continue
    raw.append(json.dumps(d))
    r = d.get("roofline") or {}
    cfg = d["config"]
    rows.append((name, d["n_gpus"], d["value"], d["ms_per_step"], r.get("bound"), r.get("frac"), r.get("kernel_ms"),
                 (d.get("e2e") or {}).get("value") or 0, (cfg.get("reshard") or cfg.get("placement") or "")[:100]))
out = [f"# Multi-GPU bench matrix (round 1, session 2; tools/multi_gpu_cycle.sh on a 4-GPU box, tag {tag})", "",
       "| run | N | tokens/s | ms/step | roofline bound | frac | loss kernel ms | e2e tokens/s | reshard / placement |",
       "|---|---|---|---|---|---|---|---|---|"]
for r in rows:
    out.append(f"| {r[0]} | {r[1]} | {r[2]:.4g} | {r[3]:.4f} | {r[4]} | {r[5]} | {r[6]} | {r[7]:.3g} | {r[8]} |")
bs = []
for f in sorted(glob.glob(os.path.join(ROOT, "gpurun_out", f"bench_store_{tag}_n*.json"))):
    try:
        bs.append(json.load(open(f)))
    except Exception:  # noqa: BLE001
        pass
if bs:
    out += ["", "C++ device DataBuffer, C4 round trip in one process (`cpp/_build/bench_store N`):", "",
            "| GPUs | ms/trip | tokens/s | bytes copied/trip | exchange s / t ms |", "|---|---|---|---|---|"]
    for d in bs:
        n = d["workload"].split(", ")[-2] if ", " in d["workload"] else "?"
        out.append(f"| {n} | {d['ms_per_trip']} | {d['tokens_per_s']:.4g} | {d['bytes_copied_per_trip']:.4g} | "
                   f"{d.get('exchange_s_ms')} / {d.get('exchange_t_ms')} |")
        raw.append(json.dumps(d))
out += ["",
        "- n1/n2/n4: the default bench (C2 per GPU, box placement W=8): zero-copy reshard, near-linear.",
        "- n2_w2 / n4_w4: the N=8 layout (one logical worker per GPU, TP partners on different GPUs) on 2 / 4 GPUs,",
        "  TP-split loss (default): each TP worker streams the rollouts it holds, the pair folds 56-byte loss rows",
        "  (NCCL all-gather + dfx_loss_combine), step captured in a CUDA graph. Projected N=8: ~0.15 ms/step, ~1.8 T",
        "  tokens/s.",
        "- n4_w4_read (--tp-read): the same layout with every TP worker streaming its whole group, the partner's",
        "  half read in place over NVLink by the multi-source loss kernel at ~73 % of the 770 GB/s peer-copy rate.",
        "- n4_store: one DataBuffer per GPU (dense slice/exchange/concat), consumers read remote slices in place.",
        "- c4_*: BASELINE config 4, the materialized DataBuffer round trip dp8 -> dp4 -> dp8 (16.8M tokens, strong",
        "  scaling), host-orchestration bound.",
        "- c5_n4: BASELINE config 5 split over 4 GPUs (strong scaling).",
        "Raw JSON lines: profiles/r01s2_multi_gpu.jsonl."]
open(os.path.join(ROOT, "profiles", "r01s2_multi_gpu.md"), "w").write("\n".join(out) + "\n")
open(os.path.join(ROOT, "profiles", "r01s2_multi_gpu.jsonl"), "w").write("\n".join(raw) + "\n")
print("\n".join(out))
