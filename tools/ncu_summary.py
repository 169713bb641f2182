"""Summarise an ncu --set full report and a launch-list CSV into profiles/ (committed evidence).

usage: python tools/ncu_summary.py REPORT.ncu-rep [LAUNCHES.csv] [--out profiles/NAME] [--bytes N]
Writes NAME.json (key metrics, dram bytes per launch) and NAME.md (human summary incl. top SASS by stall samples).
"""
from __future__ import annotations

import argparse
import csv
import io
import json
import re
import subprocess
from collections import Counter

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "smsp__inst_executed.sum", "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
    "launch__occupancy_limit_registers", "sm__cycles_elapsed.avg.per_second", "lts__t_bytes.sum",
    "l1tex__t_bytes.sum", "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_not_selected_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_lg_throttle_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_drain_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_branch_resolving_per_issue_active.ratio",
]

UNIT_SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "us": 1e-6, "ms": 1e-3, "ns": 1e-9, "s": 1}


def ncu_csv(args):
    out = subprocess.run(["ncu", "-i", *args, "--csv"], capture_output=True, text=True, check=True).stdout
    return list(csv.reader(io.StringIO(out)))


def raw_metrics(rep):
    rows = ncu_csv([rep, "--page", "raw"])
    hdr, units = rows[0], rows[1]
    kernels = []
    for vals in rows[2:]:
        d = {"kernel": vals[hdr.index("Kernel Name")] if "Kernel Name" in hdr else "?"}
        for k in KEYS:
            if k in hdr:
                i = hdr.index(k)
                d[k] = {"value": vals[i], "unit": units[i]}
        kernels.append(d)
    return kernels


def top_sass(rep, n=25):
    rows = ncu_csv([rep, "--page", "source", "--print-source", "sass"])
    hdr = rows[1]
    try:
        ia, si, ss = hdr.index("Instructions Executed"), hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)")
    except ValueError:
        return [], {}
    data = []
    for r in rows[2:]:
        try:
            data.append((int(r[ia] or 0), int(r[ss] or 0), r[si]))
        except (ValueError, IndexError):
            continue
    tot_i = sum(d[0] for d in data)
    ops = Counter()
    for d in data:
        op = d[2].split()
        if op:
            ops[op[1] if op[0].startswith("@") and len(op) > 1 else op[0]] += d[0]
    top = sorted(data, key=lambda d: -d[1])[:n]
    return top, {"instructions": tot_i, "by_opcode": ops.most_common(20)}


def launches(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr = rows[0]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    return [(r[ki], float(r[vi].replace(",", "")), r[ui]) for r in rows[1:]]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("report")
    ap.add_argument("launch_csv", nargs="?")
    ap.add_argument("--out", required=True)
    ap.add_argument("--bytes", type=float, default=None, help="algorithmic bytes per launch of the profiled kernel")
    ap.add_argument("--note", default="")
    a = ap.parse_args()
    ks = raw_metrics(a.report)
    k = ks[0]

    def val(name):
        m = k.get(name)
        if not m:
            return None
        v = float(m["value"].replace(",", ""))
        return v * UNIT_SCALE.get(m["unit"], 1)

    dram = (val("dram__bytes_read.sum") or 0) + (val("dram__bytes_write.sum") or 0)
    dur = val("gpu__time_duration.sum")
    summary = {"kernel": k["kernel"], "duration_s": dur, "dram_bytes_per_launch": dram,
               "dram_gbs": dram / dur / 1e9 if dur else None, "metrics": {n: k.get(n) for n in KEYS if n in k},
               "note": a.note}
    if a.bytes:
        summary["algorithmic_bytes_per_launch"] = a.bytes
        summary["traffic_over_algorithmic"] = dram / a.bytes
    top, ops = top_sass(a.report)
    summary["sass"] = ops
    lines = []
    if a.launch_csv:
        L = launches(a.launch_csv)
        summary["launch_list"] = [{"kernel": n[:90], "ns": v} for n, v, _ in L]
    json.dump(summary, open(a.out + ".json", "w"), indent=1)
    md = [f"# ncu summary: `{k['kernel'][:100]}`", "", a.note, "",
          "| metric | value |", "|---|---|"]
    for n in KEYS:
        if n in k:
            md.append(f"| {n} | {k[n]['value']} {k[n]['unit']} |")
    md.append(f"| dram bytes / launch | {dram:.4g} |")
    if a.bytes:
        md.append(f"| algorithmic bytes / launch | {a.bytes:.4g} (traffic/algorithmic = {dram / a.bytes:.3f}) |")
    md += ["", "## instruction mix (executed warp instructions by opcode)", "",
           f"total: {ops.get('instructions')}", ""]
    for op, c in ops.get("by_opcode", []):
        md.append(f"- {op}: {c}")
    md += ["", "## top SASS by warp-stall samples", "", "| samples | executed | sass |", "|---|---|---|"]
    for i, s, src in top:
        md.append(f"| {s} | {i} | `{src.strip()[:80]}` |")
    if a.launch_csv:
        md += ["", "## launch list (ncu --metrics gpu__time_duration.sum, cold-cache, serialised)", "",
               "| kernel | ns |", "|---|---|"]
        for n, v, _ in launches(a.launch_csv):
            md.append(f"| `{n[:80]}` | {v:.0f} |")
    open(a.out + ".md", "w").write("\n".join(md) + "\n")
    print(json.dumps({kk: summary[kk] for kk in ("kernel", "duration_s", "dram_bytes_per_launch", "dram_gbs")}))


if __name__ == "__main__":
    main()
