"""Per-source-line warp-stall samples and executed instructions from an ncu report (--import-source on).

usage: python tools/ncu_lines.py REPORT.ncu-rep [N]
"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True, check=True).stdout
stall, inst, fname = {}, {}, None
for r in csv.reader(io.StringIO(out)):
    if r and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if len(r) < 8 or not r[0] or r[0] == "Line No":
        continue
    try:
        s, ie = float(r[4] or 0), float(r[7] or 0)
    except ValueError:
        continue
    k = (fname, r[0], r[1].strip()[:96])
    stall[k] = stall.get(k, 0) + s
    inst[k] = inst.get(k, 0) + ie
ts, ti = sum(stall.values()) or 1, sum(inst.values()) or 1
print(f"stall samples {ts:.0f}, warp instructions {ti:.0f}")
for k, v in sorted(stall.items(), key=lambda x: -x[1])[:n]:
    print(f"{100 * v / ts:5.1f}% stall {100 * inst[k] / ti:5.1f}% inst  {k[0]}:{k[1]}  {k[2]}")
