"""Per-source-line stall / instruction shares of one kernel in an ncu report
(--page source --print-source cuda,sass).  usage: python scripts/ncu_lines.py REPORT [N]"""
import csv
import subprocess
import sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(txt.splitlines()))
fname, hdr, agg = "?", None, []
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
    elif r[0] == "Line No":
        hdr = r
    elif hdr and r[0].isdigit():
        off = len(r) - len(hdr)          # source text with unescaped quotes splits into extra fields
        s = float(r[off + hdr.index("Warp Stall Sampling (All Samples)")] or 0)
        i = float(r[off + hdr.index("Instructions Executed")] or 0)
        agg.append((s, i, fname, int(r[0]), ",".join(r[1:2 + off]).strip()))
ts = sum(a[0] for a in agg) or 1
ti = sum(a[1] for a in agg) or 1
for s, i, f, ln, src in sorted(agg, reverse=True)[:n]:
    print(f"{100 * s / ts:5.1f}% stall {100 * i / ti:5.1f}% inst  {f}:{ln}  {src[:90]}")
