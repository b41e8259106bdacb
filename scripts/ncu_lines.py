"""Aggregate ncu warp-stall samples of a --set full --import-source capture by
CUDA source line: python scripts/ncu_lines.py REPORT.ncu-rep [N]"""
import collections, csv, subprocess, sys
rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
cur_file = cur_line = None
agg = collections.Counter(); srcs = {}; hdr = None
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        cur_file = r[1].split('/')[-1]; continue
    if r and r[0] == "Line No":
        hdr = r; continue
    if hdr is None or len(r) < 5:
        continue
    if r[0]:
        cur_line = (cur_file, int(r[0])); srcs[cur_line] = r[1]
    else:
        try:
            agg[cur_line] += float(r[4] or 0)
        except ValueError:
            pass
T = sum(agg.values()) or 1.0
for k, v in agg.most_common(top):
    print(f"{v / T * 100:5.1f}% {k[0]}:{k[1]}  {srcs.get(k, '')[:90].strip()}")
