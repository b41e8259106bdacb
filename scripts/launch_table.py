"""Per-kernel totals of an ncu --metrics gpu__time_duration.sum,dram__bytes_*
--csv launch list: python scripts/launch_table.py LAUNCHES.csv"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
h = rows[hi]
ki, mi, vi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
agg = collections.defaultdict(lambda: collections.defaultdict(float))
cnt = collections.Counter()
for r in rows[hi + 1:]:
    if len(r) <= vi:
        continue
    name = r[ki].split("(")[0].split("::")[-1][:40]
    agg[name][r[mi]] += float(r[vi].replace(",", ""))
    if r[mi] == "gpu__time_duration.sum":
        cnt[name] += 1
tot = sum(d["gpu__time_duration.sum"] for d in agg.values())
for n, d in sorted(agg.items(), key=lambda x: -x[1]["gpu__time_duration.sum"]):
    t = d["gpu__time_duration.sum"]
    b = d.get("dram__bytes_read.sum", 0) + d.get("dram__bytes_write.sum", 0)
    print(f"{n:40s} n={cnt[n]:5d} t={t / 1e6:8.3f} ms ({100 * t / tot:4.1f}%) avg={t / cnt[n] / 1e3:8.1f} us"
          f"  dram/launch={b / cnt[n] / 1e6:8.1f} MB  {b / t if t else 0:6.0f} GB/s")
