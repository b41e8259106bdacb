"""Aggregate an ncu launch list (--metrics gpu__time_duration.sum --csv) by
kernel: launches, total ms and share of the listed device time.
usage: python scripts/ncu_share.py LAUNCHES.csv [OUT.json]"""
import csv
import json
import re
import sys


def main(path, out=None):
    rows = []
    with open(path) as fh:
        lines = [ln for ln in fh if ln.startswith('"')]
    for r in csv.DictReader(lines):
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = r["Kernel Name"]
        name = re.sub(r"\(.*", "", name)
        name = re.sub(r"^void ", "", name).replace("(anonymous namespace)::", "")
        unit = r.get("Metric Unit", "ns")
        v = float(r["Metric Value"].replace(",", ""))
        scale = {"ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0,
                 "nsecond": 1e-6, "second": 1e3}.get(unit, 1e-6)
        rows.append((name, v * scale))
    agg = {}
    for n, ms in rows:
        a = agg.setdefault(n, [0, 0.0])
        a[0] += 1
        a[1] += ms
    tot = sum(v[1] for v in agg.values()) or 1.0
    res = [{"kernel": k, "launches": v[0], "ms": round(v[1], 4), "share": round(v[1] / tot, 4)}
           for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1])]
    for r in res:
        print(f"{r['share']:7.2%} {r['ms']:10.3f} ms {r['launches']:6d}  {r['kernel'][:100]}")
    if out:
        with open(out, "w") as fh:
            json.dump({"source": path, "total_ms": tot, "kernels": res}, fh, indent=1)


if __name__ == "__main__":
    main(*sys.argv[1:])
