"""Timeline of one config-2 estimate with two run_levels calls in flight: the
band launches and the spans of the other kernels (grouped per stream while no
band launch of that stream intervenes), from a CUPTI trace (torch.profiler).
usage: python scripts/call_timeline.py [CFG=2] [OUT.json]"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2507_19246_b200.configs import get_config  # noqa: E402
from paper_2507_19246_b200.mlmc import shard_range  # noqa: E402
from paper_2507_19246_b200.models import eddy_current_family  # noqa: E402


def main():
    cfg_i = int(sys.argv[1]) if len(sys.argv) > 1 else 2
    out = sys.argv[2] if len(sys.argv) > 2 else None
    dev = torch.device("cuda", 0)
    cfg = get_config(cfg_i)
    counts = list(cfg.samples)
    fam = eddy_current_family(cfg_i, device=dev)
    est = bench.DeviceEstimate(fam, cfg, [shard_range(n, 0, 1) for n in counts], counts,
                               cfg.parareal_config(), None, dev)
    est()
    torch.cuda.synchronize()
    from torch.profiler import ProfilerActivity, profile
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        t0 = time.perf_counter()
        est()
        torch.cuda.synchronize()
        wall = time.perf_counter() - t0
    ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
    ev.sort(key=lambda e: e.time_range.start)
    base = ev[0].time_range.start
    rows = []
    open_span = {}
    for e in ev:
        name = e.name.replace("(anonymous namespace)::", "").replace("void ", "").split("(")[0]
        name = name.replace("mlmcp::", "")
        s, t = (e.time_range.start - base) / 1e3, (e.time_range.end - base) / 1e3
        strm = getattr(e, "device_index", None), getattr(e, "stream", None)
        try:
            strm = e.device_resource_id
        except Exception:
            strm = str(strm)
        if name.startswith("band_propagate"):
            open_span.pop(strm, None)
            rows.append({"kind": "band", "stream": strm, "start_ms": s, "end_ms": t})
        else:
            grp = "periodic" if name[:2] in ("ps", "pu", "pp", "pi", "pf") else "other"
            key = (strm, grp)
            sp = open_span.get(strm)
            if sp is None or sp["kind"] != grp:
                sp = {"kind": grp, "stream": strm, "start_ms": s, "end_ms": t, "kernels": 0,
                      "busy_ms": 0.0}
                open_span[strm] = sp
                rows.append(sp)
            sp["end_ms"] = max(sp["end_ms"], t)
            sp["kernels"] += 1
            sp["busy_ms"] += t - s
    rows = [r for r in rows if r["kind"] != "other" or r["busy_ms"] > 0.5]
    for r in rows:
        extra = "" if r["kind"] == "band" else f"  {r['kernels']} kernels busy {r['busy_ms']:.1f} ms"
        print(f"{r['kind']:9s} stream {r['stream']}  {r['start_ms']:9.1f} -> {r['end_ms']:9.1f} ms"
              f"  ({r['end_ms'] - r['start_ms']:8.1f}){extra}")
    print(json.dumps({"wall_ms_under_profiler": wall * 1e3}))
    if out:
        with open(out, "w") as fh:
            json.dump({"config": cfg_i, "wall_ms_under_profiler": wall * 1e3, "timeline": rows},
                      fh, indent=1)


if __name__ == "__main__":
    main()
