"""Device-time breakdown of one full MLMC estimate (bench.py's step) by kernel,
from a CUPTI trace (torch.profiler): per-kernel launches / total ms / share of
the estimate's wall time, the busy time (union of kernel intervals) and the
idle gaps between kernels.  A number taken under the profiler is never a
bench value; this is only the shares.
usage: python scripts/kernel_breakdown.py [CFG=2] [OUT.json]"""
import json
import os
import sys
import time
from collections import defaultdict

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
    with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
        t0 = time.perf_counter()
        est()
        torch.cuda.synchronize()
        wall = time.perf_counter() - t0
    ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
    agg = defaultdict(lambda: [0, 0.0])
    iv = []
    for e in ev:
        name = e.name.replace("(anonymous namespace)::", "").replace("void ", "").split("(")[0]
        if name.startswith("Memcpy") or name.startswith("Memset"):
            name = name.split(" ")[0]
        dur = e.time_range.end - e.time_range.start     # us
        agg[name][0] += 1
        agg[name][1] += dur
        iv.append((e.time_range.start, e.time_range.end))
    iv.sort()
    busy, cur_s, cur_e = 0.0, None, None
    for s, e in iv:
        if cur_e is None or s > cur_e:
            if cur_e is not None:
                busy += cur_e - cur_s
            cur_s, cur_e = s, e
        else:
            cur_e = max(cur_e, e)
    if cur_e is not None:
        busy += cur_e - cur_s
    span = (iv[-1][1] - iv[0][0]) if iv else 0.0
    rows = sorted(agg.items(), key=lambda kv: -kv[1][1])
    res = {"config": cfg_i, "wall_ms_under_profiler": wall * 1e3, "kernel_span_ms": span / 1e3,
           "busy_ms": busy / 1e3, "idle_ms": (span - busy) / 1e3, "launches": len(ev),
           "kernels": [{"name": k, "launches": v[0], "ms": v[1] / 1e3,
                        "share_of_span": v[1] / span if span else None} for k, v in rows]}
    for r in res["kernels"][:20]:
        print(f"{r['share_of_span'] * 100:6.2f}%  {r['ms']:10.2f} ms  {r['launches']:7d}  {r['name'][:90]}")
    print(json.dumps({k: v for k, v in res.items() if k != "kernels"}))
    if out:
        with open(out, "w") as fh:
            json.dump(res, fh, indent=1)


if __name__ == "__main__":
    main()
