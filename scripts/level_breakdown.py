"""Device-time breakdown (CUPTI, torch.profiler) of one level of a configuration's
estimate, e.g. config 4's Parareal level: per-kernel launches / ms / share of
the level's kernel span, busy time and idle gaps between kernels.
usage: python scripts/level_breakdown.py CFG LEVEL [N_SAMPLES] [OUT.json]"""
import json
import os
import sys
import time
from collections import defaultdict

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2507_19246_b200.configs import get_config  # noqa: E402
from paper_2507_19246_b200.mlmc import draw_level  # noqa: E402
from paper_2507_19246_b200.models import eddy_current_family  # noqa: E402


def main():
    cfg_i, lvl = int(sys.argv[1]), int(sys.argv[2])
    cfg = get_config(cfg_i)
    n = int(sys.argv[3]) if len(sys.argv) > 3 else cfg.samples[lvl]
    out = sys.argv[4] if len(sys.argv) > 4 else None
    pcfg = cfg.parareal_config()
    fam = eddy_current_family(cfg_i, device="cuda:0")
    fam.run_levels([draw_level(fam.uncertain, cfg.seed, lvl, range(1, 3))], pcfg, levels=[lvl])
    d = draw_level(fam.uncertain, cfg.seed, lvl, range(1, n + 1))
    torch.cuda.synchronize()
    from torch.profiler import ProfilerActivity, profile
    with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
        t0 = time.perf_counter()
        b = fam.run_levels([d], pcfg, levels=[lvl])[0]
        torch.cuda.synchronize()
        wall = time.perf_counter() - t0
    ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
    agg = defaultdict(lambda: [0, 0.0])
    iv = []
    for e in ev:
        name = e.name.replace("(anonymous namespace)::", "").replace("void ", "").split("(")[0]
        if name.startswith("Memcpy") or name.startswith("Memset"):
            name = name.split(" ")[0]
        agg[name][0] += 1
        agg[name][1] += e.time_range.end - e.time_range.start
        iv.append((e.time_range.start, e.time_range.end))
    iv.sort()
    busy, cs, ce = 0.0, None, None
    for s, e in iv:
        if ce is None or s > ce:
            if ce is not None:
                busy += ce - cs
            cs, ce = s, e
        else:
            ce = max(ce, e)
    if ce is not None:
        busy += ce - cs
    span = iv[-1][1] - iv[0][0] if iv else 0.0
    rows = sorted(agg.items(), key=lambda kv: -kv[1][1])
    res = {"config": cfg_i, "level": lvl, "samples": n, "wall_ms_under_profiler": wall * 1e3,
           "kernel_span_ms": span / 1e3, "busy_ms": busy / 1e3, "idle_ms": (span - busy) / 1e3,
           "launches": len(ev), "k_used": sorted({int(k) for k in b.k_used.tolist()}),
           "kernels": [{"name": k, "launches": v[0], "ms": v[1] / 1e3} for k, v in rows]}
    for r in res["kernels"][:16]:
        print(f"{r['ms']:10.2f} ms  {r['launches']:7d}  {r['name'][:90]}")
    print(json.dumps({k: v for k, v in res.items() if k != "kernels"}))
    if out:
        with open(out, "w") as fh:
            json.dump(res, fh, indent=1)


if __name__ == "__main__":
    main()
