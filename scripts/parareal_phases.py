"""Where the time of a streaming-path Parareal batch goes: device time of the
coarse sweeps, the fine-slice launches and the defect launches per Parareal
iteration (CUDA events around each phase), plus the fine PCG iterations.
usage: python scripts/parareal_phases.py [CFG=4] [S=16]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2507_19246_b200.configs import get_config  # noqa: E402
from paper_2507_19246_b200.mlmc import draw_level  # noqa: E402
from paper_2507_19246_b200.models import eddy_current_family  # noqa: E402

cfg_i = int(sys.argv[1]) if len(sys.argv) > 1 else 4
S = int(sys.argv[2]) if len(sys.argv) > 2 else 16
cfg = get_config(cfg_i)
pcfg = cfg.parareal_config()
fam = eddy_current_family(cfg_i, device="cuda:0")
top = cfg.levels - 1
d = draw_level(fam.uncertain, cfg.seed, top, range(1, S + 1))
sysobj = fam.solver.sys
ev = []


def wrap(name):
    fn = getattr(sysobj, name)

    def w(*a, **k):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        r = fn(*a, **k)
        e1.record()
        its = None
        if name == "propagate" and len(a) > 9 and a[9] is not None:
            slots = torch.from_numpy(np.asarray(a[0]["slot"], dtype=np.int64)).to(a[9].device)
            its = a[9].index_select(0, slots.clamp(min=0))     # this call's PCG iterations per task
        ev.append((name, e0, e1, its))
        return r
    setattr(sysobj, name, w)


for n in ("parareal_coarse", "propagate", "parareal_defect", "parareal_finalize"):
    wrap(n)
for rep in range(2):
    ev.clear()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    b = fam.run_levels([d], pcfg, levels=[top], _no_chunk=True)[0]
    e1.record()
    torch.cuda.synchronize()
fam.check_status()
tot = {}
per_k = []
k = 0
for name, a, z, its in ev:
    ms = a.elapsed_time(z)
    tot[name] = tot.get(name, 0.0) + ms
    if name == "parareal_coarse":
        k += 1
        per_k.append({"k": k, "coarse_ms": ms})
    elif name == "propagate" and per_k:
        per_k[-1]["fine_ms"] = per_k[-1].get("fine_ms", 0.0) + ms
        if its is not None:
            per_k[-1]["fine_tasks"] = int(its.numel())
            per_k[-1]["fine_pcg_iters"] = int(its.sum())
print(json.dumps({"config": cfg_i, "S": S, "total_ms": e0.elapsed_time(e1),
                  "phase_ms": tot, "per_k": per_k,
                  "k_used": sorted(set(b.k_used.cpu().tolist())),
                  "fine_iters": int(fam.solver._last_fine_iters) if hasattr(fam.solver, "_last_fine_iters") else None,
                  "q": b.q_l.cpu().tolist()[:4]}))
