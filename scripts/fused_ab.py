"""A/B: config-1 sequential batch through small_propagate_kernel vs the fused
scheduler with no Parareal; then the full fused estimate vs separate launches."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2507_19246_b200.configs import get_config
from paper_2507_19246_b200.mlmc import draw_level
from paper_2507_19246_b200.models import eddy_current_family

cfg = get_config(1); pcfg = cfg.parareal_config()
fam = eddy_current_family(1, device="cuda:0"); sol = fam.solver
draws = [draw_level(fam.uncertain, 0, l, range(1, n + 1)) for l, n in enumerate(cfg.samples)]
P = torch.from_numpy(np.concatenate(draws)).cuda()
M, K = sol.assemble(P)
offs = np.cumsum([0] + list(cfg.samples))
jobs = []
for l in range(3):
    rows = np.arange(offs[l], offs[l + 1])
    if l < 2: jobs.append(fam._seq_job(rows, fam.hierarchy[l].dt))
    if l > 0: jobs.append(fam._seq_job(rows, fam.hierarchy[l - 1].dt))

def timed(fn, reps=5):
    ts = []
    for r in range(reps + 2):
        torch.cuda.synchronize(); a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record(); torch.cuda.synchronize()
        if r >= 2: ts.append(a.elapsed_time(b))
    return float(np.median(ts))

print("seq via small_propagate %.2f ms" % timed(lambda: sol.run_sequential(M, K, jobs)))
print("seq via fused (no Parareal) %.2f ms" % timed(lambda: sol.run_fused(M, K, jobs, None)))
print("run_levels fused %.2f ms" % timed(lambda: fam.run_levels(draws, pcfg, params_dev=P, fused=True)))
print("run_levels separate %.2f ms" % timed(lambda: fam.run_levels(draws, pcfg, params_dev=P, fused=False)))
