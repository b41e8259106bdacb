"""Per-launch device timeline of the config-1 finest-level Parareal (32
samples, M=16) run alone: coarse sweeps, fine launches, defects, with PCG
iteration counts.  Usage: python scripts/parareal_timeline.py"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2507_19246_b200.configs import get_config
from paper_2507_19246_b200.mlmc import draw_level
from paper_2507_19246_b200.models import eddy_current_family

cfg = get_config(1); pcfg = cfg.parareal_config()
fam = eddy_current_family(1, device="cuda:0"); sol = fam.solver
P = draw_level(fam.uncertain, 0, 2, range(1, 33))
M, K = sol.assemble(torch.from_numpy(P).cuda())
marks = []
for name in ("parareal_coarse", "propagate", "parareal_defect", "parareal_finalize"):
    orig = getattr(sol.sys, name)
    def wrap(*a, _orig=orig, _name=name, **kw):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); r = _orig(*a, **kw); e1.record()
        marks.append((_name, e0, e1)); return r
    setattr(sol.sys, name, wrap)
for rep in range(3):
    marks.clear()
    t0 = torch.cuda.Event(enable_timing=True); t1 = torch.cuda.Event(enable_timing=True)
    t0.record()
    pr = sol.run_parareal(M, K, 0.0, cfg.horizon, pcfg.num_subintervals, pcfg.dt_fine,
                          pcfg.dt_coarse, pcfg.tolerance, pcfg.k_max)
    t1.record(); torch.cuda.synchronize()
print("total %.3f ms, K=%s" % (t0.elapsed_time(t1), sorted(set(pr.k_used.cpu().tolist()))))
for name, a, b in marks:
    print("  %-18s %.3f ms" % (name, a.elapsed_time(b)))
print("coarse PCG iterations per sample:", pr.coarse_iters.cpu().numpy()[:4], "fine total", int(pr.fine_iters.sum()))
fi = pr.fine_iters.cpu().numpy().reshape(32, 16)
print("fine PCG iterations per slice (sum over iterations), sample 0:", fi[0].tolist())
print("max / mean per task:", fi.max(), fi.mean())
for kmax in (1,):
    marks.clear()
    pr1 = sol.run_parareal(M, K, 0.0, cfg.horizon, 16, pcfg.dt_fine, pcfg.dt_coarse, 1e-30, 1)
    torch.cuda.synchronize()
    f1 = pr1.fine_iters.cpu().numpy().reshape(32, 16)
    print("k=1 only: fine its per slice sample0:", f1[0].tolist(), "max", f1.max(), "mean", f1.mean())
    for name, a, b in marks:
        print("  %-18s %.3f ms" % (name, a.elapsed_time(b)))
# sequential single-level launch for comparison: 32 samples x 1024 steps at dt_fine
from paper_2507_19246_b200.solver import SeqJob
import paper_2507_19246_b200._lib as L
marks.clear()
jobs = [fam._seq_job(np.arange(32), pcfg.dt_fine)]
for _ in range(2):
    marks.clear()
    r = sol.run_sequential(M, K, jobs)
torch.cuda.synchronize()
its = int(r[0].iters.sum())
for name, a, b in marks:
    ms = a.elapsed_time(b)
    print("  seq 32 x 1024 steps: %-12s %.3f ms, %d its (%.1f/step), %.0f cycles/step/task" % (name, ms, its, its/32/1024, ms*1e-3*1.965e9/1024))
