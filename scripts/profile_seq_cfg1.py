"""Run the config-1 sequential batch (all levels' sequential solves, one
launch) twice, for an ncu capture of the second launch:
  ncu --set full -k regex:small_propagate -s 1 -c 1 python scripts/profile_seq_cfg1.py"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2507_19246_b200.configs import get_config
from paper_2507_19246_b200.mlmc import draw_level
from paper_2507_19246_b200.models import eddy_current_family

cfg = get_config(1)
fam = eddy_current_family(1, device="cuda:0"); sol = fam.solver
draws = [draw_level(fam.uncertain, 0, l, range(1, n + 1)) for l, n in enumerate(cfg.samples)]
M, K = sol.assemble(torch.from_numpy(np.concatenate(draws)).cuda())
offs = np.cumsum([0] + list(cfg.samples))
jobs = []
for l in range(3):
    rows = np.arange(offs[l], offs[l + 1])
    if l < 2: jobs.append(fam._seq_job(rows, fam.hierarchy[l].dt))
    if l > 0: jobs.append(fam._seq_job(rows, fam.hierarchy[l - 1].dt))
for _ in range(2):
    res = sol.run_sequential(M, K, jobs)
torch.cuda.synchronize()
print("pcg iterations", sum(int(r.iters.to(torch.int64).sum()) for r in res))
