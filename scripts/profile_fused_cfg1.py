"""Two config-1 estimates through run_levels (fused scheduler) for an ncu
capture of the second fused launch:
  ncu --set full -k regex:fused_kernel -s 2 -c 1 python scripts/profile_fused_cfg1.py"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2507_19246_b200.configs import get_config
from paper_2507_19246_b200.mlmc import draw_level
from paper_2507_19246_b200.models import eddy_current_family
cfg = get_config(1); pcfg = cfg.parareal_config()
fam = eddy_current_family(1, device="cuda:0")
draws = [draw_level(fam.uncertain, 0, l, range(1, n + 1)) for l, n in enumerate(cfg.samples)]
P = torch.from_numpy(np.concatenate(draws)).cuda()
for _ in range(2):
    out = fam.run_levels(draws, pcfg, params_dev=P)
torch.cuda.synchronize()
print("K", sorted(set(out[-1].k_used.cpu().tolist())))
