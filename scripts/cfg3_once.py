"""One config-3 estimate (for an ncu launch list)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2507_19246_b200.configs import get_config
from paper_2507_19246_b200.mlmc import FixedSamples, mlmc_estimate
from paper_2507_19246_b200.models import eddy_current_family
cfg = get_config(3)
fam = eddy_current_family(3, device="cuda:0")
t = time.perf_counter()
res = mlmc_estimate(fam, policy=FixedSamples(tuple(cfg.samples)), parareal_cfg=cfg.parareal_config(), seed=0)
torch.cuda.synchronize()
print("wall", time.perf_counter() - t, res.expectation)
