"""Config 0 (coarse dt, short tasks): is the steady-state predictor worth its
per-(sample, dt) COCG solve there?  Times warm estimates with it on / off."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2507_19246_b200.configs import get_config
from paper_2507_19246_b200.mlmc import FixedSamples, mlmc_estimate
from paper_2507_19246_b200.models import eddy_current_family

for cfg_i in (0, 1):
    cfg = get_config(cfg_i)
    pcfg = cfg.parareal_config()
    for pred in (True, False):
        fam = eddy_current_family(cfg_i, device="cuda:0")
        fam.solver.predictor = pred
        ts = []
        for r in range(4):
            torch.cuda.synchronize(); t = time.perf_counter()
            res = mlmc_estimate(fam, policy=FixedSamples(tuple(cfg.samples)), parareal_cfg=pcfg, seed=0)
            torch.cuda.synchronize(); ts.append(time.perf_counter() - t)
        its = sum(int(r.iters.to(torch.int64).sum().item()) for r in fam._last[0])
        print(f"cfg{cfg_i} predictor={pred}: {1000*np.median(ts[1:]):.2f} ms  E={res.expectation:.12f}  seq iters={its}", flush=True)
