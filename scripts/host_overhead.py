"""Host-side cost of one config-1 estimate through mlmc_estimate: draws,
launch preparation, device time, post-processing."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2507_19246_b200.configs import get_config
from paper_2507_19246_b200.mlmc import FixedSamples, draw_level, mlmc_estimate
from paper_2507_19246_b200.models import eddy_current_family
cfg = get_config(1); pcfg = cfg.parareal_config()
fam = eddy_current_family(1, device="cuda:0")
for rep in range(4):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    draws = [draw_level(fam.uncertain, 0, l, range(1, n + 1)) for l, n in enumerate(cfg.samples)]
    t1 = time.perf_counter()
    out = fam.run_levels(draws, pcfg)
    t2 = time.perf_counter()
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    res = mlmc_estimate(fam, policy=FixedSamples(cfg.samples), parareal_cfg=pcfg, seed=0)
    torch.cuda.synchronize()
    t4 = time.perf_counter()
    print(f"draws {1e3*(t1-t0):.2f} ms, run_levels host {1e3*(t2-t1):.2f} ms, wait {1e3*(t3-t2):.2f} ms, full mlmc_estimate {1e3*(t4-t3):.2f} ms")
import cProfile, pstats
pr = cProfile.Profile(); pr.enable()
res = mlmc_estimate(fam, policy=FixedSamples(cfg.samples), parareal_cfg=pcfg, seed=0)
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(18)
