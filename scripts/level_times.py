"""Per-level wall time of one configuration's estimate (each level's coupled
batch run on its own, after a warm-up): where the time of configs 2-4 goes.
usage: python scripts/level_times.py CFG"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2507_19246_b200.configs import get_config
from paper_2507_19246_b200.mlmc import draw_level
from paper_2507_19246_b200.models import eddy_current_family
cfg_i = int(sys.argv[1])
cfg = get_config(cfg_i)
pcfg = cfg.parareal_config()
fam = eddy_current_family(cfg_i, device="cuda:0")
fam.run_levels([draw_level(fam.uncertain, cfg.seed, 0, range(1, 3))], pcfg, levels=[0])
for lvl, n in enumerate(cfg.samples):
    d = draw_level(fam.uncertain, cfg.seed, lvl, range(1, n + 1))
    torch.cuda.synchronize(); t = time.perf_counter()
    b = fam.run_levels([d], pcfg, levels=[lvl])[0]
    torch.cuda.synchronize(); w = time.perf_counter() - t
    steps = n * (cfg.steps(lvl) + (cfg.steps(lvl - 1) if lvl > 0 else 0))
    print(f"cfg{cfg_i} level {lvl}: N={n} dt=T/{round(cfg.horizon / cfg.dts[lvl] * (1 if cfg_i != 2 else 1))} "
          f"{w:.2f} s, {steps / w / 1e3:.1f} k seq-equiv sample-steps/s"
          + (f", Parareal K {sorted(set(b.k_used.cpu().tolist()))}" if pcfg is not None and lvl == cfg.levels - 1 else ""),
          flush=True)
