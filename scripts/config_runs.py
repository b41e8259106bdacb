"""One full MLMC(+Parareal) estimate of each BASELINE.json configuration on one
B200 through the public API (mlmc_estimate, host draws included): wall time and
sequential-equivalent sample-timesteps/s.  A small estimate of the same family
first initialises the context (not timed).

usage: python scripts/config_runs.py [CFG ...]   (default: 0 1 2 3 4)"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2507_19246_b200.configs import get_config
from paper_2507_19246_b200.mlmc import FixedSamples, mlmc_estimate
from paper_2507_19246_b200.models import eddy_current_family


def run(cfg_i):
    cfg = get_config(cfg_i)
    pcfg = cfg.parareal_config()
    fam = eddy_current_family(cfg_i, device="cuda:0")
    mlmc_estimate(fam, policy=FixedSamples(tuple(min(n, 2) for n in cfg.samples)),
                  parareal_cfg=pcfg, seed=cfg.seed)
    import bench
    clocks = bench.ClockSampler()     # nvidia-smi clocks / throttle reasons during the calls
    clocks.start()
    walls = []
    while True:   # configs that finish in seconds: a second (warm) call is the one reported
        torch.cuda.synchronize()
        t = time.perf_counter()
        res = mlmc_estimate(fam, policy=FixedSamples(tuple(cfg.samples)), parareal_cfg=pcfg,
                            seed=cfg.seed)
        torch.cuda.synchronize()
        walls.append(time.perf_counter() - t)
        if len(walls) == 2 or walls[0] > 5.0:
            break
    clk = clocks.stop(torch.cuda.current_device())
    wall = walls[-1]
    steps = cfg.seq_equiv_steps(1)
    ks = sorted({int(k) for lv in res.per_level for k in (getattr(lv, "parareal_k", None) or [])})
    return {"config": cfg_i, "mesh": f"{cfg.n}x{cfg.n}", "N_l": list(cfg.samples),
            "parareal": list(cfg.parareal) if cfg.parareal else None,
            "expectation": res.expectation, "rmse_estimate": res.rmse_estimate,
            "wall_s": wall, "seq_equiv_sample_timesteps": steps,
            "sample_timesteps_per_s": steps / wall, "parareal_k_values": ks,
            "calls_s": walls, "gpus": 1, "clocks": clk}


if __name__ == "__main__":
    cfgs = [int(c) for c in sys.argv[1:]] or [0, 1, 2, 3, 4]
    for c in cfgs:
        print(json.dumps(run(c)), flush=True)
