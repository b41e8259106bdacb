"""Reference-algorithm CPU rate per configuration on all host cores (bounded
sample): each worker runs the oracle port of the reference's implicit Euler
(timeint.py:88-111: one factorisation per solve — dense LU at 32^2 as
shipped, splu beyond) for a few steps of one sample at the
config's level-0 dt, including the per-solve factorisation.  Reported as
sample-timesteps/s (no Parareal redundancy, so an upper bound for the
reference on the configs that use Parareal).  Test/measurement infrastructure:
the oracle is the CPU reference here, not the product.

usage: python scripts/cpu_rates.py [CFG ...]"""
import json
import os
import sys
import time
from concurrent.futures import ProcessPoolExecutor

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")

STEPS = {0: 32, 1: 64, 2: 8, 3: 16, 4: 4}


def _init():
    try:
        from threadpoolctl import threadpool_limits
        threadpool_limits(1)
    except Exception:
        pass


def _one(args):
    from oracle import ie_oracle as ie
    from oracle import mlmc_oracle as mo
    cfg_i, k, n_steps = args
    cfg = mo.CONFIGS[cfg_i]
    prob = mo.FEProblem(cfg.n, cfg.layout)
    model = prob.model(mo.draw(cfg, 0, 0, k))
    dt = cfg.dts[0]
    t = time.perf_counter()
    ie.propagate(model, 0.0, n_steps * dt, dt, model.initial_state)
    t1 = time.perf_counter() - t
    t = time.perf_counter()
    ie.propagate(model, 0.0, 2 * n_steps * dt, dt, model.initial_state)
    t2 = time.perf_counter() - t
    return t1, t2


def main(cfgs):
    cores = os.cpu_count() or 1
    for c in cfgs:
        n = STEPS[c]
        jobs = [(c, k, n) for k in range(1, 2 * cores + 1)]
        with ProcessPoolExecutor(max_workers=cores, initializer=_init) as pool:
            list(pool.map(_one, [(c, 1, 1)] * cores))
            t = time.perf_counter()
            res = list(pool.map(_one, jobs, chunksize=1))
            wall = time.perf_counter() - t
        from oracle import mlmc_oracle as mo
        cfg = mo.CONFIGS[c]
        per_step = sum(t2 - t1 for t1, t2 in res) / (len(res) * n)   # one core
        fact = max(0.0, sum(t1 for t1, _ in res) / len(res) - n * per_step)
        n_full = int(round(cfg.horizon / cfg.dts[0]))
        rate = cores * n_full / (fact + n_full * per_step)    # a full level-0 solve per core
        print(json.dumps({"config": c, "cores": cores,
                          "sample": f"{len(jobs)} samples x ({n} + {2 * n}) steps at dt_0, "
                                    f"extrapolated to full {n_full}-step solves",
                          "per_step_s": per_step, "factorize_s": fact,
                          "sample_timesteps_per_s": rate, "wall_s": wall}), flush=True)


if __name__ == "__main__":
    main([int(a) for a in sys.argv[1:]] or [0, 1, 2, 3, 4])
