"""TEST INFRASTRUCTURE ONLY — golden fixtures at the BASELINE.json mesh sizes,
produced by the UNMODIFIED reference in the build container.

The reference's own integrators and Parareal driver are run on the oracle's
duck-typed FE models:

  timeint.implicit_euler_solve / propagate     timeint.py:88-128
  parareal.parareal_solve                      parareal.py:121-220 (jump defect :93-103)

with the module globals ``timeint._factorize`` / ``timeint.lu_solve``
(timeint.py:17,64-75,102,110,121,127) replaced by scipy's sparse ``splu`` —
the §8(c) backend substitution for meshes of 128^2 and up.  The factorisation
is cached per (model, dt): the reference refactorises the same M + dt K on every
propagator call, splu is deterministic, so the cache changes the run time and
not one bit of the arithmetic.  QoIs follow oracle/mlmc_oracle.py (1/2 a^T K a;
time average over the last period with right end points).

Written to tests/golden/:
  cfg3_l2_parareal.npz   config 3 finest level, ALL 128 samples (keys
                         (0, 2, 1..128)): Q_l by Parareal (M=32, dt_c=T/32,
                         tol 1e-8, K<=6), Q_{l-1} sequential at T/256, K,
                         defect histories
  cfg3_subset_l01.npz    config 3 levels 0/1, keys 1..16 (level statistics of
                         an N_l = (16, 16, 128) estimate together with the file
                         above)
  cfg4_l3_parareal.npz   config 4 finest level, keys (0, 3, 1..2) at 512^2:
                         Parareal M=64, dt_c=T/64, tol 1e-8, K<=6; Q_{l-1} at T/256
  cfg2_l123.npz          config 2 levels 1..3, keys 1..2 (256^2, 4 periods,
                         time-averaged energy over the last period)

Usage (build container; ~10 min on 8 cores):
    python -m oracle.make_large_goldens [--jobs 8] [--only cfg3|cfg4|cfg2]
"""

from __future__ import annotations

import argparse
import os
import sys
import time
from concurrent.futures import ProcessPoolExecutor

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
GOLDEN = os.path.join(ROOT, "tests", "golden")
REF_SRC = "/root/reference/pkg/src"

_STATE = {}


def _reference():
    """Import the unmodified reference and install the cached splu backend."""
    if "mods" in _STATE:
        return _STATE["mods"]
    if not os.path.isdir(REF_SRC):
        raise SystemExit("reference not present: make_large_goldens runs in the build container")
    os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
    sys.path.insert(0, REF_SRC)
    sys.path.insert(0, ROOT)
    import scipy.sparse as sp
    from mlmc_parareal import parareal, timeint
    from scipy.sparse.linalg import splu

    cache = {}

    def factorize(model, dt):
        # keyed by the model OBJECT (kept alive in the entry): an id() alone can
        # be reused by the next sample's model once the previous one is freed
        key = (id(model), float(dt))
        hit = cache.get(key)
        if hit is not None and hit[0] is model:
            return hit[1]
        if len(cache) > 8:
            cache.clear()
        lu = splu(sp.csc_matrix(model.mass + dt * model.stiffness))
        cache[key] = (model, lu)
        return lu

    _STATE["cache"] = cache

    timeint._factorize = factorize
    timeint.lu_solve = lambda lu, rhs: lu.solve(rhs)
    _STATE["mods"] = (timeint, parareal)
    return _STATE["mods"]


def _problem(cfg):
    from oracle import mlmc_oracle as mo
    key = (cfg.n, cfg.layout)
    if key not in _STATE:
        _STATE[key] = mo.FEProblem(cfg.n, cfg.layout)
    return _STATE[key]


def _seq_q(cfg, model, dt):
    from oracle import mlmc_oracle as mo
    timeint, _ = _reference()
    tr = timeint.implicit_euler_solve(model, 0.0, cfg.horizon, dt, model.initial_state)
    if cfg.qoi == "energy_T":
        return mo.energy(model, tr.states[-1])
    n_t = len(tr.states) - 1
    n_w = int(round(cfg.avg_window / dt))
    acc = 0.0
    for k in range(n_t - n_w + 1, n_t + 1):      # right end points of the last window
        acc += mo.energy(model, tr.states[k])
    return acc * dt / cfg.avg_window


def coupled_job(args):
    """(Q_l, Q_{l-1}, K, defects) of key (0, level, k) by the reference."""
    try:
        return _coupled_job(args)
    except Exception as exc:       # reference exception types do not unpickle in the parent
        raise RuntimeError(f"job {args} failed: {type(exc).__name__}: {exc}") from None


def _coupled_job(args):
    cfg_i, level, k = args
    from oracle import mlmc_oracle as mo
    timeint, parareal = _reference()
    _STATE["cache"].clear()
    cfg = mo.CONFIGS[cfg_i]
    prob = _problem(cfg)
    p = mo.draw(cfg, 0, level, k)
    model = prob.model(p, dense=False)
    t = time.perf_counter()
    top = len(cfg.dts) - 1
    kk, defects = -1, []
    if cfg.parareal is not None and level == top:
        m, dtc, tol, kmax = cfg.parareal
        res = parareal.parareal_solve(model, 0.0, cfg.horizon, model.initial_state,
                                      parareal.PararealConfig(m, cfg.dts[level], dtc, tol, kmax))
        q_l = mo.energy(model, res.boundary_states[-1])       # F_M (parareal.py:209-210)
        kk = res.iterations_used
        defects = list(res.defect_history)
    else:
        q_l = _seq_q(cfg, model, cfg.dts[level])
    q_lm1 = _seq_q(cfg, model, cfg.dts[level - 1]) if level > 0 else 0.0
    return cfg_i, level, k, p, q_l, q_lm1, kk, defects, time.perf_counter() - t


def _write(name, rows, kmax=0):
    rows = sorted(rows, key=lambda r: (r[1], r[2]))
    out = {"level": np.array([r[1] for r in rows]), "k": np.array([r[2] for r in rows]),
           "params": np.array([r[3] for r in rows]), "q_l": np.array([r[4] for r in rows]),
           "q_lm1": np.array([r[5] for r in rows]), "k_used": np.array([r[6] for r in rows])}
    if kmax:
        d = np.full((len(rows), kmax), np.nan)
        for i, r in enumerate(rows):
            d[i, :len(r[7])] = r[7]
        out["defects"] = d
    out["generator"] = np.array("unmodified reference (timeint/parareal) + cached splu backend")
    np.savez(os.path.join(GOLDEN, name + ".npz"), **out)
    print(f"  wrote {name}.npz ({len(rows)} samples)", flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--jobs", type=int, default=os.cpu_count() or 1)
    ap.add_argument("--only", default=None)
    args = ap.parse_args()
    os.makedirs(GOLDEN, exist_ok=True)
    groups = {
        "cfg4": [("cfg4_l3_parareal", [(4, 3, k) for k in (1, 2)], 6)],
        "cfg3": [("cfg3_l2_parareal", [(3, 2, k) for k in range(1, 129)], 6),
                 ("cfg3_subset_l01", [(3, lvl, k) for lvl in (0, 1) for k in range(1, 17)], 0)],
        "cfg2": [("cfg2_l123", [(2, lvl, k) for lvl in (1, 2, 3) for k in (1, 2)], 0)],
    }
    todo = [g for key, gs in groups.items() if args.only in (None, key) for g in gs]
    jobs = [(name, j) for name, js, _ in todo for j in js]
    # longest first (512^2 Parareal, then the 256^2 four-period levels)
    jobs.sort(key=lambda x: -({4: 100, 2: 10, 3: 1}[x[1][0]] * (x[1][1] + 1)))
    results = {name: [] for name, _, _ in todo}
    t0 = time.perf_counter()
    with ProcessPoolExecutor(max_workers=args.jobs) as pool:
        for name, r in zip([n for n, _ in jobs], pool.map(coupled_job, [j for _, j in jobs])):
            results[name].append(r)
            print(f"  {name} l={r[1]} k={r[2]} q_l={r[4]:.15e} K={r[6]} ({r[8]:.1f} s, "
                  f"{time.perf_counter() - t0:.0f} s total)", flush=True)
    for name, _, kmax in todo:
        _write(name, results[name], kmax)


if __name__ == "__main__":
    main()
