"""Command-line entry (SPEC.md [MODULE] cli): ``estimate``, ``sample`` and
``plan`` writing the SPEC's on-disk formats.

    python -m paper_2507_19246_b200 estimate CONFIG --out DIR
    python -m paper_2507_19246_b200 sample CONFIG --level L --count C --out DIR
    python -m paper_2507_19246_b200 plan [--r 10 --L 2 --nc 180,360 --K 1..10] --out DIR

CONFIG is ``cfg0`` .. ``cfg4`` (the BASELINE.json FE configurations) or a JSON
file with the SPEC ExperimentConfig fields this build supports:

    {"model": "steinmetz" | "synthetic" | "fe",  "config": 1 (fe only),
     "hierarchy": [dt_0, ...], "horizon": T, "halfwidth": h, "seed": 0,
     "n_dof": 64 (synthetic), "drive": {"amplitude", "frequency", "slip"},
     "estimator": "mlmc" | "mc",
     "policy": {"fixed": [N_0, ...]} | {"warmup": N_w, "rmse": eps},
     "parareal": {"enabled": true, "num_subintervals": M, "tolerance": tol,
                  "k_max": K, "dt_coarse": dt (default: level L-2)}}

Outputs: ``estimate.json`` (expectation, rmse, per-level stats; byte-identical
for a fixed seed), ``ledger.json`` (executor ledger: SPEC.md:497 keys),
``samples.csv`` (level,index,Q_l,Q_lm1,cost_s,parareal_K), ``figure1.csv`` /
``figure2.csv`` (n_c,K,speedup,effort_ratio).  Exit codes: 0 ok, 1 solver
error, 2 invalid configuration.
"""

from __future__ import annotations

import argparse
import json
import os
import sys

import numpy as np

from . import costmodel


class ConfigError(ValueError):
    pass


def _ranges(text: str):
    out = []
    for part in str(text).split(","):
        if ".." in part:
            a, b = part.split("..")
            out.extend(range(int(a), int(b) + 1))
        elif part:
            out.append(int(part))
    return out


def load_experiment(spec: str) -> dict:
    """Normalised experiment dict from ``cfgN`` or a JSON file."""
    if spec.startswith("cfg") and not os.path.exists(spec):
        from .configs import get_config
        try:
            c = get_config(spec)
        except (KeyError, ValueError) as exc:
            raise ConfigError(f"unknown configuration {spec!r}") from exc
        exp = {"model": "fe", "config": int(spec[3:]), "hierarchy": list(c.dts),
               "horizon": c.horizon, "seed": c.seed, "estimator": "mlmc",
               "policy": {"fixed": list(c.samples)}}
        if c.parareal is not None:
            m, dtc, tol, kmax = c.parareal
            exp["parareal"] = {"enabled": True, "num_subintervals": m, "dt_coarse": dtc,
                               "tolerance": tol, "k_max": kmax}
        return exp
    try:
        with open(spec) as fh:
            exp = json.load(fh)
    except (OSError, json.JSONDecodeError) as exc:
        raise ConfigError(f"cannot read configuration {spec!r}: {exc}") from exc
    if exp.get("model") not in ("steinmetz", "synthetic", "fe"):
        raise ConfigError("config 'model' must be steinmetz, synthetic or fe")
    if "hierarchy" not in exp and exp.get("model") != "fe":
        raise ConfigError("config needs a 'hierarchy' list of step sizes")
    return exp


def build_family(exp: dict, device=None):
    from .models import make_hierarchy
    model = exp["model"]
    try:
        if model == "fe":
            from .models import eddy_current_family
            fam = eddy_current_family(exp.get("config", 1), device=device)
            if "hierarchy" in exp and tuple(exp["hierarchy"]) != tuple(
                    lv.dt for lv in fam.hierarchy):
                fam.hierarchy = make_hierarchy(exp["hierarchy"])
            return fam
        h = make_hierarchy(exp["hierarchy"])
        from . import machines as mc
        if model == "steinmetz":
            drive = mc.DriveSettings(**exp.get("drive", {}))
            return mc.steinmetz_family(h, halfwidth=exp.get("halfwidth", 0.05), drive=drive,
                                       horizon=exp.get("horizon", 1.0), device=device)
        return mc.synthetic_family(h, n_dof=exp.get("n_dof", 64),
                                   halfwidth=exp.get("halfwidth", 0.05),
                                   horizon=exp.get("horizon", 0.16), device=device)
    except (TypeError, ValueError) as exc:
        raise ConfigError(str(exc)) from exc


def parareal_of(exp: dict, fam):
    pr = exp.get("parareal")
    if not pr or not pr.get("enabled", True):
        return None
    from .parareal import PararealConfig
    L = len(fam.hierarchy) - 1
    dtc = pr.get("dt_coarse")
    if dtc is None:
        if L < 2:
            raise ConfigError("Parareal with the L-2 coarse rule needs >= 3 levels "
                              "(or an explicit dt_coarse)")
        dtc = fam.hierarchy[L - 2].dt
    try:
        return PararealConfig(int(pr["num_subintervals"]), fam.hierarchy[L].dt, float(dtc),
                              float(pr.get("tolerance", 1e-8)), pr.get("k_max"))
    except (KeyError, ValueError) as exc:
        raise ConfigError(f"invalid parareal section: {exc}") from exc


def _policy(exp, fam):
    from .mlmc import FixedSamples, WarmupPolicy
    pol = exp.get("policy", {})
    if "fixed" in pol:
        n = list(pol["fixed"])
        if exp.get("estimator", "mlmc") == "mlmc" and len(n) != len(fam.hierarchy):
            raise ConfigError("policy.fixed needs one count per level")
        return FixedSamples(tuple(int(x) for x in n))
    if "warmup" in pol:
        return WarmupPolicy(int(pol["warmup"]), rmse=pol.get("rmse"), budget=pol.get("budget"))
    raise ConfigError("policy needs 'fixed' or 'warmup'")


def cmd_estimate(args) -> int:
    from . import executor
    from .mlmc import EstimatorResult, LevelStats, draw_level, write_estimate_json
    exp = load_experiment(args.config)
    fam = build_family(exp, args.device)
    pcfg = parareal_of(exp, fam)
    pol = _policy(exp, fam)
    seed = int(exp.get("seed", 0))
    os.makedirs(args.out, exist_ok=True)
    if exp.get("estimator", "mlmc") == "mc":
        L = len(fam.hierarchy) - 1
        n = pol.n_per_level[-1]
        if n < 2:
            raise ConfigError("mc needs N >= 2")
        P = draw_level(fam.uncertain, seed, L, range(1, n + 1))
        recs = fam.evaluate_batch(P, fam.hierarchy[L], pcfg)
        q = np.array([r.q for r in recs])
        st = LevelStats(L, n, float(np.sum(q)), float(np.sum(q * q)), recs[0].cost_s,
                        [r.parareal_iterations for r in recs] if pcfg else None)
        res = EstimatorResult(st.mean_y, [st], float(np.sqrt(max(st.var_y, 0.0) / n)),
                              {"mode": "gpu-batched"})
        led = executor.Ledger("gpu-batched", [executor.LevelLedger(L, 1, recs[0].cost_s * n,
                                                                   recs[0].cost_s * n)])
        led_d = led.to_dict()
    else:
        from .mlmc import mlmc_estimate
        res = mlmc_estimate(fam, policy=pol, parareal_cfg=pcfg, seed=seed,
                            csv_path=os.path.join(args.out, "samples.csv"), timing=True)
        led_d = res.ledger.get("executor", {"mode": "gpu-batched"})
        led_d = dict(led_d)
        for k in ("warmup", "allocation"):
            if k in res.ledger:
                led_d[k] = res.ledger[k]
    write_estimate_json(os.path.join(args.out, "estimate.json"), res)
    with open(os.path.join(args.out, "ledger.json"), "w") as fh:
        json.dump(led_d, fh, indent=1, sort_keys=True)
    print(json.dumps({"expectation": res.expectation, "rmse": res.rmse_estimate}))
    return 0


def cmd_sample(args) -> int:
    from .mlmc import draw_level
    exp = load_experiment(args.config)
    fam = build_family(exp, args.device)
    lvl = int(args.level)
    if not 0 <= lvl < len(fam.hierarchy):
        raise ConfigError(f"level {lvl} outside the hierarchy")
    pcfg = parareal_of(exp, fam) if (args.parareal and lvl == len(fam.hierarchy) - 1) else None
    os.makedirs(args.out, exist_ok=True)
    path = os.path.join(args.out, f"samples_l{lvl}.csv")
    recs = []
    if args.count > 0:
        P = draw_level(fam.uncertain, int(exp.get("seed", 0)), lvl, range(1, args.count + 1))
        recs = fam.evaluate_batch(P, fam.hierarchy[lvl], pcfg)
    with open(path, "w") as fh:
        fh.write("level,index,Q,cost_s,parareal_K\n")
        for k, r in enumerate(recs, start=1):
            kk = "" if r.parareal_iterations is None else int(r.parareal_iterations)
            fh.write(f"{lvl},{k},{r.q!r},{r.cost_s!r},{kk}\n")
    print(path)
    return 0


def cmd_plan(args) -> int:
    N = tuple(_ranges(args.N))
    p = costmodel.CostModelParams(C0=1.0, r=float(args.r), L=int(args.L), n_c=max(_ranges(args.nc)),
                                  N=N)
    rows = costmodel.figure_data(p, _ranges(args.nc), _ranges(args.K))
    os.makedirs(args.out, exist_ok=True)
    note = (f"r={args.r} L={args.L} N={list(N)} s_inf={costmodel.ideal_speedup(p.r, p.L)!r} "
            f"(rows with NaN: K > n_c,para or insufficient cores)")
    # Fig. 1 plots the speedup column, Fig. 2 the effort ratio (same rows)
    costmodel.write_figure_csv(os.path.join(args.out, "figure1.csv"), rows, note)
    costmodel.write_figure_csv(os.path.join(args.out, "figure2.csv"), rows, note)
    print(os.path.join(args.out, "figure1.csv"))
    return 0


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="python -m paper_2507_19246_b200")
    sub = ap.add_subparsers(dest="cmd", required=True)
    e = sub.add_parser("estimate")
    e.add_argument("config")
    e.add_argument("--out", required=True)
    e.add_argument("--device", default=None)
    s = sub.add_parser("sample")
    s.add_argument("config")
    s.add_argument("--level", type=int, required=True)
    s.add_argument("--count", type=int, required=True)
    s.add_argument("--parareal", action="store_true")
    s.add_argument("--out", required=True)
    s.add_argument("--device", default=None)
    p = sub.add_parser("plan")
    p.add_argument("--r", default="10")
    p.add_argument("--L", default="2")
    p.add_argument("--N", default="10303,85,10")
    p.add_argument("--nc", default="180,360,720,1440")
    p.add_argument("--K", default="1..10")
    p.add_argument("--out", required=True)
    args = ap.parse_args(argv)
    try:
        return {"estimate": cmd_estimate, "sample": cmd_sample, "plan": cmd_plan}[args.cmd](args)
    except ConfigError as exc:
        print(f"invalid configuration: {exc}", file=sys.stderr)
        return 2
    except (RuntimeError, ArithmeticError) as exc:       # SingularSystemError, PropagatorError
        print(f"solver error: {exc}", file=sys.stderr)
        return 1
