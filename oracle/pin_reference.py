"""TEST INFRASTRUCTURE ONLY — pin the oracle to the unmodified reference and
write the golden fixtures under tests/golden/.

Runs in the build container only (needs /root/reference, which does not exist
on the GPU box).  The reference package is imported from
/root/reference/pkg/src (namespace package, no __init__.py) and driven through
its public functions on the oracle's duck-typed models, exactly the way
SURVEY.md §8(c) describes:

  timeint.implicit_euler_solve / propagate     timeint.py:88-128
  parareal.parareal_solve / defect             parareal.py:93-220
  models.draw_parameters / evaluate_qoi / builders   models.py:252-344

For every case the oracle restatement (oracle/ie_oracle.py,
oracle/parareal_oracle.py) is asserted BITWISE equal to the reference before
the reference's outputs are written out.  Usage:

    python -m oracle.pin_reference            # writes tests/golden/*.npz
"""

from __future__ import annotations

import os
import sys
from dataclasses import dataclass

import numpy as np

REF_SRC = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
GOLDEN = os.path.join(os.path.dirname(HERE), "tests", "golden")


def _import_reference():
    if not os.path.isdir(REF_SRC):
        raise SystemExit("reference not present: pin_reference runs in the build container only")
    if REF_SRC not in sys.path:
        sys.path.insert(0, REF_SRC)
    from mlmc_parareal import models, parareal, timeint  # noqa: E402
    return models, timeint, parareal


@dataclass(frozen=True)
class _ZeroForcing:
    dim: int

    def __call__(self, t):
        return np.zeros(self.dim)


@dataclass(frozen=True)
class _ScalarModel:
    mass: np.ndarray
    stiffness: np.ndarray
    forcing: object
    initial_state: np.ndarray

    @property
    def dim(self):
        return self.mass.shape[0]


def _bitwise(a, b, what):
    a = np.asarray(a)
    b = np.asarray(b)
    if a.shape != b.shape or not np.array_equal(a, b):
        raise AssertionError(f"oracle restatement differs from reference: {what} "
                             f"(max abs diff {np.max(np.abs(a - b)) if a.shape == b.shape else 'shape'})")


def main():
    models, timeint, parareal = _import_reference()
    sys.path.insert(0, os.path.dirname(HERE))
    from oracle import fe_oracle as fe
    from oracle import ie_oracle, parareal_oracle
    from oracle import mlmc_oracle as mo

    os.makedirs(GOLDEN, exist_ok=True)
    T = fe.PERIOD

    # ---------------------------------------------------------- SPEC KATs
    one = np.array([[1.0]])
    scalar = _ScalarModel(one, one, _ZeroForcing(1), np.array([1.0]))
    kat = {}
    kat["one_step"] = timeint.implicit_euler_solve(scalar, 0.0, 0.5, 0.5, [1.0]).states[-1]
    kat["decay_quarter"] = timeint.propagate(scalar, 0.0, 1.0, 0.25, [1.0])
    kzero = _ScalarModel(one, np.zeros((1, 1)), _ZeroForcing(1), np.array([1.0]))
    kat["k_zero_traj"] = timeint.implicit_euler_solve(kzero, 0.0, 1.0, 0.1, [1.0]).states
    errs = []
    for dt in (1e-2, 5e-3, 2.5e-3):
        errs.append(abs(timeint.propagate(scalar, 0.0, 1.0, dt, [1.0])[0] - np.exp(-1.0)))
    kat["decay_errors"] = np.array(errs)
    kat["defect_unit"] = np.array(parareal.defect([[1.0, 0.0]], [[1.0, 1.0]]))
    for key, val in (("one_step", ie_oracle.implicit_euler(scalar, 0.0, 0.5, 0.5, [1.0]).terminal),
                     ("decay_quarter", ie_oracle.propagate(scalar, 0.0, 1.0, 0.25, [1.0])),
                     ("k_zero_traj", ie_oracle.implicit_euler(kzero, 0.0, 1.0, 0.1, [1.0]).states),
                     ("defect_unit", np.array(parareal_oracle.jump_defect([[1.0, 0.0]], [[1.0, 1.0]])))):
        _bitwise(val, kat[key], f"KAT {key}")
    np.savez(os.path.join(GOLDEN, "spec_kats.npz"), **kat)

    # ---------------------------------------------------------- draws
    nominal = mo.CONFIGS[0].nominal()
    inp = models.UncertainInput(models.ParameterVector("fe", nominal), 0.1)
    keys = [(0, lvl, k) for lvl in range(3) for k in (1, 2, 3, 17)]
    ref_draws = np.array([models.draw_parameters(inp, mo.RandomStream(*key)).values for key in keys])
    ora_draws = np.array([mo.draw_uniform(nominal, 0.1, mo.RandomStream(*key)) for key in keys])
    _bitwise(ora_draws, ref_draws, "draw_parameters")
    gauss = np.array([mo.draw_gaussian(64, mo.RandomStream(0, 2, k)) for k in (1, 2)])
    np.savez(os.path.join(GOLDEN, "draws.npz"), keys=np.array(keys), uniform=ref_draws,
             gaussian=gauss, nominal=nominal)

    # ---------------------------------------------------------- reference's own synthetic bar model
    bars = models.draw_parameters(models.UncertainInput(models.ParameterVector("synthetic", np.ones(32)), 0.05),
                                  mo.RandomStream(0, 0, 1))
    bar_model = models.build_synthetic_machine(64, bars, horizon=0.02)
    tr = timeint.implicit_euler_solve(bar_model, 0.0, 0.02, 1e-3, bar_model.initial_state)
    q_bar = models.evaluate_qoi(bar_model, tr)
    otr = ie_oracle.implicit_euler(bar_model, 0.0, 0.02, 1e-3, bar_model.initial_state)
    _bitwise(otr.states, tr.states, "synthetic bar trajectory")
    pc = parareal.PararealConfig(4, 1e-4, 1e-3, 1e-10, 4)
    pres = parareal.parareal_solve(bar_model, 0.0, 0.02, bar_model.initial_state, pc)
    opres = parareal_oracle.parareal(bar_model, 0.0, 0.02, bar_model.initial_state,
                                     parareal_oracle.OraclePararealConfig(4, 1e-4, 1e-3, 1e-10, 4))
    _bitwise(opres.boundary_states, pres.boundary_states, "synthetic bar parareal")
    np.savez(os.path.join(GOLDEN, "synthetic_bar.npz"), mass=bar_model.mass,
             stiffness=bar_model.stiffness, profile=bar_model.forcing.profile,
             frequency=bar_model.forcing.frequency, bar_scales=bars.values,
             states=tr.states, q=q_bar,
             pr_boundary=pres.boundary_states, pr_k=pres.iterations_used,
             pr_defects=np.array(pres.defect_history),
             pr_terminal=pres.fine_trajectory.states[-1])

    # ---------------------------------------------------------- FE cases
    def fe_case(tag, n, layout, params_list, dt, horizon, pr=None, qoi="energy_T", window=T):
        prob = mo.FEProblem(n, layout)
        out = {"params": np.array(params_list), "n": n, "dt": dt, "horizon": horizon}
        qs, terms, ks, defs, bnds = [], [], [], [], []
        for p in params_list:
            model = prob.model(p, dense=True)
            if pr is None:
                rtr = timeint.implicit_euler_solve(model, 0.0, horizon, dt, model.initial_state)
                otr = ie_oracle.implicit_euler(model, 0.0, horizon, dt, model.initial_state)
                _bitwise(otr.states, rtr.states, f"{tag} trajectory")
                states = rtr.states
                if qoi == "energy_T":
                    q = mo.energy(model, states[-1])
                else:
                    n_t = int(round(horizon / dt))
                    n_w = int(round(window / dt))
                    acc = 0.0
                    for k in range(n_t - n_w + 1, n_t + 1):
                        acc += mo.energy(model, states[k])
                    q = acc * dt / window
                terms.append(states[-1])
            else:
                m, dtc, tol, kmax = pr
                rres = parareal.parareal_solve(model, 0.0, horizon, model.initial_state,
                                               parareal.PararealConfig(m, dt, dtc, tol, kmax))
                ores = parareal_oracle.parareal(model, 0.0, horizon, model.initial_state,
                                                parareal_oracle.OraclePararealConfig(m, dt, dtc, tol, kmax))
                _bitwise(ores.boundary_states, rres.boundary_states, f"{tag} parareal boundary")
                _bitwise(ores.terminal, rres.fine_trajectory.states[-1], f"{tag} parareal terminal")
                assert ores.iterations_used == rres.iterations_used
                term = rres.fine_trajectory.states[-1]
                q = mo.energy(model, term)
                terms.append(term)
                ks.append(rres.iterations_used)
                d = np.full(kmax, np.nan)
                d[:len(rres.defect_history)] = rres.defect_history
                defs.append(d)
                bnds.append(rres.boundary_states)
            qs.append(q)
        out["q"] = np.array(qs)
        out["terminal"] = np.array(terms)
        if pr is not None:
            out["k_used"] = np.array(ks)
            out["defects"] = np.array(defs)
            out["boundary"] = np.array(bnds)
            out["parareal"] = np.array(pr, dtype=float)
        out["layout"] = layout
        out["qoi"] = qoi
        np.savez(os.path.join(GOLDEN, f"{tag}.npz"), **out)
        print(f"  {tag}: q={out['q']}" + (f" K={out.get('k_used')}" if pr else ""))

    cfg0, cfg1 = mo.CONFIGS[0], mo.CONFIGS[1]
    p8 = [mo.draw(cfg0, 0, 0, k) for k in (1, 2, 3)]
    fe_case("fe8_quad4_seq", 8, "quad4", p8, T / 32, T)
    fe_case("fe8_quad4_parareal", 8, "quad4", p8, T / 128, T, pr=(4, T / 16, 1e-8, 4))
    p32 = [mo.draw(cfg0, 0, 2, k) for k in (1, 2)]
    fe_case("fe32_cfg0_l2", 32, "quad4", p32, T / 128, T)
    fe_case("fe32_cfg0_l1", 32, "quad4", p32, T / 64, T)
    p32b = [mo.draw(cfg1, 0, 2, k) for k in (1, 2)]
    fe_case("fe32_cfg1_parareal", 32, "quad4", p32b, T / 1024, T, pr=cfg1.parareal)
    cfg2 = mo.CONFIGS[2]
    p16 = [mo.draw(cfg2, 0, 0, k) for k in (1, 2)]
    fe_case("fe16_blocks8_timeavg", 16, "blocks8", p16, T / 64, 4 * T, qoi="time_avg_energy")
    cfg3 = mo.CONFIGS[3]
    pkl = [mo.draw(cfg3, 0, 2, k) for k in (1, 2)]
    fe_case("fe16_kl64_parareal", 16, "kl64", pkl, T / 128, T, pr=(8, T / 8, 1e-8, 6))
    fe_case("fe16_kl64_seq", 16, "kl64", pkl, T / 64, T)
    # ---------------------------------------------------------- reference's own machine families
    # MachineFamily.evaluate (models.py:389-411) of the unmodified reference on
    # steinmetz_family / synthetic_family (models.py:431-453), sequential at
    # every level and with Parareal at the finest (coarse dt = level L-2).
    def machine_case(tag, fam, pcfg, n_per_level=3):
        out = {"dts": np.array([lv.dt for lv in fam.hierarchy]), "horizon": fam.horizon}
        L = len(fam.hierarchy) - 1
        for lvl, spec in enumerate(fam.hierarchy):
            ps = [models.draw_parameters(fam.uncertain, mo.RandomStream(0, lvl, k))
                  for k in range(1, n_per_level + 1)]
            out[f"params_l{lvl}"] = np.array([p.values for p in ps])
            out[f"q_l{lvl}"] = np.array([fam.evaluate(p, spec).q for p in ps])
            if lvl == L:
                recs = [fam.evaluate(p, spec, pcfg) for p in ps]
                out["q_pr"] = np.array([r.q for r in recs])
                out["k_pr"] = np.array([r.parareal_iterations for r in recs])
                out["pr_cfg"] = np.array([pcfg.num_subintervals, pcfg.dt_coarse, pcfg.tolerance,
                                          pcfg.max_iterations])
        # one full trajectory (the timeint mirror's dense-model parity)
        p0 = models.ParameterVector(fam.uncertain.nominal.model_id, out["params_l0"][0])
        model = fam.build(p0)
        tr = timeint.implicit_euler_solve(model, 0.0, fam.horizon, fam.hierarchy[0].dt,
                                          model.initial_state)
        out["traj0"] = tr.states
        out["traj0_q"] = models.evaluate_qoi(model, tr)
        np.savez(os.path.join(GOLDEN, f"{tag}.npz"), **out)

    h3 = models.make_hierarchy([1e-3, 1e-4, 1e-5])
    machine_case("steinmetz", models.steinmetz_family(h3, horizon=0.04),
                 parareal.PararealConfig(8, 1e-5, 1e-3, 1e-8, 8))
    hs = models.make_hierarchy([1e-3, 5e-4, 1e-4])
    machine_case("synthetic_machine", models.synthetic_family(hs, n_dof=64, horizon=0.04),
                 parareal.PararealConfig(8, 1e-4, 1e-3, 1e-8, 8))
    print("golden fixtures written to", GOLDEN)


if __name__ == "__main__":
    main()
