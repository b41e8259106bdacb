"""GPU half of the reference's own machine models: the batched families
(steinmetz_family on the direct-LU path, synthetic_family on the
SM-resident PCG path) against the unmodified reference's
MachineFamily.evaluate outputs (tests/golden/steinmetz.npz,
synthetic_machine.npz), sequential at every level and with Parareal on the
finest level, plus the timeint mirror on the dense Steinmetz model.

Tolerances: the direct path is the reference's algorithm (LU with partial
pivoting) in a different operation order; the Steinmetz step matrix
M + dt K has condition ~1e7, so QoIs agree to 1e-9 relative.  The synthetic
machine solves with Jacobi-PCG at rtol 1e-13: QoIs to 1e-8 relative.
Parareal iteration counts K must match exactly."""

import numpy as np
import pytest

from conftest import golden

pytestmark = pytest.mark.gpu

RTOL = {"steinmetz": 1e-9, "synthetic_machine": 1e-8}


def fam_of(tag):
    from paper_2507_19246_b200 import machines as mc
    from paper_2507_19246_b200.models import make_hierarchy
    g = golden(tag)
    h = make_hierarchy(list(g["dts"]))
    if tag == "steinmetz":
        return g, mc.steinmetz_family(h, horizon=float(g["horizon"]), device="cuda:0")
    return g, mc.synthetic_family(h, n_dof=64, horizon=float(g["horizon"]), device="cuda:0")


def pcfg_of(g, dt_fine):
    from paper_2507_19246_b200.parareal import PararealConfig
    m, dtc, tol, kmax = g["pr_cfg"]
    return PararealConfig(int(m), dt_fine, float(dtc), float(tol), int(kmax))


@pytest.mark.parametrize("tag", ["steinmetz", "synthetic_machine"])
def test_levels_sequential(cuda, tag):
    g, fam = fam_of(tag)
    for lvl, spec in enumerate(fam.hierarchy):
        recs = fam.evaluate_batch(g[f"params_l{lvl}"], spec)
        q = np.array([r.q for r in recs])
        np.testing.assert_allclose(q, g[f"q_l{lvl}"], rtol=RTOL[tag], atol=0)


@pytest.mark.parametrize("tag", ["steinmetz", "synthetic_machine"])
def test_finest_level_parareal(cuda, tag):
    g, fam = fam_of(tag)
    L = len(fam.hierarchy) - 1
    spec = fam.hierarchy[L]
    recs = fam.evaluate_batch(g[f"params_l{L}"], spec, pcfg_of(g, spec.dt))
    np.testing.assert_array_equal([r.parareal_iterations for r in recs], g["k_pr"])
    np.testing.assert_allclose([r.q for r in recs], g["q_pr"], rtol=RTOL[tag], atol=0)


@pytest.mark.parametrize("tag", ["steinmetz", "synthetic_machine"])
def test_per_sample_evaluate_protocol(cuda, tag):
    """MachineFamily.evaluate(params, level, parareal_cfg, pool) -> EvalRecord."""
    from paper_2507_19246_b200.models import ParameterVector
    g, fam = fam_of(tag)
    p = ParameterVector(fam.uncertain.nominal.model_id, g["params_l1"][2])
    rec = fam.evaluate(p, fam.hierarchy[1], None, pool=object())
    assert rec.parareal_iterations is None and rec.cost_s > 0
    assert rec.q == pytest.approx(float(g["q_l1"][2]), rel=RTOL[tag])


@pytest.mark.parametrize("tag", ["steinmetz", "synthetic_machine"])
def test_run_levels_coupled(cuda, tag):
    """The estimator's batched entry: Q_l and Q_{l-1} of every level at once,
    Parareal on the finest level, for the golden sample keys."""
    g, fam = fam_of(tag)
    L = len(fam.hierarchy) - 1
    draws = [g[f"params_l{lvl}"] for lvl in range(L + 1)]
    cfg = pcfg_of(g, fam.hierarchy[L].dt)
    batches = fam.run_levels(draws, cfg)
    fam.check_status()
    for lvl, b in enumerate(batches):
        want = g["q_pr"] if lvl == L else g[f"q_l{lvl}"]
        np.testing.assert_allclose(b.q_l.cpu().numpy(), want, rtol=RTOL[tag])
        if lvl == L:
            np.testing.assert_array_equal(b.k_used.cpu().numpy(), g["k_pr"])
        if lvl > 0:
            # Q_{l-1} is the level-(l-1) solve of the SAME parameters
            q_lo = np.array([r.q for r in fam.evaluate_batch(draws[lvl], fam.hierarchy[lvl - 1])])
            np.testing.assert_allclose(b.q_lm1.cpu().numpy(), q_lo, rtol=1e-13)


def test_timeint_mirror_on_dense_steinmetz(cuda):
    """implicit_euler_solve on the reference-shaped (dense, M = I,
    non-symmetric K, scaled-drive forcing) model goes through the direct path."""
    from paper_2507_19246_b200 import machines as mc
    from paper_2507_19246_b200.models import ParameterVector
    from paper_2507_19246_b200.timeint import implicit_euler_solve
    g, fam = fam_of("steinmetz")
    model = fam.build(ParameterVector("steinmetz", g["params_l0"][0]))
    tr = implicit_euler_solve(model, 0.0, fam.horizon, float(g["dts"][0]), model.initial_state)
    scale = np.max(np.abs(g["traj0"]), axis=0)
    assert np.max(np.abs(tr.states - g["traj0"]) / scale) <= 1e-9
    assert mc.evaluate_qoi(model, tr) == pytest.approx(float(g["traj0_q"]), rel=1e-9)


def test_direct_path_singular(cuda):
    """A singular step matrix raises SingularSystemError(step_index=0)
    like timeint.py:70-74."""
    from paper_2507_19246_b200.timeint import SingularSystemError, implicit_euler_solve

    class Sing:
        mass = np.array([[1.0, 1.0], [1.0, 1.0]])
        stiffness = np.zeros((2, 2))
        forcing = None
        initial_state = np.zeros(2)
        dim = 2

    with pytest.raises(SingularSystemError) as ei:
        implicit_euler_solve(Sing(), 0.0, 1.0, 0.1, np.zeros(2))
    assert ei.value.step_index == 0


def test_mlmc_estimate_steinmetz(cuda):
    """End to end: mlmc_estimate on the Steinmetz family (fixed N per level,
    Parareal on the finest) equals the telescoping sum of the golden per-sample
    QoIs for the same keys (3 samples per level, seed 0)."""
    from paper_2507_19246_b200.mlmc import FixedSamples, mlmc_estimate
    g, fam = fam_of("steinmetz")
    L = len(fam.hierarchy) - 1
    cfg = pcfg_of(g, fam.hierarchy[L].dt)
    res = mlmc_estimate(fam, policy=FixedSamples((3,) * (L + 1)), parareal_cfg=cfg, seed=0)
    # golden Q_l for keys (0, l, 1..3); Q_{l-1} on the same parameters
    want = 0.0
    for lvl in range(L + 1):
        ql = g["q_pr"] if lvl == L else g[f"q_l{lvl}"]
        if lvl > 0:
            qm = np.array([r.q for r in fam.evaluate_batch(g[f"params_l{lvl}"],
                                                            fam.hierarchy[lvl - 1])])
        else:
            qm = np.zeros(3)
        want += float(np.mean(ql - qm))
    assert res.expectation == pytest.approx(want, rel=1e-9)
    assert res.per_level[L].parareal_k == list(g["k_pr"])
