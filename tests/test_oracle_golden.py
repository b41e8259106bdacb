"""CPU: the oracle restatement (oracle/) against the golden fixtures written by
oracle/pin_reference.py from the unmodified reference (dense LU cases must be
bitwise equal).  Pins the oracle before it is trusted as the GPU checker."""

import numpy as np
import pytest

from conftest import golden
from oracle import fe_oracle as fe
from oracle import ie_oracle, parareal_oracle
from oracle import mlmc_oracle as mo


def test_spec_kats_bitwise():
    g = golden("spec_kats")

    class Scalar:
        mass = np.array([[1.0]])
        stiffness = np.array([[1.0]])
        initial_state = np.array([1.0])
        dim = 1

        @staticmethod
        def forcing(t):
            return np.zeros(1)

    assert ie_oracle.implicit_euler(Scalar, 0.0, 0.5, 0.5, [1.0]).terminal[0] == g["one_step"][0]
    assert g["one_step"][0] == 2.0 / 3.0
    assert ie_oracle.propagate(Scalar, 0.0, 1.0, 0.25, [1.0])[0] == g["decay_quarter"][0]
    assert abs(g["decay_quarter"][0] - 0.4096) < 1e-15
    assert float(parareal_oracle.jump_defect([[1.0, 0.0]], [[1.0, 1.0]])) == float(g["defect_unit"])
    p = np.log(g["decay_errors"][0] / g["decay_errors"][2]) / np.log(4.0)
    assert 0.9 <= p <= 1.1


def test_draws_match_reference():
    g = golden("draws")
    for key, row in zip(g["keys"], g["uniform"]):
        d = mo.draw_uniform(g["nominal"], 0.1, mo.RandomStream(*key))
        np.testing.assert_array_equal(d, row)
    np.testing.assert_array_equal(mo.draw_gaussian(64, mo.RandomStream(0, 2, 1)), g["gaussian"][0])


def test_synthetic_bar_bitwise():
    g = golden("synthetic_bar")

    class Bar:
        mass = g["mass"]
        stiffness = g["stiffness"]
        forcing = mo.ProfileForcing(float(g["frequency"]), g["profile"])
        initial_state = np.zeros(len(g["profile"]))
        dim = len(g["profile"])

    tr = ie_oracle.implicit_euler(Bar, 0.0, 0.02, 1e-3, Bar.initial_state)
    np.testing.assert_array_equal(tr.states, g["states"])
    res = parareal_oracle.parareal(Bar, 0.0, 0.02, Bar.initial_state,
                                   parareal_oracle.OraclePararealConfig(4, 1e-4, 1e-3, 1e-10, 4))
    np.testing.assert_array_equal(res.boundary_states, g["pr_boundary"])
    assert res.iterations_used == int(g["pr_k"])


@pytest.mark.parametrize("name", ["fe8_quad4_seq", "fe16_blocks8_timeavg", "fe16_kl64_seq"])
def test_fe_sequential_bitwise(name):
    g = golden(name)
    prob = mo.FEProblem(int(g["n"]), str(g["layout"]))
    dt, horizon = float(g["dt"]), float(g["horizon"])
    for p, q, term in zip(g["params"], g["q"], g["terminal"]):
        model = prob.model(p, dense=True)
        tr = ie_oracle.implicit_euler(model, 0.0, horizon, dt, model.initial_state)
        np.testing.assert_array_equal(tr.terminal, term)
        if str(g["qoi"]) == "energy_T":
            assert mo.energy(model, tr.terminal) == q


@pytest.mark.parametrize("name", ["fe8_quad4_parareal", "fe16_kl64_parareal"])
def test_fe_parareal_bitwise(name):
    g = golden(name)
    prob = mo.FEProblem(int(g["n"]), str(g["layout"]))
    m, dtc, tol, kmax = g["parareal"]
    for p, k, bnd in zip(g["params"], g["k_used"], g["boundary"]):
        model = prob.model(p, dense=True)
        res = parareal_oracle.parareal(model, 0.0, float(g["horizon"]), model.initial_state,
                                       parareal_oracle.OraclePararealConfig(int(m), float(g["dt"]),
                                                                            float(dtc), float(tol),
                                                                            int(kmax)))
        assert res.iterations_used == k
        np.testing.assert_array_equal(res.boundary_states, bnd)


def test_sparse_backend_agrees_with_dense():
    """The splu substitution used for >= 128^2 vs dense LU."""
    g = golden("fe8_quad4_seq")
    prob = mo.FEProblem(8, "quad4")
    p = g["params"][0]
    dense = prob.model(p, dense=True)
    sparse = prob.model(p, dense=False)
    a = ie_oracle.implicit_euler(dense, 0.0, 0.02, 0.02 / 32, dense.initial_state).terminal
    b = ie_oracle.implicit_euler(sparse, 0.0, 0.02, 0.02 / 32, sparse.initial_state).terminal
    assert np.max(np.abs(a - b)) <= 1e-12 * np.max(np.abs(a))


def test_level_statistics_formulas():
    # SPEC.md:259-260
    st = mo.level_statistics(1, [1.0, 2.0, 4.0], [0.5, 0.5, 0.5])
    y = np.array([0.5, 1.5, 3.5])
    assert st.sum_y == y.sum() and st.sum_y2 == float(np.sum(y * y))
    assert abs(st.var - np.var(y, ddof=1)) < 1e-14


def test_fe_matrices_properties():
    mesh = fe.build_mesh(8)
    geom = fe.ElementGeometry(mesh)
    sig, nu = fe.material_fields(mesh, "quad4", np.array([fe.NU0] * 4 + [fe.SIGMA0] * 4))
    M, K, prof = fe.assemble(geom, sig, nu, fe.source_elements(mesh, "quad4"))
    assert abs(M - M.T).max() == 0 and abs(K - K.T).max() == 0
    assert np.all(np.linalg.eigvalsh(K.toarray()) > 0)          # Dirichlet -> SPD
    ev = np.linalg.eigvalsh(M.toarray())
    assert ev.min() > -1e-9 * ev.max() and ev.min() < 1e-9 * ev.max()  # sigma = 0 regions: singular
    assert prof.sum() > 0


def test_oracle_matches_reference_goldens_at_baseline_meshes():
    """The oracle restatement (splu backend, one factorisation per propagator
    call as timeint.py:64-75) reproduces BITWISE the reference-generated
    fixtures at the BASELINE mesh sizes (oracle/make_large_goldens.py): a
    config-3 level-1 coupled sample at 128^2 and one finest-level Parareal
    sample (M=32, K<=6) — the oracle that checks the GPU at these sizes is
    pinned to the reference there too."""
    from oracle import mlmc_oracle as mo
    cfg = mo.CONFIGS[3]
    prob = mo.FEProblem(128, "kl64")
    g = golden("cfg3_subset_l01")
    i = int(np.nonzero((g["level"] == 1) & (g["k"] == 1))[0][0])
    q_l, q_lm1, _ = mo.coupled(prob, cfg, 1, g["params"][i])
    assert (q_l, q_lm1) == (g["q_l"][i], g["q_lm1"][i])
    g2 = golden("cfg3_l2_parareal")
    j = 46                                           # key 47
    rec = mo.evaluate(prob, cfg, g2["params"][j], cfg.dts[2], True)
    assert rec.k_used == g2["k_used"][j]
    assert rec.q == g2["q_l"][j]
    np.testing.assert_array_equal(np.array(rec.defects), g2["defects"][j][:rec.k_used])
