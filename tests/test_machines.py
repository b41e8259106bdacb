"""The reference's own machine models (Steinmetz circuit, synthetic bar
machine; models.py:217-302) — CPU half: builders and host QoI pinned to the
unmodified reference through the golden fixtures (tests/golden/steinmetz.npz,
synthetic_machine.npz written by oracle/pin_reference.py), the batched CSR
values against the dense builders, and the device-independent validation."""

import numpy as np
import pytest

from conftest import golden
from oracle import ie_oracle
from paper_2507_19246_b200 import machines as mc
from paper_2507_19246_b200.models import ParameterVector, make_hierarchy


def fam_of(tag):
    g = golden(tag)
    h = make_hierarchy(list(g["dts"]))
    if tag == "steinmetz":
        return g, mc.steinmetz_family(h, horizon=float(g["horizon"]))
    return g, mc.synthetic_family(h, n_dof=64, horizon=float(g["horizon"]))


@pytest.mark.parametrize("tag", ["steinmetz", "synthetic_machine"])
def test_builder_trajectory_pinned_to_reference(tag):
    """Our host builders + the oracle's LU integrator reproduce the reference's
    own trajectory and evaluate_qoi (bitwise: same operations)."""
    g, fam = fam_of(tag)
    p = ParameterVector(fam.uncertain.nominal.model_id, g["params_l0"][0])
    model = fam.build(p)
    tr = ie_oracle.implicit_euler(model, 0.0, fam.horizon, float(g["dts"][0]), model.initial_state)
    np.testing.assert_array_equal(tr.states, g["traj0"])
    from paper_2507_19246_b200.timeint import Trajectory
    q = mc.evaluate_qoi(model, Trajectory(tr.times, tr.states, float(g["dts"][0])))
    assert q == float(g["traj0_q"])


@pytest.mark.parametrize("tag", ["steinmetz", "synthetic_machine"])
def test_batched_values_match_dense_builder(tag):
    import scipy.sparse as sp
    g, fam = fam_of(tag)
    P = g["params_l1"]
    Mv, Kv = fam.values(P)
    row_ptr, col, profile, freq = fam._pattern()
    for i, pv in enumerate(P):
        model = fam.build(ParameterVector(fam.uncertain.nominal.model_id, pv))
        M = sp.csr_matrix((Mv[i], col, row_ptr)).toarray()
        K = sp.csr_matrix((Kv[i], col, row_ptr)).toarray()
        if tag == "steinmetz":
            # first equation scaled by L_s1 (machines.py docstring)
            scale = np.array([pv[3], 1.0, 1.0])[:, None]
            np.testing.assert_allclose(M, scale * model.mass, rtol=0, atol=0)
            np.testing.assert_allclose(K, scale * model.stiffness, rtol=1e-15)
            np.testing.assert_allclose(profile * 1.0, model.forcing.drive.amplitude
                                       * model.forcing.direction * pv[3], rtol=1e-15)
        else:
            np.testing.assert_array_equal(M, model.mass)
            np.testing.assert_array_equal(K, model.stiffness)
            np.testing.assert_array_equal(profile, model.forcing.profile)
        assert freq == 50.0


def test_validation_mirrors_reference():
    with pytest.raises(ValueError):
        ParameterVector("steinmetz", np.ones(5))
    with pytest.raises(ValueError):
        ParameterVector("synthetic", np.ones(31))
    with pytest.raises(ValueError):
        mc.DriveSettings(slip=0.0)
    with pytest.raises(ValueError):
        mc.DriveSettings(frequency=-1.0)
    with pytest.raises(ValueError):
        mc.synthetic_family(make_hierarchy([1e-3]), n_dof=48)
    with pytest.raises(ValueError):
        mc.build_steinmetz(ParameterVector("synthetic", np.ones(32)), mc.DriveSettings())


def test_timeint_rejects_nonsymmetric_large_system():
    """PCG needs symmetric M, K above MLMCP_DIRECT_MAX_ROWS states; the check
    runs before any device work."""
    from paper_2507_19246_b200.timeint import implicit_euler_solve

    class M6:
        mass = np.eye(6)
        stiffness = np.eye(6) + np.diag(np.ones(5), 1)
        forcing = None
        initial_state = np.zeros(6)
        dim = 6

    with pytest.raises(ValueError, match="symmetric"):
        implicit_euler_solve(M6(), 0.0, 1.0, 0.1, np.zeros(6))
