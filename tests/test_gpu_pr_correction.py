"""Correction fine solves of the streaming Parareal (MLMCP_TASK_CORRECTION).

The fine propagator is affine, so from iteration 2 on the tile path computes
F(U^k_{n-1}) = F(U^{k-1}_{n-1}) + Phi(U^k_{n-1} - U^{k-1}_{n-1}), Phi the
propagator without source, instead of re-solving the forced problem from
scratch as parareal.py:185-188 does.  The correction is solved to the absolute
accuracy of a full solve (stopping reference max(b.D^-1.b, sum (M_ii F_i)^2 /
A_ii)), so K, Q and the defect histories stay those of the reference.

Checked against the reference's own golden fixtures (oracle/make_large_goldens.py:
config 3's finest level, Parareal M=32, K<=6; config 4 at 512^2 in
test_gpu_large_parity.py runs the same code by default) and against the
full-solve mode (MLMCP_PR_CORRECTION=0) on the same samples.
"""

import numpy as np
import pytest

from conftest import golden

pytestmark = pytest.mark.gpu


def _run_cfg3(n, monkeypatch, corr: str):
    from paper_2507_19246_b200.configs import get_config
    from paper_2507_19246_b200.models import eddy_current_family
    monkeypatch.setenv("MLMCP_STREAM_IMPL", "4")      # the tile path on the 128^2 mesh
    monkeypatch.setenv("MLMCP_PR_CORRECTION", corr)
    g = golden("cfg3_l2_parareal")
    fam = eddy_current_family(3, device="cuda:0")
    b = fam.run_levels([g["params"][:n]], get_config(3).parareal_config(), levels=[2])[0]
    fam.check_status()
    return g, fam, b


def test_correction_mode_matches_reference_goldens(cuda, monkeypatch):
    n = 6
    g, fam, b = _run_cfg3(n, monkeypatch, "1")
    assert fam.solver._last_pr_corr, "correction fine solves were not used"
    assert b.k_used.cpu().numpy().tolist() == g["k_used"][:n].tolist()
    q = b.q_l.cpu().numpy()
    rel = np.abs(q - g["q_l"][:n]) / np.abs(g["q_l"][:n])
    assert rel.max() <= 1e-8, rel
    d = b.defects.cpu().numpy()
    ref = g["defects"][:n]
    both = np.isfinite(ref)
    assert (np.isfinite(d) == both).all()
    assert np.max(np.abs(d[both] - ref[both])) <= 1e-10


def test_correction_mode_agrees_with_full_fine_solves(cuda, monkeypatch):
    n = 4
    _, fam1, b1 = _run_cfg3(n, monkeypatch, "1")
    _, fam0, b0 = _run_cfg3(n, monkeypatch, "0")
    assert not fam0.solver._last_pr_corr
    assert b1.k_used.cpu().tolist() == b0.k_used.cpu().tolist()
    q1, q0 = b1.q_l.cpu().numpy(), b0.q_l.cpu().numpy()
    assert np.max(np.abs(q1 - q0) / np.abs(q0)) <= 1e-10
    d1, d0 = b1.defects.cpu().numpy(), b0.defects.cpu().numpy()
    f = np.isfinite(d0)
    assert np.max(np.abs(d1[f] - d0[f])) <= 1e-11


def test_correction_flag_rejected_off_the_tile_path(cuda):
    """A correction task on the SM-resident path reports ST_UNSUPPORTED
    (-> ValueError), never a silently wrong solve."""
    import torch
    from paper_2507_19246_b200 import _lib
    from paper_2507_19246_b200.configs import T
    from paper_2507_19246_b200.engine import new_tasks
    from paper_2507_19246_b200.solver import FESolver, raise_on_status
    sol = FESolver(16, "quad4", device="cuda:0")
    p = torch.tensor([[7.9e5] * 4 + [1e6] * 4], dtype=torch.float64, device="cuda:0")
    M, K = sol.assemble(p)
    t = new_tasks(1)
    t["sample"], t["n_steps"], t["dt"], t["x_in"], t["x_out"] = 0, 2, T / 32, 0, sol.N
    t["flags"] = _lib.TASK_CORRECTION
    t["qoi_slot"], t["qoi_mode"], t["ss_slot"], t["traj"], t["group"], t["slot"] = \
        -1, _lib.QOI_NONE, -1, -1, -1, 0
    xbuf = torch.zeros(2 * sol.N, dtype=torch.float64, device="cuda:0")
    status = torch.zeros((1, _lib.STATUS_INTS), dtype=torch.int32, device="cuda:0")
    sol.sys.propagate(t, M, K, sol.profile, sol.omega, 1e-13, 1000, xbuf, status=status)
    torch.cuda.synchronize()
    assert int(status[0, 0]) == _lib.ST_UNSUPPORTED
    with pytest.raises(ValueError):
        raise_on_status(status, "propagate")
