"""GPU FE path vs the reference (golden fixtures from pin_reference.py: the
unmodified reference integrators on the oracle's FE models) and vs the live
CPU oracle.

Parity bar (BASELINE.json north_star): per-sample QoI within 1e-8 relative;
Parareal K equal per sample.  PCG tolerance: ||r||_2 <= 1e-13 ||b||_2.
"""

import numpy as np
import pytest

from conftest import golden

pytestmark = pytest.mark.gpu

RTOL_Q = 1e-8


def family(n, layout, dts, horizon, qoi="energy_T", window=0.0, path="auto"):
    from paper_2507_19246_b200 import fe
    from paper_2507_19246_b200.models import (EddyCurrentFamily, GaussianInput, ParameterVector,
                                              QoIKind, UncertainInput, make_hierarchy)
    if layout == "kl64":
        unc = GaussianInput("kl64", 64)
    else:
        P = fe.n_params(layout)
        unc = UncertainInput(ParameterVector(layout, np.array([fe.NU0] * (P // 2) +
                                                              [fe.SIGMA0] * (P // 2))), 0.1)
    kind = QoIKind.MAGNETIC_ENERGY_T if qoi == "energy_T" else QoIKind.TIME_AVG_MAGNETIC_ENERGY
    return EddyCurrentFamily(layout, unc, make_hierarchy(dts), horizon, n, layout, kind, window,
                             device="cuda:0", path=path)


def check_seq_case(name, path="auto"):
    import torch
    g = golden(name)
    n, dt, horizon = int(g["n"]), float(g["dt"]), float(g["horizon"])
    qoi = str(g["qoi"])
    fam = family(n, str(g["layout"]), [dt], horizon, qoi, window=0.02, path=path)
    sol = fam.solver
    M, K = sol.assemble(torch.from_numpy(g["params"]).to(sol.device))
    r = sol.run_sequential(M, K, [fam._seq_job(np.arange(len(g["params"])), dt)])[0]
    q = fam._finish_q(r.qoi, dt).cpu().numpy()
    np.testing.assert_allclose(q, g["q"], rtol=RTOL_Q, atol=0)
    xb = sol._last_xbuf.view(len(g["params"]), -1).cpu().numpy()
    scale = np.max(np.abs(g["terminal"]))
    assert np.max(np.abs(xb - g["terminal"])) <= 1e-9 * scale
    assert int(r.status[:, 0].abs().sum().item()) == 0


@pytest.mark.parametrize("name", ["fe8_quad4_seq", "fe32_cfg0_l1", "fe32_cfg0_l2",
                                  "fe16_blocks8_timeavg", "fe16_kl64_seq"])
def test_sequential_golden(cuda, name):
    check_seq_case(name)


@pytest.mark.parametrize("name", ["fe8_quad4_seq", "fe16_kl64_seq"])
def test_streaming_path_golden(cuda, name):
    """The HBM-streaming path (used for >1024 rows) on the same cases."""
    check_seq_case(name, path="stream")


def check_parareal_case(name, path="auto"):
    import torch
    g = golden(name)
    n, dt, horizon = int(g["n"]), float(g["dt"]), float(g["horizon"])
    m, dtc, tol, kmax = g["parareal"]
    fam = family(n, str(g["layout"]), [dt], horizon, path=path)
    sol = fam.solver
    M, K = sol.assemble(torch.from_numpy(g["params"]).to(sol.device))
    pr = sol.run_parareal(M, K, 0.0, horizon, int(m), dt, float(dtc), float(tol), int(kmax))
    np.testing.assert_array_equal(pr.k_used.cpu().numpy(), g["k_used"])
    np.testing.assert_allclose(pr.qoi.cpu().numpy(), g["q"], rtol=RTOL_Q, atol=0)
    U = pr.U.cpu().numpy()
    scale = np.max(np.abs(g["boundary"]))
    assert np.max(np.abs(U - g["boundary"])) <= 1e-8 * scale
    d = pr.defects.cpu().numpy()
    for i, k in enumerate(g["k_used"]):
        # early defects are O(1e-2..1e-7) jumps between iterates whose states carry
        # the PCG tolerance (~1e-11 relative after a slice): relative + absolute slack
        np.testing.assert_allclose(d[i, :k - 1], g["defects"][i, :k - 1], rtol=1e-5, atol=1e-10)
        assert d[i, k - 1] <= tol


@pytest.mark.parametrize("name", ["fe8_quad4_parareal", "fe16_kl64_parareal", "fe32_cfg1_parareal"])
def test_parareal_golden(cuda, name):
    check_parareal_case(name)


def test_parareal_streaming_path(cuda):
    check_parareal_case("fe8_quad4_parareal", path="stream")


def test_batch_invariance_bitwise(cuda):
    """A sample's result does not depend on the batch it runs in."""
    import torch
    g = golden("fe32_cfg0_l2")
    fam = family(32, "quad4", [float(g["dt"])], float(g["horizon"]))
    sol = fam.solver
    p = np.repeat(g["params"], 3, axis=0)[:5]
    M, K = sol.assemble(torch.from_numpy(p).to(sol.device))
    r5 = sol.run_sequential(M, K, [fam._seq_job(np.arange(5), float(g["dt"]))])[0].qoi.cpu().numpy()
    M1, K1 = sol.assemble(torch.from_numpy(p[:1]).to(sol.device))
    r1 = sol.run_sequential(M1, K1, [fam._seq_job(np.arange(1), float(g["dt"]))])[0].qoi.cpu().numpy()
    assert r5[0] == r1[0] and r5[2] == r1[0] and r5[3] == r5[4]


def test_zero_source_gives_zero(cuda):
    """b == 0 every step -> a == 0 exactly (edge case of the stopping rule)."""
    import torch
    fam = family(8, "quad4", [0.02 / 32], 0.02)
    sol = fam.solver
    sol.profile.zero_()
    g = golden("fe8_quad4_seq")
    M, K = sol.assemble(torch.from_numpy(g["params"]).to(sol.device))
    r = sol.run_sequential(M, K, [fam._seq_job(np.arange(3), 0.02 / 32)])[0]
    assert np.all(r.qoi.cpu().numpy() == 0.0)
    assert np.all(sol._last_xbuf.cpu().numpy() == 0.0)


def test_empty_batch(cuda):
    from paper_2507_19246_b200.models import ParameterVector  # noqa: F401
    fam = family(8, "quad4", [0.02 / 32, 0.02 / 64], 0.02)
    out = fam.run_levels([np.zeros((0, 8)), np.zeros((0, 8))])
    assert all(len(b.q_l) == 0 for b in out)


@pytest.mark.parametrize("impl", ["1", "4"])
def test_streaming_batch_invariance_bitwise(cuda, impl, monkeypatch):
    """Streaming paths (two-launch ELL, tile): per-task reductions in fixed
    order, so a sample's result is bitwise independent of the batch it runs in
    (full 256x256 config-2 mesh, 6 steps)."""
    import torch
    from paper_2507_19246_b200.mlmc import draw_level
    from paper_2507_19246_b200.models import eddy_current_family
    monkeypatch.setenv("MLMCP_STREAM_IMPL", impl)
    fam = eddy_current_family(2, device="cuda:0")
    sol = fam.solver
    p = draw_level(fam.uncertain, 0, 0, range(1, 4))
    dt = fam.hierarchy[0].dt

    def run(params):
        M, K = sol.assemble(torch.from_numpy(params).to(sol.device))
        job = fam._seq_job(np.arange(len(params)), dt)
        job.n_steps = 6
        r = sol.run_sequential(M, K, [job])[0]
        return (sol._last_xbuf.view(len(params), -1).cpu().numpy().copy(),
                r.iters.cpu().numpy().copy())

    x3, it3 = run(p)
    x1, it1 = run(p[1:2])
    assert np.array_equal(x3[1], x1[0]) and it3[1] == it1[0]


def test_streaming_paths_agree_full_mesh(cuda, monkeypatch):
    """Two-launch ELL kernels and the tile kernel on the full 512x512 config-4
    mesh: same iterates to the PCG tolerance (states within 1e-10 of max|x|)."""
    import torch
    from paper_2507_19246_b200.mlmc import draw_level
    from paper_2507_19246_b200.models import eddy_current_family
    fam = eddy_current_family(4, device="cuda:0")
    sol = fam.solver
    p = draw_level(fam.uncertain, 0, 0, range(1, 3))
    M, K = sol.assemble(torch.from_numpy(p).to(sol.device))
    out = {}
    for impl in ("1", "4"):
        monkeypatch.setenv("MLMCP_STREAM_IMPL", impl)
        job = fam._seq_job(np.arange(2), fam.hierarchy[0].dt)
        job.n_steps = 4
        sol.run_sequential(M, K, [job])
        out[impl] = sol._last_xbuf.view(2, -1).cpu().numpy().copy()
    scale = np.max(np.abs(out["1"]))
    assert scale > 0 and np.max(np.abs(out["1"] - out["4"])) <= 1e-10 * scale
