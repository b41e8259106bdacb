"""GPU estimator path vs the CPU oracle: per-sample Q_l / Q_{l-1}, Parareal K,
level sums and the MLMC estimate (parity bar: 1e-8 relative per sample;
level statistics with an absolute tolerance of 1e-8 |E|);
bitwise independence of the sample partitioning (emulated ranks on one GPU);
large meshes through the HBM-streaming path vs the splu oracle; failures map
to the reference's exception types."""

import numpy as np
import pytest

from oracle import mlmc_oracle as mo

pytestmark = pytest.mark.gpu

T = mo.T


def small_family(n=8, dts=(T / 32, T / 64, T / 128), **kw):
    from paper_2507_19246_b200 import fe
    from paper_2507_19246_b200.models import (EddyCurrentFamily, ParameterVector, QoIKind,
                                              UncertainInput, make_hierarchy)
    nominal = np.array([fe.NU0] * 4 + [fe.SIGMA0] * 4)
    return EddyCurrentFamily("quad4", UncertainInput(ParameterVector("quad4", nominal), 0.1),
                             make_hierarchy(list(dts)), T, n, "quad4",
                             QoIKind.MAGNETIC_ENERGY_T, device="cuda:0", **kw)


def oracle_levels(n, dts, counts, pr, seed=0):
    cfg = mo.OracleConfig("t", n, "quad4", T, tuple(dts), tuple(counts), "energy_T", parareal=pr)
    prob = mo.FEProblem(n, "quad4")
    out = []
    for lvl, N in enumerate(counts):
        rows = [mo.coupled(prob, cfg, lvl, mo.draw(cfg, seed, lvl, k), dense=True)
                for k in range(1, N + 1)]
        out.append(rows)
    return out


def check_estimate(n, dts, counts, pr):
    from paper_2507_19246_b200.mlmc import FixedSamples, mlmc_estimate
    from paper_2507_19246_b200.parareal import PararealConfig
    fam = small_family(n, dts)
    pcfg = PararealConfig(pr[0], dts[-1], pr[1], pr[2], pr[3]) if pr else None
    res = mlmc_estimate(fam, policy=FixedSamples(tuple(counts)), parareal_cfg=pcfg, seed=0)
    ora = oracle_levels(n, dts, counts, pr)
    stats = [mo.level_statistics(lvl, [r[0] for r in rows], [r[1] for r in rows])
             for lvl, rows in enumerate(ora)]
    E = sum(st.mean for st in stats)
    for lvl, st in enumerate(stats):
        g = res.per_level[lvl]
        assert g.n == st.n
        assert abs(g.mean_y - st.mean) <= 1e-8 * abs(E)
        assert abs(g.var_y - st.var) <= 1e-8 * abs(E)          # V_l, same absolute bar
        if lvl == len(counts) - 1 and pr:
            assert g.parareal_k == [r[2] for r in ora[lvl]]
    assert abs(res.expectation - E) <= 1e-8 * abs(E)
    return fam, ora


def test_estimator_small_mesh_with_parareal(cuda):
    check_estimate(8, (T / 32, T / 64, T / 128), (6, 4, 3), (4, T / 16, 1e-8, 4))


def test_estimator_config1_subset(cuda):
    """Config-1 settings on the 32x32 mesh (Parareal M=16, K<=5, tol 1e-8)."""
    from paper_2507_19246_b200.parareal import PararealConfig
    fam, ora = check_estimate(32, (T / 256, T / 512, T / 1024), (3, 2, 1), (16, T / 16, 1e-8, 5))
    # per-sample parity through the batched family entry point
    draws = [np.array([mo.draw(mo.CONFIGS[1], 0, lvl, k) for k in range(1, N + 1)])
             for lvl, N in enumerate((3, 2, 1))]
    out = fam.run_levels(draws, PararealConfig(16, T / 1024, T / 16, 1e-8, 5))
    for lvl, b in enumerate(out):
        ql, qm = b.q_l.cpu().numpy(), b.q_lm1.cpu().numpy()
        for i, (hi, lo, k) in enumerate(ora[lvl]):
            assert abs(ql[i] - hi) <= 1e-8 * abs(hi)
            if lvl:
                assert abs(qm[i] - lo) <= 1e-8 * abs(lo)
        if lvl == 2:
            assert b.k_used.cpu().numpy().tolist() == [r[2] for r in ora[lvl]]


def test_partition_bitwise_independent(cuda):
    """Emulated 3-rank run (contiguous shards, slot buffers summed, fixed-order
    reduction) equals the 1-rank run bitwise."""
    import torch
    from paper_2507_19246_b200.engine import level_reduce
    from paper_2507_19246_b200.mlmc import draw_level, shard_range
    from paper_2507_19246_b200.parareal import PararealConfig
    fam = small_family()
    pcfg = PararealConfig(4, T / 128, T / 16, 1e-8, 4)
    counts = (7, 5, 4)
    full = fam.run_levels([draw_level(fam.uncertain, 0, l, range(1, n + 1))
                           for l, n in enumerate(counts)], pcfg)
    slots = [torch.zeros((n, 4), dtype=torch.float64, device="cuda") for n in counts]
    for rank in range(3):
        rngs = [shard_range(n, rank, 3) for n in counts]
        part = fam.run_levels([draw_level(fam.uncertain, 0, l, range(a + 1, b + 1))
                               for l, (a, b) in enumerate(rngs)], pcfg)
        for l, (b, (a, e)) in enumerate(zip(part, rngs)):
            slots[l][a:e, 0] += b.q_l
            slots[l][a:e, 1] += b.q_lm1
            slots[l][a:e, 2] += b.k_used.to(torch.float64)
    for l, b in enumerate(full):
        np.testing.assert_array_equal(slots[l][:, 0].cpu().numpy(), b.q_l.cpu().numpy())
        np.testing.assert_array_equal(slots[l][:, 1].cpu().numpy(), b.q_lm1.cpu().numpy())
        s1 = level_reduce(slots[l][:, 0].contiguous(), slots[l][:, 1].contiguous()).cpu().numpy()
        s2 = level_reduce(b.q_l, b.q_lm1).cpu().numpy()
        np.testing.assert_array_equal(s1, s2)


def test_level_reduce_kernel_formulas(cuda):
    import torch
    from paper_2507_19246_b200.engine import level_reduce
    rng = np.random.default_rng(0)
    a, b = rng.random(1000), rng.random(1000)
    out = level_reduce(torch.tensor(a, device="cuda"), torch.tensor(b, device="cuda")).cpu().numpy()
    y = a - b
    np.testing.assert_allclose(out[:2], [y.sum(), (y * y).sum()], rtol=1e-13)
    assert abs(out[2] - y.mean()) < 1e-15 and abs(out[3] - y.var(ddof=1)) < 1e-14


def test_failures_map_to_reference_errors(cuda):
    from paper_2507_19246_b200.parareal import PararealConfig, PropagatorError
    from paper_2507_19246_b200.timeint import SingularSystemError
    fam = small_family(max_it=2)
    draws = [np.array([mo.draw(mo.CONFIGS[0], 0, 0, 1)])]
    fam.run_levels(draws, levels=[0])
    with pytest.raises(SingularSystemError):
        fam.check_status()
    fam.run_levels([np.array([mo.draw(mo.CONFIGS[0], 0, 2, 1)])],
                   PararealConfig(4, T / 128, T / 16, 1e-8, 4), levels=[2])
    with pytest.raises((PropagatorError, SingularSystemError)):
        fam.check_status()


# ---------------------------------------------------------------- large meshes
def large_family(cfg_i):
    from paper_2507_19246_b200.models import eddy_current_family
    return eddy_current_family(cfg_i, device="cuda:0")


@pytest.mark.slow
def test_cfg3_128_kl_sequential_and_parareal(cuda):
    """128x128 lognormal KL field (config 3): streaming path vs splu oracle."""
    import torch
    from paper_2507_19246_b200.parareal import PararealConfig
    fam = large_family(3)
    assert not fam.solver.sys.sm_resident
    cfg = mo.CONFIGS[3]
    prob = mo.FEProblem(128, "kl64")
    p = np.array([mo.draw(cfg, 0, 0, k) for k in (1, 2)])
    out = fam.run_levels([p], levels=[0])[0]
    for i in range(2):
        q = mo.evaluate(prob, cfg, p[i], T / 128, False).q
        assert abs(out.q_l[i].item() - q) <= 1e-8 * abs(q)
    pp = np.array([mo.draw(cfg, 0, 2, 1)])
    b = fam.run_levels([pp], PararealConfig(32, T / 512, T / 32, 1e-8, 6), levels=[2])[0]
    rec = mo.evaluate(prob, cfg, pp[0], T / 512, True)
    assert int(b.k_used[0].item()) == rec.k_used
    assert abs(b.q_l[0].item() - rec.q) <= 1e-8 * abs(rec.q)
    del torch


@pytest.mark.slow
def test_cfg2_256_time_averaged(cuda):
    fam = large_family(2)
    cfg = mo.CONFIGS[2]
    p = np.array([mo.draw(cfg, 0, 0, 1)])
    out = fam.run_levels([p], levels=[0])[0]
    q = mo.evaluate(mo.FEProblem(256, "blocks8"), cfg, p[0], cfg.dts[0], False).q
    assert abs(out.q_l[0].item() - q) <= 1e-8 * abs(q)


@pytest.mark.slow
def test_cfg4_512_level0(cuda):
    fam = large_family(4)
    cfg = mo.CONFIGS[4]
    p = np.array([mo.draw(cfg, 0, 0, 1)])
    out = fam.run_levels([p], levels=[0])[0]
    q = mo.evaluate(mo.FEProblem(512, "blocks8"), cfg, p[0], cfg.dts[0], False).q
    assert abs(out.q_l[0].item() - q) <= 1e-8 * abs(q)


@pytest.mark.parametrize("impl", ["auto", "twolaunch", "coop", "cluster", "tile"])
def test_streaming_64_mesh_vs_oracle(cuda, impl, monkeypatch):
    """64x64 mesh (3969 rows) forced onto the streaming path: every kernel
    family of it (MLMCP_STREAM_IMPL: two-launch ELL kernels, grid-resident
    cooperative, thread-block cluster, fused tile kernel), sequential and
    Parareal, vs the splu oracle."""
    from paper_2507_19246_b200 import fe
    from paper_2507_19246_b200.models import (EddyCurrentFamily, ParameterVector, QoIKind,
                                              UncertainInput, make_hierarchy)
    from paper_2507_19246_b200.parareal import PararealConfig
    code = {"auto": None, "twolaunch": "1", "coop": "2", "cluster": "3", "tile": "4"}[impl]
    if code is None:
        monkeypatch.delenv("MLMCP_STREAM_IMPL", raising=False)
    else:
        monkeypatch.setenv("MLMCP_STREAM_IMPL", code)   # read by libmlmcp on every call
    nominal = np.array([fe.NU0] * 4 + [fe.SIGMA0] * 4)
    fam = EddyCurrentFamily("quad4", UncertainInput(ParameterVector("quad4", nominal), 0.1),
                            make_hierarchy([T / 64, T / 128]), T, 64, "quad4",
                            QoIKind.MAGNETIC_ENERGY_T, device="cuda:0", path="stream")
    cfg = mo.OracleConfig("t64", 64, "quad4", T, (T / 64, T / 128), (3, 1), "energy_T",
                          parareal=(8, T / 8, 1e-8, 4))
    prob = mo.FEProblem(64, "quad4")
    p = np.array([mo.draw(cfg, 0, 0, k) for k in (1, 2, 3)])
    out = fam.run_levels([p], levels=[0])[0]
    fam.check_status()
    for i in range(3):
        q = mo.evaluate(prob, cfg, p[i], T / 64, False, dense=False).q
        assert abs(out.q_l[i].item() - q) <= 1e-8 * abs(q)
    pp = np.array([mo.draw(cfg, 0, 1, 1)])
    b = fam.run_levels([pp], PararealConfig(8, T / 128, T / 8, 1e-8, 4), levels=[1])[0]
    fam.check_status()
    rec = mo.evaluate(prob, cfg, pp[0], T / 128, True, dense=False)
    assert int(b.k_used[0].item()) == rec.k_used
    assert abs(b.q_l[0].item() - rec.q) <= 1e-8 * abs(rec.q)


def test_device_draws_bitwise(cuda):
    """mlmcp_draw_uniform (device) == draw_level (host) == numpy RandomStream."""
    import torch

    from paper_2507_19246_b200.mlmc import RandomStream, draw_level, draw_level_device
    from paper_2507_19246_b200.models import ParameterVector, UncertainInput
    nominal = np.array([795.77] * 4 + [1e6] * 4)
    inp = UncertainInput(ParameterVector("quad4", nominal), 0.1)
    for seed, lvl, kf, n in ((0, 0, 1, 1000), (5, 2, 2 ** 32 - 3, 7), (2 ** 40, 1, 17, 33)):
        out = torch.empty((n, 8), dtype=torch.float64, device="cuda")
        draw_level_device(inp, seed, lvl, kf, n, out)
        host = draw_level(inp, seed, lvl, range(kf, kf + n))
        np.testing.assert_array_equal(out.cpu().numpy(), host)
        np.testing.assert_array_equal(
            host[-1], RandomStream(seed, lvl, kf + n - 1).generator().uniform(nominal * 0.9,
                                                                                 nominal * 1.1))


@pytest.mark.parametrize("cfg_id,counts", [(1, (24, 12, 8)), (0, (16, 8, 4))])
def test_fused_launch_matches_separate_launches(cuda, cfg_id, counts):
    """The scheduled persistent launch (mlmcp_run_fused) vs separate launches:
    the sequential solves run the same per-task code (bitwise equal Q); the
    Parareal coarse sweep is pipelined per slice there (each coarse slice a
    task with its own PCG start), so the finest level agrees to the solver
    tolerance with identical iteration counts K."""
    from paper_2507_19246_b200.mlmc import draw_level
    from paper_2507_19246_b200.models import eddy_current_family
    from paper_2507_19246_b200.configs import get_config
    fam = eddy_current_family(cfg_id, device="cuda:0")
    draws = [draw_level(fam.uncertain, 0, lvl, range(1, n + 1)) for lvl, n in enumerate(counts)]
    pcfg = get_config(1).parareal_config()
    a = fam.run_levels(draws, pcfg, fused=True)
    fam.check_status()
    b = fam.run_levels(draws, pcfg, fused=False)
    fam.check_status()
    top = len(counts) - 1
    for lvl, (x, y) in enumerate(zip(a, b)):
        np.testing.assert_array_equal(x.q_lm1.cpu().numpy(), y.q_lm1.cpu().numpy())
        np.testing.assert_array_equal(x.k_used.cpu().numpy(), y.k_used.cpu().numpy())
        if lvl < top:
            np.testing.assert_array_equal(x.q_l.cpu().numpy(), y.q_l.cpu().numpy())
        else:
            np.testing.assert_allclose(x.q_l.cpu().numpy(), y.q_l.cpu().numpy(), rtol=1e-10)
            np.testing.assert_allclose(x.defects.cpu().numpy(), y.defects.cpu().numpy(),
                                       rtol=1e-6, atol=1e-11)


def test_graph_replay_matches_eager(cuda):
    """mlmc_estimate's CUDA-graph replay (run_levels_graphed) gives the same
    per-level sums as the eager launch sequence, across repeated estimates
    with different draws (seeds)."""
    from paper_2507_19246_b200.configs import get_config
    from paper_2507_19246_b200.mlmc import draw_level
    from paper_2507_19246_b200.models import eddy_current_family
    fam = eddy_current_family(1, device="cuda:0")
    pcfg = get_config(1).parareal_config()
    counts = (20, 10, 6)
    for seed in (0, 1, 0):
        draws = [draw_level(fam.uncertain, seed, lvl, range(1, n + 1))
                 for lvl, n in enumerate(counts)]
        g = fam.run_levels_graphed(draws, pcfg)
        gq = [(b.q_l.cpu().numpy().copy(), b.q_lm1.cpu().numpy().copy(), b.k_used.cpu().numpy().copy())
              for b in g]
        e = fam.run_levels(draws, pcfg)
        for (ql, qm, ku), b in zip(gq, e):
            np.testing.assert_array_equal(ql, b.q_l.cpu().numpy())
            np.testing.assert_array_equal(qm, b.q_lm1.cpu().numpy())
            np.testing.assert_array_equal(ku, b.k_used.cpu().numpy())


def test_chunked_estimate_bitwise(cuda, monkeypatch):
    """Full-size streaming configs run the rank's samples in several
    run_levels calls (max_samples_per_call); per-sample results do not depend
    on the batch composition, so the chunked estimate is bitwise the single-
    call one (forced here with a cap of 5 samples on a small mesh)."""
    from paper_2507_19246_b200.mlmc import FixedSamples, mlmc_estimate
    from paper_2507_19246_b200.parareal import PararealConfig
    fam = small_family()
    pr = PararealConfig(4, T / 128, T / 16, 1e-8, 4)
    counts = (12, 7, 5)
    ref = mlmc_estimate(fam, policy=FixedSamples(counts), parareal_cfg=pr, seed=3)
    monkeypatch.setattr(type(fam), "max_samples_per_call", lambda self, cfg=None, level=None: 5)
    got = mlmc_estimate(fam, policy=FixedSamples(counts), parareal_cfg=pr, seed=3)
    assert got.expectation == ref.expectation
    for a, b in zip(got.per_level, ref.per_level):
        assert (a.sum_y, a.sum_y2) == (b.sum_y, b.sum_y2)
    assert got.per_level[-1].parareal_k == ref.per_level[-1].parareal_k


def test_fused_scheduler_coarse_failure_ends_chains(cuda):
    """A Parareal batch whose coarse solves cannot converge (max_it below the
    coarse step's PCG count): every chain ends at its first coarse slice with
    the reference's PropagatorError(interval=1, iteration=1) status, the
    scheduler terminates, and no fine slice beyond the failure runs."""
    import torch

    from paper_2507_19246_b200 import _lib
    from paper_2507_19246_b200.parareal import PropagatorError, raise_parareal_status
    fam = small_family(n=32, max_it=20)
    sol = fam.solver
    P = np.array([mo.draw(mo.CONFIGS[1], 0, 2, k) for k in range(1, 5)])
    M, K = sol.assemble(torch.from_numpy(P).cuda())
    spec = dict(row0=0, S=4, t0=0.0, t1=T, m=16, dt_fine=T / 1024, dt_coarse=T / 16,
                tol=1e-8, k_max=5, qoi_mode=_lib.QOI_FINAL_ENERGY)
    _, pr = sol.run_fused(M, K, [], spec)
    st = pr.status.cpu().numpy()
    assert (st[:, 0] == _lib.ST_NOCONV).all()
    assert (st[:, 2] == 1).all() and (st[:, 3] == 1).all()      # interval 1, iteration 1
    fi = pr.fine_iters.cpu().numpy().reshape(4, 16)
    assert (fi[:, 0] > 0).all() and (fi[:, 1:] == 0).all()
    with pytest.raises(PropagatorError) as ei:
        raise_parareal_status(st, pr.fine_status.cpu().numpy())
    assert (ei.value.interval, ei.value.iteration) == (1, 1)


@pytest.mark.parametrize("n,env", [
    (40, {"MLMCP_STREAM_IMPL": "4"}),                               # one ragged tile column
    (72, {"MLMCP_STREAM_IMPL": "4"}),                               # 64 + 7 columns
    (72, {"MLMCP_STREAM_IMPL": "4", "MLMCP_TILE_CFG": "3"}),        # 8-row tiles
    (40, {"MLMCP_STREAM_IMPL": "5"}),                               # band path: 13 empty CTAs
    (72, {"MLMCP_STREAM_IMPL": "5"}),                               # band path, ragged rows
    (72, {"MLMCP_STREAM_IMPL": "4", "MLMCP_STREAM_GRAPH": "1"}),    # device-driven step loop
    (72, {"MLMCP_STREAM_IMPL": "1", "MLMCP_STREAM_GRAPH": "1"}),
])
def test_tile_path_ragged_grids_vs_oracle(cuda, n, env, monkeypatch):
    """The tile kernels on grids whose width / height are not multiples of the
    tile (edge tiles, halo clamping), every variant and the graph-driven step
    loop, and the band path on grids that leave part of its 16 x 16-row
    cluster empty: sequential and Parareal vs the splu oracle (QoI 1e-8, K equal)."""
    from paper_2507_19246_b200 import fe
    from paper_2507_19246_b200.models import (EddyCurrentFamily, ParameterVector, QoIKind,
                                              UncertainInput, make_hierarchy)
    from paper_2507_19246_b200.parareal import PararealConfig
    for k in ("MLMCP_STREAM_IMPL", "MLMCP_TILE_CFG", "MLMCP_STREAM_GRAPH"):
        monkeypatch.delenv(k, raising=False)
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    nominal = np.array([fe.NU0] * 8 + [fe.SIGMA0] * 8)
    fam = EddyCurrentFamily("blocks8", UncertainInput(ParameterVector("blocks8", nominal), 0.1),
                            make_hierarchy([T / 32, T / 64]), T, n, "blocks8",
                            QoIKind.MAGNETIC_ENERGY_T, device="cuda:0", path="stream")
    cfg = mo.OracleConfig(f"t{n}", n, "blocks8", T, (T / 32, T / 64), (3, 1), "energy_T",
                          parareal=(4, T / 4, 1e-8, 3))
    prob = mo.FEProblem(n, "blocks8")
    p = np.array([mo.draw(cfg, 0, 0, k) for k in (1, 2, 3)])
    out = fam.run_levels([p], levels=[0])[0]
    fam.check_status()
    for i in range(3):
        q = mo.evaluate(prob, cfg, p[i], T / 32, False, dense=False).q
        assert abs(out.q_l[i].item() - q) <= 1e-8 * abs(q)
    pp = np.array([mo.draw(cfg, 0, 1, 1)])
    b = fam.run_levels([pp], PararealConfig(4, T / 64, T / 4, 1e-8, 3), levels=[1])[0]
    fam.check_status()
    rec = mo.evaluate(prob, cfg, pp[0], T / 64, True, dense=False)
    assert int(b.k_used[0].item()) == rec.k_used
    assert abs(b.q_l[0].item() - rec.q) <= 1e-8 * abs(rec.q)


@pytest.mark.parametrize("impl", ["3", "4"])
def test_streaming_coarse_failure_maps_to_propagator_error(cuda, impl, monkeypatch):
    """Coarse solves that cannot converge within max_it on the cluster sweep
    (impl 3) and on the tile path (impl 4): the sample is deactivated with the
    reference's PropagatorError(interval=1, iteration=1) (parareal.py:151-152)."""
    from paper_2507_19246_b200 import fe
    from paper_2507_19246_b200.models import (EddyCurrentFamily, ParameterVector, QoIKind,
                                              UncertainInput, make_hierarchy)
    from paper_2507_19246_b200.parareal import PararealConfig, PropagatorError
    monkeypatch.setenv("MLMCP_STREAM_IMPL", impl)
    nominal = np.array([fe.NU0] * 8 + [fe.SIGMA0] * 8)
    fam = EddyCurrentFamily("blocks8", UncertainInput(ParameterVector("blocks8", nominal), 0.1),
                            make_hierarchy([T / 32]), T, 64, "blocks8",
                            QoIKind.MAGNETIC_ENERGY_T, device="cuda:0", path="stream",
                            max_it=12)
    cfg = mo.OracleConfig("t64f", 64, "blocks8", T, (T / 32,), (2,), "energy_T",
                          parareal=(4, T / 4, 1e-8, 3))
    pp = np.array([mo.draw(cfg, 0, 0, k) for k in (1, 2)])
    fam.run_levels([pp], PararealConfig(4, T / 32, T / 4, 1e-8, 3), levels=[0])
    with pytest.raises(PropagatorError) as ei:
        fam.check_status()
    assert (ei.value.interval, ei.value.iteration) == (1, 1)


def test_pipelined_calls_bitwise(cuda, monkeypatch):
    """Config 2 (256^2, band path) with its calls two in flight on two streams
    (mlmc.run_level_calls: finest level first, balanced chunks) against one
    call at a time (MLMCP_PIPELINE=0): level sums and the estimate bitwise
    equal, and the plan covers every sample exactly once."""
    from paper_2507_19246_b200.mlmc import FixedSamples, mlmc_estimate, plan_calls
    from paper_2507_19246_b200.models import EddyCurrentFamily
    monkeypatch.delenv("MLMCP_PIPELINE", raising=False)
    fam = large_family(2)
    monkeypatch.setattr(EddyCurrentFamily, "max_samples_per_call",
                        lambda self, parareal_cfg=None, level=None: 3)
    counts = (7, 4, 2, 1)
    assert fam.call_streams(None) is not None and len(fam.call_streams(None)) == 2
    calls = plan_calls([(0, n) for n in counts], [3] * 4, pipelined=True)
    assert [c[0] for c in calls] == sorted((c[0] for c in calls), reverse=True)
    for lvl, n in enumerate(counts):
        cover = sorted((c0, c1) for l, c0, c1 in calls if l == lvl)
        assert cover[0][0] == 0 and cover[-1][1] == n
        assert all(a[1] == b[0] for a, b in zip(cover, cover[1:]))
        assert all(c1 - c0 <= 2 for c0, c1 in cover)      # 0.8 of the cap
    piped = mlmc_estimate(fam, policy=FixedSamples(counts), seed=0)
    monkeypatch.setenv("MLMCP_PIPELINE", "0")
    assert fam.call_streams(None) is None
    serial = mlmc_estimate(fam, policy=FixedSamples(counts), seed=0)
    assert piped.expectation == serial.expectation
    for a, b in zip(piped.per_level, serial.per_level):
        assert (a.n, a.mean_y, a.var_y) == (b.n, b.mean_y, b.var_y)


def test_periodic_region_vs_csr(cuda, monkeypatch):
    """Periodic steady states on a region-linear grid: the class-table COCG
    kernels (region parameters passed) against the kernels that stream the CSR
    values of M and K, both solved to 1e-12."""
    import torch
    from paper_2507_19246_b200.mlmc import draw_level
    fam = large_family(2)
    sol = fam.solver
    S = 3
    pd = torch.from_numpy(draw_level(fam.uncertain, 0, 1, range(1, S + 1))).cuda()
    M = torch.empty((S, sol.nnz), dtype=torch.float64, device="cuda")
    K = torch.empty_like(M)
    rp = sol.new_region_params(S)
    sol.assemble(pd, out=(M, K), rp_out=rp)
    sidx = torch.tensor([0, 1, 2, 0], dtype=torch.int32, device="cuda")
    dts = torch.tensor([T / 64, T / 64, T / 128, T / 512], dtype=torch.float64, device="cuda")
    kw = dict(rtol=1e-12, max_it=2000)
    x_rg = sol.sys.periodic_state(sidx, dts, M, K, sol.profile, sol.omega, rp=rp, **kw)
    x_csr = sol.sys.periodic_state(sidx, dts, M, K, sol.profile, sol.omega, rp=None, **kw)
    monkeypatch.setenv("MLMCP_PERIODIC_REGION", "0")
    x_off = sol.sys.periodic_state(sidx, dts, M, K, sol.profile, sol.omega, rp=rp, **kw)
    torch.cuda.synchronize()
    assert torch.equal(x_csr, x_off)                      # the knob selects the CSR kernels
    scale = x_csr.abs().amax(dim=(1, 2), keepdim=True)
    assert float(((x_rg - x_csr).abs() / scale).max()) <= 1e-9
    assert float(scale.min()) > 0.0


def test_run_levels_direct_chunking_bitwise(cuda, monkeypatch):
    """run_levels called directly with more samples than the per-call cap
    (_run_levels_chunked): per-sample Q_l, Q_{l-1}, K and iteration counts
    bitwise those of one call."""
    from paper_2507_19246_b200.mlmc import draw_level
    from paper_2507_19246_b200.parareal import PararealConfig
    fam = small_family()
    pcfg = PararealConfig(4, T / 128, T / 16, 1e-8, 4)
    draws = [draw_level(fam.uncertain, 0, lvl, range(1, n + 1)) for lvl, n in enumerate((7, 5, 4))]
    ref = fam.run_levels(draws, pcfg)
    ref = [(b.q_l.cpu().numpy(), b.q_lm1.cpu().numpy(), b.k_used.cpu().numpy(),
            b.iters.cpu().numpy()) for b in ref]
    monkeypatch.setattr(type(fam), "max_samples_per_call", lambda self, cfg=None, level=None: 3)
    got = fam.run_levels(draws, pcfg)
    fam.check_status()
    for b, (ql, qm, ku, its) in zip(got, ref):
        np.testing.assert_array_equal(b.q_l.cpu().numpy(), ql)
        np.testing.assert_array_equal(b.q_lm1.cpu().numpy(), qm)
        np.testing.assert_array_equal(b.k_used.cpu().numpy(), ku)
        np.testing.assert_array_equal(b.iters.cpu().numpy(), its)
