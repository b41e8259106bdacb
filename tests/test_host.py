"""CPU: host-side logic of the product package — configs, grids, validation,
draws, FE setup vs the oracle, the estimator with the closed-form toy family
(SPEC.md KATs for the mlmc / parareal host pieces)."""

import numpy as np
import pytest

from conftest import golden
from oracle import mlmc_oracle as mo
from paper_2507_19246_b200 import fe
from paper_2507_19246_b200.configs import CONFIGS, T
from paper_2507_19246_b200.mlmc import (FixedSamples, RandomStream, draw_level, mlmc_estimate,
                                        optimal_allocation, shard_range)
from paper_2507_19246_b200.models import (GaussianInput, LevelSpec, ParameterVector, UncertainInput,
                                          draw_parameters, make_hierarchy, toy_family)
from paper_2507_19246_b200.parareal import PararealConfig, defect
from paper_2507_19246_b200.solver import parareal_grid
from paper_2507_19246_b200.timeint import step_count


def test_seq_equivalent_steps():
    assert CONFIGS[1].seq_equiv_steps() == 278528
    assert CONFIGS[0].seq_equiv_steps() == 67520
    assert CONFIGS[2].seq_equiv_steps() == 2424832
    assert CONFIGS[3].seq_equiv_steps() == 557056
    assert CONFIGS[4].seq_equiv_steps() == 1212416


def test_step_count_rules():
    assert step_count(0.0, T, T / 256) == 256
    with pytest.raises(ValueError):
        step_count(0.0, 1.0, 0.3)
    with pytest.raises(ValueError):
        step_count(0.0, 1.0, 0.0)


def test_parareal_config_validation():
    with pytest.raises(ValueError):
        PararealConfig(0, 1e-3, 1e-2)
    with pytest.raises(ValueError):
        PararealConfig(4, 1e-2, 1e-3)        # dt_coarse < dt_fine
    with pytest.raises(ValueError):
        PararealConfig(4, 1e-3, 1e-2, max_iterations=5)
    with pytest.raises(ValueError):
        PararealConfig(4, 1e-3, 1e-2, tolerance=-1.0)
    c = PararealConfig(4, 1e-3, 1e-2)
    assert c.k_max == 4 and c.with_dt_fine(1e-3) is c and c.with_dt_fine(5e-4).dt_fine == 5e-4


def test_parareal_grid_config1():
    bounds, fk0, fst, ck0, cst = parareal_grid(0.0, T, 16, T / 1024, T / 16)
    assert np.all(fst == 64) and np.all(cst == 1)
    np.testing.assert_array_equal(fk0, np.arange(16) * 64)
    np.testing.assert_array_equal(ck0, np.arange(16))
    with pytest.raises(ValueError):
        parareal_grid(0.0, T, 3, T / 1024, T / 16)


def test_defect_examples():
    # SPEC.md:218-220
    assert defect([[1.0, 2.0]], [[1.0, 2.0]]) == 0.0
    assert abs(defect([[1.0, 0.0]], [[1.0, 1.0]]) - 2 ** -0.5) < 1e-15
    a, b = np.random.default_rng(1).random((2, 3, 5))
    assert abs(defect(a * 1e3, b * 1e3) - defect(a, b)) <= 1e-12 * defect(a, b)
    assert defect(np.zeros((0, 3)), np.zeros((0, 3))) == 0.0


def test_draws_identical_to_reference_and_oracle():
    g = golden("draws")
    inp = UncertainInput(ParameterVector("quad4", g["nominal"]), 0.1)
    for key, row in zip(g["keys"], g["uniform"]):
        np.testing.assert_array_equal(draw_parameters(inp, RandomStream(*key)).values, row)
    gi = GaussianInput("kl64", 64)
    np.testing.assert_array_equal(draw_parameters(gi, RandomStream(0, 2, 1)).values, g["gaussian"][0])
    d = draw_level(inp, 0, 1, [1, 2, 3])
    np.testing.assert_array_equal(d[1], mo.draw(mo.CONFIGS[0], 0, 1, 2))


def test_draw_halfwidth_zero_and_positivity():
    inp = UncertainInput(ParameterVector("quad4", np.ones(8)), 0.0)
    np.testing.assert_array_equal(draw_parameters(inp, RandomStream(0, 0, 1)).values, np.ones(8))
    with pytest.raises(ValueError):
        ParameterVector("quad4", -np.ones(8))
    with pytest.raises(ValueError):
        ParameterVector("quad4", np.ones(7))
    with pytest.raises(ValueError):
        UncertainInput(ParameterVector("quad4", np.ones(8)), 1.0)


def test_hierarchy():
    h = make_hierarchy([T / 32, T / 64])
    assert h[1] == LevelSpec(1, T / 64)
    with pytest.raises(ValueError):
        make_hierarchy([T / 64, T / 32])


@pytest.mark.parametrize("n,layout", [(8, "quad4"), (16, "blocks8"), (16, "kl64"), (32, "quad4")])
def test_product_fe_setup_matches_oracle(n, layout):
    """Pattern, gather map and source profile of fe.py vs the oracle's element
    loop (independent implementations)."""
    m = fe.structured_mesh(n)
    cfg = {"quad4": mo.CONFIGS[0], "blocks8": mo.CONFIGS[2], "kl64": mo.CONFIGS[3]}[layout]
    p = mo.draw(cfg, 0, 1, 5)
    model = mo.FEProblem(n, layout).model(p, dense=False)
    if layout == "kl64":
        sig = np.exp(np.log(fe.SIGMA0) + fe.KL_SCALE * (p @ fe.kl_basis(m)))
        nu = np.full(m.n_elem, fe.NU0)
    else:
        reg = fe.region_map(m, layout)
        R = len(fe.conducting_mask(layout))
        nu = p[:R][reg]
        sig = (p[R:2 * R] * fe.conducting_mask(layout))[reg]
    Mv = np.add.reduceat(sig[m.celem] * m.cmw, m.cptr[:-1])
    Kv = np.add.reduceat(nu[m.celem] * m.ckw, m.cptr[:-1])
    Mo, Ko = model.mass.tocsr(), model.stiffness.tocsr()
    Mo.sort_indices()
    Ko.sort_indices()
    np.testing.assert_array_equal(Mo.indptr, m.row_ptr)
    np.testing.assert_array_equal(Mo.indices, m.col)
    np.testing.assert_allclose(Mv, Mo.data, rtol=1e-13, atol=1e-13 * np.abs(Mo.data).max())
    np.testing.assert_allclose(Kv, Ko.data, rtol=1e-13, atol=1e-13 * np.abs(Ko.data).max())
    np.testing.assert_allclose(fe.source_profile(m, layout), model.forcing.profile, rtol=1e-13)
    assert int(np.diff(m.row_ptr).max()) == 7


def test_shard_range_covers_exactly():
    for n in (0, 1, 7, 512):
        for world in (1, 2, 3, 8):
            parts = [shard_range(n, r, world) for r in range(world)]
            assert parts[0][0] == 0 and parts[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(parts, parts[1:]))


def test_optimal_allocation_examples():
    # SPEC.md:296-298
    V, C = [1.0, 1e-2, 1e-4], [1.0, 10.0, 100.0]
    n = optimal_allocation(V, C, rmse=1e-3)
    w = np.sqrt(np.array(V) / np.array(C))
    np.testing.assert_allclose(w / w[0], [1.0, 0.0316228, 0.001], rtol=1e-5)
    assert n[0] > n[1] > n[2] >= 2
    assert optimal_allocation([0.0, 0.0], [1.0, 1.0], rmse=1.0) == [2, 2]
    assert optimal_allocation([2.0], [1.0], rmse=0.1) == [int(np.ceil(2 * 2.0 / 0.01))]
    a = optimal_allocation(V, C, rmse=1e-2)
    b = optimal_allocation(V, [c * 7 for c in C], rmse=1e-2)   # homogeneous in C
    assert a == b


def test_toy_estimator_telescoping_and_coupling():
    fam = toy_family(make_hierarchy([0.1, 0.05, 0.025]), halfwidth=0.05)
    res = mlmc_estimate(fam, policy=FixedSamples((200, 50, 20)), seed=3)
    assert abs(res.expectation - sum(st.mean_y for st in res.per_level)) < 1e-15
    # E[Q_L] = 1 + dt_L for xi ~ U[0.95, 1.05]
    assert abs(res.expectation - 1.025) < 4 * res.rmse_estimate + 1e-3
    # level-0 mean equals a plain MC mean of the same keys
    qs = [draw_parameters(fam.uncertain, RandomStream(3, 0, k)).values[0] * 1.1 for k in range(1, 201)]
    assert abs(res.per_level[0].mean_y - np.mean(qs)) < 1e-14


def test_toy_estimator_equal_dt_levels_zero():
    # SPEC.md:287 / :309: identical dt on two levels -> Y = 0 on level 1
    fam = toy_family([LevelSpec(0, 0.1), LevelSpec(1, 0.1)])
    res = mlmc_estimate(fam, policy=FixedSamples((10, 10)), seed=0)
    assert res.per_level[1].sum_y == 0.0 and res.per_level[1].var_y == 0.0


def test_toy_estimator_constant_qoi():
    fam = toy_family(make_hierarchy([0.1, 0.05]), nominal=2.0, halfwidth=0.0)
    res = mlmc_estimate(fam, policy=FixedSamples((5, 5)), seed=0)
    assert abs(res.expectation - 2.0 * 1.05) <= 1e-15 * 2.1 and res.rmse_estimate == 0.0


def test_bench_reports_one_workload_for_both_arms():
    """bench.py: the headline workload is config 2 (the largest single-GPU
    configuration) with its full N_l; both arms name the same workload, and
    the CPU legs use the same method (model-based extrapolation from level-0
    solves for the splu-sized meshes, a proportional subset at 32^2)."""
    import bench
    from paper_2507_19246_b200.configs import get_config
    args = bench.parse.__wrapped__() if hasattr(bench.parse, "__wrapped__") else None
    del args
    cfg = get_config(2)
    w = bench.workload_name(2, cfg, list(cfg.samples), cfg.parareal_config())
    assert w.startswith("cfg2: 256x256") and "N_l=[4096, 1024, 256, 64]" in w
    assert "no Parareal" in w and "4 period(s)" in w and "T/64..T/512" in w
    c1 = get_config(1)
    w1 = bench.workload_name(1, c1, list(c1.samples), c1.parareal_config())
    assert w1.startswith("cfg1: 32x32") and "Parareal M=16" in w1
    assert cfg.seq_equiv_steps() == 2424832


def test_level_costs_follow_level_work():
    """each level gets its own cost per sample, the
    wall time split by solver work, so optimal_allocation sees C_l grow with
    the level's steps (and the Parareal level's redundant fine work)."""
    from paper_2507_19246_b200.mlmc import _level_costs
    from paper_2507_19246_b200.models import make_hierarchy
    from paper_2507_19246_b200.parareal import PararealConfig
    h = make_hierarchy([0.02 / 64, 0.02 / 128, 0.02 / 256])
    c = _level_costs(h, [100, 50, 10], None, None, 1.0)
    assert abs(sum(ci * n for ci, n in zip(c, [100, 50, 10])) - 1.0) < 1e-12
    assert abs(c[1] / c[0] - 3.0) < 1e-12 and abs(c[2] / c[1] - 2.0) < 1e-12
    pc = PararealConfig(16, 0.02 / 256, 0.02 / 16, 1e-8, 5)
    cp = _level_costs(h, [100, 50, 10], pc, [3] * 10, 1.0)
    assert cp[2] / cp[1] > c[2] / c[1]          # Parareal redundancy (K=3: 45/16 fine work)


def test_toy_family_chunked_estimate_bitwise():
    from paper_2507_19246_b200.mlmc import FixedSamples, mlmc_estimate
    from paper_2507_19246_b200.models import make_hierarchy, toy_family
    h = make_hierarchy([0.1, 0.05, 0.025])
    a = mlmc_estimate(toy_family(h), policy=FixedSamples((23, 9, 4)), seed=5)
    b = mlmc_estimate(toy_family(h, cap=3), policy=FixedSamples((23, 9, 4)), seed=5)
    assert a.expectation == b.expectation
    assert [(s.sum_y, s.sum_y2) for s in a.per_level] == [(s.sum_y, s.sum_y2) for s in b.per_level]


def test_plan_calls_cover_and_order():
    """mlmc.plan_calls: every sample of every level in exactly one call; one
    call at a time keeps the level order and the caps; the pipelined plan keeps
    each call within 0.8 of its cap, balances a level's chunks and starts with
    the finest level."""
    from paper_2507_19246_b200.mlmc import plan_calls
    ranges = [(0, 4096), (10, 1034), (0, 0), (5, 69)]
    caps = [3335, 2620, 2620, 2620]
    for pipelined in (False, True):
        calls = plan_calls(ranges, caps, pipelined)
        for lvl, (a, b) in enumerate(ranges):
            mine = sorted((c0, c1) for l, c0, c1 in calls if l == lvl)
            if b <= a:
                assert not mine
                continue
            assert mine[0][0] == a and mine[-1][1] == b
            assert all(x[1] == y[0] for x, y in zip(mine, mine[1:]))
            lim = int(caps[lvl] * 0.8) if pipelined else caps[lvl]
            assert all(0 < c1 - c0 <= lim for c0, c1 in mine)
        lv = [c[0] for c in calls]
        assert lv == sorted(lv, reverse=pipelined)
    piped = plan_calls(ranges, caps, True)
    sizes0 = [c1 - c0 for l, c0, c1 in piped if l == 0]
    assert sizes0 == [2048, 2048]                      # balanced, not 2668 + 1428


def test_run_level_calls_without_streams_checks_each_call():
    """run_level_calls on a family without call streams: calls in plan order,
    the status check after each one."""
    from paper_2507_19246_b200.mlmc import run_level_calls

    class Fam:
        def __init__(self):
            self.log = []

        def check_status(self, token=None):
            self.log.append("check")

    fam = Fam()
    run_level_calls(fam, [(0, 0, 2), (1, 0, 1)], lambda l, a, b: fam.log.append((l, a, b)))
    assert fam.log == [(0, 0, 2), "check", (1, 0, 1), "check"]
