"""Cost model and executor accounting (SPEC.md [MODULE] costmodel :335-445 and
[MODULE] executor :447-500): the SPEC's worked examples and invariants."""

import math
import random

import numpy as np
import pytest

from paper_2507_19246_b200 import costmodel as cm
from paper_2507_19246_b200 import executor as ex


def test_parareal_time_examples():
    assert cm.parareal_time(100, 1, 10, 1) == pytest.approx(10.9, rel=1e-12)
    assert cm.parareal_time(100, 1, 10, 2) == pytest.approx(21.7, rel=1e-12)
    assert cm.parareal_time(100, 0.0, 7, 7) == pytest.approx(100.0, rel=1e-15)
    with pytest.raises(ValueError):
        cm.parareal_time(1, 1, 3, 4)


def test_parareal_effort_examples():
    assert cm.parareal_effort(100, 1, 10, 2) == pytest.approx(191.7, rel=1e-12)
    assert cm.parareal_effort(100, 1, 1, 1) == pytest.approx(100.0, rel=1e-15)
    e = cm.parareal_effort(100, 0.0, 10, 2)
    assert e == pytest.approx(190.0) and e > 100.0


def test_closed_forms_equal_iteration_sums():
    rng = random.Random(0)
    for _ in range(200):
        M = rng.randint(1, 64)
        K = rng.randint(1, M)
        tf, tc = rng.uniform(0, 1e3), rng.uniform(0, 10)
        assert cm.parareal_time(tf, tc, M, K) == pytest.approx(cm.parareal_time_sum(tf, tc, M, K),
                                                                rel=1e-12)
        assert cm.parareal_effort(tf, tc, M, K) == pytest.approx(
            cm.parareal_effort_sum(tf, tc, M, K), rel=1e-12)


def test_ideal_speedup():
    assert cm.ideal_speedup(10, 2) == pytest.approx(999 / 189, rel=1e-14)
    assert cm.ideal_speedup(2, 2) == pytest.approx(1.4, rel=1e-14)
    rng = random.Random(1)
    for _ in range(100):
        r, L = rng.uniform(1.1, 20), rng.randint(1, 6)
        C = [r ** l for l in range(L + 1)]
        sigma = sum(C) / (sum(C[:L]) + C[L - 1])
        assert cm.ideal_speedup(r, L) == pytest.approx(sigma, rel=1e-12)
        assert cm.ideal_speedup(r, L) > 1.0


def test_kappa_examples_and_scan():
    assert cm.kappa(10, 16) == 1
    assert cm.kappa(10, 180) == 6
    for r in range(2, 13):
        for n in range(1, 257):
            assert cm.kappa(r, n) == cm.kappa_scan(r, n), (r, n)
    rng = random.Random(2)
    for _ in range(200):
        r, n = rng.uniform(1.01, 30), rng.randint(1, 4096)
        assert cm.kappa(r, n) <= r


def test_batch_and_cores():
    assert cm.batch_count(10303, 0.0, 180) == 58
    assert cm.batch_count(10, 0.1, 180) == 1
    assert cm.batch_count(0, 0.1, 180) == 0
    assert cm.cores_per_sample(180, 10, 0.1) == 16
    assert cm.cores_per_sample(10, 10, 0.0) == 1
    assert cm.cores_per_sample(1000, 10, 0.1) == 90
    with pytest.raises(ValueError):
        cm.cores_per_sample(5, 10, 0.1)


def test_effort_ratio():
    p = cm.CostModelParams(N=(10303, 85, 0))
    assert cm.effort_ratio_infinite(p, 1, M=16) == 1.0
    p = cm.CostModelParams()
    # term-by-term summation oracle
    C = [1.0, 10.0, 100.0]
    ref = 10303 * C[0] + 85 * C[1] + 10 * C[2]
    e_para = (1 / 16) * (16 - 1) * (C[2] + C[0]) + (1 / 16) * C[2]
    comb = 10303 * C[0] + 85 * C[1] + 10 * e_para
    assert cm.effort_ratio_infinite(p, 1, M=16) == pytest.approx(comb / ref, rel=1e-12)
    for K in range(1, 17):
        assert cm.effort_ratio_infinite(p, K) >= 1.0
    assert cm.effort_ratio_max(p) == cm.effort_ratio_infinite(p, cm.kappa(10, 16))


def test_finite_speedup_oracle_and_monotone():
    p = cm.CostModelParams(n_c=180)
    b = [58, 1, 1]
    C = [1.0, 10.0, 100.0]
    n = 16
    num = sum(bi * ci for bi, ci in zip(b, C))
    den = b[0] * C[0] + b[1] * C[1] + (1 / n) * (100 + (n - 1) * 1)
    assert cm.finite_speedup(p, 1) == pytest.approx(num / den, rel=1e-12)
    s = [cm.finite_speedup(p, K) for K in range(1, 17)]
    assert all(a > b for a, b in zip(s, s[1:]))


def test_figure_data(tmp_path):
    p = cm.CostModelParams()
    rows = cm.figure_data(p, [180, 360, 720, 1440], range(1, 11))
    by = {(n, K): (s, e) for n, K, s, e in rows}
    for n, K, s, e in rows:
        if not math.isnan(s):
            q = cm.CostModelParams(n_c=n)
            assert s == cm.finite_speedup(q, K)
    for K in range(1, 11):
        vals = [by[(n, K)][0] for n in (180, 360, 720, 1440)]
        vals = [v for v in vals if not math.isnan(v)]
        assert all(b >= a for a, b in zip(vals, vals[1:]))
    for n in (180, 360, 720, 1440):
        eps = [by[(n, K)][1] for K in range(1, 11) if not math.isnan(by[(n, K)][1])]
        assert all(b >= a for a, b in zip(eps, eps[1:]))
    out = tmp_path / "f.csv"
    cm.write_figure_csv(str(out), rows, note="s_inf=%r" % cm.ideal_speedup(10, 2))
    text = out.read_text().splitlines()
    assert text[1] == "n_c,K,speedup,effort_ratio"
    assert len(text) == 2 + len(rows)


def test_schedule_level():
    tasks = [ex.SequentialSolve(0, k, cost_s=1.0) for k in range(10303)]
    assert len(ex.schedule_level(tasks, 180)) == 58
    tasks = ([ex.PararealSolve(2, k, width=16, tau_F=100, tau_C=1, K=2) for k in range(10)]
             + [ex.SequentialSolve(2, k, cost_s=10) for k in range(10)])
    assert len(ex.schedule_level(tasks, 180)) == 1
    assert ex.schedule_level([], 180) == []
    with pytest.raises(ValueError):
        ex.schedule_level([ex.PararealSolve(2, 0, width=200)], 180)


def test_simulated_table2():
    rt = (10.02, 47.87, 397.45)
    N = (10303, 85, 10)
    ref = ex.simulate(ex.plan_tasks(N, rt), 180)
    comb = ex.simulate(ex.plan_tasks(N, rt, (16, 1, rt[0], 147.93)), 180)
    assert [lv.batches for lv in ref.levels] == [58, 1, 1]
    oracle_ref = 58 * 10.02 + 1 * 47.87 + 1 * 397.45
    oracle_comb = 58 * 10.02 + 1 * 47.87 + 1 * 147.93
    assert ref.total_wall_s == pytest.approx(oracle_ref, rel=1e-12)
    assert comb.total_wall_s == pytest.approx(oracle_comb, rel=1e-12)
    assert ref.total_wall_s / comb.total_wall_s == pytest.approx(oracle_ref / oracle_comb,
                                                                 rel=1e-9)
    # ledger identity: Parareal level effort = N_L E_para + coupled coarse costs
    e2 = comb.levels[2].effort_core_s
    assert e2 == pytest.approx(10 * cm.parareal_effort(397.45, 10.02, 16, 1) + 10 * 47.87,
                               rel=1e-12)
    for lv in ref.levels:
        assert lv.effort_core_s >= lv.wall_s
    single = ex.simulate([[ex.SequentialSolve(0, 0, cost_s=3.0)]], 4)
    assert single.total_wall_s == single.total_effort_core_s == 3.0
    d = comb.to_dict()
    assert set(d) >= {"mode", "levels", "total_wall_s", "total_effort_core_s"}
    assert set(d["levels"][0]) == {"level", "batches", "wall_s", "effort_core_s"}
    assert np.isclose(d["total_effort_core_s"], sum(x["effort_core_s"] for x in d["levels"]))
