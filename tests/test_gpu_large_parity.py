"""GPU path vs golden fixtures produced by the UNMODIFIED reference at the
BASELINE.json mesh sizes (oracle/make_large_goldens.py: the reference's own
implicit_euler_solve / parareal_solve, timeint.py:88-128 / parareal.py:121-220,
with the splu backend of SURVEY §8(c)).

Covers what round 1 left unchecked: every one of config 3's 128 finest-level
samples (Parareal M=32, K<=6: K equal per sample, defect histories), config 4's
finest level at 512^2 (Parareal M=64, K<=6), config 2's levels 1-3 (256^2,
four periods, time-averaged QoI) and config 3's level statistics (mean_Y and
V_l with an absolute tolerance of 1e-8 |E|).

Tolerances: per-sample Q within 1e-8 relative (the north-star bar); defect
histories within 1e-10 absolute (the stopping test compares them with 1e-8);
PCG stopping rule ||r||_{D^-1} <= 1e-13 ||b||_{D^-1}.
"""

import numpy as np
import pytest

from conftest import golden

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

RTOL = 1e-8


def _family(cfg_i):
    from paper_2507_19246_b200.models import eddy_current_family
    return eddy_current_family(cfg_i, device="cuda:0")


def _check_q(got, want, what):
    got = np.asarray(got, dtype=float)
    want = np.asarray(want, dtype=float)
    rel = np.abs(got - want) / np.maximum(np.abs(want), 1e-300)
    i = int(np.argmax(rel))
    assert rel[i] <= RTOL, f"{what}: sample {i}: {got[i]!r} vs {want[i]!r} (rel {rel[i]:.2e})"
    return float(rel.max())


def _draws_match(fam, g, level):
    """The product's host draws of the golden keys are the golden parameters."""
    from paper_2507_19246_b200.mlmc import draw_level
    sel = g["level"] == level
    p = draw_level(fam.uncertain, 0, level, g["k"][sel].tolist())
    np.testing.assert_array_equal(p, g["params"][sel])
    return p


def test_cfg3_finest_level_all_samples(cuda):
    """All 128 finest-level samples of config 3 (128^2 KL field, Parareal M=32,
    K<=6, tol 1e-8 on the jump defect parareal.py:198-207): K equal for every
    sample, Q_l / Q_{l-1} within 1e-8, defect histories within 1e-10."""
    from paper_2507_19246_b200.configs import get_config
    g = golden("cfg3_l2_parareal")
    fam = _family(3)
    p = _draws_match(fam, g, 2)
    b = fam.run_levels([p], get_config(3).parareal_config(), levels=[2])[0]
    fam.check_status()
    k = b.k_used.cpu().numpy()
    bad = np.nonzero(k != g["k_used"])[0]
    assert len(bad) == 0, f"K differs for samples {bad.tolist()}: {k[bad]} vs {g['k_used'][bad]}"
    _check_q(b.q_l.cpu().numpy(), g["q_l"], "cfg3 Q_l (Parareal)")
    _check_q(b.q_lm1.cpu().numpy(), g["q_lm1"], "cfg3 Q_{l-1}")
    d = b.defects.cpu().numpy()
    ref = g["defects"]
    both = np.isfinite(ref)
    assert (np.isfinite(d) == both).all()
    assert np.max(np.abs(d[both] - ref[both])) <= 1e-10


def test_cfg3_level_statistics_subset(cuda):
    """mlmc_estimate on config 3 with N_l = (16, 16, 128): mean_Y, V_l and the
    estimate against the reference-generated per-sample values reduced in
    sample order, absolute tolerance 1e-8 |E|."""
    from oracle import mlmc_oracle as mo
    from paper_2507_19246_b200.configs import get_config
    from paper_2507_19246_b200.mlmc import FixedSamples, mlmc_estimate
    g01 = golden("cfg3_subset_l01")
    g2 = golden("cfg3_l2_parareal")
    fam = _family(3)
    res = mlmc_estimate(fam, policy=FixedSamples((16, 16, 128)),
                        parareal_cfg=get_config(3).parareal_config(), seed=0)
    stats = []
    for lvl in range(3):
        g = g2 if lvl == 2 else g01
        sel = g["level"] == lvl
        stats.append(mo.level_statistics(lvl, g["q_l"][sel], g["q_lm1"][sel]))
    E = sum(st.mean for st in stats)
    for lvl, st in enumerate(stats):
        got = res.per_level[lvl]
        assert got.n == st.n
        assert abs(got.mean_y - st.mean) <= 1e-8 * abs(E), lvl
        assert abs(got.var_y - st.var) <= 1e-8 * abs(E), lvl
    assert abs(res.expectation - E) <= 1e-8 * abs(E)
    assert res.per_level[2].parareal_k == g2["k_used"].tolist()


def test_cfg4_finest_level_parareal_512(cuda):
    """Config 4's finest level at 512^2 (Parareal M=64, 8 fine steps per slice,
    K<=6) on the HBM-streaming tile path, two samples: K, Q_l, Q_{l-1}, defects."""
    from paper_2507_19246_b200.configs import get_config
    g = golden("cfg4_l3_parareal")
    fam = _family(4)
    p = _draws_match(fam, g, 3)
    b = fam.run_levels([p], get_config(4).parareal_config(), levels=[3])[0]
    fam.check_status()
    assert b.k_used.cpu().numpy().tolist() == g["k_used"].tolist()
    _check_q(b.q_l.cpu().numpy(), g["q_l"], "cfg4 Q_l (Parareal)")
    _check_q(b.q_lm1.cpu().numpy(), g["q_lm1"], "cfg4 Q_{l-1}")
    d = b.defects.cpu().numpy()
    ref = g["defects"]
    both = np.isfinite(ref)
    assert (np.isfinite(d) == both).all()
    assert np.max(np.abs(d[both] - ref[both])) <= 1e-10


@pytest.mark.parametrize("level", [1, 2, 3])
def test_cfg2_levels_time_averaged(cuda, level):
    """Config 2's levels 1-3 (dt = T/128 .. T/512 over four periods, QoI the
    time average of W over the last period, right end points): Q_l and Q_{l-1}
    of two samples per level on the tile path with the steady-state predictor
    and the least-squares guesses."""
    g = golden("cfg2_l123")
    fam = _family(2)
    p = _draws_match(fam, g, level)
    sel = g["level"] == level
    b = fam.run_levels([p], levels=[level])[0]
    fam.check_status()
    _check_q(b.q_l.cpu().numpy(), g["q_l"][sel], f"cfg2 level {level} Q_l")
    _check_q(b.q_lm1.cpu().numpy(), g["q_lm1"][sel], f"cfg2 level {level} Q_{{l-1}}")
