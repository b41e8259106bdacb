"""Sample draws: the native restatement of numpy's SeedSequence -> PCG64 ->
Generator.uniform (libmlmcp mlmcp_draw_uniform_host, used by
mlmc.draw_level) is bitwise equal to RandomStream(seed, l, k).generator()
.uniform(lo, hi) (models.py:305-318) over a spread of keys,
including multi-word seeds and keys; the golden draws of the reference pin
the whole chain."""

import numpy as np
import pytest

from conftest import golden
from paper_2507_19246_b200.mlmc import RandomStream, _draw_uniform_host, draw_level
from paper_2507_19246_b200.models import ParameterVector, UncertainInput


@pytest.mark.parametrize("seed", [0, 1, 7, 2 ** 32 - 1, 2 ** 32 + 5, 2 ** 63 + 11])
@pytest.mark.parametrize("level", [0, 1, 3, 2 ** 32 + 1])
def test_native_uniform_matches_numpy(seed, level):
    nominal = np.array([795.77, 795.77, 1e6, 2.5e-3, 1.0, 3.0, 17.0, 1e-6])
    lo, hi = nominal * 0.9, nominal * 1.1
    k_first, n = 2 ** 31 - 3, 6           # crosses 2^31 and 2^32 word boundaries later
    for kf in (1, k_first, 2 ** 32 - 2):
        out = np.empty((n, len(nominal)))
        _draw_uniform_host(seed, level, kf, lo, hi - lo, out)
        ref = np.array([RandomStream(seed, level, k).generator().uniform(lo, hi)
                        for k in range(kf, kf + n)])
        np.testing.assert_array_equal(out, ref)


def test_draw_level_matches_reference_golden():
    g = golden("draws")
    inp = UncertainInput(ParameterVector("fe", g["nominal"]), 0.1)
    for key, row in zip(g["keys"], g["uniform"]):
        seed, lvl, k = (int(v) for v in key)
        np.testing.assert_array_equal(draw_level(inp, seed, lvl, [k])[0], row)
    # contiguous block (native path) == per-key rows
    blk = draw_level(inp, 0, 1, range(1, 4))
    rows = [draw_level(inp, 0, 1, [k])[0] for k in (1, 2, 3)]
    np.testing.assert_array_equal(blk, np.array(rows))
    np.testing.assert_array_equal(blk[0], g["uniform"][list(map(tuple, g["keys"])).index((0, 1, 1))])


def test_draw_level_zero_halfwidth_and_empty():
    inp = UncertainInput(ParameterVector("fe", np.array([1.0, 2.0])), 0.0)
    np.testing.assert_array_equal(draw_level(inp, 0, 0, range(1, 4)), np.array([[1.0, 2.0]] * 3))
    assert draw_level(UncertainInput(ParameterVector("fe", np.array([1.0])), 0.1), 0, 0,
                      []).shape == (0, 1)
