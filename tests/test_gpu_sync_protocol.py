"""The mbarrier exchange / all-reduce protocol of the cluster-resident paths.

compute-sanitizer (racecheck / synccheck) is not available on the GPU pool, so
the synchronisation of the band path (band_path.cu, 256^2 grids, 16-CTA
clusters) and of the cluster path (cluster_path.cu, <= 128^2 grids) is checked
by what a race would break:

* determinism: the same batch twice gives bitwise identical QoIs and PCG
  iteration counts (the all-reduce sums fixed partials in a fixed order, so
  any run-to-run difference would come from a value read before it was
  written or after it was overwritten);
* the barrier-serialised debug mode (MLMCP_BAND_SYNC=1 / MLMCP_CLUSTER_SYNC=1:
  a cluster barrier before and after every exchange and all-reduce, so no CTA
  can run ahead of another) gives the same bits;
* the device-side-checked build (make checked, MLMCP_DCHECK bounds asserts of
  the exchange buffers, class tables and ring offsets) runs the same batches
  in a subprocess without a trap and with the same results.

The reference's contract these protect is bitwise independence of the
evaluation order (parareal.py:125-128)."""

import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _level(cfg_i, lvl, n):
    from paper_2507_19246_b200.configs import get_config
    from paper_2507_19246_b200.mlmc import draw_level
    from paper_2507_19246_b200.models import eddy_current_family
    cfg = get_config(cfg_i)
    fam = eddy_current_family(cfg_i, device="cuda:0")
    d = draw_level(fam.uncertain, cfg.seed, lvl, range(1, n + 1))
    b = fam.run_levels([d], cfg.parareal_config(), levels=[lvl])[0]
    return (b.q_l.cpu().numpy(), b.q_lm1.cpu().numpy(),
            None if b.iters is None else b.iters.cpu().numpy())


def _same(a, b, what):
    for x, y, name in zip(a, b, ("Q_l", "Q_l-1", "iterations")):
        if x is None and y is None:
            continue
        assert np.array_equal(x, y), f"{what}: {name} differ"


@pytest.mark.parametrize("cfg_i,lvl,n,env", [(2, 1, 10, "MLMCP_BAND_SYNC"),
                                             (3, 0, 24, "MLMCP_CLUSTER_SYNC")])
def test_cluster_protocol_deterministic_and_serialisable(cfg_i, lvl, n, env, monkeypatch):
    a = _level(cfg_i, lvl, n)
    b = _level(cfg_i, lvl, n)
    _same(a, b, f"config {cfg_i} run-to-run")
    monkeypatch.setenv(env, "1")
    c = _level(cfg_i, lvl, n)
    _same(a, c, f"config {cfg_i} vs {env}=1")


_CHILD = r"""
import json, sys
sys.path.insert(0, sys.argv[1])
import numpy as np
from paper_2507_19246_b200.configs import get_config
from paper_2507_19246_b200.mlmc import draw_level
from paper_2507_19246_b200.models import eddy_current_family
out = {}
for cfg_i, lvl, n in ((2, 1, 6), (3, 2, 2), (4, 0, 4), (1, 2, 3)):
    cfg = get_config(cfg_i)
    fam = eddy_current_family(cfg_i, device="cuda:0")
    d = draw_level(fam.uncertain, cfg.seed, lvl, range(1, n + 1))
    b = fam.run_levels([d], cfg.parareal_config(), levels=[lvl])[0]
    out[f"{cfg_i}/{lvl}"] = [b.q_l.cpu().tolist(), b.q_lm1.cpu().tolist()]
print("RESULT " + json.dumps(out))
"""


def _child(lib):
    env = dict(os.environ)
    if lib:
        env["MLMCP_LIB"] = lib
    p = subprocess.run([sys.executable, "-c", _CHILD, ROOT], env=env, capture_output=True,
                       text=True, timeout=900)
    assert p.returncode == 0, f"{lib or 'libmlmcp.so'} failed:\n{p.stdout[-2000:]}\n{p.stderr[-2000:]}"
    line = [ln for ln in p.stdout.splitlines() if ln.startswith("RESULT ")][-1]
    import json
    return json.loads(line[len("RESULT "):])


def test_checked_build_runs_clean():
    lib = os.path.join(ROOT, "paper_2507_19246_b200", "libmlmcp_checked.so")
    if not os.path.exists(lib):
        pytest.skip("libmlmcp_checked.so not built (make checked)")
    want = _child(None)
    got = _child(lib)
    for key, (ql, qm) in want.items():
        gl, gm = got[key]
        np.testing.assert_allclose(gl, ql, rtol=1e-12, atol=0, err_msg=key)
        np.testing.assert_allclose(gm, qm, rtol=1e-12, atol=0, err_msg=key)
