"""CLI on the GPU (SPEC.md cmd_estimate / cmd_sample examples) with the
Steinmetz family: byte-identical estimate.json for a fixed seed, ledger keys,
per-sample CSV consistent with the family API."""

import json

import numpy as np
import pytest

from paper_2507_19246_b200.cli import main

pytestmark = pytest.mark.gpu

CFG = {"model": "steinmetz", "hierarchy": [1e-3, 1e-4, 1e-5], "horizon": 0.04,
       "seed": 0, "estimator": "mlmc", "policy": {"fixed": [6, 4, 2]},
       "parareal": {"enabled": True, "num_subintervals": 8, "tolerance": 1e-8}}


def run(tmp_path, name, cfg, *extra):
    path = tmp_path / f"{name}.json"
    path.write_text(json.dumps(cfg))
    out = tmp_path / name
    return main([extra[0], str(path), "--out", str(out), *extra[1:]]), out


def test_estimate_deterministic_and_ledger(cuda, tmp_path):
    rc1, o1 = run(tmp_path, "a", CFG, "estimate")
    rc2, o2 = run(tmp_path, "b", CFG, "estimate")
    assert rc1 == rc2 == 0
    assert (o1 / "estimate.json").read_bytes() == (o2 / "estimate.json").read_bytes()
    est = json.loads((o1 / "estimate.json").read_text())
    assert est["expectation"] == pytest.approx(sum(lv["mean_y"] for lv in est["levels"]),
                                               rel=1e-15)
    led = json.loads((o1 / "ledger.json").read_text())
    assert {"mode", "levels", "total_wall_s", "total_effort_core_s"} <= set(led)
    assert [lv["level"] for lv in led["levels"]] == [0, 1, 2]
    for lv in led["levels"]:
        assert lv["effort_core_s"] >= lv["wall_s"] > 0
    rows = (o1 / "samples.csv").read_text().splitlines()
    assert rows[0] == "level,index,Q_l,Q_lm1,cost_s,parareal_K"
    assert len(rows) == 1 + 6 + 4 + 2


def test_estimate_with_without_parareal_agree(cuda, tmp_path):
    cfg = dict(CFG)
    cfg["parareal"] = {"enabled": False}
    _, o1 = run(tmp_path, "pr", CFG, "estimate")
    _, o2 = run(tmp_path, "seq", cfg, "estimate")
    e1 = json.loads((o1 / "estimate.json").read_text())
    e2 = json.loads((o2 / "estimate.json").read_text())
    # Parareal at tol 1e-8 vs sequential: within 10*tol relative per sample
    assert e1["expectation"] == pytest.approx(e2["expectation"], rel=1e-6)


def test_sample_command(cuda, tmp_path):
    rc, out = run(tmp_path, "s0", CFG, "sample", "--level", "1", "--count", "0")
    assert rc == 0
    assert (out / "samples_l1.csv").read_text().splitlines() == ["level,index,Q,cost_s,parareal_K"]
    rc, out = run(tmp_path, "s2", CFG, "sample", "--level", "2", "--count", "2", "--parareal")
    rows = [r.split(",") for r in (out / "samples_l2.csv").read_text().splitlines()[1:]]
    assert len(rows) == 2 and all(int(r[4]) >= 1 for r in rows)
    from paper_2507_19246_b200 import machines as mc
    from paper_2507_19246_b200.mlmc import draw_level
    from paper_2507_19246_b200.models import make_hierarchy
    fam = mc.steinmetz_family(make_hierarchy(CFG["hierarchy"]), horizon=0.04)
    P = draw_level(fam.uncertain, 0, 2, range(1, 3))
    q = [r.q for r in fam.evaluate_batch(P, fam.hierarchy[2])]
    np.testing.assert_allclose([float(r[2]) for r in rows], q, rtol=1e-6)
