"""CLI (SPEC.md [MODULE] cli): plan output, configuration errors (exit 2);
the GPU half (estimate / sample on the Steinmetz family) is in
test_gpu_cli.py."""

import json
import math

import pytest

from paper_2507_19246_b200 import costmodel
from paper_2507_19246_b200.cli import main


def test_plan_writes_consistent_figures(tmp_path):
    assert main(["plan", "--out", str(tmp_path)]) == 0
    lines = (tmp_path / "figure1.csv").read_text().splitlines()
    assert "5.2857142857" in lines[0]                 # s_inf note, SPEC.md cmd_plan example
    assert lines[1] == "n_c,K,speedup,effort_ratio"
    p = costmodel.CostModelParams()
    for row in lines[2:]:
        n_c, K, s, e = row.split(",")
        if s != "nan":
            q = costmodel.CostModelParams(n_c=int(n_c))
            assert float(s) == costmodel.finite_speedup(q, int(K))
            assert float(e) == costmodel.effort_ratio_infinite(q, int(K))
    assert (tmp_path / "figure2.csv").exists()
    del p


def test_plan_guard_rows(tmp_path):
    # n_c below N_L (1 + 1/r): no core per level-L sample -> NaN rows, still exit 0
    assert main(["plan", "--nc", "5", "--K", "1", "--out", str(tmp_path)]) == 0
    row = (tmp_path / "figure1.csv").read_text().splitlines()[2].split(",")
    assert math.isnan(float(row[2]))


@pytest.mark.parametrize("cfg", [
    {"model": "nope"},
    {"model": "steinmetz"},                                        # no hierarchy
    {"model": "steinmetz", "hierarchy": [1e-3, 1e-4], "policy": {"fixed": [2]}},
    {"model": "steinmetz", "hierarchy": [1e-4, 1e-3], "policy": {"fixed": [2, 2]}},
    {"model": "steinmetz", "hierarchy": [1e-3, 1e-4], "policy": {"fixed": [2, 2]},
     "parareal": {"num_subintervals": 4}},                         # L-2 rule needs 3 levels
])
def test_invalid_configs_exit_2(tmp_path, cfg):
    path = tmp_path / "c.json"
    path.write_text(json.dumps(cfg))
    assert main(["estimate", str(path), "--out", str(tmp_path / "o")]) == 2


def test_unknown_baseline_config_exit_2(tmp_path):
    assert main(["estimate", "cfg9", "--out", str(tmp_path)]) == 2
