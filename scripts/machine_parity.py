"""Print the achieved relative errors of the GPU machine families against the
reference golden fixtures (DESIGN.md parity table)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
from conftest import golden
from paper_2507_19246_b200 import machines as mc
from paper_2507_19246_b200.models import make_hierarchy
from paper_2507_19246_b200.parareal import PararealConfig
for tag in ("steinmetz", "synthetic_machine"):
    g = golden(tag)
    h = make_hierarchy(list(g["dts"]))
    fam = (mc.steinmetz_family(h, horizon=float(g["horizon"])) if tag == "steinmetz"
           else mc.synthetic_family(h, horizon=float(g["horizon"])))
    for lvl, spec in enumerate(fam.hierarchy):
        q = np.array([r.q for r in fam.evaluate_batch(g[f"params_l{lvl}"], spec)])
        print(tag, "level", lvl, "max rel err", np.max(np.abs(q / g[f"q_l{lvl}"] - 1)))
    m, dtc, tol, kmax = g["pr_cfg"]
    L = len(h) - 1
    recs = fam.evaluate_batch(g[f"params_l{L}"], h[L], PararealConfig(int(m), h[L].dt, dtc, tol, int(kmax)))
    q = np.array([r.q for r in recs])
    print(tag, "parareal max rel err", np.max(np.abs(q / g["q_pr"] - 1)), "K", [r.parareal_iterations for r in recs], "ref K", list(g["k_pr"]))
