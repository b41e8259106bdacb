"""Defect-history parity of the config-1 Parareal golden case (diagnostic)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np, torch
from conftest import golden
from test_gpu_fe_parity import family
for name in ("fe32_cfg1_parareal", "fe16_kl64_parareal", "fe8_quad4_parareal"):
    g = golden(name)
    n, dt, horizon = int(g["n"]), float(g["dt"]), float(g["horizon"])
    m, dtc, tol, kmax = g["parareal"]
    fam = family(n, str(g["layout"]), [dt], horizon)
    sol = fam.solver
    M, K = sol.assemble(torch.from_numpy(g["params"]).to(sol.device))
    pr = sol.run_parareal(M, K, 0.0, horizon, int(m), dt, float(dtc), float(tol), int(kmax))
    d = pr.defects.cpu().numpy(); ku = pr.k_used.cpu().numpy()
    U = pr.U.cpu().numpy()
    print(name, "K", ku.tolist(), "ref", g["k_used"].tolist(), "pred", sol.use_predictor(), "rtol", sol.step_rtol())
    for i, k in enumerate(g["k_used"]):
        print("   defect abs diff", np.abs(d[i, :k] - g["defects"][i, :k]).tolist())
    print("   max boundary err / scale", np.max(np.abs(U - g["boundary"])) / np.max(np.abs(g["boundary"])),
          " q rel err", np.max(np.abs(pr.qoi.cpu().numpy() / g["q"] - 1)))
