"""Diagnostic: first-iteration Parareal fine end states (GPU vs oracle dense LU)
for the golden fe32_cfg1_parareal sample, with and without extrapolation."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from oracle import mlmc_oracle as mo, ie_oracle
from paper_2507_19246_b200 import _lib
from paper_2507_19246_b200.models import eddy_current_family
from paper_2507_19246_b200.engine import new_tasks
T = mo.T
g = np.load("tests/golden/fe32_cfg1_parareal.npz")
p = g["params"][0]
prob = mo.FEProblem(32, "quad4"); model = prob.model(p, dense=True)
# oracle: 16 slices from the coarse-seeded boundaries, dt = T/1024
m = 16; dtf = T / 1024; dtc = T / 16
U = [model.initial_state]
for n in range(1, m):
    U.append(ie_oracle.propagate(model, (n - 1) * T / 16, n * T / 16, dtc, U[-1], time_origin=0.0))
F = [ie_oracle.propagate(model, (n - 1) * T / 16, n * T / 16, dtf, U[n - 1], time_origin=0.0) for n in range(1, m + 1)]
fam = eddy_current_family(1, device="cuda:0")
sol = fam.solver
M, K = sol.assemble(torch.from_numpy(p[None]).cuda())
N = sol.N
for flags, rtol in ((_lib.TASK_NO_EXTRAPOLATION, 1e-12), (0, 1e-12), (0, 1e-13), (0, 1e-14), (_lib.TASK_NO_EXTRAPOLATION, 1e-13)):
    t = new_tasks(m)
    t["sample"] = 0; t["n_steps"] = 64; t["k0"] = np.arange(m) * 64; t["dt"] = dtf; t["t_base"] = 0.0
    t["x_in"] = np.arange(m) * N; t["x_out"] = (m + np.arange(m)) * N; t["slot"] = np.arange(m); t["flags"] = flags
    xb = torch.zeros(2 * m * N, dtype=torch.float64, device="cuda")
    xb[:m * N] = torch.from_numpy(np.concatenate(U)).cuda()
    its = torch.zeros(m, dtype=torch.int32, device="cuda")
    sol.sys.propagate(t, M, K, sol.profile, sol.omega, rtol, 20000, xb, None, its, None)
    out = xb[m * N:].view(m, N).cpu().numpy()
    err = [np.linalg.norm(out[n] - F[n]) / np.linalg.norm(F[n]) for n in range(m)]
    print(f"flags={flags} rtol={rtol:g}: its/slice {its.cpu().numpy().mean():.0f} fine-end rel err max {max(err):.2e} median {np.median(err):.2e}")
