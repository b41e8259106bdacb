"""One launch of 148 tasks x 1024 steps at rtol = 1 (per-step fixed work
only), for an ncu source-level capture of the per-step overhead."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2507_19246_b200.configs import get_config
from paper_2507_19246_b200.engine import F64, I32, new_tasks, tasks_to_device
from paper_2507_19246_b200.mlmc import draw_level
from paper_2507_19246_b200.models import eddy_current_family
rtol = float(sys.argv[1]) if len(sys.argv) > 1 else 1.0
cfg = get_config(1)
fam = eddy_current_family(1, device="cuda:0"); sol = fam.solver
S = 148
P = draw_level(fam.uncertain, 0, 0, range(1, S + 1))
M, K = sol.assemble(torch.from_numpy(P).cuda())
dt = cfg.horizon / 1024; N = sol.N
tasks = new_tasks(S)
tasks["sample"] = np.arange(S); tasks["n_steps"] = 1024; tasks["dt"] = dt
tasks["x_in"] = np.arange(S) * N; tasks["x_out"] = np.arange(S) * N; tasks["slot"] = np.arange(S)
tasks["ss_slot"] = np.arange(S)
xss = sol.steady_states(np.arange(S), np.full(S, dt), M, K)
td = tasks_to_device(tasks, sol.device)
for rep in range(2):
    x = torch.zeros(S * N, dtype=F64, device=sol.device)
    sol.sys.propagate(tasks, M, K, sol.profile, sol.omega, rtol, 20000, x, None, None, None,
                      None, tasks_dev=td, xss=xss)
torch.cuda.synchronize()
print("done")
