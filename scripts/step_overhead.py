"""Per-step overhead vs per-iteration cost of the SM-resident kernel:
S tasks x 1024 steps (config-1 mesh, T/1024) at rtol = 1 (no PCG iteration:
the step's fixed work only) and at the production tolerance, with and
without the steady-state predictor.  Cycles per step per task and per PCG
iteration are derived from the launch time."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2507_19246_b200 import _lib
from paper_2507_19246_b200.configs import get_config
from paper_2507_19246_b200.engine import F64, I32, new_tasks, tasks_to_device
from paper_2507_19246_b200.mlmc import draw_level
from paper_2507_19246_b200.models import eddy_current_family

cfg = get_config(1)
fam = eddy_current_family(1, device="cuda:0"); sol = fam.solver
clock = 1.965e9
for S in (148, 296):
    P = draw_level(fam.uncertain, 0, 0, range(1, S + 1))
    M, K = sol.assemble(torch.from_numpy(P).cuda())
    dt = cfg.horizon / 1024
    N = sol.N
    for pred in (False, True):
        tasks = new_tasks(S)
        tasks["sample"] = np.arange(S); tasks["n_steps"] = 1024; tasks["dt"] = dt
        tasks["x_in"] = np.arange(S) * N; tasks["x_out"] = np.arange(S) * N; tasks["slot"] = np.arange(S)
        xss = None
        if pred:
            tasks["ss_slot"] = np.arange(S)
            xss = sol.steady_states(np.arange(S), np.full(S, dt), M, K)
        td = tasks_to_device(tasks, sol.device)
        for rtol in (1.0, 1e-14):
            its = torch.zeros(S, dtype=I32, device=sol.device)
            st = torch.zeros((S, 4), dtype=I32, device=sol.device)
            ms = []
            for rep in range(3):
                x = torch.zeros(S * N, dtype=F64, device=sol.device)
                a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
                a.record()
                sol.sys.propagate(tasks, M, K, sol.profile, sol.omega, rtol, 20000, x, None, its, st,
                                  None, tasks_dev=td, xss=xss)
                b.record(); torch.cuda.synchronize(); ms.append(a.elapsed_time(b))
            t = min(ms) * 1e-3
            it = int(its.sum())
            per_step = t * clock / 1024 / (1 if S <= 148 else 2) * (1 if S <= 148 else 1)
            print(f"S={S} pred={pred} rtol={rtol:g}: {min(ms):.3f} ms, {it / S / 1024:.2f} its/step, "
                  f"{t * clock / 1024:.0f} cycles/step (wall per task-step, {S // 148} CTA/SM)")
