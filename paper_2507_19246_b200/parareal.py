"""Drop-in mirror of ``mlmc_parareal.parareal`` (parareal.py:1-220) whose
iteration runs on the GPU.

Same names, fields and errors as the reference:
  ``PropagatorError(interval, iteration)``  parareal.py:37-43
  ``PararealConfig``                        parareal.py:46-79 (validation, k_max,
                                            with_dt_fine)
  ``PararealResult``                        parareal.py:82-90
  ``defect``                                parareal.py:93-103 (host helper; the
                                            solver uses the device kernel K5)
  ``parareal_solve``                        parareal.py:121-220

Semantics kept exactly: iteration k runs the coarse/update sweep on intervals
k..M-1 (k=1 seeds), fine solves on k..M anchored at t0, the *jump* defect
max_n |F_n - U_n| / max(|F_n|, 1e-30) over n=k..M-1 (0 when k == M), stop at
defect <= tolerance, and boundary_states[k_used:] = fine_end[k_used:].
``pool`` is accepted and ignored (all slices of an iteration already run
concurrently on the device).
"""

from __future__ import annotations

from dataclasses import dataclass, replace

import numpy as np

from .timeint import Trajectory, step_count

__all__ = ["PararealConfig", "PararealResult", "PropagatorError", "defect", "parareal_solve"]

_DEFECT_FLOOR = 1e-30


class PropagatorError(RuntimeError):
    def __init__(self, message: str, interval: int, iteration: int):
        super().__init__(f"{message} (interval {interval}, iteration {iteration})")
        self.interval = interval
        self.iteration = iteration


@dataclass(frozen=True)
class PararealConfig:
    num_subintervals: int
    dt_fine: float
    dt_coarse: float
    tolerance: float = 1e-6
    max_iterations: int | None = None

    def __post_init__(self):
        if self.num_subintervals < 1:
            raise ValueError(f"need at least one sub-interval, got {self.num_subintervals}")
        if self.dt_fine <= 0.0 or self.dt_coarse <= 0.0:
            raise ValueError("step sizes must be positive")
        if self.dt_coarse < self.dt_fine:
            raise ValueError(f"dt_coarse ({self.dt_coarse}) must be >= dt_fine ({self.dt_fine})")
        if self.tolerance < 0.0:
            raise ValueError(f"tolerance must be >= 0, got {self.tolerance}")
        if not 1 <= self.k_max <= self.num_subintervals:
            raise ValueError(f"max_iterations must lie in [1, M={self.num_subintervals}], "
                             f"got {self.k_max}")

    @property
    def k_max(self) -> int:
        return self.max_iterations if self.max_iterations is not None else self.num_subintervals

    def with_dt_fine(self, dt: float) -> "PararealConfig":
        return self if dt == self.dt_fine else replace(self, dt_fine=dt)


@dataclass(frozen=True)
class PararealResult:
    boundary_times: np.ndarray
    boundary_states: np.ndarray
    fine_trajectory: Trajectory
    iterations_used: int
    defect_history: list
    fine_solves_per_iter: list
    coarse_solves_per_iter: list


def defect(boundary_states_prev, boundary_states_next) -> float:
    prev = np.atleast_2d(np.asarray(boundary_states_prev, dtype=float))
    nxt = np.atleast_2d(np.asarray(boundary_states_next, dtype=float))
    if prev.shape != nxt.shape:
        raise ValueError(f"boundary lists differ in shape: {prev.shape} vs {nxt.shape}")
    if prev.shape[0] == 0:
        return 0.0
    jumps = np.linalg.norm(nxt - prev, axis=1)
    scales = np.maximum(np.linalg.norm(nxt, axis=1), _DEFECT_FLOOR)
    return float(np.max(jumps / scales))


def raise_parareal_status(coarse_status: np.ndarray, fine_status: np.ndarray):
    """Device status rows -> PropagatorError (parareal.py:151-152,189-192)."""
    from . import _lib
    for row in np.atleast_2d(coarse_status):
        if row[0] != _lib.ST_OK:
            raise PropagatorError(f"coarse propagator failed: "
                                  f"{_lib.STATUS_NAMES.get(int(row[0]))} at step {int(row[1])}",
                                  int(row[2]), int(row[3]))
    for row in np.atleast_2d(fine_status):
        if row[0] != _lib.ST_OK:
            raise PropagatorError(f"fine propagator failed: "
                                  f"{_lib.STATUS_NAMES.get(int(row[0]))} at step {int(row[1])}",
                                  int(row[2]), int(row[3]))


def parareal_solve(model, t0: float, t1: float, x0, cfg: PararealConfig, pool=None, *,
                   rtol: float = 1e-13, max_it: int = 20000, device=None) -> PararealResult:
    """parareal.py:121-220 for one duck-typed model, on the device."""
    import torch

    from .engine import F64, I32
    from .solver import parareal_grid
    from .timeint import _ModelOnDevice

    m = cfg.num_subintervals
    if t1 <= t0:
        raise ValueError(f"need t1 > t0, got [{t0}, {t1}]")
    bounds, fk0, fst, ck0, cst = parareal_grid(t0, t1, m, cfg.dt_fine, cfg.dt_coarse)
    x0 = np.asarray(x0, dtype=float)
    dev = _ModelOnDevice(model, device)
    sysd = dev.sys
    N = dev.n
    S = 1
    k_max = cfg.k_max
    from . import _lib
    from .engine import new_tasks, tasks_to_device
    uf = S * (m + 1) * N
    steps = int(fst.max()) + 1
    buf = torch.zeros(2 * uf + m * steps * N, dtype=F64, device=sysd.device)
    U = buf[:uf].view(S, m + 1, N)
    F = buf[uf:2 * uf].view(S, m + 1, N)
    U[0, 0] = torch.from_numpy(x0).to(sysd.device)
    C = torch.zeros((S, m, N), dtype=F64, device=sysd.device)
    active = torch.ones(S, dtype=I32, device=sysd.device)
    k_used = torch.zeros(S, dtype=I32, device=sysd.device)
    defects = torch.full((S, k_max), float("nan"), dtype=F64, device=sysd.device)
    status = torch.zeros((S, _lib.STATUS_INTS), dtype=I32, device=sysd.device)
    fstatus = torch.zeros((m, _lib.STATUS_INTS), dtype=I32, device=sysd.device)
    fiters = torch.zeros(m, dtype=I32, device=sysd.device)
    citers = torch.zeros(S, dtype=I32, device=sysd.device)
    ck0_d = torch.tensor(ck0, device=sysd.device)
    cst_d = torch.tensor(cst, device=sysd.device)
    n_idx = np.arange(1, m + 1)
    tasks = new_tasks(m)
    tasks["sample"] = 0
    tasks["n_steps"] = fst
    tasks["k0"] = fk0
    tasks["dt"] = cfg.dt_fine
    tasks["t_base"] = t0
    tasks["x_in"] = (n_idx - 1) * N
    tasks["x_out"] = uf + n_idx * N
    tasks["traj"] = 2 * uf + (n_idx - 1) * steps * N
    tasks["group"] = 0
    tasks["slot"] = n_idx - 1
    tasks["flags"] = _lib.TASK_NO_EXTRAPOLATION
    for k in range(1, k_max + 1):
        sysd.parareal_coarse(S, k, m, dev.M, dev.K, dev.profile, dev.omega, cfg.dt_coarse, t0,
                             ck0_d, cst_d, rtol, max_it, U, F, C, citers, status, active)
        sel = tasks[n_idx >= k].copy()
        sel["tag"] = k
        sysd.propagate(sel, dev.M, dev.K, dev.profile, dev.omega, rtol, max_it, buf, None, fiters,
                       fstatus, active, tasks_dev=tasks_to_device(sel, sysd.device))
        sysd.parareal_defect(S, k, m, k_max, U, F, cfg.tolerance, active, k_used, defects)
    sysd.parareal_finalize(S, m, U, F, k_used)
    raise_parareal_status(status.cpu().numpy(), fstatus.cpu().numpy())
    ku = int(k_used.cpu().item())
    hist = [float(d) for d in defects.cpu().numpy()[0, :ku]]
    traj_all = buf[2 * uf:].view(m, steps, N).cpu().numpy()
    parts = [traj_all[0, :fst[0] + 1]] + [traj_all[n, 1:fst[n] + 1] for n in range(1, m)]
    states = np.vstack(parts)
    times = np.concatenate([t0 + (fk0[0] + np.arange(fst[0] + 1)) * cfg.dt_fine] +
                           [t0 + (fk0[n] + np.arange(1, fst[n] + 1)) * cfg.dt_fine for n in range(1, m)])
    return PararealResult(
        boundary_times=bounds,
        boundary_states=U[0].cpu().numpy(),
        fine_trajectory=Trajectory(times=times, states=states, dt=cfg.dt_fine),
        iterations_used=ku,
        defect_history=hist,
        fine_solves_per_iter=[m - k + 1 for k in range(1, ku + 1)],
        coarse_solves_per_iter=[m - k for k in range(1, ku + 1)],
    )
