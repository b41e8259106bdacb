"""TEST INFRASTRUCTURE ONLY — restatement of the reference Parareal driver,
/root/reference/pkg/src/mlmc_parareal/parareal.py:93-220.

Kept exactly (arithmetic order included, so the dense backend is bitwise equal
to the reference):
  * iteration k=1 seeds U_n = C(U_{n-1}) for n=1..M-1           (:168-171)
  * k>=2 freezes U_{k-1}=F_{k-1}, then U_n = (F_n + C_new) - C_prev
    for n=k..M-1 and U_M = F_M                                   (:173-178)
  * fine solves on intervals k..M, anchored at time origin t0    (:182-196)
  * stop on the *jump* defect max_n |F_n-U_n| / max(|F_n|,1e-30)
    over n=k..M-1 (0 when k == M)                                (:93-103,198-207)
  * result boundary = U with [k_used:] replaced by F             (:209-210)

``keep_fine`` controls whether per-interval fine trajectories are stored (the
reference always stores them; 512^2 oracle runs only need the terminal state).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .ie_oracle import implicit_euler, propagate, step_count

DEFECT_FLOOR = 1e-30  # parareal.py:34


class PropagatorError(RuntimeError):
    """parareal.py:37-43."""

    def __init__(self, message: str, interval: int, iteration: int):
        super().__init__(f"{message} (interval {interval}, iteration {iteration})")
        self.interval = interval
        self.iteration = iteration


@dataclass(frozen=True)
class OraclePararealConfig:
    num_subintervals: int
    dt_fine: float
    dt_coarse: float
    tolerance: float = 1e-6
    max_iterations: int | None = None

    @property
    def k_max(self) -> int:
        return self.num_subintervals if self.max_iterations is None else self.max_iterations


@dataclass
class OraclePararealResult:
    boundary_times: np.ndarray
    boundary_states: np.ndarray
    iterations_used: int
    defect_history: list = field(default_factory=list)
    fine_counts: list = field(default_factory=list)
    coarse_counts: list = field(default_factory=list)
    fine_trajectories: list | None = None   # per interval 1..M, final solve
    terminal: np.ndarray | None = None


def jump_defect(prev, nxt) -> float:
    """parareal.py:93-103."""
    prev = np.atleast_2d(np.asarray(prev, dtype=float))
    nxt = np.atleast_2d(np.asarray(nxt, dtype=float))
    if prev.shape != nxt.shape:
        raise ValueError(f"shape mismatch {prev.shape} vs {nxt.shape}")
    if prev.shape[0] == 0:
        return 0.0
    num = np.linalg.norm(nxt - prev, axis=1)
    den = np.maximum(np.linalg.norm(nxt, axis=1), DEFECT_FLOOR)
    return float(np.max(num / den))


def parareal(model, t0: float, t1: float, x0, cfg: OraclePararealConfig,
             keep_fine: bool = True) -> OraclePararealResult:
    m = cfg.num_subintervals
    if t1 <= t0:
        raise ValueError(f"need t1 > t0, got [{t0}, {t1}]")
    nf = step_count(t0, t1, cfg.dt_fine)
    nc = step_count(t0, t1, cfg.dt_coarse)
    if nf % m or nc % m:
        raise ValueError("sub-interval grid incompatible with dt_fine / dt_coarse")
    per = nf // m
    x0 = np.asarray(x0, dtype=float)
    edges = t0 + (np.arange(m + 1) * per) * cfg.dt_fine

    def coarse(n, value, it):
        try:
            return propagate(model, edges[n - 1], edges[n], cfg.dt_coarse, value,
                             time_origin=t0)
        except Exception as exc:
            raise PropagatorError(f"coarse propagator failed: {exc}", n, it) from exc

    dim = model.dim
    U = np.empty((m + 1, dim))
    U[0] = x0
    C = np.empty((m, dim))            # C[n-1] belongs to boundary n
    F = np.empty((m + 1, dim))
    fine = [None] * (m + 1)
    res = OraclePararealResult(boundary_times=edges, boundary_states=U,
                               iterations_used=cfg.k_max)
    k_used = cfg.k_max
    for k in range(1, cfg.k_max + 1):
        if k == 1:
            for n in range(1, m):
                U[n] = coarse(n, U[n - 1], k)
                C[n - 1] = U[n]
        else:
            U[k - 1] = F[k - 1]
            for n in range(k, m):
                c_new = coarse(n, U[n - 1], k)
                U[n] = F[n] + c_new - C[n - 1]
                C[n - 1] = c_new
            U[m] = F[m]
        res.coarse_counts.append(m - k)
        for n in range(k, m + 1):
            try:
                tr = implicit_euler(model, edges[n - 1], edges[n], cfg.dt_fine,
                                    U[n - 1], time_origin=t0, keep_states=keep_fine)
            except Exception as exc:
                raise PropagatorError(f"fine propagator failed: {exc}", k, k) from exc
            fine[n] = tr
            F[n] = tr.terminal
        res.fine_counts.append(m - k + 1)
        d = jump_defect(U[k:m], F[k:m]) if k < m else 0.0
        res.defect_history.append(d)
        k_used = k
        if d <= cfg.tolerance:
            break
    out = U.copy()
    out[k_used:] = F[k_used:]
    res.boundary_states = out
    res.iterations_used = k_used
    res.terminal = F[m].copy()
    res.fine_trajectories = fine[1:] if keep_fine else None
    return res


def concatenate_states(fine_trajectories) -> np.ndarray:
    """parareal.py:111-118 — states of the concatenated fine trajectory."""
    parts = [fine_trajectories[0].states]
    for tr in fine_trajectories[1:]:
        parts.append(tr.states[1:])
    return np.vstack(parts)
