"""TEST INFRASTRUCTURE ONLY — restatement of the reference implicit-Euler
integrator, /root/reference/pkg/src/mlmc_parareal/timeint.py.

Arithmetic is kept in the reference's order so the dense backend is bitwise
equal to the unmodified reference (checked by ``pin_reference.py`` and
``tests/test_oracle_golden.py``):

    operator     = M + dt*K                       (timeint.py:65)
    rhs_k        = M @ a_k + dt*r(t_{k+1})        (timeint.py:109,127)
    a_{k+1}      = solve(operator, rhs_k)         (timeint.py:110,127)
    grid         = origin + (k0 + arange)*dt      (timeint.py:78-85)

Backends: ``dense`` (scipy lu_factor / lu_solve, as shipped) and ``sparse``
(scipy splu), the latter being the SURVEY.md §8(c) substitution for meshes of
128^2 and up.  ``keep_states=False`` keeps only the running state and hands
each new state to ``observer(k, t_{k+1}, a_{k+1})`` (memory for 512^2 runs).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import scipy.sparse as sp
from scipy.linalg import lu_factor, lu_solve
from scipy.sparse.linalg import splu

GRID_RTOL = 1e-9  # timeint.py:22


class SingularSystemError(RuntimeError):
    """timeint.py:25-30 — factorisation failure, carries a step index."""

    def __init__(self, message: str, step_index: int = 0):
        super().__init__(message)
        self.step_index = step_index


@dataclass(frozen=True)
class OracleTrajectory:
    times: np.ndarray
    states: np.ndarray | None
    dt: float
    terminal: np.ndarray


def step_count(t0: float, t1: float, dt: float) -> int:
    """timeint.py:49-61."""
    if dt <= 0.0:
        raise ValueError(f"dt must be positive, got {dt}")
    raw = (t1 - t0) / dt
    n = int(round(raw))
    if n < 1 or abs(raw - n) > GRID_RTOL * max(1.0, abs(raw)):
        raise ValueError(f"[{t0}, {t1}] is not an integer number of steps of {dt}")
    return n


def time_grid(t0: float, dt: float, n: int, origin: float | None) -> np.ndarray:
    """timeint.py:78-85."""
    if origin is None:
        return t0 + np.arange(n + 1) * dt
    k0 = int(round((t0 - origin) / dt))
    return origin + (k0 + np.arange(n + 1)) * dt


class _DenseSolver:
    def __init__(self, op):
        try:
            self.lu = lu_factor(op)
        except Exception as exc:  # timeint.py:66-69
            raise SingularSystemError(f"factorization failed: {exc}") from exc
        piv = np.abs(np.diag(self.lu[0]))
        if not np.all(np.isfinite(self.lu[0])) or np.any(piv == 0.0):
            raise SingularSystemError("operator is singular", step_index=0)

    def __call__(self, rhs):
        return lu_solve(self.lu, rhs)


class _SparseSolver:
    def __init__(self, op):
        try:
            self.lu = splu(sp.csc_matrix(op))
        except Exception as exc:
            raise SingularSystemError(f"factorization failed: {exc}") from exc

    def __call__(self, rhs):
        return self.lu.solve(rhs)


def factorize(model, dt: float):
    """timeint.py:64-75 with the backend chosen by the matrix storage."""
    op = model.mass + dt * model.stiffness
    if sp.issparse(op):
        return _SparseSolver(op)
    return _DenseSolver(op)


def implicit_euler(model, t0: float, t1: float, dt: float, x0,
                   time_origin: float | None = None, keep_states: bool = True,
                   observer=None) -> OracleTrajectory:
    """timeint.py:88-111 (and propagate, :114-128, via ``.terminal``)."""
    if t1 <= t0:
        raise ValueError(f"need t1 > t0, got [{t0}, {t1}]")
    n = step_count(t0, t1, dt)
    x = np.asarray(x0, dtype=float)
    if x.shape != (model.dim,):
        raise ValueError(f"x0 has shape {x.shape}, expected ({model.dim},)")
    solve = factorize(model, dt)
    times = time_grid(t0, dt, n, time_origin)
    mass, forcing = model.mass, model.forcing
    states = None
    if keep_states:
        states = np.empty((n + 1, model.dim))
        states[0] = x
    for k in range(n):
        x = solve(mass @ x + dt * forcing(times[k + 1]))
        if keep_states:
            states[k + 1] = x
        if observer is not None:
            observer(k, times[k + 1], x)
    return OracleTrajectory(times=times, states=states, dt=dt, terminal=x)


def propagate(model, t_start: float, t_end: float, dt: float, x0,
              time_origin: float | None = None) -> np.ndarray:
    """timeint.py:114-128."""
    x0 = np.asarray(x0, dtype=float)
    if t_end == t_start:
        return x0.copy()
    return implicit_euler(model, t_start, t_end, dt, x0, time_origin,
                          keep_states=False).terminal
