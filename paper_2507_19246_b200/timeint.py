"""Drop-in mirror of ``mlmc_parareal.timeint`` (timeint.py:1-128) running on
the GPU.

Same names, argument meaning and errors as the reference:
  ``Trajectory``              timeint.py:33-46
  ``SingularSystemError``     timeint.py:25-30 (carries ``step_index``)
  ``step_count``              timeint.py:49-61 (ValueError on non-integer grids)
  ``implicit_euler_solve``    timeint.py:88-111
  ``propagate``               timeint.py:114-128

Difference by design: for systems with more than MLMCP_DIRECT_MAX_ROWS (4)
states each step's linear solve is Jacobi-PCG on the device (tolerance
``rtol``, default 1e-13 — the stated PCG tolerance; M and K must be
symmetric) instead of a dense LU factorisation; smaller systems (the
Steinmetz circuit, scalar tests) use the device's direct LU path, the
reference's own algorithm.  The model is duck-typed like the reference
(``mass``, ``stiffness`` as dense or scipy-sparse operators with <= 8
entries per row of their union pattern; ``forcing`` of the form
sin(2*pi*f*t) * profile, i.e. an object with ``frequency`` and ``profile``
like models.py:171-179, a scaled drive ``drive(t) * direction`` like
models.py:160-168, or ``None`` for r = 0).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

__all__ = ["Trajectory", "SingularSystemError", "step_count", "implicit_euler_solve",
           "propagate"]

_GRID_RTOL = 1e-9


class SingularSystemError(RuntimeError):
    """The per-step solve failed (PCG breakdown / non-convergence)."""

    def __init__(self, message: str, step_index: int = 0):
        super().__init__(message)
        self.step_index = step_index


@dataclass(frozen=True)
class Trajectory:
    times: np.ndarray
    states: np.ndarray
    dt: float

    @property
    def n_steps(self) -> int:
        return len(self.times) - 1

    def terminal_state(self) -> np.ndarray:
        return self.states[-1]


def step_count(t0: float, t1: float, dt: float) -> int:
    if dt <= 0.0:
        raise ValueError(f"dt must be positive, got {dt}")
    raw = (t1 - t0) / dt
    n = int(round(raw))
    if n < 1 or abs(raw - n) > _GRID_RTOL * max(1.0, abs(raw)):
        raise ValueError(f"interval [{t0}, {t1}] is not an integer number of steps of dt={dt} "
                         f"(got {raw})")
    return n


def _grid_origin(t0: float, dt: float, time_origin: float | None):
    """(t_base, k0) such that t_g = t_base + (k0 + g)*dt reproduces
    timeint.py:78-85 bitwise."""
    if time_origin is None:
        return float(t0), 0
    return float(time_origin), int(round((t0 - time_origin) / dt))


def _csr(a):
    import scipy.sparse as sp
    m = sp.csr_matrix(a, dtype=np.float64)
    m.sum_duplicates()
    m.sort_indices()
    return m


def operator_pattern(mass, stiffness):
    """Union CSR pattern (sorted, diagonal included) and the aligned values."""
    import scipy.sparse as sp
    Mc, Kc = _csr(mass), _csr(stiffness)
    if Mc.shape != Kc.shape or Mc.shape[0] != Mc.shape[1]:
        raise ValueError(f"inconsistent dimensions: mass {Mc.shape}, stiffness {Kc.shape}")
    n = Mc.shape[0]
    pat = (abs(Mc) + abs(Kc) + sp.identity(n, format="csr")).tocsr()
    pat.sort_indices()
    row_ptr = pat.indptr.astype(np.int32)
    col = pat.indices.astype(np.int32)

    def values(m):
        out = np.zeros(len(col))
        for i in range(n):
            a, b = row_ptr[i], row_ptr[i + 1]
            pos = {int(c): q for q, c in enumerate(col[a:b], start=a)}
            for q in range(m.indptr[i], m.indptr[i + 1]):
                out[pos[int(m.indices[q])]] = m.data[q]
        return out

    return row_ptr, col, values(Mc), values(Kc)


def _symmetric(a) -> bool:
    m = _csr(a)
    d = m - m.T
    return d.nnz == 0 or float(abs(d).max()) <= 1e-14 * max(float(abs(m).max()), 1e-300)


def forcing_profile(model, n: int):
    f = getattr(model, "forcing", None)
    if f is None:
        return 0.0, np.zeros(n)
    drive = getattr(f, "drive", None)
    if drive is not None and hasattr(f, "direction") and hasattr(drive, "amplitude"):
        # u(t) * direction with u = amplitude sin(2 pi f t) (models.py:160-168)
        prof = float(drive.amplitude) * np.asarray(f.direction, dtype=float)
        if prof.shape != (n,):
            raise ValueError(f"forcing direction has shape {prof.shape}, expected ({n},)")
        return float(drive.frequency), prof
    if hasattr(f, "frequency") and hasattr(f, "profile"):
        prof = np.asarray(f.profile, dtype=float)
        if prof.shape != (n,):
            raise ValueError(f"forcing profile has shape {prof.shape}, expected ({n},)")
        return float(f.frequency), prof
    probe = [np.asarray(f(t), dtype=float) for t in (0.0, 0.37, 1.3)]
    if all(np.all(p == 0.0) for p in probe):
        return 0.0, np.zeros(n)
    raise ValueError("GPU propagator supports forcings r(t) = sin(2*pi*f*t)*profile "
                     "(objects with .frequency and .profile) or r = 0")


class _ModelOnDevice:
    """Uploads one duck-typed model (pattern, M/K values, forcing profile)."""

    _cache: dict = {}

    def __init__(self, model, device=None):
        import torch

        from .engine import DeviceSystem, F64
        row_ptr, col, mv, kv = operator_pattern(model.mass, model.stiffness)
        from . import _lib
        if len(row_ptr) - 1 > _lib.DIRECT_MAX_ROWS and not (_symmetric(model.mass) and
                                                            _symmetric(model.stiffness)):
            raise ValueError("systems with more than "
                             f"{_lib.DIRECT_MAX_ROWS} states need symmetric M and K "
                             "(Jacobi-PCG path); smaller ones use the direct LU path")
        key = (row_ptr.tobytes(), col.tobytes(), str(device))
        sys = _ModelOnDevice._cache.get(key)
        if sys is None:
            sys = DeviceSystem(row_ptr, col, device)
            _ModelOnDevice._cache[key] = sys
        self.sys = sys
        self.n = len(row_ptr) - 1
        self.M = torch.tensor(mv, dtype=F64, device=sys.device)[None, :].contiguous()
        self.K = torch.tensor(kv, dtype=F64, device=sys.device)[None, :].contiguous()
        freq, prof = forcing_profile(model, self.n)
        self.omega = 2.0 * np.pi * freq
        self.profile = torch.tensor(prof, dtype=F64, device=sys.device)

    def run(self, x0: np.ndarray, dt: float, n_steps: int, t_base: float, k0: int,
            keep_traj: bool, rtol: float, max_it: int):
        import torch

        from . import _lib
        from .engine import F64, I32, new_tasks
        N = self.n
        tasks = new_tasks(1)
        tasks["sample"] = 0
        tasks["n_steps"] = n_steps
        tasks["k0"] = k0
        tasks["dt"] = dt
        tasks["t_base"] = t_base
        tasks["x_in"] = 0
        tasks["x_out"] = N
        tasks["slot"] = 0
        tasks["flags"] = _lib.TASK_NO_EXTRAPOLATION   # one-step method, as the reference
        if keep_traj:
            tasks["traj"] = 2 * N
        size = 2 * N + ((n_steps + 1) * N if keep_traj else 0)
        xbuf = torch.zeros(size, dtype=F64, device=self.sys.device)
        xbuf[:N] = torch.from_numpy(np.ascontiguousarray(x0, dtype=np.float64)).to(self.sys.device)
        iters = torch.zeros(1, dtype=I32, device=self.sys.device)
        status = torch.zeros((1, _lib.STATUS_INTS), dtype=I32, device=self.sys.device)
        self.sys.propagate(tasks, self.M, self.K, self.profile, self.omega, rtol, max_it, xbuf,
                           None, iters, status)
        st = status.cpu().numpy()[0]
        if st[0] != _lib.ST_OK:
            raise SingularSystemError(
                f"(M + dt K) solve failed for dt={dt}: {_lib.STATUS_NAMES.get(int(st[0]))}",
                step_index=int(st[1]))
        host = xbuf.cpu().numpy()
        term = host[N:2 * N].copy()
        states = host[2 * N:].reshape(n_steps + 1, N) if keep_traj else None
        return term, states


def implicit_euler_solve(model, t0: float, t1: float, dt: float, x0,
                         time_origin: float | None = None, *, rtol: float = 1e-13,
                         max_it: int = 20000, device=None) -> Trajectory:
    """timeint.py:88-111 on the GPU; returns the full trajectory."""
    if t1 <= t0:
        raise ValueError(f"need t1 > t0, got [{t0}, {t1}]")
    n = step_count(t0, t1, dt)
    x0 = np.asarray(x0, dtype=float)
    if x0.shape != (model.dim,):
        raise ValueError(f"x0 has shape {x0.shape}, expected ({model.dim},)")
    dev = _ModelOnDevice(model, device)
    t_base, k0 = _grid_origin(t0, dt, time_origin)
    if time_origin is None:
        times = t0 + np.arange(n + 1) * dt
    else:
        times = time_origin + (k0 + np.arange(n + 1)) * dt
    _, states = dev.run(x0, dt, n, t_base, k0, True, rtol, max_it)
    return Trajectory(times=times, states=states, dt=dt)


def propagate(model, t_start: float, t_end: float, dt: float, x0,
              time_origin: float | None = None, *, rtol: float = 1e-13, max_it: int = 20000,
              device=None) -> np.ndarray:
    """timeint.py:114-128 on the GPU; x0 itself for an empty span."""
    x0 = np.asarray(x0, dtype=float)
    if t_end == t_start:
        return x0.copy()
    n = step_count(t_start, t_end, dt)
    dev = _ModelOnDevice(model, device)
    t_base, k0 = _grid_origin(t_start, dt, time_origin)
    term, _ = dev.run(x0, dt, n, t_base, k0, False, rtol, max_it)
    return term
