"""The reference's own machine models on the GPU:
the Steinmetz equivalent circuit (3 states, non-symmetric) and the synthetic
conductor-bar machine (n_dof states, SPD), as batched families behind the
same family protocol as ``MachineFamily`` (models.py:376-411).

Drop-in names (same fields, defaults, validation and errors):
  ``STEINMETZ_PARAM_NAMES`` / ``STEINMETZ_NOMINAL``   models.py:34-45
  ``NUM_BARS`` / ``SIGMA_NOMINAL``                    models.py:47-48
  ``SinusoidalDrive`` / ``DriveSettings``             models.py:116-144
  ``QoIDefinition`` / ``LinearSystemModel``           models.py:147-214
  ``build_steinmetz``                                 models.py:217-249
  ``build_synthetic_machine``                         models.py:262-302
  ``evaluate_qoi``                                    models.py:321-344
  ``steinmetz_family`` / ``synthetic_family``         models.py:431-453

Device mapping:
  * Steinmetz: n = 3 <= MLMCP_DIRECT_MAX_ROWS, so every solve runs on the
    direct path (dense LU with partial pivoting per task, one thread per
    task, like the reference's lu_factor/lu_solve, timeint.py:64-75).  The
    forcing u(t)/L_s1 e_1 (models.py:245-248) differs per sample while the
    ABI has one shared profile, so the first equation is scaled by L_s1:
    M' = diag(L_s1, 1, 1), K' row 0 = L_s1 K row 0 = (R1 + R_fe, -R_fe,
    -R_fe/L_h), profile = amplitude e_1 — the same implicit-Euler iterate in
    exact arithmetic (row scaling of the step system), one rounding apart.
    QoI ELECTRICAL_ENERGY = amplitude * dt * sum_g sin(w t_g) i1(t_g)
    (models.py:337-339) accumulated on the device (MLMCP_QOI_ELECTRICAL).
  * Synthetic machine: tridiagonal SPD M + dt K (block-tridiagonal mass,
    models.py:252-259, 285-289): SM-resident Jacobi-PCG.  QoI
    MEAN_JOULE_LOSS = sum_k d_k^T M d_k dt / T with d_k = (a_{k+1}-a_k)/dt
    (models.py:340-343) = sum_k (da)^T M (da) / (dt T), the sum accumulated
    on the device (MLMCP_QOI_JOULE).
Host code here only builds per-sample operator values (a few floats per
sample) and scales QoIs; every time step runs in libmlmcp.so.
"""

from __future__ import annotations

import enum
from dataclasses import dataclass, field
from typing import Callable

import numpy as np

from . import _lib
from .models import (EvalRecord, ParameterVector, QoIKind, UncertainInput, _BatchedFamily,
                     make_hierarchy)

__all__ = ["STEINMETZ_PARAM_NAMES", "STEINMETZ_NOMINAL", "NUM_BARS", "SIGMA_NOMINAL",
           "SinusoidalDrive", "DriveSettings", "QoIDefinition", "LinearSystemModel",
           "build_steinmetz", "build_synthetic_machine", "evaluate_qoi", "MachineFamily",
           "steinmetz_family", "synthetic_family", "make_hierarchy", "EvalRecord"]

STEINMETZ_PARAM_NAMES = ("R1", "R2", "R_fe", "L_s1", "L_s2", "L_h")
STEINMETZ_NOMINAL = (1.111140e-01, 7.158602e-02, 1.736354e+06, 1.649983e-03, 1.063014e-03,
                     6.407774e-02)
NUM_BARS = 32
SIGMA_NOMINAL = 26.7e6
_COND_LIMIT = 1e12


@dataclass(frozen=True)
class SinusoidalDrive:
    """u(t) = amplitude * sin(2 pi frequency t)."""

    amplitude: float
    frequency: float

    def __call__(self, t):
        return self.amplitude * np.sin(2.0 * np.pi * self.frequency * t)


@dataclass(frozen=True)
class DriveSettings:
    amplitude: float = 230.0 * np.sqrt(2.0)
    frequency: float = 50.0
    slip: float = 0.05

    def __post_init__(self):
        if self.amplitude < 0.0:
            raise ValueError(f"drive amplitude must be >= 0, got {self.amplitude}")
        if self.frequency <= 0.0:
            raise ValueError(f"drive frequency must be > 0, got {self.frequency}")
        if not 0.0 < self.slip <= 1.0:
            raise ValueError(f"slip must lie in (0, 1], got {self.slip}")

    def voltage(self) -> SinusoidalDrive:
        return SinusoidalDrive(self.amplitude, self.frequency)


@dataclass(frozen=True)
class QoIDefinition:
    kind: QoIKind
    horizon: float
    drive: SinusoidalDrive | None = None
    current_index: int | None = None
    mass: np.ndarray | None = None

    def __post_init__(self):
        if self.horizon <= 0.0:
            raise ValueError(f"QoI horizon must be positive, got {self.horizon}")


@dataclass(frozen=True)
class _ScaledDriveForcing:
    """r(t) = u(t) * direction (timeint mirror: profile = amplitude * direction)."""

    drive: SinusoidalDrive
    direction: np.ndarray

    def __call__(self, t):
        return self.drive(t) * self.direction


@dataclass(frozen=True)
class _ProfileForcing:
    frequency: float
    profile: np.ndarray

    def __call__(self, t):
        return np.sin(2.0 * np.pi * self.frequency * t) * self.profile


@dataclass(frozen=True)
class LinearSystemModel:
    """(M, K, r) with initial state and QoI; dense host arrays, validated like
    models.py:182-214 (consumed by the GPU timeint / parareal mirrors)."""

    mass: np.ndarray
    stiffness: np.ndarray
    forcing: Callable
    initial_state: np.ndarray
    qoi: QoIDefinition

    def __post_init__(self):
        mass = np.asarray(self.mass, dtype=float)
        stiff = np.asarray(self.stiffness, dtype=float)
        x0 = np.asarray(self.initial_state, dtype=float)
        object.__setattr__(self, "mass", mass)
        object.__setattr__(self, "stiffness", stiff)
        object.__setattr__(self, "initial_state", x0)
        n = mass.shape[0]
        if mass.shape != (n, n) or stiff.shape != (n, n) or x0.shape != (n,):
            raise ValueError(f"inconsistent dimensions: mass {mass.shape}, stiffness "
                             f"{stiff.shape}, initial state {x0.shape}")
        r0 = np.asarray(self.forcing(0.0), dtype=float)
        if r0.shape != (n,):
            raise ValueError(f"forcing returns shape {r0.shape}, expected ({n},)")
        cond = np.linalg.cond(mass)
        if not np.isfinite(cond) or cond > _COND_LIMIT:
            raise ValueError(f"mass matrix is not safely invertible (cond={cond:.3e})")

    @property
    def dim(self) -> int:
        return self.mass.shape[0]


def _check_model_id(params: ParameterVector, want: str):
    if params.model_id != want:
        raise ValueError(f"expected {want} parameters, got '{params.model_id}'")


def _steinmetz_stiffness(v: np.ndarray, slip: float) -> np.ndarray:
    """K of x = (i1, i2, lam_h) for parameter rows v [..., 6] (models.py:231-238)."""
    r1, r2, r_fe, l_s1, l_s2, l_h = (v[..., i] for i in range(6))
    r2s = r2 / slip
    K = np.empty(v.shape[:-1] + (3, 3))
    K[..., 0, 0] = (r1 + r_fe) / l_s1
    K[..., 0, 1] = -r_fe / l_s1
    K[..., 0, 2] = -r_fe / (l_s1 * l_h)
    K[..., 1, 0] = -r_fe / l_s2
    K[..., 1, 1] = (r_fe + r2s) / l_s2
    K[..., 1, 2] = r_fe / (l_s2 * l_h)
    K[..., 2, 0] = -r_fe
    K[..., 2, 1] = r_fe
    K[..., 2, 2] = r_fe / l_h
    return K


def build_steinmetz(params: ParameterVector, drive: DriveSettings,
                    horizon: float = 1.0) -> LinearSystemModel:
    _check_model_id(params, "steinmetz")
    v = params.values
    voltage = drive.voltage()
    qoi = QoIDefinition(kind=QoIKind.ELECTRICAL_ENERGY, horizon=horizon, drive=voltage,
                        current_index=0)
    return LinearSystemModel(mass=np.eye(3), stiffness=_steinmetz_stiffness(v, drive.slip),
                             forcing=_ScaledDriveForcing(voltage, np.array([1.0 / v[3], 0.0, 0.0])),
                             initial_state=np.zeros(3), qoi=qoi)


def _bar_mass_diag(n_dof: int, scales: np.ndarray):
    """Diagonal and super-diagonal of the block-diagonal bar mass for parameter
    rows ``scales`` [..., NUM_BARS] (models.py:252-259, 285-289)."""
    bs = n_dof // NUM_BARS
    h = 1.0 / n_dof
    s = SIGMA_NOMINAL * np.asarray(scales, dtype=float)          # [..., NUM_BARS]
    per_dof = np.repeat(s, bs, axis=-1)                             # [..., n_dof]
    diag = per_dof * (h * (2.0 / 3.0))
    off = per_dof[..., :-1] * (h * (1.0 / 6.0))
    same_bar = (np.arange(n_dof - 1) // bs) == (np.arange(1, n_dof) // bs)
    off = np.where(same_bar, off, 0.0)
    return diag, off


def _synthetic_check(n_dof: int):
    if n_dof < 2 * NUM_BARS or n_dof % NUM_BARS != 0:
        raise ValueError(f"n_dof must be >= {2 * NUM_BARS} and divisible by {NUM_BARS}, "
                         f"got {n_dof}")


def build_synthetic_machine(n_dof: int, bar_scales: ParameterVector, horizon: float = 0.16,
                            frequency: float = 50.0) -> LinearSystemModel:
    _synthetic_check(n_dof)
    _check_model_id(bar_scales, "synthetic")
    h = 1.0 / n_dof
    diag, off = _bar_mass_diag(n_dof, bar_scales.values)
    mass = np.diag(diag) + np.diag(off, 1) + np.diag(off, -1)
    stiffness = np.zeros((n_dof, n_dof))
    np.fill_diagonal(stiffness, 2.0 / h ** 2)
    idx = np.arange(n_dof - 1)
    stiffness[idx, idx + 1] = -1.0 / h ** 2
    stiffness[idx + 1, idx] = -1.0 / h ** 2
    profile = np.sin(np.pi * np.arange(1, n_dof + 1) / (n_dof + 1))
    qoi = QoIDefinition(kind=QoIKind.MEAN_JOULE_LOSS, horizon=horizon, mass=mass)
    return LinearSystemModel(mass=mass, stiffness=stiffness,
                             forcing=_ProfileForcing(frequency, profile),
                             initial_state=np.zeros(n_dof), qoi=qoi)


def evaluate_qoi(model: LinearSystemModel, trajectory) -> float:
    """models.py:321-344 on a host trajectory (the device families accumulate
    the same sums inside the time-stepping kernels instead)."""
    qoi = model.qoi
    dt = trajectory.dt
    covered = trajectory.times[-1] - trajectory.times[0]
    if covered < qoi.horizon * (1.0 - 1e-9):
        raise ValueError(f"trajectory covers {covered} s but the QoI horizon is {qoi.horizon} s")
    n_t = int(round(qoi.horizon / dt))
    if qoi.kind is QoIKind.ELECTRICAL_ENERGY:
        u = qoi.drive(trajectory.times[1:n_t + 1])
        i1 = trajectory.states[1:n_t + 1, qoi.current_index]
        return float(np.sum(u * i1) * dt)
    if qoi.kind is QoIKind.MEAN_JOULE_LOSS:
        d = np.diff(trajectory.states[:n_t + 1], axis=0) / dt
        quad = np.einsum("ki,ij,kj->k", d, qoi.mass, d)
        return float(np.sum(quad) * dt / qoi.horizon)
    raise ValueError(f"unknown QoI kind {qoi.kind}")


class _Kind(enum.Enum):
    STEINMETZ = "steinmetz"
    SYNTHETIC = "synthetic"


@dataclass
class MachineFamily(_BatchedFamily):
    """A parametrized machine model plus its level hierarchy on one GPU
    (models.py:376-411 protocol: ``uncertain``, ``hierarchy``, ``evaluate``;
    plus ``build``, ``evaluate_batch``, ``coupled_batch``, ``run_levels``)."""

    model_id: str
    uncertain: UncertainInput
    hierarchy: tuple
    horizon: float
    drive: DriveSettings | None = None
    n_dof: int = 0
    frequency: float = 50.0
    device: object = None
    rtol: float = 1e-13
    max_it: int = 20000
    _solver: object = field(default=None, repr=False, compare=False)

    # ------------------------------------------------------------ host model
    def build(self, params: ParameterVector) -> LinearSystemModel:
        if self.model_id == "steinmetz":
            return build_steinmetz(params, self.drive, horizon=self.horizon)
        return build_synthetic_machine(self.n_dof, params, horizon=self.horizon,
                                       frequency=self.frequency)

    # ------------------------------------------------------------ device
    def _pattern(self):
        if self.model_id == "steinmetz":
            row_ptr = np.array([0, 3, 6, 9], dtype=np.int32)
            col = np.tile(np.arange(3, dtype=np.int32), 3)
            profile = np.array([self.drive.amplitude, 0.0, 0.0])
            return row_ptr, col, profile, self.drive.frequency
        n = self.n_dof
        rows = [[j for j in (i - 1, i, i + 1) if 0 <= j < n] for i in range(n)]
        row_ptr = np.concatenate([[0], np.cumsum([len(r) for r in rows])]).astype(np.int32)
        col = np.concatenate(rows).astype(np.int32)
        profile = np.sin(np.pi * np.arange(1, n + 1) / (n + 1))
        return row_ptr, col, profile, self.frequency

    @property
    def solver(self):
        if self._solver is None:
            from .solver import SystemSolver
            row_ptr, col, profile, freq = self._pattern()
            self._solver = SystemSolver(row_ptr, col, profile, freq, self.device, self.rtol,
                                        self.max_it)
        return self._solver

    def _n_params(self) -> int:
        return 6 if self.model_id == "steinmetz" else NUM_BARS

    def values(self, params: np.ndarray):
        """Per-sample CSR values (M, K) [S, nnz] on the device pattern."""
        p = np.asarray(params, dtype=float).reshape(-1, self._n_params())
        S = len(p)
        if self.model_id == "steinmetz":
            K = _steinmetz_stiffness(p, self.drive.slip)
            r1, r_fe, l_s1, l_h = p[:, 0], p[:, 2], p[:, 3], p[:, 5]
            # first equation scaled by L_s1 (module docstring)
            K[:, 0, 0] = r1 + r_fe
            K[:, 0, 1] = -r_fe
            K[:, 0, 2] = -r_fe / l_h
            M = np.zeros((S, 3, 3))
            M[:, 0, 0] = l_s1
            M[:, 1, 1] = 1.0
            M[:, 2, 2] = 1.0
            return M.reshape(S, 9), K.reshape(S, 9)
        n = self.n_dof
        h = 1.0 / n
        diag, off = _bar_mass_diag(n, p)
        nnz = 3 * n - 2
        Mv = np.zeros((S, nnz))
        Kv = np.zeros((S, nnz))
        # CSR order per row: (i-1, i, i+1)
        first = np.concatenate([[0], 3 * np.arange(1, n) - 1])     # position of (i, i-1) or (0, 0)
        dpos = first + (np.arange(n) > 0)
        Mv[:, dpos] = diag
        Mv[:, dpos[:-1] + 1] = off                 # (i, i+1)
        Mv[:, dpos[1:] - 1] = off                  # (i+1, i)
        Kv[:, dpos] = 2.0 / h ** 2
        Kv[:, dpos[:-1] + 1] = -1.0 / h ** 2
        Kv[:, dpos[1:] - 1] = -1.0 / h ** 2
        return Mv, Kv

    def _assemble_host(self, params, M, K, rp=None):
        import torch
        Mv, Kv = self.values(params)
        M.copy_(torch.from_numpy(Mv).pin_memory(), non_blocking=True)
        K.copy_(torch.from_numpy(Kv).pin_memory(), non_blocking=True)

    def _seq_job(self, rows, dt):
        from .solver import SeqJob
        from .timeint import step_count
        n = step_count(0.0, self.horizon, dt)
        mode = _lib.QOI_ELECTRICAL if self.model_id == "steinmetz" else _lib.QOI_JOULE
        return SeqJob(rows, dt, n, mode, 0, 0)

    def _finish_q(self, acc, dt):
        if self.model_id == "steinmetz":
            return acc * (self.drive.amplitude * dt)
        return acc / (dt * self.horizon)


def steinmetz_family(hierarchy, nominal=STEINMETZ_NOMINAL, halfwidth: float = 0.05,
                     drive: DriveSettings = DriveSettings(), horizon: float = 1.0,
                     device=None, **kw) -> MachineFamily:
    """models.py:431-441 on the GPU (direct path)."""
    nominal_pv = ParameterVector("steinmetz", np.asarray(nominal, dtype=float))
    return MachineFamily(model_id="steinmetz", uncertain=UncertainInput(nominal_pv, halfwidth),
                         hierarchy=tuple(hierarchy), horizon=horizon, drive=drive,
                         device=device, **kw)


def synthetic_family(hierarchy, n_dof: int = 64, halfwidth: float = 0.05,
                     horizon: float = 0.16, frequency: float = 50.0, device=None,
                     **kw) -> MachineFamily:
    """models.py:444-453 on the GPU (SM-resident PCG path)."""
    _synthetic_check(n_dof)
    nominal_pv = ParameterVector("synthetic", np.ones(NUM_BARS))
    return MachineFamily(model_id="synthetic", uncertain=UncertainInput(nominal_pv, halfwidth),
                         hierarchy=tuple(hierarchy), horizon=horizon, n_dof=n_dof,
                         frequency=frequency, device=device, **kw)

