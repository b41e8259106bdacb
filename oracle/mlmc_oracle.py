"""TEST INFRASTRUCTURE ONLY — CPU oracle for the sampler, the FE family, the
QoIs and the MLMC level statistics.

* ``RandomStream``: the SPEC.md:250-254 contract (pure function of
  (seed, level, index)); ``np.random.default_rng(SeedSequence(seed,
  spawn_key=(level, index)))``.
* ``draw_uniform``: models.py:305-318 (``rng.uniform(nom*(1-h), nom*(1+h))``,
  nominal returned unchanged when h == 0).  ``draw_gaussian``: config 3's
  xi ~ N(0,1)^64 (``rng.standard_normal``), a new input kind.
* ``OracleFEModel``: the duck type the reference integrators consume
  (``mass``, ``stiffness``, ``forcing``, ``initial_state``, ``dim``;
  timeint.py:65,99,104-109; parareal.py:154), with a picklable
  ``ProfileForcing`` shaped like models.py:171-179.
* QoIs (new kinds, quadrature conventions of models.py:335-343):
  MAGNETIC_ENERGY_T  = 1/2 a(T)^T K a(T);
  TIME_AVG_MAGNETIC_ENERGY = (1/T_w) sum_{t_{k+1} in last window} W(a_{k+1}) dt
  (right end points, like ELECTRICAL_ENERGY at models.py:337-339).
* ``evaluate`` mirrors MachineFamily.evaluate (models.py:389-411);
  ``level_statistics`` the SPEC.md:256-266,280-288 estimator with a fixed
  N per level (Q_{-1} = 0; sums accumulated in sample order k = 1..N).
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from . import fe_oracle as fe
from .ie_oracle import implicit_euler
from .parareal_oracle import OraclePararealConfig, parareal


# ----------------------------------------------------------------- sampling
class RandomStream:
    def __init__(self, seed: int, level: int, index: int):
        self.key = (int(seed), int(level), int(index))

    def generator(self) -> np.random.Generator:
        seed, level, index = self.key
        return np.random.default_rng(np.random.SeedSequence(seed, spawn_key=(level, index)))


def draw_uniform(nominal: np.ndarray, halfwidth: float, stream) -> np.ndarray:
    nominal = np.asarray(nominal, dtype=float)
    if halfwidth == 0.0:
        return nominal.copy()
    rng = stream.generator() if hasattr(stream, "generator") else stream
    return rng.uniform(nominal * (1.0 - halfwidth), nominal * (1.0 + halfwidth))


def draw_gaussian(dim: int, stream) -> np.ndarray:
    rng = stream.generator() if hasattr(stream, "generator") else stream
    return rng.standard_normal(dim)


# ----------------------------------------------------------------- configs
@dataclass(frozen=True)
class OracleConfig:
    name: str
    n: int
    layout: str
    horizon: float
    dts: tuple
    samples: tuple
    qoi: str                         # "energy_T" | "time_avg_energy"
    avg_window: float = 0.0
    parareal: tuple | None = None    # (M, dt_coarse, tol, K_max)
    halfwidth: float = 0.1

    @property
    def n_params(self) -> int:
        return {"quad4": 8, "blocks8": 16, "kl64": fe.KL_MODES}[self.layout]

    def nominal(self) -> np.ndarray:
        if self.layout == "quad4":
            return np.array([fe.NU0] * 4 + [fe.SIGMA0] * 4)
        if self.layout == "blocks8":
            return np.array([fe.NU0] * 8 + [fe.SIGMA0] * 8)
        return np.zeros(fe.KL_MODES)


T = fe.PERIOD
CONFIGS = {
    0: OracleConfig("cfg0", 32, "quad4", T, (T / 32, T / 64, T / 128), (1000, 250, 60),
                    "energy_T"),
    1: OracleConfig("cfg1", 32, "quad4", T, (T / 256, T / 512, T / 1024), (512, 128, 32),
                    "energy_T", parareal=(16, T / 16, 1e-8, 5)),
    2: OracleConfig("cfg2", 256, "blocks8", 4 * T, (T / 64, T / 128, T / 256, T / 512),
                    (4096, 1024, 256, 64), "time_avg_energy", avg_window=T),
    3: OracleConfig("cfg3", 128, "kl64", T, (T / 128, T / 256, T / 512), (2048, 512, 128),
                    "energy_T", parareal=(32, T / 32, 1e-8, 6)),
    4: OracleConfig("cfg4", 512, "blocks8", T, (T / 64, T / 128, T / 256, T / 512),
                    (8192, 2048, 512, 128), "energy_T", parareal=(64, T / 64, 1e-8, 6)),
}


def draw(cfg: OracleConfig, seed: int, level: int, index: int) -> np.ndarray:
    stream = RandomStream(seed, level, index)
    if cfg.layout == "kl64":
        return draw_gaussian(fe.KL_MODES, stream)
    return draw_uniform(cfg.nominal(), cfg.halfwidth, stream)


# ----------------------------------------------------------------- FE model
@dataclass(frozen=True)
class ProfileForcing:
    frequency: float
    profile: np.ndarray

    def __call__(self, t):
        return np.sin(2.0 * np.pi * self.frequency * t) * self.profile


@dataclass(frozen=True)
class OracleFEModel:
    mass: object
    stiffness: object
    forcing: ProfileForcing
    initial_state: np.ndarray

    @property
    def dim(self) -> int:
        return self.mass.shape[0]


class FEProblem:
    """Mesh + element geometry cached per (n, layout)."""

    def __init__(self, n: int, layout: str):
        self.n = n
        self.layout = layout
        self.mesh = fe.build_mesh(n)
        self.geom = fe.ElementGeometry(self.mesh)
        self.src = fe.source_elements(self.mesh, layout)

    def model(self, params: np.ndarray, dense: bool | None = None) -> OracleFEModel:
        sigma, nu = fe.material_fields(self.mesh, self.layout, params)
        mass, stiff, prof = fe.assemble(self.geom, sigma, nu, self.src)
        if dense is None:
            dense = self.mesh.n_interior <= 1100
        if dense:
            mass, stiff = mass.toarray(), stiff.toarray()
        return OracleFEModel(mass=mass, stiffness=stiff,
                             forcing=ProfileForcing(fe.FREQ, prof),
                             initial_state=np.zeros(self.mesh.n_interior))


def energy(model, a) -> float:
    return 0.5 * float(a @ (model.stiffness @ a))


@dataclass
class OracleRecord:
    q: float
    k_used: int | None = None
    defects: list | None = None


def evaluate(problem: FEProblem, cfg: OracleConfig, params, dt: float,
             use_parareal: bool, dense: bool | None = None) -> OracleRecord:
    """models.py:389-411 with the FE model and the new QoIs."""
    model = problem.model(params, dense=dense)
    n_t = int(round(cfg.horizon / dt))
    if use_parareal:
        m, dtc, tol, kmax = cfg.parareal
        pcfg = OraclePararealConfig(m, dt, dtc, tol, kmax)
        res = parareal(model, 0.0, cfg.horizon, model.initial_state, pcfg,
                       keep_fine=cfg.qoi != "energy_T")
        if cfg.qoi == "energy_T":
            return OracleRecord(energy(model, res.terminal), res.iterations_used,
                                list(res.defect_history))
        raise NotImplementedError("time-averaged QoI under Parareal is not configured")
    if cfg.qoi == "energy_T":
        tr = implicit_euler(model, 0.0, cfg.horizon, dt, model.initial_state,
                            keep_states=False)
        return OracleRecord(energy(model, tr.terminal))
    n_w = int(round(cfg.avg_window / dt))
    acc = [0.0]

    def obs(k, t, a):
        if k + 1 > n_t - n_w:
            acc[0] += energy(model, a)

    implicit_euler(model, 0.0, cfg.horizon, dt, model.initial_state,
                   keep_states=False, observer=obs)
    return OracleRecord(acc[0] * dt / cfg.avg_window)


# ----------------------------------------------------------------- estimator
@dataclass
class OracleLevelStats:
    level: int
    n: int
    sum_y: float
    sum_y2: float

    @property
    def mean(self) -> float:
        return self.sum_y / self.n

    @property
    def var(self) -> float:
        if self.n < 2:
            return 0.0
        return (self.sum_y2 - self.n * self.mean ** 2) / (self.n - 1)


def level_statistics(level: int, q_l, q_lm1) -> OracleLevelStats:
    """SPEC.md:256-260; accumulation in sample order."""
    sy = 0.0
    sy2 = 0.0
    for a, b in zip(q_l, q_lm1):
        y = float(a) - float(b)
        sy += y
        sy2 += y * y
    return OracleLevelStats(level, len(q_l), sy, sy2)


def coupled(problem: FEProblem, cfg: OracleConfig, level: int, params,
            dense: bool | None = None):
    """(Q_l, Q_{l-1}, K) with Q_{-1} = 0."""
    top = len(cfg.dts) - 1
    use_pr = cfg.parareal is not None and level == top
    hi = evaluate(problem, cfg, params, cfg.dts[level], use_pr, dense)
    lo = 0.0 if level == 0 else evaluate(problem, cfg, params, cfg.dts[level - 1],
                                         False, dense).q
    return hi.q, lo, hi.k_used
