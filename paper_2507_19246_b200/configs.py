"""The five BASELINE.json configurations as data.

Decisions BASELINE.json leaves open: region layouts and
conducting regions (fe.py), J0 = 1e6 A/m^2, source region, KL ordering /
normalisation, config-3/4 coarse propagator = one implicit-Euler step per
slice, Parareal tolerance 1e-8 with the reference's *jump* criterion
(parareal.py:198-207), config-4 horizon = one period, config-4 K_max = 6.
"""

from __future__ import annotations

from dataclasses import dataclass

from . import fe

T = fe.PERIOD


@dataclass(frozen=True)
class ExperimentConfig:
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
    seed: int = 0

    @property
    def levels(self) -> int:
        return len(self.dts)

    def steps(self, level: int) -> int:
        return int(round(self.horizon / self.dts[level]))

    def seq_equiv_steps(self, scale: int = 1) -> int:
        """sum_l N_l (n_l + n_{l-1}) — sequential-equivalent sample-timesteps."""
        tot = 0
        for lvl, n in enumerate(self.samples):
            tot += n * scale * (self.steps(lvl) + (self.steps(lvl - 1) if lvl > 0 else 0))
        return tot

    def parareal_config(self):
        if self.parareal is None:
            return None
        from .parareal import PararealConfig
        m, dtc, tol, kmax = self.parareal
        return PararealConfig(m, self.dts[-1], dtc, tol, kmax)


CONFIGS = {
    0: ExperimentConfig("cfg0", 32, "quad4", T, (T / 32, T / 64, T / 128), (1000, 250, 60),
                        "energy_T"),
    1: ExperimentConfig("cfg1", 32, "quad4", T, (T / 256, T / 512, T / 1024), (512, 128, 32),
                        "energy_T", parareal=(16, T / 16, 1e-8, 5)),
    2: ExperimentConfig("cfg2", 256, "blocks8", 4 * T, (T / 64, T / 128, T / 256, T / 512),
                        (4096, 1024, 256, 64), "time_avg_energy", avg_window=T),
    3: ExperimentConfig("cfg3", 128, "kl64", T, (T / 128, T / 256, T / 512), (2048, 512, 128),
                        "energy_T", parareal=(32, T / 32, 1e-8, 6)),
    4: ExperimentConfig("cfg4", 512, "blocks8", T, (T / 64, T / 128, T / 256, T / 512),
                        (8192, 2048, 512, 128), "energy_T", parareal=(64, T / 64, 1e-8, 6)),
}


def get_config(c) -> ExperimentConfig:
    if isinstance(c, ExperimentConfig):
        return c
    if isinstance(c, str):
        c = int(c.replace("cfg", ""))
    return CONFIGS[int(c)]
