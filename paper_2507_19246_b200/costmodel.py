"""Closed-form cost, speedup and effort model of the combined MLMC+Parareal
method (§II-C/§II-D; SPEC.md [MODULE] costmodel, lines 335-445).

Host-only arithmetic (the planning side of the executor); the measured side
is ``executor.gpu_ledger``, which feeds device-timed costs into the same
formulas.  Sums run small-to-large as SPEC.md's design decision asks.

  parareal_time        tau_para
  parareal_effort      E_para
  ideal_speedup        s_inf
  kappa                K <= kappa
  effort_ratio_*       eps_inf
  batch_count          b_l
  cores_per_sample     n_c,para
  finite_speedup       s_nc
  figure_data          Figs. 1-2
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import Callable, Sequence

__all__ = ["CostModelParams", "parareal_time", "parareal_effort", "parareal_time_sum",
           "parareal_effort_sum", "ideal_speedup", "kappa", "kappa_scan",
           "effort_ratio_infinite", "effort_ratio_max", "batch_count", "cores_per_sample",
           "finite_speedup", "figure_data", "write_figure_csv"]


def _default_variance(level: int) -> float:
    return 10.0 ** (-2 * level)


@dataclass(frozen=True)
class CostModelParams:
    """C_l = C0 r^l; V_l = 10^-2l by default."""

    C0: float = 1.0
    r: float = 10.0
    L: int = 2
    n_c: int = 180
    N: tuple = (10303, 85, 10)
    variance_model: Callable[[int], float] = field(default=_default_variance, compare=False)

    def __post_init__(self):
        if not self.r > 1.0:
            raise ValueError(f"refinement rate r must be > 1, got {self.r}")
        if self.L < 1:
            raise ValueError(f"L must be >= 1, got {self.L}")
        if self.n_c < 1:
            raise ValueError(f"n_c must be >= 1, got {self.n_c}")
        if len(self.N) != self.L + 1:
            raise ValueError(f"need L+1 = {self.L + 1} sample counts, got {len(self.N)}")
        if any(int(n) < 0 for n in self.N):
            raise ValueError("sample counts must be >= 0")

    def cost(self, level: int) -> float:
        return self.C0 * self.r ** level

    def ratio_prev(self, level: int) -> float:
        return 0.0 if level == 0 else 1.0 / self.r


def _check_km(M: int, K: int):
    if M < 1:
        raise ValueError(f"M must be >= 1, got {M}")
    if not 1 <= K <= M:
        raise ValueError(f"need 1 <= K <= M, got K={K}, M={M}")


def parareal_time(tau_F: float, tau_C: float, M: int, K: int) -> float:
    """(K/M) [tau_F + (M - (K+1)/2) tau_C]."""
    _check_km(M, K)
    if tau_F < 0 or tau_C < 0:
        raise ValueError("costs must be >= 0")
    return K / M * (tau_F + (M - (K + 1) / 2.0) * tau_C)


def parareal_effort(tau_F: float, tau_C: float, M: int, K: int) -> float:
    """(K/M)[M - (K+1)/2](tau_F + tau_C) + (K/M) tau_F."""
    _check_km(M, K)
    if tau_F < 0 or tau_C < 0:
        raise ValueError("costs must be >= 0")
    return K / M * (M - (K + 1) / 2.0) * (tau_F + tau_C) + K / M * tau_F


def parareal_time_sum(tau_F, tau_C, M, K) -> float:
    """Per-iteration form sum_k tau_F/M + (M-k)/M tau_C."""
    _check_km(M, K)
    return math.fsum(tau_F / M + (M - k) / M * tau_C for k in range(1, K + 1))


def parareal_effort_sum(tau_F, tau_C, M, K) -> float:
    """Per-iteration form sum_k (M-k+1)/M tau_F + (M-k)/M tau_C."""
    _check_km(M, K)
    return math.fsum((M - k + 1) / M * tau_F + (M - k) / M * tau_C for k in range(1, K + 1))


def ideal_speedup(r: float, L: int) -> float:
    """s_inf = (r^{L+1} - 1) / (2 r^L - r^{L-1} - 1)."""
    if not r > 1.0 or L < 1:
        raise ValueError("need r > 1 and L >= 1")
    return (r ** (L + 1) - 1.0) / (2.0 * r ** L - r ** (L - 1) - 1.0)


def kappa(r: float, n_c_para: int) -> int:
    """Largest K with tau_para <= C_{L-1} for tau_F = C_L, tau_C = C_{L-2}."""
    if not r > 1.0 or n_c_para < 1:
        raise ValueError("need r > 1 and n_c_para >= 1")
    a = 2.0 * r * r + 2.0 * n_c_para - 1.0
    disc = a * a - 8.0 * n_c_para * r
    if disc < 0:
        raise ValueError(f"negative discriminant {disc} (r={r}, n={n_c_para})")
    k = int(math.floor((a - math.sqrt(disc)) / 2.0))
    if k > r:
        raise ValueError(f"kappa {k} exceeds r {r}")
    return k


def kappa_scan(r: float, n_c_para: int, L: int = 2) -> int:
    """Scan oracle: largest K in 1..n with parareal_time(r^L, r^{L-2}, n, K) <= r^{L-1}."""
    best = 0
    for K in range(1, n_c_para + 1):
        if parareal_time(r ** L, r ** (L - 2), n_c_para, K) <= r ** (L - 1) * (1 + 1e-12):
            best = K
    return best


def batch_count(N_l: int, cost_ratio_prev: float, n_c: int) -> int:
    """ceil(N_l (1 + C_{l-1}/C_l) / n_c), exact for rational ratios 1/r."""
    if N_l < 0 or n_c < 1:
        raise ValueError("need N_l >= 0 and n_c >= 1")
    if N_l == 0:
        return 0
    return int(math.ceil(N_l * (1.0 + cost_ratio_prev) / n_c - 1e-12))


def cores_per_sample(n_c: int, N_L: int, cost_ratio_prev: float) -> int:
    """floor(n_c / (N_L (1 + C_{L-1}/C_L)))."""
    if N_L < 1:
        raise ValueError("need N_L >= 1")
    n = int(math.floor(n_c / (N_L * (1.0 + cost_ratio_prev)) + 1e-12))
    if n < 1:
        raise ValueError("insufficient cores for per-sample parallelism")
    return n


def _M(params: CostModelParams, M):
    if M is not None:
        return int(M)
    return cores_per_sample(params.n_c, int(params.N[-1]), params.ratio_prev(params.L))


def effort_ratio_infinite(params: CostModelParams, K: int, M: int | None = None) -> float:
    """E_comb,inf / E_ref,inf with E_comb = sum_{l<L} N_l C_l + N_L E_para(C_L, C_{L-2}, M, K);
    M defaults to n_c,para (SPEC.md:435 identifies M with n_c,para)."""
    L = params.L
    ref = math.fsum(int(params.N[l]) * params.cost(l) for l in range(L + 1))
    if int(params.N[L]) == 0:
        return 1.0
    m = _M(params, M)
    tau_c = params.cost(L - 2) if L >= 2 else 0.0
    comb = math.fsum([int(params.N[l]) * params.cost(l) for l in range(L)]
                     + [int(params.N[L]) * parareal_effort(params.cost(L), tau_c, m, K)])
    return comb / ref


def effort_ratio_max(params: CostModelParams, M: int | None = None) -> float:
    m = _M(params, M)
    return effort_ratio_infinite(params, min(kappa(params.r, m), m), m)


def finite_speedup(params: CostModelParams, K: int) -> float:
    """s_nc = sum_l b_l C_l / (sum_{l<L} b_l C_l + (K/n)[r^L + (n - (K+1)/2) r^{L-2}] C0)."""
    L, r = params.L, params.r
    b = [batch_count(int(params.N[l]), params.ratio_prev(l), params.n_c) for l in range(L + 1)]
    n = cores_per_sample(params.n_c, int(params.N[L]), params.ratio_prev(L))
    _check_km(n, K)
    num = math.fsum(b[l] * params.cost(l) for l in range(L + 1))
    den = math.fsum([b[l] * params.cost(l) for l in range(L)]
                    + [params.C0 * K / n * (r ** L + (n - (K + 1) / 2.0) * r ** (L - 2))])
    return num / den


def figure_data(params: CostModelParams, n_c_list: Sequence[int], K_range: Sequence[int]):
    """Rows (n_c, K, s_nc, eps) for Figs. 1-2; rows whose K exceeds n_c,para
    (or whose n_c cannot give every level-L sample a core) carry NaN."""
    rows = []
    for n_c in n_c_list:
        p = CostModelParams(params.C0, params.r, params.L, int(n_c), tuple(params.N),
                            params.variance_model)
        for K in K_range:
            try:
                s = finite_speedup(p, int(K))
                e = effort_ratio_infinite(p, int(K))
            except ValueError:
                s = e = float("nan")
            rows.append((int(n_c), int(K), s, e))
    return rows


def write_figure_csv(path: str, rows, note: str | None = None):
    with open(path, "w") as fh:
        if note:
            fh.write(f"# {note}\n")
        fh.write("n_c,K,speedup,effort_ratio\n")
        for n_c, K, s, e in rows:
            fh.write(f"{n_c},{K},{s!r},{e!r}\n")
