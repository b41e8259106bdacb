"""Executor accounting: sampling plans under a core budget and the Ledger
(SPEC.md [MODULE] executor, lines 447-500).

Two modes, as the SPEC asks:
  * ``simulate`` — the simulated clock: batches from greedy packing
    (``schedule_level``), batch wall time = max task time, Parareal tasks
    timed by costmodel.parareal_time / parareal_effort.
  * ``gpu_ledger`` — the real mode of this framework: one batched device
    launch per estimate, timed on the device.  Effort is counted in device
    task-slot seconds from per-task device timers (each task holds one CTA
    slot of an SM, or one thread on the direct path, for its duration), the
    GPU analogue of "the sum of the time spent over all active processor
    cores".

Ledger JSON keys follow SPEC.md:497: ``mode``, ``levels[{level, batches,
wall_s, effort_core_s}]``, ``total_wall_s``, ``total_effort_core_s``.
"""

from __future__ import annotations

import json
from dataclasses import dataclass, field

from . import costmodel

__all__ = ["Task", "SequentialSolve", "CoupledPair", "PararealSolve", "schedule_level",
           "LevelLedger", "Ledger", "simulate", "plan_tasks", "gpu_ledger"]


@dataclass(frozen=True)
class Task:
    level: int
    index: int = 0

    width: int = 1

    def wall(self) -> float:
        raise NotImplementedError

    def effort(self) -> float:
        raise NotImplementedError


@dataclass(frozen=True)
class SequentialSolve(Task):
    cost_s: float = 0.0

    def wall(self):
        return self.cost_s

    def effort(self):
        return self.cost_s


@dataclass(frozen=True)
class CoupledPair(Task):
    """Q_l and Q_{l-1} of one sample solved concurrently on two cores."""

    cost_hi_s: float = 0.0
    cost_lo_s: float = 0.0
    width: int = 2

    def wall(self):
        return max(self.cost_hi_s, self.cost_lo_s)

    def effort(self):
        return self.cost_hi_s + self.cost_lo_s


@dataclass(frozen=True)
class PararealSolve(Task):
    """Finest-level Parareal solve on n_c_para cores (width); ``K`` recorded
    iterations.  ``wall_hint_s`` overrides the closed form (measured runs)."""

    tau_F: float = 0.0
    tau_C: float = 0.0
    K: int = 1
    wall_hint_s: float | None = None

    def wall(self):
        if self.wall_hint_s is not None:
            return self.wall_hint_s
        return costmodel.parareal_time(self.tau_F, self.tau_C, self.width, self.K)

    def effort(self):
        return costmodel.parareal_effort(self.tau_F, self.tau_C, self.width, self.K)


def schedule_level(tasks, n_c: int) -> list[list[Task]]:
    """Greedy in-order packing into batches of at most n_c core slots."""
    if n_c < 1:
        raise ValueError("n_c must be >= 1")
    batches: list[list[Task]] = []
    used = n_c
    levels = {t.level for t in tasks}
    if len(levels) > 1:
        raise ValueError(f"schedule_level needs tasks of one level, got {sorted(levels)}")
    for t in tasks:
        if t.width > n_c:
            raise ValueError(f"task of width {t.width} does not fit n_c={n_c}")
        if used + t.width > n_c:
            batches.append([])
            used = 0
        batches[-1].append(t)
        used += t.width
    return batches


@dataclass
class LevelLedger:
    level: int
    batches: int
    wall_s: float
    effort_core_s: float


@dataclass
class Ledger:
    mode: str
    levels: list = field(default_factory=list)
    extra: dict = field(default_factory=dict)

    @property
    def total_wall_s(self) -> float:
        if "total_wall_s" in self.extra:
            return float(self.extra["total_wall_s"])
        return sum(lv.wall_s for lv in self.levels)

    @property
    def total_effort_core_s(self) -> float:
        return sum(lv.effort_core_s for lv in self.levels)

    def to_dict(self) -> dict:
        d = {"mode": self.mode,
             "levels": [{"level": lv.level, "batches": lv.batches, "wall_s": lv.wall_s,
                         "effort_core_s": lv.effort_core_s} for lv in self.levels],
             "total_wall_s": self.total_wall_s,
             "total_effort_core_s": self.total_effort_core_s}
        d.update({k: v for k, v in self.extra.items() if k != "total_wall_s"})
        return d

    def dump(self, path: str):
        with open(path, "w") as fh:
            json.dump(self.to_dict(), fh, indent=1, sort_keys=True)


def simulate(plan, n_c: int) -> Ledger:
    """plan: per level a list of Tasks (levels run one after another)."""
    led = Ledger("simulated")
    for lvl, tasks in enumerate(plan):
        batches = schedule_level(tasks, n_c) if tasks else []
        wall = sum(max(t.wall() for t in b) for b in batches)
        effort = sum(t.effort() for t in tasks)
        led.levels.append(LevelLedger(lvl, len(batches), wall, effort))
    return led


def plan_tasks(N, costs, parareal=None):
    """Per-level task lists for sample counts N and per-level costs C_l:
    level 0 single solves, level l > 0 coupled pairs; with
    ``parareal = (n_c_para, K, tau_C[, wall_hint])`` the finest level runs
    Parareal plus a separate level-(L-1) solve per sample."""
    L = len(N) - 1
    plan = []
    for lvl, n in enumerate(N):
        if lvl == 0:
            plan.append([SequentialSolve(0, k, cost_s=costs[0]) for k in range(n)])
        elif lvl == L and parareal is not None:
            n_para, K, tau_c = parareal[:3]
            hint = parareal[3] if len(parareal) > 3 else None
            tasks = []
            for k in range(n):
                tasks.append(PararealSolve(lvl, k, width=n_para, tau_F=costs[lvl], tau_C=tau_c,
                                           K=K, wall_hint_s=hint))
            tasks += [SequentialSolve(lvl, k, cost_s=costs[lvl - 1]) for k in range(n)]
            plan.append(tasks)
        else:
            plan.append([CoupledPair(lvl, k, cost_hi_s=costs[lvl], cost_lo_s=costs[lvl - 1])
                         for k in range(n)])
    return plan


def gpu_ledger(batches, wall_s: float, dist=None) -> Ledger:
    """Real-mode ledger of one batched device estimate (mlmc_estimate with
    ``timing=True``).  All levels run in one batched launch (plus the finest
    level's Parareal on a second stream), so per level: ``batches`` = 1,
    ``wall_s`` = the longest task of the level (its critical path inside the
    launch; for the Parareal level the longest coarse sweep or fine slice
    accumulated over iterations), ``effort_core_s`` = the sum over the
    level's tasks of the device time each held its execution slot (one CTA
    on the SM-resident path, one thread on the direct path).  Over ranks:
    effort summed, wall maxed.  ``total_wall_s`` is the measured host wall
    time of the whole estimate."""
    import torch
    led = Ledger("gpu-batched", extra={"total_wall_s": float(wall_s),
                                       "effort_unit": "device task-slot seconds"})
    rows = []
    for b in batches:
        eff, longest = 0.0, 0.0
        for t in b.elapsed:
            if t.numel():
                eff += float(t.to(torch.float64).sum().item()) * 1e-9
                longest = max(longest, float(t.max().item()) * 1e-9)
        rows.append((eff, longest))
    if dist is not None and dist.get_world_size() > 1 and rows:
        dev = batches[0].q_l.device
        e = torch.tensor([r[0] for r in rows], dtype=torch.float64, device=dev)
        w = torch.tensor([r[1] for r in rows], dtype=torch.float64, device=dev)
        dist.all_reduce(e, op=dist.ReduceOp.SUM)
        dist.all_reduce(w, op=dist.ReduceOp.MAX)
        rows = list(zip(e.tolist(), w.tolist()))
    for b, (eff, longest) in zip(batches, rows):
        led.levels.append(LevelLedger(b.level, 1, longest, eff))
    return led
