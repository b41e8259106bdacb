"""Sampler / level / family API (drop-in for ``mlmc_parareal.models``) with the
2D eddy-current FE family whose solves run batched on the GPU.

Kept from the reference with the same names, fields and errors:
  ``ParameterVector``   models.py:54-74 (strict positivity)
  ``UncertainInput``    models.py:77-88
  ``LevelSpec``         models.py:91-100
  ``make_hierarchy``    models.py:103-108
  ``QoIKind``           models.py:111-113 (+ the two FE kinds below)
  ``draw_parameters``   models.py:305-318 (uniform; nominal when h == 0)
  ``EvalRecord``        models.py:347-353
  ``LinearToyFamily``   models.py:414-428 / ``toy_family`` :456-461
The family protocol (``uncertain``, ``hierarchy``, ``evaluate``) of
``MachineFamily`` (models.py:376-411) is implemented by ``EddyCurrentFamily``,
which adds the batched entry points ``evaluate_batch`` / ``coupled_batch`` /
``run_levels`` used by the estimator.

New (no reference counterpart; BASELINE.json configs):
  ``GaussianInput``     xi ~ N(0,1)^d for the config-3 KL field
  QoIKind.MAGNETIC_ENERGY_T         1/2 a(T)^T K a(T)
  QoIKind.TIME_AVG_MAGNETIC_ENERGY  (1/T_w) sum_{t_k in last window} W(a_k) dt
                                    (right end points, like models.py:337-339)
"""

from __future__ import annotations

import enum
import time
from dataclasses import dataclass, field

import numpy as np

from . import fe
from .parareal import PararealConfig

__all__ = ["ParameterVector", "UncertainInput", "GaussianInput", "LevelSpec", "make_hierarchy",
           "QoIKind", "draw_parameters", "EvalRecord", "EddyCurrentFamily", "CoupledBatch",
           "LinearToyFamily", "toy_family", "eddy_current_family"]


_PARAM_COUNTS = {"steinmetz": 6, "synthetic": 32}   # models.py:50


@dataclass(frozen=True)
class ParameterVector:
    model_id: str
    values: np.ndarray

    def __post_init__(self):
        vals = np.atleast_1d(np.asarray(self.values, dtype=float))
        object.__setattr__(self, "values", vals)
        expected = (fe.n_params(self.model_id) if self.model_id in fe.LAYOUTS
                    else _PARAM_COUNTS.get(self.model_id))
        if expected is not None and len(vals) != expected:
            raise ValueError(f"model '{self.model_id}' takes {expected} parameters, got {len(vals)}")
        if self.model_id != "kl64" and not np.all(vals > 0.0):
            bad = int(np.argmin(vals))
            raise ValueError(f"parameter {bad} of '{self.model_id}' must be strictly positive, "
                             f"got {vals[bad]}")


@dataclass(frozen=True)
class UncertainInput:
    nominal: ParameterVector
    relative_halfwidth: float

    def __post_init__(self):
        if not 0.0 <= self.relative_halfwidth < 1.0:
            raise ValueError(f"relative_halfwidth must lie in [0, 1), got {self.relative_halfwidth}")

    @property
    def dim(self) -> int:
        return len(self.nominal.values)


@dataclass(frozen=True)
class GaussianInput:
    """Independent standard normals (KL coefficients of config 3)."""

    model_id: str
    dim: int


@dataclass(frozen=True, order=True)
class LevelSpec:
    level: int
    dt: float

    def __post_init__(self):
        if self.level < 0 or self.dt <= 0.0:
            raise ValueError(f"invalid level spec (level={self.level}, dt={self.dt})")


def make_hierarchy(dts) -> tuple[LevelSpec, ...]:
    dts = [float(dt) for dt in dts]
    if any(b >= a for a, b in zip(dts, dts[1:])):
        raise ValueError(f"step sizes must be strictly decreasing, got {dts}")
    return tuple(LevelSpec(level=i, dt=dt) for i, dt in enumerate(dts))


class QoIKind(enum.Enum):
    ELECTRICAL_ENERGY = "electrical_energy"
    MEAN_JOULE_LOSS = "mean_joule_loss"
    MAGNETIC_ENERGY_T = "magnetic_energy_T"
    TIME_AVG_MAGNETIC_ENERGY = "time_avg_magnetic_energy"


def draw_parameters(inp, stream) -> ParameterVector:
    """models.py:305-318 (uniform) and the Gaussian input of config 3."""
    if isinstance(inp, GaussianInput):
        rng = stream.generator() if hasattr(stream, "generator") else stream
        return ParameterVector(inp.model_id, rng.standard_normal(inp.dim))
    nominal = inp.nominal.values
    if inp.relative_halfwidth == 0.0:
        return ParameterVector(inp.nominal.model_id, nominal.copy())
    rng = stream.generator() if hasattr(stream, "generator") else stream
    lo = nominal * (1.0 - inp.relative_halfwidth)
    hi = nominal * (1.0 + inp.relative_halfwidth)
    return ParameterVector(inp.nominal.model_id, rng.uniform(lo, hi))


@dataclass(frozen=True)
class EvalRecord:
    q: float
    cost_s: float
    parareal_iterations: int | None = None


@dataclass
class CoupledBatch:
    """Device results of one level: Q_l, Q_{l-1} (0 on level 0) and Parareal K."""

    level: int
    q_l: object
    q_lm1: object
    k_used: object
    iters: object = None
    wall_s: float = 0.0
    defects: object = None
    elapsed: list = field(default_factory=list)   # int64 device-ns tensors (timing on)


@dataclass
class LinearToyFamily:
    """models.py:414-428: Q_l(xi) = xi (1 + dt_l); CPU, closed form (tests)."""

    uncertain: UncertainInput
    hierarchy: tuple
    cap: int | None = None      # samples per run_levels call (chunked-path tests)

    def evaluate(self, params: ParameterVector, level: LevelSpec, parareal_cfg=None,
                 pool=None) -> EvalRecord:
        return EvalRecord(q=float(params.values[0]) * (1.0 + level.dt), cost_s=1e-9)

    def max_samples_per_call(self, parareal_cfg=None, level=None):
        return self.cap

    def run_levels(self, draws, parareal_cfg=None, levels=None, **_):
        import torch
        levels = list(range(len(draws))) if levels is None else levels
        out = []
        for lvl, p in zip(levels, draws):
            p = p.get() if hasattr(p, "get") else p
            xi = torch.as_tensor(np.asarray(p, dtype=float)[:, 0] if len(p) else np.zeros(0))
            ql = xi * (1.0 + self.hierarchy[lvl].dt)
            qm = xi * (1.0 + self.hierarchy[lvl - 1].dt) if lvl > 0 else torch.zeros_like(xi)
            out.append(CoupledBatch(lvl, ql, qm, torch.zeros(len(xi), dtype=torch.int32)))
        return out


def toy_family(hierarchy, nominal: float = 1.0, halfwidth: float = 0.05,
               cap: int | None = None) -> LinearToyFamily:
    return LinearToyFamily(UncertainInput(ParameterVector("toy", np.array([nominal])), halfwidth),
                           tuple(hierarchy), cap)


class _BatchedFamily:
    """Batched level evaluation shared by the GPU families.  Subclasses set
    ``solver`` (a solver.BatchSolver), ``hierarchy``, ``horizon`` and provide
    the hooks ``_n_params``, ``_assemble_host`` / ``_assemble_dev`` (per-sample
    operator values into [S, nnz] slices), ``_seq_job`` / ``_finish_q`` (QoI
    task mode and its host-side scale; ``_pr_qoi`` derives the Parareal
    level's QoI from them)."""

    def _pr_stream(self, device):
        import torch
        st = getattr(self, "_side_stream", None)
        if st is None:
            lo, hi = torch.cuda.Stream.priority_range()
            st = torch.cuda.Stream(device=device, priority=hi)
            self._side_stream = st
        return st

    def _level_index(self, level) -> int:
        if isinstance(level, LevelSpec):
            return level.level
        return int(level)

    def _pr_qoi(self, dt_fine) -> dict:
        """QoI of the Parareal level as run_parareal keywords: the sequential
        job's task mode over the fine trajectory (final-state energy when
        the mode is QOI_FINAL_ENERGY)."""
        j = self._seq_job(np.zeros(0, dtype=np.int64), dt_fine)
        return {"qoi_mode": j.qoi_mode, "qoi_index": j.qoi_index, "qoi_from": j.qoi_from}

    def _assemble_dev(self, params_dev, M, K, rp=None):
        self._assemble_host(params_dev.cpu().numpy(), M, K)

    def _new_rp(self, S: int):
        """Region-parameter buffer of the region-linear operator (None: the
        family streams its operator)."""
        fn = getattr(self.solver, "new_region_params", None)
        return fn(S) if fn is not None else None

    # ------------------------------------------------------------ batched
    def run_levels(self, draws, parareal_cfg: PararealConfig | None = None, levels=None,
                   concurrent: bool = True, params_dev=None,
                   fused: bool | None = None, _no_chunk: bool = False) -> list[CoupledBatch]:
        """Coupled (Q_l, Q_{l-1}) for every level at once.

        draws[i]: [N_i, P] parameters of level ``levels[i]`` (default 0..L).
        All levels' operators are assembled up front.  On the SM-resident path
        (``fused``, default) every sequential solve of every level and the
        finest level's Parareal run in ONE persistent launch whose device-side
        scheduler advances each Parareal chain as soon as its inputs are ready
        (mlmcp_run_fused); otherwise the sequential solves go into one batched
        launch (longest first) and the Parareal runs concurrently on a
        high-priority second stream.  Returns device tensors (no host sync)."""
        import torch
        sol = self.solver
        levels = list(range(len(draws))) if levels is None else list(levels)
        top = len(self.hierarchy) - 1
        sizes = [len(d) for d in draws]
        if not _no_chunk and params_dev is None:
            # HBM budget, computed ONCE per call: each level's footprint per
            # sample differs (tasks per launch, Parareal buffers on the top
            # level), so the batch is chunked level by level with per-level caps
            caps = self.level_caps(levels, parareal_cfg)
            if caps is not None and sum(s / c for s, c in zip(sizes, caps)) > 1.0:
                return self._run_levels_chunked(draws, levels, parareal_cfg, caps,
                                                concurrent=concurrent, fused=fused)
        offs = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
        nnz = sol.nnz
        M = torch.empty((int(offs[-1]), nnz), dtype=torch.float64, device=sol.device)
        K = torch.empty_like(M)
        RP = self._new_rp(int(offs[-1]))

        def assemble_level(i):
            a, b = int(offs[i]), int(offs[i + 1])
            if b == a:
                return
            rp = RP[a:b] if RP is not None else None
            if params_dev is not None:
                self._assemble_dev(params_dev[a:b], M[a:b], K[a:b], rp=rp)   # resident in HBM
            else:
                d = draws[i].get() if hasattr(draws[i], "get") else draws[i]
                host = np.ascontiguousarray(np.asarray(d, dtype=float).reshape(b - a, -1))
                self._assemble_host(host, M[a:b], K[a:b], rp=rp)

        pr_level = None
        if parareal_cfg is not None:
            for i, lvl in enumerate(levels):
                if lvl == top and sizes[i] > 0:
                    pr_level = i
        if fused is None:
            fused = concurrent and sol.sys.sm_resident and not sol.sys.direct
        if fused:
            return self._run_levels_fused(levels, sizes, offs, M, K, assemble_level, pr_level,
                                          parareal_cfg)
        main = torch.cuda.current_stream()
        pr = None
        side = main
        if pr_level is not None:
            # the finest level's Parareal is the critical path: assemble and
            # launch it first (host draws of the other levels overlap with it)
            assemble_level(pr_level)
            cfg = parareal_cfg.with_dt_fine(self.hierarchy[levels[pr_level]].dt)
            a, b = offs[pr_level], offs[pr_level + 1]
            # Parareal gets the higher-priority stream so its CTAs are dispatched
            # ahead of the big sequential launch as SMs free up
            side = self._pr_stream(sol.device) if (concurrent and sol.sys.sm_resident) else main
            if side is not main:
                side.wait_stream(main)
            with torch.cuda.stream(side):
                pr = sol.run_parareal(M[a:b], K[a:b], 0.0, self.horizon, cfg.num_subintervals,
                                      cfg.dt_fine, cfg.dt_coarse, cfg.tolerance, cfg.k_max,
                                      stream=side, rp=RP[a:b] if RP is not None else None,
                                      **self._pr_qoi(cfg.dt_fine))
                pr_q = self._finish_q(pr.qoi, cfg.dt_fine)
        for i in range(len(levels)):
            if i != pr_level:
                assemble_level(i)
        jobs, where = self._level_jobs(levels, offs, pr_level)
        res = sol.run_sequential(M, K, jobs, rp=RP) if jobs else []
        if pr is not None and side is not main:
            main.wait_stream(side)
            for t in (pr.qoi, pr.k_used, pr.defects):
                t.record_stream(main)
        self._last = (res, pr, M, K)
        return self._collect(levels, sizes, where, res, pr_level, pr,
                             pr_q if pr is not None else None)

    def _level_jobs(self, levels, offs, pr_level):
        jobs, where = [], []
        for i, lvl in enumerate(levels):
            rows = np.arange(offs[i], offs[i + 1])
            if len(rows) == 0:
                continue
            dt = self.hierarchy[lvl].dt
            if i != pr_level:
                jobs.append(self._seq_job(rows, dt))
                where.append((i, "hi", dt))
            if lvl > 0:
                dtm = self.hierarchy[lvl - 1].dt
                jobs.append(self._seq_job(rows, dtm))
                where.append((i, "lo", dtm))
        return jobs, where

    def _collect(self, levels, sizes, where, res, pr_level, pr, pr_q):
        import torch
        sol = self.solver
        out = []
        for i, lvl in enumerate(levels):
            S = sizes[i]
            dev = sol.device
            ql = torch.zeros(S, dtype=torch.float64, device=dev)
            qm = torch.zeros(S, dtype=torch.float64, device=dev)
            ku = torch.zeros(S, dtype=torch.int32, device=dev)
            its = torch.zeros(S, dtype=torch.int64, device=dev)
            defects = None
            elapsed = []
            for (j, kind, dt), r in zip(where, res):
                if j != i:
                    continue
                if r.elapsed is not None:
                    elapsed.append(r.elapsed)
                q = self._finish_q(r.qoi, dt)
                if kind == "hi":
                    ql = q
                else:
                    qm = q
                its = its + r.iters.to(torch.int64)
            if i == pr_level:
                ql = pr_q
                ku = pr.k_used
                defects = pr.defects
                if pr.elapsed is not None:
                    elapsed.extend(pr.elapsed)
            out.append(CoupledBatch(lvl, ql, qm, ku, its, defects=defects, elapsed=elapsed))
        return out

    def _pr_ctas(self, jobs, pr_spec) -> int:
        """SM slots for the Parareal chains: the share of the resident CTA
        slots proportional to the Parareal batch's expected step work (K ~ 3)
        against the sequential batch's (MLMCP_PR_CTAS overrides)."""
        import os

        import torch
        env = os.environ.get("MLMCP_PR_CTAS")
        slots = 2 * torch.cuda.get_device_properties(self.solver.device).multi_processor_count
        if env:
            return max(1, min(int(env), slots))
        from .timeint import step_count
        w_seq = sum(len(j.rows) * j.n_steps for j in jobs)
        m = pr_spec["m"]
        k_est = min(3, pr_spec["k_max"])
        fine_steps = step_count(0.0, pr_spec["t1"], pr_spec["dt_fine"]) // m
        w_pr = pr_spec["S"] * sum(m - k + 1 for k in range(1, k_est + 1)) * fine_steps
        share = w_pr / max(1, w_pr + w_seq)
        return int(min(slots - 32, max(pr_spec["S"], round(slots * share))))

    def _run_levels_fused(self, levels, sizes, offs, M, K, assemble_level, pr_level,
                          parareal_cfg):
        """Every sequential solve and the finest level's Parareal in ONE
        persistent device-scheduled launch (mlmcp_run_fused): each Parareal
        chain step starts as soon as its own inputs are ready instead of
        waiting for SM slots held by long sequential tasks, and sequential
        tasks fill the rest.  MLMCP_FUSED=split: the sequential batch as its
        own launch and the Parareal as a persistent launch on a fixed share of
        the slots on a second stream (sensitive to which launch the hardware
        dispatches first)."""
        import os

        import torch
        sol = self.solver
        for i in range(len(levels)):
            assemble_level(i)
        jobs, where = self._level_jobs(levels, offs, pr_level)
        pr_spec = None
        cfg = None
        if pr_level is not None:
            cfg = parareal_cfg.with_dt_fine(self.hierarchy[levels[pr_level]].dt)
            pr_spec = dict(row0=int(offs[pr_level]), S=int(sizes[pr_level]), t0=0.0,
                           t1=self.horizon, m=cfg.num_subintervals, dt_fine=cfg.dt_fine,
                           dt_coarse=cfg.dt_coarse, tol=cfg.tolerance, k_max=cfg.k_max,
                           **self._pr_qoi(cfg.dt_fine))
        if pr_spec is None or os.environ.get("MLMCP_FUSED", "all") != "split":
            res, pr = sol.run_fused(M, K, jobs, pr_spec)
        else:
            main = torch.cuda.current_stream()
            side = self._pr_stream(sol.device)
            side.wait_stream(main)
            with torch.cuda.stream(side):
                _, pr = sol.run_fused(M, K, [], pr_spec, stream=side,
                                      grid_ctas=self._pr_ctas(jobs, pr_spec))
            res = sol.run_sequential(M, K, jobs) if jobs else []
            main.wait_stream(side)
            for t in (pr.qoi, pr.k_used, pr.defects):
                t.record_stream(main)
        pr_q = self._finish_q(pr.qoi, cfg.dt_fine) if pr is not None else None
        self._last = (res, pr, M, K)
        return self._collect(levels, sizes, where, res, pr_level, pr, pr_q)

    def level_caps(self, levels, parareal_cfg=None):
        """Per-level sample caps of one run_levels call (None: unbounded).
        Computed once per call from the reclaimable HBM; families without
        ``max_samples_per_call`` are unbounded."""
        cap_fn = getattr(self, "max_samples_per_call", None)
        if cap_fn is None:
            return None
        caps = [cap_fn(parareal_cfg, level=lvl) for lvl in levels]
        if any(c is None for c in caps):
            return None
        return [max(1, int(c)) for c in caps]

    def _run_levels_chunked(self, draws, levels, parareal_cfg, caps, concurrent: bool = True,
                            fused: bool | None = None):
        """run_levels over batches larger than HBM holds: each level in calls of
        <= caps[i] samples (per-sample results are bitwise independent of the
        batch), statuses checked per call, results concatenated."""
        import torch
        out = []
        for d, lvl, cap in zip(draws, levels, caps):
            d = d.get() if hasattr(d, "get") else d          # LazyDraw: materialise first
            parts = []
            for c0 in range(0, len(d), cap):
                parts.append(self.run_levels([d[c0:c0 + cap]], parareal_cfg, levels=[lvl],
                                             concurrent=concurrent, fused=fused,
                                             _no_chunk=True)[0])
                self.check_status()
            if not parts:
                parts.append(self.run_levels([d], parareal_cfg, levels=[lvl],
                                             concurrent=concurrent, fused=fused,
                                             _no_chunk=True)[0])

            def cat(xs):
                if all(isinstance(x, torch.Tensor) for x in xs):
                    return torch.cat(xs)
                if all(isinstance(x, np.ndarray) for x in xs):
                    return np.concatenate(xs)
                raise TypeError(f"cannot concatenate chunk results of types "
                                f"{sorted({type(x).__name__ for x in xs})}")

            out.append(CoupledBatch(
                level=lvl, q_l=cat([b.q_l for b in parts]), q_lm1=cat([b.q_lm1 for b in parts]),
                k_used=cat([b.k_used for b in parts]),
                iters=cat([b.iters for b in parts]) if parts[0].iters is not None else None,
                wall_s=sum(b.wall_s for b in parts),
                defects=cat([b.defects for b in parts]) if parts[0].defects is not None else None,
                elapsed=[e for b in parts for e in b.elapsed]))
        return out

    def run_levels_graphed(self, draws, parareal_cfg: PararealConfig | None = None,
                           params_dev=None):
        """run_levels through a captured CUDA graph: the whole launch sequence
        (assembly, steady states, the device-scheduled estimate launch,
        result collection) is captured once per (sample counts, Parareal
        config) and replayed, so a repeated estimate costs one host memcpy of
        the draws into a pinned staging buffer, one H2D copy and one graph
        launch instead of ~1 ms of host-side launch preparation.  Same results
        as run_levels (same kernels, same inputs).  Falls back to run_levels
        when the path is not graph-capturable (streaming / direct paths,
        MLMCP_GRAPHS=0)."""
        import os

        import torch

        from . import _lib
        sol = self.solver
        self._graph_launches = 0
        if (os.environ.get("MLMCP_GRAPHS", "1") == "0" or not sol.sys.sm_resident
                or sol.sys.direct or sol.timing):
            return self.run_levels(draws, parareal_cfg, params_dev=params_dev)
        rows = [np.asarray(d.get() if hasattr(d, "get") else d, dtype=np.float64) for d in draws]
        sizes = tuple(len(r) for r in rows)
        if sum(sizes) == 0:
            return self.run_levels(draws, parareal_cfg)
        host = None
        if params_dev is None:
            host = np.concatenate([r.reshape(len(r), -1) for r in rows if len(r)], axis=0)
        pkey = None if parareal_cfg is None else (parareal_cfg.num_subintervals,
                                                  parareal_cfg.dt_coarse, parareal_cfg.tolerance,
                                                  parareal_cfg.k_max)
        width = host.shape[1] if host is not None else int(params_dev.shape[1])
        key = (sizes, width, pkey, None if params_dev is None else params_dev.data_ptr())
        cache = self.__dict__.setdefault("_graphs", {})
        entry = cache.get(key)
        if entry is None:
            pinned = None
            if params_dev is None:
                static_in = torch.empty(host.shape, dtype=torch.float64, device=sol.device)
                pinned = torch.empty(host.shape, dtype=torch.float64, pin_memory=True)
                pinned.numpy()[:] = host
                static_in.copy_(pinned, non_blocking=True)
            else:
                static_in = params_dev
            self.run_levels(rows, parareal_cfg, params_dev=static_in, fused=True)   # warm caches
            torch.cuda.synchronize()
            g = torch.cuda.CUDAGraph()
            l0 = _lib.launch_count()
            with torch.cuda.graph(g):
                out = self.run_levels(rows, parareal_cfg, params_dev=static_in, fused=True)
            n_launch = _lib.launch_count() - l0          # libmlmcp kernels per replay
            entry = (g, static_in, pinned, out, self._last, n_launch)
            cache[key] = entry
        g, static_in, pinned, out, last, n_launch = entry
        if pinned is not None:
            pinned.numpy()[:] = host        # previous replay finished (its results were read)
            static_in.copy_(pinned, non_blocking=True)
        g.replay()
        self._last = last
        self._graph_launches = n_launch
        return out

    def status_flag(self, token=None):
        """0-d device tensor: any failed task in the last run, or in the run
        ``token`` (take_last) stands for (no host sync)."""
        import torch
        last = token if token is not None else getattr(self, "_last", None)
        if last is None:
            return None
        res, pr, _, _ = last
        sts = [r.status for r in res]
        if pr is not None:
            sts += [pr.status, pr.fine_status]
        sts = [st for st in sts if st.numel()]
        if not sts:
            return None
        return torch.stack([(st[:, 0] != 0).any() for st in sts]).any()

    def check_status(self, token=None):
        """Raise SingularSystemError / PropagatorError for failed samples of the
        last run (or of the run ``token`` stands for)."""
        from .parareal import raise_parareal_status
        from .solver import raise_on_status
        last = token if token is not None else getattr(self, "_last", None)
        if last is None:
            return
        res, pr, _, _ = last
        for r in res:
            raise_on_status(r.status, "implicit Euler solve")
        if pr is not None:
            raise_parareal_status(pr.status.cpu().numpy(), pr.fine_status.cpu().numpy())

    def take_last(self):
        """Detach the last run's statuses and operator buffers as a token for
        status_flag / check_status, so that the next run_levels call can be
        issued before this one has been checked (mlmc.run_level_calls)."""
        tok = getattr(self, "_last", None)
        self._last = None
        return tok

    def call_streams(self, parareal_cfg=None):
        """CUDA streams on which run_levels calls may be in flight together
        (mlmc.run_level_calls), or None when calls run one after the other."""
        return None

    def coupled_batch(self, params, level, parareal_cfg=None) -> CoupledBatch:
        lvl = self._level_index(level)
        return self.run_levels([np.asarray(params, dtype=float)], parareal_cfg, levels=[lvl])[0]

    def evaluate_batch(self, params, level: LevelSpec, parareal_cfg=None) -> list[EvalRecord]:
        """Q at one level for a batch of samples (no coupling)."""
        import torch
        lvl = self._level_index(level)
        params = np.asarray(params, dtype=float).reshape(-1, self._n_params())
        sol = self.solver
        t = time.perf_counter()
        M = torch.empty((len(params), sol.nnz), dtype=torch.float64, device=sol.device)
        K = torch.empty_like(M)
        RP = self._new_rp(len(params))
        self._assemble_host(params, M, K, rp=RP)
        top = len(self.hierarchy) - 1
        dt = self.hierarchy[lvl].dt
        ks = None
        if parareal_cfg is not None:
            cfg = parareal_cfg.with_dt_fine(dt)
            pr = sol.run_parareal(M, K, 0.0, self.horizon, cfg.num_subintervals, cfg.dt_fine,
                                  cfg.dt_coarse, cfg.tolerance, cfg.k_max, rp=RP,
                                  **self._pr_qoi(cfg.dt_fine))
            from .parareal import raise_parareal_status
            raise_parareal_status(pr.status.cpu().numpy(), pr.fine_status.cpu().numpy())
            q = self._finish_q(pr.qoi, cfg.dt_fine).cpu().numpy()
            ks = pr.k_used.cpu().numpy()
        else:
            from .solver import raise_on_status
            r = sol.run_sequential(M, K, [self._seq_job(np.arange(len(params)), dt)], rp=RP)[0]
            raise_on_status(r.status, "implicit Euler solve")
            q = self._finish_q(r.qoi, dt).cpu().numpy()
        wall = time.perf_counter() - t
        del top
        cost = wall / max(1, len(params))
        return [EvalRecord(float(q[i]), cost, None if ks is None else int(ks[i]))
                for i in range(len(params))]

    def evaluate(self, params: ParameterVector, level: LevelSpec, parareal_cfg=None,
                 pool=None) -> EvalRecord:
        """models.py:389-411 (``pool`` accepted and ignored)."""
        vals = params.values if isinstance(params, ParameterVector) else np.asarray(params)
        return self.evaluate_batch(np.asarray(vals, dtype=float)[None, :], level, parareal_cfg)[0]


@dataclass
class EddyCurrentFamily(_BatchedFamily):
    """2D linear eddy-current P1 FE family; one sample = one transient solve.

    ``evaluate`` follows MachineFamily.evaluate (models.py:389-411): a
    Parareal configuration switches the solve to Parareal with
    ``parareal_cfg.with_dt_fine(level.dt)``; the QoI is evaluated from the
    device-resident solution.  Batched entry points run many samples in one
    launch.
    """

    model_id: str
    uncertain: object
    hierarchy: tuple
    horizon: float
    n: int
    layout: str
    qoi: QoIKind = QoIKind.MAGNETIC_ENERGY_T
    avg_window: float = 0.0
    device: object = None
    rtol: float = 1e-13
    max_it: int = 20000
    path: str = "auto"
    _solver: object = field(default=None, repr=False, compare=False)

    # ------------------------------------------------------------ setup
    @property
    def solver(self):
        if self._solver is None:
            from .solver import FESolver
            self._solver = FESolver(self.n, self.layout, self.device, self.rtol, self.max_it,
                                    self.path)
            self._solver.periods = self.horizon * self._solver.omega / (2.0 * np.pi)
        return self._solver

    def _seq_job(self, rows, dt):
        from . import _lib
        from .solver import SeqJob
        from .timeint import step_count
        n = step_count(0.0, self.horizon, dt)
        if self.qoi is QoIKind.MAGNETIC_ENERGY_T:
            return SeqJob(rows, dt, n, _lib.QOI_FINAL_ENERGY, 0)
        if self.qoi is QoIKind.TIME_AVG_MAGNETIC_ENERGY:
            n_w = int(round(self.avg_window / dt))
            return SeqJob(rows, dt, n, _lib.QOI_SUM_ENERGY, n - n_w)
        raise ValueError(f"QoI kind {self.qoi} is not defined for the FE family")

    def _finish_q(self, acc, dt):
        if self.qoi is QoIKind.TIME_AVG_MAGNETIC_ENERGY:
            return acc * dt / self.avg_window
        return acc

    def max_samples_per_call(self, parareal_cfg=None, level=None):
        """Samples of ``level`` one run_levels call may hold on this GPU: None
        on the SM-resident path (a config-1 estimate needs ~0.2 GB); on the
        streaming path (128^2..512^2) half of the reclaimable HBM divided by
        that level's per-sample footprint, so full-size configs 2-4 run as a
        sequence of calls.  The footprint counts what the level's launches
        hold per sample: the M/K values, the per-task workspace of ONE
        propagate launch (one task per sample and dt; m fine tasks per sample
        on the Parareal level) and the states of every task (2 per sample
        above level 0; U, F, C, D on the Parareal level), plus the steady states
        of the predictor.  ``level`` None: the most demanding sequential level."""
        import torch
        sol = self.solver
        if sol.sys.sm_resident:
            return None
        lib, ctx = sol.sys.lib, sol.sys.ctx
        ws = lambda tasks, S: int(lib.mlmcp_workspace_bytes(ctx, tasks, S))
        per_task = ws(2, 1) - ws(1, 1)
        per_op = ws(2, 2) - ws(2, 1)
        N8 = 8 * sol.N
        top = len(self.hierarchy) - 1
        lvl = 1 if level is None else int(level)
        if parareal_cfg is not None and lvl == top:
            m = parareal_cfg.num_subintervals
            # U, F, C and the increments D of the correction fine solves
            tasks, states, ss = m, (4 * m + 3) * N8, 2
        else:
            tasks, states, ss = 1, (2 if lvl > 0 else 1) * N8, (2 if lvl > 0 else 1)
        per = 16 * sol.nnz + per_op + tasks * per_task + states
        if sol.use_predictor():
            per += ss * (int(lib.mlmcp_periodic_workspace_bytes(ctx, 2))
                         - int(lib.mlmcp_periodic_workspace_bytes(ctx, 1)) + 2 * N8)
        free, _ = torch.cuda.mem_get_info(sol.device)
        # memory torch's caching allocator holds but no tensor uses, and the
        # engine workspace (replaced, not added, by the next call) are free too
        reclaim = torch.cuda.memory_reserved(sol.device) - torch.cuda.memory_allocated(sol.device)
        cur_ws = sol.sys.workspace_bytes_held()
        avail = free + max(0, reclaim) + cur_ws
        return max(1, int(0.5 * avail // max(per, 1)))

    def call_streams(self, parareal_cfg=None):
        """Two streams for the band path (region-linear grids up to 256^2
        without Parareal: config 2).  A band launch is one asynchronous kernel
        that holds 112 of the 148 SMs (seven 16-CTA clusters, one per GPC that
        has 16 SMs), so the next call's assembly and periodic steady-state
        solves (grid-wide streaming kernels, host-synchronised on their own
        stream) run on the idle SMs meanwhile, and its band clusters take over
        cluster slots as the previous launch's last tasks drain.
        MLMCP_PIPELINE=0 keeps one call at a time."""
        import os

        import torch

        from . import _lib
        sol = self.solver
        if (os.environ.get("MLMCP_PIPELINE", "1") == "0" or parareal_cfg is not None
                or sol.sys.sm_resident or not getattr(sol, "region_mode", False)):
            return None
        if sol.sys.propagate_path(16, 16, sol.use_predictor(), True) != _lib.PATH_BAND:
            return None
        st = getattr(self, "_call_streams", None)
        if st is None:
            _, hi = torch.cuda.Stream.priority_range()
            st = [torch.cuda.Stream(device=sol.device, priority=hi) for _ in range(2)]
            self._call_streams = st
            sol.sys.band_low_priority = True
        return st

    def _n_params(self) -> int:
        return fe.n_params(self.layout)

    def _assemble_host(self, params, M, K, rp=None):
        import torch
        p = torch.from_numpy(np.ascontiguousarray(params, dtype=np.float64)).pin_memory()
        self.solver.assemble(p.to(self.solver.device, non_blocking=True), out=(M, K), rp_out=rp)

    def _assemble_dev(self, params_dev, M, K, rp=None):
        self.solver.assemble(params_dev, out=(M, K), rp_out=rp)


def eddy_current_family(config: int | str, device=None, **kw) -> EddyCurrentFamily:
    """The family of one BASELINE.json config (see configs.py)."""
    from .configs import get_config
    c = get_config(config)
    if c.layout == "kl64":
        unc = GaussianInput("kl64", fe.KL_MODES)
    else:
        nominal = np.array([fe.NU0] * (fe.n_params(c.layout) // 2)
                           + [fe.SIGMA0] * (fe.n_params(c.layout) // 2))
        unc = UncertainInput(ParameterVector(c.layout, nominal), c.halfwidth)
    qoi = QoIKind.TIME_AVG_MAGNETIC_ENERGY if c.qoi == "time_avg_energy" else QoIKind.MAGNETIC_ENERGY_T
    return EddyCurrentFamily(model_id=c.layout, uncertain=unc, hierarchy=make_hierarchy(c.dts),
                             horizon=c.horizon, n=c.n, layout=c.layout, qoi=qoi,
                             avg_window=c.avg_window, device=device, **kw)
