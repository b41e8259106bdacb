"""MLMC estimator over the temporal level hierarchy (the
reference ships no ``mlmc`` module — ``models.py:308,315`` refers to it).

  ``RandomStream``        SPEC.md:250-254: generator = pure function of
                          (seed, level, index) via SeedSequence spawn keys
  ``LevelStats``          SPEC.md:256-260 (mean = sum_Y/N,
                          var = (sum_Y2 - N mean^2)/(N-1))
  ``EstimatorResult``     SPEC.md:262-266 (expectation = sum_l mean_Y)
  ``coupled_sample``      SPEC.md:280-288 (Q_{-1} = 0; Parareal only on the
                          finest level, the coarser solve stays sequential)
  ``mc_estimate``
  ``optimal_allocation``  SPEC.md:290-298 (rmse split eps^2/2; N_l >= 2)
  ``mlmc_estimate``       SPEC.md:300-314 with a fixed-N policy (the BASELINE
                          configs) or a warm-up + allocation policy

Batched device path: for a family with ``run_levels`` (EddyCurrentFamily)
every level's samples run in one batched launch; each rank of a
``torch.distributed`` group takes a contiguous slice of every level's sample
indices (keys stay (seed, l, k) with k the global index), fills
its slots of a per-sample buffer [N_l, 4] = (Q_l, Q_{l-1}, K, PCG iters),
one all-reduce(SUM) per level combines the buffers (exactly one non-zero
contributor per slot, so the sum is exact), and the K7 kernel reduces in
fixed sample order — the estimate is bitwise independent of the GPU count
(SPEC.md:313).
"""

from __future__ import annotations

import math
import time
from dataclasses import dataclass, field

import numpy as np

from .models import EvalRecord, LevelSpec, draw_parameters

__all__ = ["RandomStream", "LevelStats", "EstimatorResult", "FixedSamples", "WarmupPolicy",
           "coupled_sample", "mc_estimate", "optimal_allocation", "mlmc_estimate",
           "draw_level", "draw_level_device", "shard_range", "LazyDraw", "estimate_dict",
           "write_estimate_json"]


class RandomStream:
    def __init__(self, master_seed: int, level: int, index: int):
        self.master_seed = int(master_seed)
        self.level = int(level)
        self.index = int(index)

    def generator(self) -> np.random.Generator:
        return np.random.default_rng(
            np.random.SeedSequence(self.master_seed, spawn_key=(self.level, self.index)))


@dataclass
class LevelStats:
    level: int
    n: int
    sum_y: float
    sum_y2: float
    cost_per_sample: float = 0.0
    parareal_k: list | None = None

    @property
    def mean_y(self) -> float:
        return self.sum_y / self.n if self.n else 0.0

    @property
    def var_y(self) -> float:
        if self.n < 2:
            return 0.0
        return (self.sum_y2 - self.n * self.mean_y ** 2) / (self.n - 1)


@dataclass
class EstimatorResult:
    expectation: float
    per_level: list
    rmse_estimate: float
    ledger: dict = field(default_factory=dict)


@dataclass(frozen=True)
class FixedSamples:
    """SPEC.md:527 'fixed N per level' policy."""

    n_per_level: tuple


@dataclass(frozen=True)
class WarmupPolicy:
    n_warmup: int = 20
    rmse: float | None = None
    budget: float | None = None


def shard_range(n: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous slice [a, b) of 0..n-1 owned by ``rank``."""
    base, rem = divmod(n, world)
    a = rank * base + min(rank, rem)
    return a, a + base + (1 if rank < rem else 0)


def draw_level(uncertain, seed: int, level: int, indices) -> np.ndarray:
    """Host draws for sample keys (seed, level, k), k in ``indices`` (1-based).

    Row k equals ``draw_parameters(uncertain, RandomStream(seed, level, k)).values``
    bitwise (same generator, same call, same arithmetic, models.py:305-318).
    Uniform inputs run through libmlmcp's native restatement of SeedSequence /
    PCG64 / ``uniform`` (``mlmcp_draw_uniform_host``, ~300x faster than one
    numpy Generator per sample; tests/test_draws.py pins it to numpy); the
    per-sample ParameterVector validation is done once on the whole block."""
    from .models import GaussianInput, ParameterVector
    idx = [int(k) for k in indices]
    if isinstance(uncertain, GaussianInput):
        out = np.empty((len(idx), uncertain.dim))
        for i, k in enumerate(idx):
            out[i] = RandomStream(seed, level, k).generator().standard_normal(uncertain.dim)
        return out
    nominal = uncertain.nominal.values
    h = uncertain.relative_halfwidth
    out = np.empty((len(idx), len(nominal)))
    if h == 0.0:
        out[:] = nominal
        return out
    lo = nominal * (1.0 - h)
    hi = nominal * (1.0 + h)
    if len(idx) and idx == list(range(idx[0], idx[0] + len(idx))) and min(seed, level, idx[0]) >= 0:
        _draw_uniform_host(int(seed), int(level), idx[0], lo, hi - lo, out)
    else:
        for i, k in enumerate(idx):
            out[i] = RandomStream(seed, level, k).generator().uniform(lo, hi)
    if len(idx) and not np.all(out > 0.0):
        ParameterVector(uncertain.nominal.model_id, out[np.argmin(out.min(axis=1))])  # raises
    return out


def _draw_uniform_host(seed: int, level: int, k_first: int, lo, rng, out):
    from . import _lib
    lo = np.ascontiguousarray(lo, dtype=np.float64)
    rng = np.ascontiguousarray(rng, dtype=np.float64)
    _lib.check(_lib.load().mlmcp_draw_uniform_host(seed, level, k_first, out.shape[0],
                                                   out.shape[1], _lib.np_ptr(lo),
                                                   _lib.np_ptr(rng), _lib.np_ptr(out)),
               "mlmcp_draw_uniform_host")


def draw_level_device(uncertain, seed: int, level: int, k_first: int, n: int, out):
    """Device draws (``mlmcp_draw_uniform``) of keys (seed, level, k_first..)
    into the [n, P] float64 CUDA tensor ``out`` — bitwise equal to
    ``draw_level``; uniform inputs only."""
    import torch

    from . import _lib
    from .engine import stream_handle
    nominal = uncertain.nominal.values
    h = uncertain.relative_halfwidth
    if h == 0.0:
        out.copy_(torch.from_numpy(np.broadcast_to(nominal, (n, len(nominal))).copy()))
        return out
    lo = nominal * (1.0 - h)
    rng = nominal * (1.0 + h) - lo
    lr = torch.from_numpy(np.stack([lo, rng])).to(out.device)
    _lib.check(_lib.load().mlmcp_draw_uniform(int(seed), int(level), int(k_first), int(n),
                                              len(nominal), _lib.ptr(lr[0]), _lib.ptr(lr[1]),
                                              _lib.ptr(out), stream_handle()),
               "mlmcp_draw_uniform")
    return out


class LazyDraw:
    """Level draws evaluated on first use (``len`` is known up front), so a
    batched family can launch the finest level before the host draws the
    rest (host RNG overlaps device work)."""

    def __init__(self, n: int, fn):
        self.n = int(n)
        self._fn = fn
        self._v = None

    def __len__(self):
        return self.n

    def get(self) -> np.ndarray:
        if self._v is None:
            self._v = self._fn()
        return self._v


def coupled_sample(family, params, level: LevelSpec, hierarchy, parareal_cfg=None):
    """SPEC.md:280-288 through the per-sample family API."""
    top = hierarchy[-1].level
    hi = family.evaluate(params, level, parareal_cfg if (parareal_cfg is not None and
                                                         level.level == top) else None)
    if level.level == 0:
        return hi.q, 0.0, (hi.cost_s, 0.0), hi.parareal_iterations
    lo = family.evaluate(params, hierarchy[level.level - 1])
    return hi.q, lo.q, (hi.cost_s, lo.cost_s), hi.parareal_iterations


def mc_estimate(family, level: LevelSpec, n: int, seed: int) -> EstimatorResult:
    if n < 2:
        raise ValueError("need N >= 2")
    qs = []
    for k in range(1, n + 1):
        p = draw_parameters(family.uncertain, RandomStream(seed, level.level, k))
        qs.append(family.evaluate(p, level).q)
    st = LevelStats(level.level, n, float(np.sum(qs)), float(np.sum(np.square(qs))))
    return EstimatorResult(st.mean_y, [st], math.sqrt(max(st.var_y, 0.0) / n))


def optimal_allocation(V, C, rmse: float | None = None, budget: float | None = None):
    V = np.asarray(V, dtype=float)
    C = np.asarray(C, dtype=float)
    if np.any(V < 0) or np.any(C <= 0):
        raise ValueError("need V >= 0 and C > 0")
    if np.all(V == 0):
        return [2] * len(V)
    w = np.sqrt(V / C)
    if rmse is not None:
        if rmse <= 0:
            raise ValueError("rmse must be > 0")
        n = np.ceil(2.0 / rmse ** 2 * w * np.sum(np.sqrt(V * C)))
    elif budget is not None:
        if budget <= 0:
            raise ValueError("budget must be > 0")
        n = np.floor(budget * w / np.sum(w * C))
    else:
        raise ValueError("need an rmse or a budget target")
    return [int(max(2, x)) for x in n]


def _dist():
    try:
        import torch.distributed as dist
        if dist.is_available() and dist.is_initialized():
            return dist
    except Exception:
        pass
    return None


def torch_device_type(device) -> str:
    import torch
    return torch.device(device).type


def _fill_slots(slots, batch, a: int, b: int):
    import torch
    dev = slots.device
    if b > a:
        slots[a:b, 0] = batch.q_l.to(dev, torch.float64)
        slots[a:b, 1] = batch.q_lm1.to(dev, torch.float64)
        slots[a:b, 2] = batch.k_used.to(dev, torch.float64)
        if batch.iters is not None:
            slots[a:b, 3] = batch.iters.to(dev, torch.float64)


def _family_caps(family, n_levels: int, parareal_cfg):
    """Per-level sample caps of one run_levels call (None: one call)."""
    if hasattr(family, "level_caps"):
        return family.level_caps(list(range(n_levels)), parareal_cfg)
    fn = getattr(family, "max_samples_per_call", None)
    if fn is None:
        return None
    caps = [fn(parareal_cfg, level=lvl) for lvl in range(n_levels)]
    return None if any(c is None for c in caps) else [max(1, int(c)) for c in caps]


def plan_calls(ranges, caps, pipelined: bool = False):
    """The run_levels calls of one estimate as (level, c0, c1) sample ranges.
    One call at a time: level by level in chunks of <= caps[l].  Pipelined (two
    calls in flight, family.call_streams): each call may hold 0.8 of its cap
    (the caps budget half of the free HBM per call), a level's chunks are
    balanced, and the finest level goes first — its few long tasks start
    early and the later calls' short tasks fill the cluster slots they leave.
    Per-sample results do not depend on the plan."""
    calls = []
    for lvl, (a, b) in enumerate(ranges):
        if b <= a:
            continue
        cap = max(1, int(caps[lvl] * 0.8)) if pipelined else caps[lvl]
        if pipelined:
            n = -(-(b - a) // cap)
            size = -(-(b - a) // n)
        else:
            size = cap
        calls += [(lvl, c0, min(b, c0 + size)) for c0 in range(a, b, size)]
    if pipelined:
        calls.sort(key=lambda c: -c[0])
    return calls


def run_level_calls(family, calls, launch, parareal_cfg=None, on_token=None):
    """Issue ``launch(lvl, c0, c1)`` for every planned call.  With
    family.call_streams() the calls alternate between two streams so that one
    call's host-synchronised preparation (assembly, periodic steady states)
    overlaps the previous call's asynchronous propagate launch; a stream's
    previous call is completed (synchronised, statuses checked or handed to
    ``on_token``) before the stream is reused, so at most two calls hold
    memory.  ``launch`` runs under the call's stream and must leave its
    results in buffers the caller reduces after this function returns (the
    current stream waits for both streams at the end)."""
    streams = None
    if len(calls) > 1 and hasattr(family, "call_streams"):
        streams = family.call_streams(parareal_cfg)

    def done(tok):
        if tok is None:
            return
        if on_token is not None:
            on_token(tok)
        else:
            family.check_status(tok)

    if not streams:
        for c in calls:
            launch(*c)
            if on_token is not None and hasattr(family, "take_last"):
                on_token(family.take_last())
            elif hasattr(family, "check_status"):
                family.check_status()
        return
    import torch
    main = torch.cuda.current_stream()
    inflight = [None] * len(streams)
    try:
        for i, c in enumerate(calls):
            k = i % len(streams)
            s = streams[k]
            if inflight[k] is not None:
                s.synchronize()
                tok, inflight[k] = inflight[k], None
                done(tok)
                del tok
            s.wait_stream(main)
            with torch.cuda.stream(s):
                launch(*c)
                inflight[k] = family.take_last()
        for k, s in enumerate(streams):
            if inflight[k] is not None:
                s.synchronize()
                tok, inflight[k] = inflight[k], None
                done(tok)
                del tok
    finally:
        for s in streams:
            main.wait_stream(s)


def _run_chunked(family, ranges, counts, caps, seed: int, parareal_cfg, dev):
    """Evaluate the rank's sample ranges in run_levels calls of <= caps[l]
    samples (keys unchanged) into per-level slot buffers.  The caps are
    computed once by the caller (no per-call re-sizing); the calls follow
    plan_calls / run_level_calls (two in flight where the family allows)."""
    import torch
    slots = [torch.zeros((n, 4), dtype=torch.float64, device=dev) for n in counts]
    pipelined = bool(hasattr(family, "call_streams") and family.call_streams(parareal_cfg))
    last = [None]

    def launch(lvl, c0, c1):
        d = draw_level(family.uncertain, seed, lvl, range(c0 + 1, c1 + 1))
        out = family.run_levels([d], parareal_cfg, levels=[lvl], _no_chunk=True)
        _fill_slots(slots[lvl], out[0], c0, c1)
        last[0] = out

    run_level_calls(family, plan_calls(ranges, caps, pipelined), launch, parareal_cfg)
    return slots, last[0]


def _level_costs(hierarchy, counts, parareal_cfg, ks, wall: float):
    """Per-level cost per sample C_l (measured per level during
    the warm-up): the batched call's wall time split by each level's solver
    work — N_l (1/dt_l + 1/dt_{l-1}) time steps, the Parareal level's fine
    steps counted with its redundancy sum_{k<=K} (M - k + 1) / M at the mean K
    used (parareal.py:182-196) plus one coarse step per slice and iteration."""
    top = len(hierarchy) - 1
    work = []
    for lvl, n in enumerate(counts):
        hi = 1.0 / hierarchy[lvl].dt
        if parareal_cfg is not None and lvl == top:
            m = parareal_cfg.num_subintervals
            kbar = float(np.mean(ks)) if ks is not None and len(ks) else float(parareal_cfg.k_max)
            kk = max(1, int(round(kbar)))
            hi = hi * sum(m - k + 1 for k in range(1, kk + 1)) / m + kk * m
        lo = 1.0 / hierarchy[lvl - 1].dt if lvl > 0 else 0.0
        work.append(n * (hi + lo))
    tot = sum(work)
    return [(wall * w / tot / n) if (n and tot > 0) else 0.0 for w, n in zip(work, counts)]


def _reduce_slots(slots, dist, device):
    """all-reduce of a filled slot buffer, then the fixed-order reduction."""
    import torch
    if dist is not None and dist.get_world_size() > 1:
        dist.all_reduce(slots, op=dist.ReduceOp.SUM)
    if slots.device.type == "cuda":
        from .engine import level_reduce
        return level_reduce(slots[:, 0].contiguous(), slots[:, 1].contiguous())
    # CPU families (tests) — same fixed order as the kernel's definition
    y = (slots[:, 0] - slots[:, 1]).numpy()
    return torch.tensor([float(np.sum(y)), float(np.sum(y * y)), 0.0, 0.0], dtype=torch.float64)


def _reduce_level(batch, n_global: int, a: int, b: int, dist, device):
    """Slot buffer -> all-reduce -> fixed-order K7 reduction."""
    import torch
    on_gpu = device is not None and torch.device(device).type == "cuda"
    slots = torch.zeros((n_global, 4), dtype=torch.float64, device=device if on_gpu else "cpu")
    _fill_slots(slots, batch, a, b)
    return slots, _reduce_slots(slots, dist, device)


def mlmc_estimate(family, hierarchy=None, policy=None, parareal_cfg=None, seed: int = 0,
                  device=None, draws=None, csv_path: str | None = None,
                  timing: bool = False) -> EstimatorResult:
    """SPEC.md:300-314.  ``policy``: FixedSamples (all levels at once) or
    WarmupPolicy (warm-up, optimal allocation, then the remainder).
    ``timing``: record per-task device time and attach the executor ledger
    (executor.gpu_ledger) as ``result.ledger["executor"]``."""
    hierarchy = tuple(hierarchy or family.hierarchy)
    dist = _dist()
    rank = dist.get_rank() if dist else 0
    world = dist.get_world_size() if dist else 1
    if policy is None:
        raise ValueError("need a sampling policy")
    if isinstance(policy, WarmupPolicy):
        return _mlmc_warmup(family, hierarchy, policy, parareal_cfg, seed, device, timing)
    counts = list(policy.n_per_level)
    if len(counts) != len(hierarchy):
        raise ValueError("one sample count per level is required")
    t_start = time.perf_counter()
    ranges = [shard_range(n, rank, world) for n in counts]
    if draws is None:
        draws = [LazyDraw(b - a, (lambda lvl=lvl, a=a, b=b: draw_level(
            family.uncertain, seed, lvl, range(a + 1, b + 1))))
            for lvl, (a, b) in enumerate(ranges)]
    dev = device
    if dev is None and hasattr(family, "solver"):
        dev = family.solver.device
    sol = None
    caps = _family_caps(family, len(hierarchy), parareal_cfg)
    if caps is not None and sum((b - a) / c for (a, b), c in zip(ranges, caps)) > 1.0:
        # full-size streaming configs: the rank's samples in calls of <= cap_l
        # samples, filling the per-sample slot buffers (same keys, same result)
        all_slots, batches = _run_chunked(family, ranges, counts, caps, seed, parareal_cfg, dev)
        sums_dev = [_reduce_slots(slots, dist, dev) for slots in all_slots]
    else:
        sol = getattr(family, "solver", None) if timing else None
        if sol is not None:
            sol.timing = True
        try:
            if hasattr(family, "run_levels_graphed"):
                batches = family.run_levels_graphed(draws, parareal_cfg)
            else:
                batches = family.run_levels(draws, parareal_cfg)
        finally:
            if sol is not None:
                sol.timing = False
        all_slots, sums_dev = [], []
        for lvl, (batch, (a, b)) in enumerate(zip(batches, ranges)):
            slots, sums = _reduce_level(batch, counts[lvl], a, b, dist, dev)
            all_slots.append(slots)
            sums_dev.append(sums)
    per_level = []
    top = len(hierarchy) - 1
    want_k = parareal_cfg is not None
    flag = family.status_flag() if hasattr(family, "status_flag") else None
    if dev is not None and torch_device_type(dev) == "cuda":
        # one device->host read for the level sums, the Parareal K slots and the
        # failure flag (the detailed status check only runs when a task failed)
        import torch
        parts = [s.to(torch.float64) for s in sums_dev]
        if want_k:
            parts.append(all_slots[top][:, 2])
        if flag is not None:
            parts.append(flag.to(torch.float64).reshape(1))
        pack = torch.cat([p.reshape(-1) for p in parts]).cpu().numpy()
        if flag is not None and pack[-1] != 0.0:
            family.check_status()
        host = [pack[4 * i:4 * i + 4] for i in range(len(sums_dev))]
        ks_host = pack[4 * len(sums_dev):4 * len(sums_dev) + counts[top]] if want_k else None
    else:
        if hasattr(family, "check_status"):
            family.check_status()
        host = [s.cpu().numpy() for s in sums_dev]
        ks_host = all_slots[top][:, 2].cpu().numpy() if want_k else None
    wall = time.perf_counter() - t_start
    costs = _level_costs(hierarchy, counts, parareal_cfg,
                         ks_host if want_k else None, wall)
    for lvl, sums in enumerate(host):
        ks = None
        if want_k and lvl == top:
            ks = ks_host.astype(int).tolist()
        per_level.append(LevelStats(lvl, counts[lvl], float(sums[0]), float(sums[1]),
                                    costs[lvl], ks))
    expectation = float(sum(st.mean_y for st in per_level))
    rmse = math.sqrt(sum(max(st.var_y, 0.0) / st.n for st in per_level if st.n > 0))
    ledger = {"wall_time_s": wall, "world_size": world,
              "samples": counts, "mode": "gpu-batched"}
    if sol is not None:
        from .executor import gpu_ledger
        ledger["executor"] = gpu_ledger(batches, wall, dist).to_dict()
    if csv_path and rank == 0:
        _write_csv(csv_path, all_slots, per_level)
    return EstimatorResult(expectation, per_level, rmse, ledger)


def _write_csv(path, all_slots, per_level):
    """SPEC.md:326 per-sample records: level,index,Q_l,Q_lm1,cost_s,parareal_K."""
    with open(path, "w") as fh:
        fh.write("level,index,Q_l,Q_lm1,cost_s,parareal_K\n")
        for lvl, slots in enumerate(all_slots):
            s = slots.cpu().numpy()
            for k in range(len(s)):
                fh.write(f"{lvl},{k + 1},{s[k, 0]!r},{s[k, 1]!r},"
                         f"{per_level[lvl].cost_per_sample!r},{int(s[k, 2])}\n")


def _mlmc_warmup(family, hierarchy, policy: WarmupPolicy, parareal_cfg, seed, device,
                 timing=False):
    n_w = max(2, policy.n_warmup)
    warm = mlmc_estimate(family, hierarchy, FixedSamples((n_w,) * len(hierarchy)), parareal_cfg,
                         seed, device)
    V = [st.var_y for st in warm.per_level]
    C = [max(st.cost_per_sample, 1e-12) for st in warm.per_level]
    target = optimal_allocation(V, C, rmse=policy.rmse, budget=policy.budget)
    counts = tuple(max(n_w, t) for t in target)
    res = mlmc_estimate(family, hierarchy, FixedSamples(counts), parareal_cfg, seed, device,
                        timing=timing)
    res.ledger["warmup"] = [n_w] * len(hierarchy)
    res.ledger["allocation"] = list(counts)
    return res


def evaluate_records(family, params, level, parareal_cfg=None) -> list[EvalRecord]:
    return family.evaluate_batch(params, level, parareal_cfg)


def estimate_dict(res: EstimatorResult) -> dict:
    """estimate.json content (SPEC.md cmd_estimate: expectation, rmse, per-level
    stats); deterministic for a fixed seed (no timings)."""
    return {"expectation": res.expectation, "rmse_estimate": res.rmse_estimate,
            "levels": [{"level": st.level, "n": st.n, "sum_y": st.sum_y, "sum_y2": st.sum_y2,
                        "mean_y": st.mean_y, "var_y": st.var_y,
                        "parareal_k": st.parareal_k} for st in res.per_level]}


def write_estimate_json(path: str, res: EstimatorResult):
    import json
    with open(path, "w") as fh:
        json.dump(estimate_dict(res), fh, indent=1, sort_keys=True)

