"""Benchmark: one 'step' = one complete MLMC+Parareal estimate of BASELINE.json
config 1 (32x32 P1 eddy-current mesh, 3 levels dt = T/256, T/512, T/1024,
N_l = 512, 128, 32 per GPU, finest level by Parareal M=16 / K<=5 / tol 1e-8),
i.e. every coupled implicit-Euler solve of every sample plus the level
reductions.

  value  sequential-equivalent sample-timesteps/s, sum_l N_l (n_l + n_{l-1})
         over all ranks / device time per estimate (params resident in HBM,
         CUDA events on the launching stream, max over ranks, L2 flushed
         between steps)
  e2e    the same metric through the public API ``mlmc.mlmc_estimate`` from
         host draws (RandomStream keys), pinned H2D of the parameters, D2H of
         the level statistics / statuses, wall clock around each call
  --impl reference   the CPU oracle port of the reference path (dense LU as
         shipped, timeint.py:64-75) on all host cores, bounded sample

Multi-GPU (torchrun): weak scaling — every rank owns N_l samples per level
(global keys), one NCCL all-reduce per level on the per-sample slot buffer.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

# the CPU legs run one dense-LU solve per process: one BLAS thread each
# (more threads make the per-step solve slower) — set before numpy loads
os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
os.environ.setdefault("OMP_NUM_THREADS", "1")

import numpy as np  # noqa: E402

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "sample-timesteps/s (batched FE implicit-Euler solves); MLMC+Parareal wall time"
UNIT = "sample-timesteps/s"
FALLBACK_HBM = 6650.0


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="mlmcp", choices=["mlmcp", "reference"])
    ap.add_argument("--config", type=int, default=1)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true", help="skip the e2e leg (profiling runs)")
    ap.add_argument("--no-streaming", action="store_true",
                    help="skip the HBM-streaming roofline legs (configs 2 and 4)")
    ap.add_argument("--cpu-seconds", type=float, default=6.0,
                    help="target wall seconds of the bounded CPU-baseline sample")
    return ap.parse_args()


# ---------------------------------------------------------------- CPU side
_PROB = {}


def _cpu_init():
    try:
        from threadpoolctl import threadpool_limits
        threadpool_limits(1)
    except Exception:
        pass


def _cpu_task(args):
    """One coupled sample through the oracle (reference algorithm, dense LU)."""
    from oracle import mlmc_oracle as mo
    cfg_i, level, k, seed = args
    cfg = mo.CONFIGS[cfg_i]
    key = (cfg.n, cfg.layout)
    if key not in _PROB:
        _PROB[key] = mo.FEProblem(cfg.n, cfg.layout)
    p = mo.draw(cfg, seed, level, k)
    return mo.coupled(_PROB[key], cfg, level, p)


def cpu_sample_counts(cfg, cores: int, target_s: float):
    """Per-level sample counts of a bounded, proportional subset of the job."""
    # single-core dense-LU cost model of the reference path at 32^2:
    # ~0.73 ms per step, Parareal sample ~4.7 s at config 1
    per_step = 0.73e-3
    full = 0.0
    for lvl, n in enumerate(cfg.samples):
        steps = cfg.steps(lvl) + (cfg.steps(lvl - 1) if lvl > 0 else 0)
        if cfg.parareal is not None and lvl == cfg.levels - 1:
            # ~K=3 iterations of fine slices + one dense LU per propagator call
            steps = 7 * cfg.steps(lvl) + (cfg.steps(lvl - 1) if lvl > 0 else 0)
        full += n * steps * per_step
    frac = min(1.0, cores * target_s / full)
    return [max(1, int(math.ceil(n * frac))) for n in cfg.samples]


def run_cpu_subset(cfg_i: int, counts, seed: int, cores: int):
    from concurrent.futures import ProcessPoolExecutor
    from paper_2507_19246_b200.configs import get_config
    cfg = get_config(cfg_i)
    jobs = [(cfg_i, lvl, k, seed) for lvl in reversed(range(cfg.levels))
            for k in range(1, counts[lvl] + 1)]          # longest (Parareal) first
    steps = sum(counts[lvl] * (cfg.steps(lvl) + (cfg.steps(lvl - 1) if lvl > 0 else 0))
                for lvl in range(cfg.levels))
    with ProcessPoolExecutor(max_workers=cores, initializer=_cpu_init) as pool:
        list(pool.map(_cpu_task, [(cfg_i, 0, 1, seed + 99)] * cores))   # warm the workers
        t = time.perf_counter()
        list(pool.map(_cpu_task, jobs, chunksize=1))
        wall = time.perf_counter() - t
    return steps, wall


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def workload_name(cfg_i, cfg, counts, pcfg):
    """The workload string both arms report (config.workload)."""
    par = ("Parareal M=%d K<=%d tol=%g" % (pcfg.num_subintervals, pcfg.k_max, pcfg.tolerance)
           if pcfg else "no Parareal")
    return (f"cfg{cfg_i}: {cfg.n}x{cfg.n} P1 eddy-current, levels "
            f"dt=T/{round(cfg.horizon / cfg.dts[0])}..T/{round(cfg.horizon / cfg.dts[-1])}, "
            f"N_l={list(counts)} ({par}), full MLMC estimate per step")


def reference_arm(args):
    """--impl reference: the reference algorithm (oracle port; the reference is
    pure Python and cannot travel) on all host cores."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    os.environ["OPENBLAS_NUM_THREADS"] = "1"
    from paper_2507_19246_b200.configs import get_config
    cfg = get_config(args.config)
    cores = os.cpu_count() or 1
    counts = cpu_sample_counts(cfg, cores, 2.0)
    for w in range(args.warmup):
        run_cpu_subset(args.config, counts, 1000 + w, cores)
    times, steps_done = [], 0
    for s in range(args.steps):
        st, wall = run_cpu_subset(args.config, counts, s, cores)
        times.append(wall)
        steps_done = st
    ms = 1000.0 * float(np.mean(times))
    value = steps_done / (ms / 1000.0)
    sample = (f"per step: config-{args.config} subset N_l={counts} (global keys 1..N_l, "
              f"seed varies per step), {steps_done} seq-equivalent sample-timesteps, "
              f"dense LU as shipped, ProcessPool x{cores}, OPENBLAS_NUM_THREADS=1, CPU {cpu_model()}")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": workload_name(args.config, cfg, [n * args.gpus for n in cfg.samples],
                                                 cfg.parareal_config()),
                       "seq_equiv_sample_timesteps": cfg.seq_equiv_steps(args.gpus),
                       "sampled_per_step": f"N_l={counts} of it (bounded CPU sample, rate extrapolated)",
                       "parallelism": f"{cores} host processes"},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "port",
                             "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------- clocks
class ClockSampler:
    def __init__(self):
        self.proc = None
        self.lines = []

    def start(self):
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={q}", "--format=csv,noheader",
                                          "-lms", "100"], stdout=subprocess.PIPE,
                                         stderr=subprocess.DEVNULL, text=True)
            self.th = threading.Thread(target=self._read, daemon=True)
            self.th.start()
        except OSError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self, gpu_index: int):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9 or not f[0].isdigit() or int(f[0]) != gpu_index:
                continue
            try:
                sm.append(float(f[1].split()[0]))
                mx = float(f[2].split()[0])
            except ValueError:
                continue
            for name, val in zip(names, f[5:9]):
                if val.lower().startswith("active"):
                    reasons.add(name)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------- GPU arm
def measured_peak():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return float(json.load(fh)["hbm_gbs"]), "measured"
    except Exception:
        return FALLBACK_HBM, "fallback"


def ncu_sm_internal():
    """SM-internal utilisation of the top kernel from the committed ncu capture
    (the bound of the SM-resident config-1 kernel: fp64 pipe / issue slots)."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_top_kernel.json")) as fh:
            src = json.load(fh).get("source")
        with open(os.path.join(ROOT, src)) as fh:
            d = json.load(fh)
        d = d["kernels"][0] if "kernels" in d else d
        f = lambda k: float(d[k]["value"]) / 100.0
        return {"fp64_pipe_active": f("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"),
                "issue_active": f("smsp__issue_active.avg.pct_of_peak_sustained_active"),
                "source": src}
    except Exception:
        return None


def ncu_traffic():
    """dram bytes per launch of the top kernel from the committed ncu capture."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_top_kernel.json")) as fh:
            d = json.load(fh)
        return d.get("dram_bytes_per_launch")
    except Exception:
        return None


def streaming_roofline(dev, peak, flush):
    """HBM roofline of the streaming path (meshes > 1024 rows, where the batch's
    working set is far larger than L2): one level-0 batch of config 2 (256^2)
    and of config 4 (512^2).  achieved = PCG iterations x B_it / device time of
    the PCG-iteration launches (CUDA events on their stream, inside the
    library); call_achieved the same over the whole propagate call."""
    import torch

    from paper_2507_19246_b200.mlmc import draw_level
    from paper_2507_19246_b200.models import eddy_current_family
    out = []
    for cfg_i, S, steps in ((2, 512, 8), (4, 128, 4)):
        fam = eddy_current_family(cfg_i, device=dev)
        sol = fam.solver
        sol.predictor = False   # the PCG kernels alone (no steady-state COCG solves)
        p = draw_level(fam.uncertain, 0, 0, range(1, S + 1))
        M, K = sol.assemble(torch.from_numpy(p).to(dev))
        job = fam._seq_job(np.arange(S), fam.hierarchy[0].dt)
        job.n_steps = steps
        times = []
        for r in range(3):
            flush.zero_()
            if r == 1:
                sol.sys.stream_timing(1)    # events around the PCG-iteration launches
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            res = sol.run_sequential(M, K, [job])[0]
            e1.record()
            torch.cuda.synchronize()
            if r:
                times.append(e0.elapsed_time(e1) / 1000.0)
        it_ms, it_launches = sol.sys.stream_timing(0)
        its = int(res.iters.to(torch.int64).sum().item())
        b_it = 8 * sol.mesh.nnz + 56 * sol.N
        t = float(np.mean(times))
        ach = its * b_it / (it_ms / 2 / 1000.0) / 1e9     # 2 timed calls
        call = its * b_it / t / 1e9
        out.append({"workload": f"cfg{cfg_i} level-0 batch: {S} samples x {steps} implicit-Euler "
                                f"steps, {sol.n}x{sol.n} mesh (N={sol.N})",
                    "kernel": "tile_iter_kernel<16,4,3> (one fused launch per PCG iteration)",
                    "achieved": ach, "peak": peak, "unit": "GB/s", "frac": ach / peak,
                    "kernel_ms": it_ms / 2, "launches": it_launches // 2,
                    "pcg_iterations": its, "call_ms": 1000 * t, "call_achieved": call,
                    "call_frac": call / peak,
                    "algorithmic_bytes": f"{its} PCG iterations x (8 nnz + 56 N) = {its} x {b_it} B",
                    "note": "achieved / frac: the iteration kernel's launches (CUDA events on its "
                            "stream, mlmcp_stream_timing); call_*: the whole propagate call "
                            "(step starts, guesses, QoI included)"})
        del M, K, res, sol, fam
        torch.cuda.empty_cache()
    return out


def main():
    args = parse()
    if args.impl == "reference":
        reference_arm(args)
        return
    import torch
    import torch.distributed as dist

    from paper_2507_19246_b200 import _lib
    from paper_2507_19246_b200.configs import get_config
    from paper_2507_19246_b200.engine import level_reduce
    from paper_2507_19246_b200.mlmc import FixedSamples, draw_level, mlmc_estimate, shard_range
    from paper_2507_19246_b200.models import eddy_current_family

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    cfg = get_config(args.config)
    pcfg = cfg.parareal_config()
    counts = [n * world for n in cfg.samples]                 # weak scaling
    ranges = [shard_range(n, rank, world) for n in counts]
    fam = eddy_current_family(args.config, device=dev)
    draws = [draw_level(fam.uncertain, cfg.seed, lvl, range(a + 1, b + 1))
             for lvl, (a, b) in enumerate(ranges)]
    params_dev = torch.from_numpy(np.concatenate(draws, axis=0)).to(dev)
    sol = fam.solver
    N = sol.N
    nnz = sol.mesh.nnz
    b_it = 8 * nnz + 56 * N                                   # SURVEY §8(d) bytes / PCG iteration
    flush = torch.empty(512 * 1024 * 1024, dtype=torch.uint8, device=dev)   # > 126 MB L2

    graph_launches = [0]

    def one_step(rec, graphed=True):
        # the estimate's launch sequence replays as a captured CUDA graph
        # (libmlmcp kernels counted at capture: graph_launches)
        if graphed:
            batches = fam.run_levels_graphed(draws, pcfg, params_dev=params_dev)
            graph_launches[0] += fam._graph_launches
        else:
            batches = fam.run_levels(draws, pcfg, params_dev=params_dev)
        sums = []
        for lvl, (b, (a, e)) in enumerate(zip(batches, ranges)):
            slots = torch.zeros((counts[lvl], 4), dtype=torch.float64, device=dev)
            slots[a:e, 0] = b.q_l
            slots[a:e, 1] = b.q_lm1
            slots[a:e, 2] = b.k_used.to(torch.float64)
            if world > 1:
                dist.all_reduce(slots)
            sums.append(level_reduce(slots[:, 0].contiguous(), slots[:, 1].contiguous()))
        if rec is not None:
            rec.append(batches)
        return sums

    for _ in range(args.warmup):
        one_step(None)
    torch.cuda.synchronize()
    fam.check_status()
    seq_start = torch.cuda.Event(enable_timing=True)
    seq_end = torch.cuda.Event(enable_timing=True)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    seq_ms, batches_rec = [], []
    graph_launches[0] = 0
    clocks = ClockSampler()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clocks.start()
    l0 = _lib.launch_count()
    wall0 = time.perf_counter()
    for s in range(args.steps):
        flush.zero_()                                         # L2 flush, outside the events
        ev[s][0].record()
        one_step(batches_rec)
        ev[s][1].record()
        torch.cuda.synchronize()
    torch.cuda.synchronize()
    wall = time.perf_counter() - wall0
    launches = (_lib.launch_count() - l0 + graph_launches[0]) // max(1, args.steps)
    if world > 1:
        dist.barrier()
    clk = clocks.stop(local)
    fam.check_status()
    # roofline: the estimate launch timed with events on its stream (eager runs,
    # same work as a replay)
    sol.events = (seq_start, seq_end)
    for _ in range(3):
        flush.zero_()
        one_step(None, graphed=False)
        torch.cuda.synchronize()
        seq_ms.append(seq_start.elapsed_time(seq_end))
    sol.events = None
    step_ms = [a.elapsed_time(b) for a, b in ev]
    ms_local = float(np.mean(step_ms))
    ms = torch.tensor([ms_local], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    ms = float(ms.item())
    total_steps = cfg.seq_equiv_steps(world)
    value = total_steps / (ms / 1000.0)

    # roofline of the dominant kernel (SM-resident batched IE/PCG launch)
    its = 0
    for batches in batches_rec[-1:]:
        res = sol._last_xbuf  # noqa: F841  (keeps the last launch's buffers alive)
    res_seq = fam._last[0]
    its = int(sum(int(r.iters.to(torch.int64).sum().item()) for r in res_seq))
    pr = fam._last[1]
    pr_fine_its = int(pr.fine_iters.to(torch.int64).sum().item()) if pr is not None else 0
    pr_coarse_its = int(pr.coarse_iters.to(torch.int64).sum().item()) if pr is not None else 0
    k_used = pr.k_used.cpu().numpy().tolist() if pr is not None else []
    seq_kernel_ms = float(np.mean(seq_ms))
    # default: the timed launch runs the sequential solves AND the Parareal batch
    # (device-scheduled); MLMCP_FUSED=split: the events bracket the sequential
    # launch only (the Parareal runs in its own launch on a second stream)
    fused = bool(sol.sys.sm_resident and not sol.sys.direct
                 and os.environ.get("MLMCP_FUSED", "all") != "split")
    kern_its = its + (pr_fine_its + pr_coarse_its if fused else 0)
    achieved = kern_its * b_it / (seq_kernel_ms / 1000.0) / 1e9
    peak, peak_kind = measured_peak()

    # e2e through the public API (host draws, H2D, all kernels, D2H)
    e2e_times = []
    if world > 1:
        dist.barrier()
    for s in range(0 if args.no_e2e else max(2, args.steps // 2) + 1):
        torch.cuda.synchronize()
        t = time.perf_counter()
        res = mlmc_estimate(fam, policy=FixedSamples(tuple(counts)), parareal_cfg=pcfg,
                            seed=cfg.seed)
        torch.cuda.synchronize()
        if s > 0:                                             # first call = warm-up
            e2e_times.append(time.perf_counter() - t)
    e2e_s = torch.tensor([float(np.mean(e2e_times)) if e2e_times else float("nan")],
                         dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(e2e_s, op=dist.ReduceOp.MAX)
    e2e_s = float(e2e_s.item())
    n_local = sum(b - a for a, b in ranges)
    h2d = n_local * draws[0].shape[1] * 8                     # pinned parameter upload
    n_pr = (ranges[-1][1] - ranges[-1][0]) if pcfg is not None else 0
    n_seq = sum((b - a) * ((0 if (pcfg is not None and lvl == cfg.levels - 1) else 1) + (lvl > 0))
                for lvl, (a, b) in enumerate(ranges))
    m_sl = pcfg.num_subintervals if pcfg is not None else 0
    # level sums + per-task status rows (16 B) + Parareal K slots read back by the API
    d2h = 32 * cfg.levels + 16 * (n_seq + n_pr + n_pr * m_sl) + (8 * counts[-1] if pcfg else 0)

    out = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
           "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
           "vs_baseline": None, "dtype": "f64", "data": "synthetic",
           "config": {"workload": workload_name(args.config, cfg, counts, pcfg),
                      "seq_equiv_sample_timesteps": total_steps, "mlmc_parareal_wall_ms": ms,
                      "pcg_rtol": sol.step_rtol(), "predictor": sol.use_predictor(), "parareal_k": sorted(set(k_used)),
                      "l2": "flushed between steps (512 MiB write)", "parallelism": f"samples x{world}"},
           "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                        "frac": achieved / peak, "traffic": ncu_traffic(),
                        "kernel": ("fused_kernel<GridOp,2> (every sequential solve of every level + the "
                                   "finest level's Parareal, one persistent launch)" if fused else
                                   "small_propagate_kernel<GridOp,2> (all sequential solves of all "
                                   "levels, one launch; the Parareal runs concurrently in a "
                                   "persistent device-scheduled launch)"),
                        "algorithmic_bytes": f"{kern_its} PCG iterations x (8 nnz + 56 N) = {kern_its} x {b_it} B",
                        "kernel_ms": seq_kernel_ms, "peak_kind": peak_kind,
                        "sm_internal": ncu_sm_internal(),
                        "note": "32x32 operators live in registers/SMEM (SM-resident CTA per task): "
                                "frac > 1 means the kernel runs faster than streaming its algorithmic "
                                "bytes from HBM would allow; ncu dram bytes are the actual traffic"},
           "e2e": {"value": total_steps / e2e_s, "unit": UNIT, "h2d_bytes_per_step": int(h2d),
                   "d2h_bytes_per_step": int(d2h), "wall_ms": 1000 * e2e_s,
                   "api": "paper_2507_19246_b200.mlmc.mlmc_estimate (host RandomStream draws)"},
           "gpu_launches": int(launches),
           "clocks": clk,
           "detail": {"pcg_iterations_sequential": its, "pcg_iterations_parareal_fine": pr_fine_its,
                      "pcg_iterations_parareal_coarse": pr_coarse_its,
                      "host_wall_ms_per_step": 1000 * wall / args.steps}}
    if rank == 0 and not args.no_streaming:
        out["roofline"]["streaming"] = streaming_roofline(dev, peak, flush)
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        os.environ["OPENBLAS_NUM_THREADS"] = "1"
        cores = os.cpu_count() or 1
        cc = cpu_sample_counts(cfg, cores, args.cpu_seconds)
        st, w = run_cpu_subset(args.config, cc, cfg.seed, cores)
        out["cpu_baseline"] = {"value": st / w, "unit": UNIT, "cores": cores, "kind": "port",
                               "sample": f"config-{args.config} subset N_l={cc} (keys 1..N_l), "
                                         f"{st} seq-equivalent sample-timesteps in {w:.2f} s; oracle "
                                         f"port of the reference (dense LU as shipped), "
                                         f"ProcessPool x{cores}, CPU {cpu_model()}"}
    if rank == 0:
        print(json.dumps(out), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
