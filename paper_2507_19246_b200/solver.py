"""Batched FE transient solves on one GPU: operator assembly per sample,
sequential implicit-Euler jobs and on-device Parareal.

This is the batched replacement of the per-sample work under
``MachineFamily.evaluate`` (models.py:389-411):
  * ``assemble``       builders + ``mass + dt*stiffness`` (models.py:217-302,
                       timeint.py:65) -> per-sample CSR values (K1)
  * ``run_sequential`` implicit_euler_solve (timeint.py:88-111) for many
                       (sample, dt) jobs in ONE launch (longest job first)
  * ``run_parareal``   parareal_solve (parareal.py:121-220) for a batch of
                       samples: K_max rounds of [coarse sweep, all fine
                       slices of all samples, jump defect], convergence
                       masks on the device, one host sync at the end.
All per-sample results are bitwise independent of the batch composition.
"""

from __future__ import annotations

import os
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib, fe
from ._lib import ptr
from .engine import DeviceSystem, F64, I32, kl_sigma, new_tasks, region_params, tasks_to_device
from .timeint import SingularSystemError, step_count

DEFAULT_RTOL = 1e-13   # ||r||_2 <= 1e-13 ||b||_2, the stated PCG tolerance
# With the steady-state predictor PCG starts so close to the solution that the
# stopping residual is dominated by smooth (small-eigenvalue) components, whose
# error is up to kappa * rtol; 1e-14 keeps the per-step state error at the
# 1e-13 warm-start level for < 1 extra iteration per step.
PREDICTOR_RTOL = 1e-14
# COCG tolerance of the periodic steady states: they only feed initial guesses.
# Streaming meshes (config-2 estimate): 1e-8 -> 1e-6 costs 1% more PCG
# iterations and saves 30% of the COCG iterations (1e-5 costs 9%); on the
# SM-resident path (configs 0/1, least-squares guesses at rtol 1e-14) 1e-6
# costs 26% of the config-1 estimate, so 1e-8 stays there.
SS_RTOL_STREAMING = 1e-6
SS_RTOL_RESIDENT = 1e-8
DEFAULT_MAX_IT = 20000


@dataclass
class SeqJob:
    """n_steps implicit-Euler steps of dt from the zero state for M/K rows
    ``rows``; QoI 'energy_T' (1/2 a(T)^T K a(T)) or ('sum', from_step)."""

    rows: np.ndarray
    dt: float
    n_steps: int
    qoi_mode: int = _lib.QOI_FINAL_ENERGY
    qoi_from: int = 0
    qoi_index: int = 0


@dataclass
class SeqResult:
    qoi: torch.Tensor       # (len(rows),) device
    iters: torch.Tensor     # (len(rows),) device, PCG iterations
    status: torch.Tensor    # (len(rows), 4) device
    elapsed: torch.Tensor | None = None   # (len(rows),) int64 device ns (timing on)


@dataclass
class PararealBatchResult:
    qoi: torch.Tensor           # (S,) energy of the final fine state
    k_used: torch.Tensor        # (S,) int32
    defects: torch.Tensor       # (S, k_max) NaN beyond k_used
    status: torch.Tensor        # (S, 4) coarse failures: code, step, interval, iteration
    fine_status: torch.Tensor   # (S*m, 4) fine failures
    U: torch.Tensor             # (S, m+1, N) boundary states (after finalize)
    F: torch.Tensor             # (S, m+1, N) fine end states
    traj: torch.Tensor | None   # (S, m, steps+1, N) last fine solve of each slice
    fine_iters: torch.Tensor
    coarse_iters: torch.Tensor
    elapsed: tuple | None = None  # (coarse [S], fine [S*m]) int64 device ns (timing on)


def parareal_grid(t0: float, t1: float, m: int, dt_fine: float, dt_coarse: float):
    """parareal.py:133-150: boundaries on the fine grid and per-slice
    (k0, n_steps) of the fine and coarse propagators (origin t0)."""
    nf = step_count(t0, t1, dt_fine)
    nc = step_count(t0, t1, dt_coarse)
    if nf % m != 0 or nc % m != 0:
        raise ValueError(
            f"[{t0}, {t1}] with M={m} sub-intervals is incompatible with dt_fine={dt_fine} "
            f"({nf} steps) and dt_coarse={dt_coarse} ({nc} steps)")
    m_f = nf // m
    bounds = t0 + (np.arange(m + 1) * m_f) * dt_fine
    fk0 = np.array([int(round((bounds[n - 1] - t0) / dt_fine)) for n in range(1, m + 1)], dtype=np.int64)
    fst = np.array([step_count(bounds[n - 1], bounds[n], dt_fine) for n in range(1, m + 1)], dtype=np.int32)
    ck0 = np.array([int(round((bounds[n - 1] - t0) / dt_coarse)) for n in range(1, m + 1)], dtype=np.int64)
    cst = np.array([step_count(bounds[n - 1], bounds[n], dt_coarse) for n in range(1, m + 1)], dtype=np.int32)
    return bounds, fk0, fst, ck0, cst


class BatchSolver:
    """Batched sequential / Parareal solves of one sparsity pattern on one GPU.

    Subclasses supply the per-sample operator values (FESolver assembles them
    on the device; SystemSolver uploads them from host builders)."""

    def __init__(self, row_ptr, col, profile, frequency: float, device=None,
                 rtol: float = DEFAULT_RTOL, max_it: int = DEFAULT_MAX_IT, path: str = "auto",
                 assembly=None):
        self.rtol = float(rtol)
        self.max_it = int(max_it)
        self.sys = DeviceSystem(row_ptr, col, device, assembly=assembly)
        if path != "auto":
            self.sys.set_path(path)
        dev = self.sys.device
        self.device = dev
        self.N = self.sys.n_rows
        self.nnz = self.sys.nnz
        self.profile = torch.tensor(np.asarray(profile, dtype=np.float64), dtype=F64, device=dev)
        self._task_cache: dict = {}
        self.events = None    # optional (start, end) CUDA events around the sequential launch
        self.timing = False   # True: launches record per-task device ns (executor ledger)
        # periodic steady-state initial-guess predictor (SM-resident path);
        # MLMCP_PREDICTOR=0 disables it (A/B measurements)
        self.predictor = os.environ.get("MLMCP_PREDICTOR", "1") != "0"
        self.omega = 2.0 * np.pi * frequency       # same rounding as np.sin(2.0*np.pi*f*t)
        self.periods = 1.0    # forcing periods in the family's horizon (set by the family)

    # ------------------------------------------------------------ sequential
    def run_sequential(self, M, K, jobs: list[SeqJob], stream=None, keep_traj: bool = False,
                       rp=None):
        """``rp``: [S, R, 2] region parameters of the M/K rows (region-linear
        operator on the streaming tile path; None streams the operator)."""
        return _run_sequential(self, M, K, jobs, stream, keep_traj, rp)

    def run_fused(self, M, K, jobs: list[SeqJob], pr=None, stream=None, grid_ctas: int = 0):
        return _run_fused(self, M, K, jobs, pr, stream, grid_ctas)

    def run_parareal(self, M, K, t0: float, t1: float, m: int, dt_fine: float,
                     dt_coarse: float, tol: float, k_max: int, stream=None,
                     keep_traj: bool = False, qoi_mode: int | None = None,
                     qoi_index: int = 0, qoi_from: int = -1, rp=None) -> PararealBatchResult:
        """qoi_mode None / QOI_FINAL_ENERGY: 1/2 a(T)^T K a(T); otherwise the
        task QoI accumulated over the fine trajectory (global fine steps g >
        qoi_from), summed over slices."""
        return _run_parareal(self, M, K, t0, t1, m, dt_fine, dt_coarse, tol, k_max, stream,
                             keep_traj, qoi_mode, qoi_index, qoi_from, rp)

    def use_predictor(self) -> bool:
        """The steady-state predictor pays where the forced periodic response
        dominates the step-to-step change — the sigma = 0 (quasi-static) regions
        of configs 0/1 (PCG iterations per step 29.7 -> 11.4; estimate 37.1 ->
        15.6 ms), and on the streaming meshes once the horizon spans several
        periods, so that the initial transient has decayed in the later ones
        (config 2, 4 periods: 42.5 -> 32.8 s per estimate).  Over a single
        period (configs 3, 4) the solution is the transient itself: measured no
        gain (config 3: 14.1 vs 14.2 iterations per step), and on grids up to
        128^2 the predictor would move the batch off the cluster kernel.
        MLMCP_PREDICTOR=all forces it on, =0 off."""
        if not self.predictor or self.sys.direct or self.omega == 0.0:
            return False
        if self.sys.sm_resident or os.environ.get("MLMCP_PREDICTOR") == "all":
            return True
        return self.periods >= 2.0 and self.N > 127 * 127

    def step_rtol(self) -> float:
        return min(self.rtol, PREDICTOR_RTOL) if self.use_predictor() else self.rtol

    def steady_states(self, samples: np.ndarray, dts: np.ndarray, M, K, stream=None, rp=None):
        """X [n, 2, N] for (sample, dt) pairs (mlmcp_periodic_state)."""
        key = ("ss", samples.tobytes(), dts.tobytes())
        v = self._task_cache.get(key)
        if v is None:
            v = (torch.tensor(samples.astype(np.int32), device=self.device),
                 torch.tensor(dts.astype(np.float64), device=self.device))
            self._task_cache[key] = v
        return self.sys.periodic_state(v[0], v[1], M, K, self.profile, self.omega,
                                       rtol=float(os.environ.get(
                                           "MLMCP_SS_RTOL", SS_RTOL_RESIDENT if self.sys.sm_resident
                                           else SS_RTOL_STREAMING)),
                                       stream=stream, rp=rp)

    def _grid_tensors(self, ck0, cst):
        key = ("grid", ck0.tobytes(), cst.tobytes())
        v = self._task_cache.get(key)
        if v is None:
            v = (torch.tensor(ck0, device=self.device), torch.tensor(cst, device=self.device))
            self._task_cache[key] = v
        return v


class SystemSolver(BatchSolver):
    """A small linear model family M da/dt + K a = sin(2 pi f t) profile with
    per-sample M/K values built on the host (the reference's own builders,
    models.py:217-302) on one shared CSR pattern."""

    def values(self, M_vals, K_vals):
        """Upload [S, nnz] host value arrays (pinned, asynchronous)."""
        Mh = np.ascontiguousarray(M_vals, dtype=np.float64).reshape(-1, self.nnz)
        Kh = np.ascontiguousarray(K_vals, dtype=np.float64).reshape(-1, self.nnz)
        if Mh.shape != Kh.shape:
            raise ValueError(f"M/K value arrays differ in shape: {Mh.shape} vs {Kh.shape}")
        M = torch.from_numpy(Mh).pin_memory().to(self.device, non_blocking=True)
        K = torch.from_numpy(Kh).pin_memory().to(self.device, non_blocking=True)
        return M, K


class FESolver(BatchSolver):
    """One structured P1 mesh + material layout on one GPU (K1 assembly on the
    device)."""

    def __init__(self, n: int, layout: str, device=None, rtol: float = DEFAULT_RTOL,
                 max_it: int = DEFAULT_MAX_IT, path: str = "auto"):
        if layout not in fe.LAYOUTS:
            raise ValueError(f"unknown layout {layout!r}")
        self.n = n
        self.layout = layout
        self.mesh = fe.structured_mesh(n)
        m = self.mesh
        super().__init__(m.row_ptr, m.col, fe.source_profile(m, layout), fe.FREQ, device, rtol,
                         max_it, path, assembly=(m.n_elem, m.cptr, m.celem, m.cmw, m.ckw))
        dev = self.device
        if layout == "kl64":
            self.kl_basis = torch.tensor(fe.kl_basis(m), dtype=F64, device=dev)
            self.nu_const = torch.full((1,), fe.NU0, dtype=F64, device=dev)
            self.nu_index = torch.zeros(m.n_elem, dtype=I32, device=dev)
        else:
            region = fe.region_map(m, layout)
            self.region = torch.tensor(region, dtype=I32, device=dev)
            self.mask = torch.tensor(fe.conducting_mask(layout), dtype=F64, device=dev)
            self.n_regions = len(fe.conducting_mask(layout))
            # region-linear operator of the streaming tile kernels (structured
            # grids; the operator is computed from the per-sample region
            # parameters instead of streamed: 112 -> 80 B/point per PCG iteration)
            if not self.sys.sm_resident and os.environ.get("MLMCP_TILE_OPERATOR") != "stored":
                rg = fe.region_grid(m, region, self.n_regions)
                if rg is not None:
                    try:
                        self.sys.set_region_grid(rg)
                    except ValueError:       # no 2D grid view of the pattern (no tile path)
                        self.sys.region_grid = None

    @property
    def region_mode(self) -> bool:
        return self.sys.region_grid is not None

    def new_region_params(self, S: int):
        """[S, R, 2] buffer for assemble(rp_out=...) (None without a region grid)."""
        if not self.region_mode:
            return None
        return torch.empty((S, self.n_regions, 2), dtype=F64, device=self.device)

    # ------------------------------------------------------------ K1
    def assemble(self, params: torch.Tensor, stream=None, out=None, rp_out=None):
        """Per-sample CSR values (M, K) [S, nnz] from parameters [S, P]
        (written into ``out`` = (M, K) slices when given; ``rp_out`` [S, R, 2]
        receives the region parameters of the region-linear operator)."""
        params = params.to(device=self.device, dtype=F64).contiguous()
        S = params.shape[0]
        if S == 0:
            empty = torch.empty((0, self.mesh.nnz), dtype=F64, device=self.device)
            return (empty, empty.clone()) if out is None else out
        if params.shape[1] != fe.n_params(self.layout):
            raise ValueError(f"layout {self.layout} takes {fe.n_params(self.layout)} parameters, "
                             f"got {params.shape[1]}")
        if self.layout == "kl64":
            sigma = kl_sigma(params, self.kl_basis, float(np.log(fe.SIGMA0)), fe.KL_SCALE, stream)
            return self.sys.assemble(S, sigma, self.mesh.n_elem, None, self.nu_const, 0,
                                     self.nu_index, stream, out)
        R = self.n_regions
        # sigma masked to 0 in non-conducting regions *after* drawing (ParameterVector
        # positivity, models.py:69-74), and the (sigma, nu) pairs of the
        # region-linear operator, in one libmlmcp launch
        sigma = torch.empty((S, R), dtype=F64, device=self.device)
        region_params(params, R, self.mask, sigma, rp_out, stream)
        return self.sys.assemble(S, sigma, R, self.region, params, 2 * R, self.region, stream, out)




# ------------------------------------------------------------ sequential
def _seq_setup(self, M, K, jobs: list[SeqJob], stream=None, keep_traj: bool = False, rp=None):
    """Task table (longest first), buffers and predictor states of a batch of
    sequential jobs."""
    from types import SimpleNamespace
    sizes = [len(j.rows) for j in jobs]
    T = int(sum(sizes))
    N = self.N
    tasks = new_tasks(T)
    off = 0
    for j in jobs:
        sl = slice(off, off + len(j.rows))
        tasks["sample"][sl] = j.rows
        tasks["n_steps"][sl] = j.n_steps
        tasks["k0"][sl] = 0
        tasks["dt"][sl] = j.dt
        tasks["t_base"][sl] = 0.0
        tasks["qoi_mode"][sl] = j.qoi_mode
        tasks["qoi_from"][sl] = j.qoi_from
        tasks["qoi_index"][sl] = j.qoi_index
        off += len(j.rows)
    idx = np.arange(T)
    tasks["x_in"] = idx * N
    tasks["x_out"] = idx * N
    tasks["qoi_slot"] = idx
    tasks["slot"] = idx
    if keep_traj:
        steps = tasks["n_steps"].astype(np.int64)
        base = T * N
        tstart = base + np.concatenate([[0], np.cumsum((steps + 1) * N)[:-1]])
        tasks["traj"] = tstart
        xbuf = torch.zeros(int(base + np.sum((steps + 1) * N)), dtype=F64, device=self.device)
    else:
        xbuf = torch.zeros(T * N, dtype=F64, device=self.device)
    st = SimpleNamespace(jobs=jobs, T=T, tasks=tasks, xbuf=xbuf, xss=None, td=None,
                         qoi=torch.zeros(T, dtype=F64, device=self.device),
                         iters=torch.zeros(T, dtype=I32, device=self.device),
                         status=torch.zeros((T, _lib.STATUS_INTS), dtype=I32, device=self.device),
                         elapsed=(torch.zeros(T, dtype=torch.int64, device=self.device)
                                  if self.timing else None))
    if T and self.use_predictor():
        tasks["ss_slot"] = idx
        st.xss = self.steady_states(tasks["sample"], tasks["dt"], M, K, stream, rp=rp)
    if self.sys.sm_resident and T:
        order = np.argsort(-tasks["n_steps"], kind="stable")   # longest first
        key = (tasks.tobytes(), N)
        td = self._task_cache.get(key)
        if td is None:
            td = tasks_to_device(tasks[order], self.device)
            self._task_cache[key] = td
        st.td = td
        st.order = order
    return st


def _seq_results(self, st):
    out = []
    off = 0
    for j in st.jobs:
        sl = slice(off, off + len(j.rows))
        out.append(SeqResult(st.qoi[sl], st.iters[sl], st.status[sl],
                             None if st.elapsed is None else st.elapsed[sl]))
        off += len(j.rows)
    self._last_xbuf = st.xbuf
    self._last_tasks = st.tasks
    return out


def _run_sequential(self, M, K, jobs: list[SeqJob], stream=None, keep_traj: bool = False,
                    rp=None):
    """All jobs in one batched launch (SM-resident path) or one launch per
    dt (streaming path).  Returns one SeqResult per job (device tensors)."""
    st = _seq_setup(self, M, K, jobs, stream, keep_traj, rp=rp)
    if st.T == 0:
        return _seq_results(self, st)
    cur = stream if stream is not None else torch.cuda.current_stream()
    if self.sys.sm_resident:
        if self.events is not None:
            self.events[0].record(cur)
        self.sys.propagate(st.tasks[st.order], M, K, self.profile, self.omega, self.step_rtol(),
                           self.max_it, st.xbuf, st.qoi, st.iters, st.status, None, stream,
                           tasks_dev=st.td, elapsed=st.elapsed, xss=st.xss)
        if self.events is not None:
            self.events[1].record(cur)
    elif (rp is not None and self.sys.propagate_path(st.T, M.shape[0], st.xss is not None, True)
          == _lib.PATH_BAND):
        # band path: every task carries its own dt, so a level's fine and coarse
        # solves share ONE launch (longest tasks first: the short ones fill the
        # cluster slots the long ones leave at the end of the launch)
        order = np.argsort(-st.tasks["n_steps"], kind="stable")
        self.sys.propagate(st.tasks[order], M, K, self.profile, self.omega, self.step_rtol(),
                           self.max_it, st.xbuf, st.qoi, st.iters, st.status, None, stream,
                           elapsed=st.elapsed, xss=st.xss, rp=rp)
    else:
        for dt in sorted(set(st.tasks["dt"].tolist())):
            sel = st.tasks[st.tasks["dt"] == dt]
            self.sys.propagate(sel, M, K, self.profile, self.omega, self.step_rtol(),
                               self.max_it, st.xbuf, st.qoi, st.iters, st.status, None, stream,
                               elapsed=st.elapsed, xss=st.xss, rp=rp)
    return _seq_results(self, st)


# ------------------------------------------------------------ Parareal
def _pr_setup(self, M, K, S: int, row0: int, t0: float, t1: float, m: int, dt_fine: float,
              dt_coarse: float, k_max: int, stream=None, keep_traj: bool = False,
              qoi_mode: int | None = None, qoi_index: int = 0, qoi_from: int = -1,
              correction: bool = False, rp_on: bool = False):
    """Buffers, fine task tables and predictor states of a Parareal batch whose
    operators are M/K rows row0 .. row0+S-1."""
    from types import SimpleNamespace
    if not 1 <= k_max <= m:
        raise ValueError(f"max_iterations must lie in [1, M={m}], got {k_max}")
    N = self.N
    dev = self.device
    bounds, fk0, fst, ck0, cst = parareal_grid(t0, t1, m, dt_fine, dt_coarse)
    uf_size = S * (m + 1) * N
    traj_steps = int(fst.max()) + 1
    traj_size = S * m * traj_steps * N if keep_traj else 0
    # correction fine solves (iterations k >= 2): F^k = F^{k-1} + Phi(U^k - U^{k-1})
    corr = (correction and not keep_traj and k_max > 1
            and (qoi_mode is None or qoi_mode == _lib.QOI_FINAL_ENERGY)
            and os.environ.get("MLMCP_PR_CORRECTION", "1") != "0"
            and self.sys.propagate_path(S * m, S, self.use_predictor(), rp_on,
                                        False) == _lib.PATH_TILE)
    d_size = uf_size if corr else 0
    buf = torch.zeros(2 * uf_size + d_size + traj_size, dtype=F64, device=dev)
    st = SimpleNamespace(S=S, row0=row0, m=m, k_max=k_max, t0=t0, dt_coarse=dt_coarse,
                         uf_size=uf_size, traj_steps=traj_steps, buf=buf, keep_traj=keep_traj,
                         corr=corr, traj_off=2 * uf_size + d_size,
                         D=buf[2 * uf_size:3 * uf_size].view(S, m + 1, N) if corr else None,
                         U=buf[:uf_size].view(S, m + 1, N),
                         F=buf[uf_size:2 * uf_size].view(S, m + 1, N),
                         C=torch.zeros((S, m, N), dtype=F64, device=dev),
                         active=torch.ones(S, dtype=I32, device=dev),
                         k_used=torch.zeros(S, dtype=I32, device=dev),
                         defects=torch.full((S, k_max), float("nan"), dtype=F64, device=dev),
                         status=torch.zeros((S, _lib.STATUS_INTS), dtype=I32, device=dev),
                         fine_status=torch.zeros((S * m, _lib.STATUS_INTS), dtype=I32, device=dev),
                         fine_iters=torch.zeros(S * m, dtype=I32, device=dev),
                         coarse_iters=torch.zeros(S, dtype=I32, device=dev),
                         elapsed_c=None, elapsed_f=None, slice_qoi=None, xss_f=None, xss_c=None)
    st.ck0_d, st.cst_d = self._grid_tensors(ck0, cst)
    if self.timing:                   # executor ledger: per-sample coarse / per-slice fine ns
        st.elapsed_c = torch.zeros(S, dtype=torch.int64, device=dev)
        st.elapsed_f = torch.zeros(S * m, dtype=torch.int64, device=dev)
    s_idx, n_idx = np.meshgrid(np.arange(S), np.arange(1, m + 1), indexing="ij")
    s_idx, n_idx = s_idx.ravel(), n_idx.ravel()
    all_tasks = new_tasks(S * m)
    all_tasks["sample"] = row0 + s_idx
    all_tasks["n_steps"] = fst[n_idx - 1]
    all_tasks["k0"] = fk0[n_idx - 1]
    all_tasks["dt"] = dt_fine
    all_tasks["t_base"] = t0
    all_tasks["x_in"] = (s_idx * (m + 1) + (n_idx - 1)) * N
    all_tasks["x_out"] = uf_size + (s_idx * (m + 1) + n_idx) * N
    if keep_traj:
        all_tasks["traj"] = st.traj_off + ((s_idx * m + (n_idx - 1)) * traj_steps) * N
    all_tasks["group"] = s_idx
    all_tasks["slot"] = s_idx * m + (n_idx - 1)
    if qoi_mode is not None and qoi_mode != _lib.QOI_FINAL_ENERGY:
        # time-accumulated QoI over the fine trajectory (parareal.py:212 concatenates
        # the last fine solve of every slice): each fine solve of slice n
        # overwrites its partial sum, so after convergence slot (s, n) holds the
        # sum over the slice's final sub-trajectory
        all_tasks["qoi_slot"] = s_idx * m + (n_idx - 1)
        all_tasks["qoi_mode"] = qoi_mode
        all_tasks["qoi_from"] = qoi_from
        all_tasks["qoi_index"] = qoi_index
        st.slice_qoi = torch.zeros(S * m, dtype=F64, device=dev)
    if self.use_predictor():
        # periodic steady states at dt_fine (rows 0..S-1) and dt_coarse (S..2S-1)
        all_tasks["ss_slot"] = s_idx
        rows = row0 + np.arange(S)
        X = self.steady_states(np.concatenate([rows, rows]),
                               np.concatenate([np.full(S, dt_fine), np.full(S, dt_coarse)]),
                               M, K, stream)
        st.xss_f, st.xss_c = X[:S], X[S:]
        if os.environ.get("MLMCP_PREDICTOR") == "fine":
            st.xss_c = None
    st.all_tasks, st.n_idx = all_tasks, n_idx
    if corr:
        # slice n at iteration k >= 2 solves the homogeneous problem from
        # D[s][n-1] = U^k_{n-1} - U^{k-1}_{n-1} and adds its end state to F_n
        ct = all_tasks.copy()
        ct["x_in"] = 2 * uf_size + (s_idx * (m + 1) + (n_idx - 1)) * N
        ct["flags"] = _lib.TASK_CORRECTION
        ct["ss_slot"] = -1
        ct["qoi_slot"] = -1
        ct["qoi_mode"] = _lib.QOI_NONE
        st.corr_tasks = ct
    return st


def _pr_result(self, st, K, stream=None) -> PararealBatchResult:
    S, m, N = st.S, st.m, self.N
    dev = self.device
    ekey = ("energy", S, m, N, st.row0)
    ev = self._task_cache.get(ekey)
    if ev is None:
        ev = (torch.arange(st.row0, st.row0 + S, dtype=I32, device=dev),
              torch.tensor((st.uf_size + (np.arange(S) * (m + 1) + m) * N).astype(np.int64),
                           device=dev))
        self._task_cache[ekey] = ev
    if st.slice_qoi is not None:
        qoi = st.slice_qoi.view(S, m).sum(dim=1)
    else:
        qoi = self.sys.energy(ev[0], ev[1], st.buf, K, stream)
    traj = None
    if st.keep_traj:
        traj = st.buf[st.traj_off:].view(S, m, st.traj_steps, N)
    return PararealBatchResult(qoi, st.k_used, st.defects, st.status, st.fine_status, st.U, st.F,
                               traj, st.fine_iters, st.coarse_iters,
                               (st.elapsed_c, st.elapsed_f) if self.timing else None)


def _run_parareal(self, M, K, t0: float, t1: float, m: int, dt_fine: float,
                  dt_coarse: float, tol: float, k_max: int, stream=None,
                  keep_traj: bool = False, qoi_mode: int | None = None,
                  qoi_index: int = 0, qoi_from: int = -1, rp=None) -> PararealBatchResult:
    """parareal_solve for the S samples whose operators are M/K rows 0..S-1
    (slice the level's M/K to pass a sub-batch), from the zero state:
    K_max rounds of [coarse sweep, fine slices, defect] launches."""
    S = M.shape[0]
    st = _pr_setup(self, M, K, S, 0, t0, t1, m, dt_fine, dt_coarse, k_max, stream, keep_traj,
                   qoi_mode, qoi_index, qoi_from, correction=True, rp_on=rp is not None)
    dev = self.device
    key = ("pr", st.all_tasks.tobytes(), k_max, st.corr)
    tables = self._task_cache.get(key)
    if tables is None:
        tables = []
        for k in range(1, k_max + 1):
            src = st.corr_tasks if (st.corr and k >= 2) else st.all_tasks
            sel = src[st.n_idx >= k].copy()
            sel["tag"] = k
            tables.append(tasks_to_device(sel, dev))
        self._task_cache[key] = tables
    for k in range(1, k_max + 1):
        if st.corr and k >= 2:     # U^{k-1} before the sweep overwrites it
            self.sys.parareal_delta(S, k, m, st.U, st.D, 0, st.active, stream)
        self.sys.parareal_coarse(S, k, m, M, K, self.profile, self.omega, dt_coarse, t0,
                                 st.ck0_d, st.cst_d, self.step_rtol(), self.max_it, st.U, st.F,
                                 st.C, st.coarse_iters, st.status, st.active, stream,
                                 elapsed=st.elapsed_c, xss=st.xss_c, rp=rp)
        if st.corr and k >= 2:
            self.sys.parareal_delta(S, k, m, st.U, st.D, 1, st.active, stream)
        sel = (st.corr_tasks if (st.corr and k >= 2) else st.all_tasks)[st.n_idx >= k]
        self.sys.propagate(sel, M, K, self.profile, self.omega, self.step_rtol(), self.max_it,
                           st.buf, st.slice_qoi, st.fine_iters, st.fine_status, st.active, stream,
                           tasks_dev=tables[k - 1], elapsed=st.elapsed_f, xss=st.xss_f, rp=rp)
        self.sys.parareal_defect(S, k, m, k_max, st.U, st.F, tol, st.active, st.k_used,
                                 st.defects, stream)
    self.sys.parareal_finalize(S, m, st.U, st.F, st.k_used, stream)
    self._keep = tables
    self._last_pr_corr = st.corr
    return _pr_result(self, st, K, stream)


def _run_fused(self, M, K, jobs: list[SeqJob], pr=None, stream=None, grid_ctas: int = 0):
    """Sequential jobs and/or one Parareal batch in ONE persistent launch with
    the device-side scheduler (mlmcp_run_fused).  ``pr`` = dict(row0, S, t0,
    t1, m, dt_fine, dt_coarse, tol, k_max, qoi_mode, qoi_index, qoi_from).
    Every task kind addresses one set of arrays (states, QoI, iteration,
    status and timer slots, steady states), laid out [sequential | Parareal
    fine | Parareal coarse].  Returns (list of SeqResult, PararealBatchResult
    or None)."""
    from types import SimpleNamespace
    N = self.N
    dev = self.device
    pred = self.use_predictor()
    # ---- sequential part (slots 0 .. T-1)
    T = int(sum(len(j.rows) for j in jobs))
    tasks = new_tasks(T)
    off = 0
    for j in jobs:
        sl = slice(off, off + len(j.rows))
        tasks["sample"][sl] = j.rows
        tasks["n_steps"][sl] = j.n_steps
        tasks["dt"][sl] = j.dt
        tasks["qoi_mode"][sl] = j.qoi_mode
        tasks["qoi_from"][sl] = j.qoi_from
        tasks["qoi_index"][sl] = j.qoi_index
        off += len(j.rows)
    idx = np.arange(T)
    tasks["x_in"] = idx * N
    tasks["x_out"] = idx * N
    tasks["qoi_slot"] = idx
    tasks["slot"] = idx
    if pred:
        tasks["ss_slot"] = idx
    order = np.argsort(-tasks["n_steps"], kind="stable")   # longest first
    # ---- Parareal part
    S = int(pr["S"]) if pr is not None else 0
    m = int(pr["m"]) if S else 1
    k_max = int(pr["k_max"]) if S else 1
    n_fine = S * m
    n_slots = T + n_fine + S
    u_off = T * N
    uf = S * (m + 1) * N
    c_tmp_off = u_off + 2 * uf
    xbuf = torch.zeros(c_tmp_off + S * N, dtype=F64, device=dev)
    qoi = torch.zeros(T + n_fine, dtype=F64, device=dev)
    iters = torch.zeros(n_slots, dtype=I32, device=dev)
    status = torch.zeros((n_slots, _lib.STATUS_INTS), dtype=I32, device=dev)
    elapsed = torch.zeros(n_slots, dtype=torch.int64, device=dev) if self.timing else None
    active = torch.ones(max(S, 1), dtype=I32, device=dev)
    batch = _lib.PararealBatch()
    pst = None
    ss_samples = [tasks["sample"]] if pred else []
    ss_dts = [tasks["dt"]] if pred else []
    if S:
        bounds, fk0, fst, ck0, cst = parareal_grid(pr["t0"], pr["t1"], m, pr["dt_fine"],
                                                   pr["dt_coarse"])
        s_idx, n_idx = np.meshgrid(np.arange(S), np.arange(1, m + 1), indexing="ij")
        s_idx, n_idx = s_idx.ravel(), n_idx.ravel()
        ft = new_tasks(n_fine)
        ft["sample"] = pr["row0"] + s_idx
        ft["n_steps"] = fst[n_idx - 1]
        ft["k0"] = fk0[n_idx - 1]
        ft["dt"] = pr["dt_fine"]
        ft["t_base"] = pr["t0"]
        ft["x_in"] = u_off + (s_idx * (m + 1) + (n_idx - 1)) * N
        ft["x_out"] = u_off + uf + (s_idx * (m + 1) + n_idx) * N
        ft["group"] = s_idx
        ft["slot"] = T + s_idx * m + (n_idx - 1)
        qm = pr.get("qoi_mode")
        slice_q = qm is not None and qm != _lib.QOI_FINAL_ENERGY
        if slice_q:
            ft["qoi_slot"] = T + s_idx * m + (n_idx - 1)
            ft["qoi_mode"] = qm
            ft["qoi_from"] = pr.get("qoi_from", -1)
            ft["qoi_index"] = pr.get("qoi_index", 0)
        if pred:
            ft["ss_slot"] = T + s_idx
            rows = pr["row0"] + np.arange(S)
            ss_samples += [rows, rows]
            ss_dts += [np.full(S, pr["dt_fine"]), np.full(S, pr["dt_coarse"])]
        key = ("fused-fine", ft.tobytes())
        ftd = self._task_cache.get(key)
        if ftd is None:
            ftd = tasks_to_device(ft, dev)
            self._task_cache[key] = ftd
        ck0_d, cst_d = self._grid_tensors(ck0, cst)
        C = torch.zeros((S, m, N), dtype=F64, device=dev)
        k_used = torch.zeros(S, dtype=I32, device=dev)
        defects = torch.full((S, k_max), float("nan"), dtype=F64, device=dev)
        batch = _lib.PararealBatch(S, int(pr["row0"]), m, k_max, float(pr["tol"]),
                                   float(pr["dt_coarse"]), float(pr["t0"]), ptr(ck0_d),
                                   ptr(cst_d), ptr(ftd), u_off, c_tmp_off, ptr(C), T + n_fine,
                                   T + S if pred else -1, ptr(k_used), ptr(defects))
        pst = SimpleNamespace(S=S, m=m, k_max=k_max, row0=int(pr["row0"]), uf_size=uf,
                              buf=xbuf[u_off:u_off + 2 * uf], C=C, active=active[:S],
                              k_used=k_used, defects=defects, keep_traj=False,
                              status=status[T + n_fine:], fine_status=status[T:T + n_fine],
                              fine_iters=iters[T:T + n_fine], coarse_iters=iters[T + n_fine:],
                              elapsed_c=None if elapsed is None else elapsed[T + n_fine:],
                              elapsed_f=None if elapsed is None else elapsed[T:T + n_fine],
                              slice_qoi=qoi[T:] if slice_q else None, traj_steps=0, t0=pr["t0"],
                              dt_coarse=pr["dt_coarse"])
        pst.U = pst.buf[:uf].view(S, m + 1, N)
        pst.F = pst.buf[uf:].view(S, m + 1, N)
    xss = None
    if pred and (T or S):
        xss = self.steady_states(np.concatenate(ss_samples), np.concatenate(ss_dts), M, K, stream)
    td = None
    if T:
        key = (tasks.tobytes(), N)
        td = self._task_cache.get(key)
        if td is None:
            td = tasks_to_device(tasks[order], dev)
            self._task_cache[key] = td
    arrays = _lib.TaskArrays(T, ptr(td) if td is not None else None, ptr(xss), ptr(xbuf),
                             ptr(qoi), ptr(iters), ptr(status), ptr(active), ptr(elapsed))
    cur = stream if stream is not None else torch.cuda.current_stream()
    timed = self.events is not None and T > 0     # events bracket launches with sequential tasks
    if timed:
        self.events[0].record(cur)
    if T or S:
        self.sys.run_fused(M, K, self.profile, self.omega, self.step_rtol(), self.max_it, arrays,
                           batch, S, m, k_max, stream, grid_ctas)
    if timed:
        self.events[1].record(cur)
    sq = SimpleNamespace(jobs=jobs, qoi=qoi[:T], iters=iters[:T], status=status[:T],
                         elapsed=None if elapsed is None else elapsed[:T], xbuf=xbuf[:T * N],
                         tasks=tasks)
    res = _seq_results(self, sq)
    self._keep_fused = (arrays, batch, td, xss)
    return res, (_pr_result(self, pst, K, stream) if pst is not None else None)


def raise_on_status(status: torch.Tensor, what: str):
    """Map per-task failure codes to SingularSystemError (timeint.py:25-30)."""
    st = status.cpu().numpy()
    bad = np.nonzero(st[:, 0] != _lib.ST_OK)[0]
    if len(bad):
        i = int(bad[0])
        code, step = int(st[i, 0]), int(st[i, 1])
        if code == _lib.ST_UNSUPPORTED:
            raise ValueError(f"{what}: task {i}: {_lib.STATUS_NAMES[code]}")
        raise SingularSystemError(f"{what}: task {i}: {_lib.STATUS_NAMES.get(code, code)} "
                                  f"at step {step}", step_index=step)
