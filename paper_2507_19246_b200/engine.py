"""Device engine: one ``mlmcp_ctx`` per (sparsity pattern, GPU) plus the
torch-owned buffers and the task tables the C ABI consumes.

PyTorch is plumbing here: it owns device memory (caching allocator), streams
and ``torch.distributed``; every arithmetic step of the hot path is a
libmlmcp.so kernel launched through ``_lib``.  There is no CPU fallback — a
missing library or GPU raises.
"""

from __future__ import annotations

import ctypes

import numpy as np
import torch

from . import _lib
from ._lib import TASK_DTYPE, check, np_ptr, ptr

F64 = torch.float64
I32 = torch.int32


def require_cuda(device=None) -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2507_19246_b200 needs a CUDA device (sm_100a); "
                           "there is no CPU fallback")
    if device is None:
        return torch.device("cuda", torch.cuda.current_device())
    dev = torch.device(device)
    if dev.type != "cuda":
        raise ValueError(f"device must be a CUDA device, got {dev}")
    return torch.device("cuda", dev.index if dev.index is not None else torch.cuda.current_device())


def stream_handle(stream=None) -> ctypes.c_void_p:
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


def new_tasks(n: int) -> np.ndarray:
    t = np.zeros(n, dtype=TASK_DTYPE)
    t["traj"] = -1
    t["qoi_slot"] = -1
    t["group"] = -1
    t["slot"] = -1
    t["ss_slot"] = -1
    return t


def tasks_to_device(tasks: np.ndarray, device) -> torch.Tensor:
    raw = np.ascontiguousarray(tasks).view(np.uint8)
    return torch.from_numpy(raw.copy()).to(device, non_blocking=False)


class DeviceSystem:
    """A CSR sparsity pattern bound to one GPU (``mlmcp_ctx``).

    ``assembly`` = (n_elem, cptr, celem, cmw, ckw) enables ``assemble``.
    """

    def __init__(self, row_ptr, col, device=None, assembly=None):
        self.device = require_cuda(device)
        self.lib = _lib.load()
        row_ptr = np.ascontiguousarray(row_ptr, dtype=np.int32)
        col = np.ascontiguousarray(col, dtype=np.int32)
        self.n_rows = len(row_ptr) - 1
        self.nnz = int(row_ptr[-1])
        self.row_ptr_h = row_ptr
        self.col_h = col
        handle = ctypes.c_void_p()
        check(self.lib.mlmcp_ctx_create(self.device.index, self.n_rows, self.nnz, np_ptr(row_ptr),
                                        np_ptr(col), ctypes.byref(handle)), "mlmcp_ctx_create")
        self.ctx = handle
        w = ctypes.c_int()
        small = ctypes.c_int()
        check(self.lib.mlmcp_ctx_info(self.ctx, ctypes.byref(w), ctypes.byref(small)), "mlmcp_ctx_info")
        self.max_row_nnz = w.value
        self.small_max_rows = small.value
        self._path = 0
        if assembly is not None:
            n_elem, cptr, celem, cmw, ckw = assembly
            cptr = np.ascontiguousarray(cptr, dtype=np.int32)
            celem = np.ascontiguousarray(celem, dtype=np.int32)
            cmw = np.ascontiguousarray(cmw, dtype=np.float64)
            ckw = np.ascontiguousarray(ckw, dtype=np.float64)
            check(self.lib.mlmcp_ctx_set_assembly(self.ctx, int(n_elem), len(celem), np_ptr(cptr),
                                                  np_ptr(celem), np_ptr(cmw), np_ptr(ckw)),
                  "mlmcp_ctx_set_assembly")
        self._ws_by_stream = {}     # streaming workspace of each stream that launches
        self.band_low_priority = False   # set by families that keep two calls in flight
        self._band_streams = {}
        self._fused_ws = {}
        self.region_grid = None

    # ------------------------------------------------------------ lifecycle
    def close(self):
        if getattr(self, "ctx", None) is not None and self.lib is not None:
            self.lib.mlmcp_ctx_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ------------------------------------------------------------ config
    def set_path(self, path: str):
        code = {"auto": 0, "small": 1, "stream": 2, "direct": 3}[path]
        check(self.lib.mlmcp_ctx_set_path(self.ctx, code), "mlmcp_ctx_set_path")
        self._path = code

    def stream_timing(self, mode: int) -> tuple[float, int]:
        """mlmcp_stream_timing: (ms, launches) of the streaming PCG-iteration
        launches; mode 1 resets and starts, 0 stops."""
        ms = ctypes.c_double()
        n = ctypes.c_int64()
        check(self.lib.mlmcp_stream_timing(self.ctx, int(mode), ctypes.byref(ms), ctypes.byref(n)),
              "mlmcp_stream_timing")
        return float(ms.value), int(n.value)

    @property
    def direct(self) -> bool:
        return self._path == 3 or (self._path == 0 and self.n_rows <= _lib.DIRECT_MAX_ROWS)

    @property
    def sm_resident(self) -> bool:
        """True when every launch is stream-ordered and workspace-free (SM-resident
        or direct path), so concurrent launches on several streams are safe."""
        if self._path in (1, 3):
            return True
        if self._path == 2:
            return False
        return self.n_rows <= self.small_max_rows

    def workspace(self, n_tasks: int, S: int, stream=None) -> torch.Tensor | None:
        """The streaming workspace of ``stream`` (default: the current stream).
        One buffer per launching stream, grown on demand and kept between
        calls, so calls in flight on different streams never share one."""
        nbytes = int(self.lib.mlmcp_workspace_bytes(self.ctx, int(n_tasks), int(S)))
        if nbytes == 0:
            return None
        s = stream if stream is not None else torch.cuda.current_stream()
        key = s.cuda_stream
        ws = self._ws_by_stream.get(key)
        if ws is None or ws.numel() < nbytes:
            self._ws_by_stream.pop(key, None)
            ws = None
            with torch.cuda.stream(s):      # owned by the stream's allocator pool
                ws = torch.empty(nbytes, dtype=torch.uint8, device=self.device)
            self._ws_by_stream[key] = ws
        return ws

    def workspace_bytes_held(self) -> int:
        return sum(w.numel() for w in self._ws_by_stream.values())

    # ------------------------------------------------------------ K1
    def assemble(self, S: int, sigma: torch.Tensor, sigma_stride: int, sigma_index,
                 nu: torch.Tensor, nu_stride: int, nu_index, stream=None, out=None):
        if out is not None:
            M, K = out
            if M.shape != (S, self.nnz) or K.shape != (S, self.nnz) or not (
                    M.is_contiguous() and K.is_contiguous()):
                raise ValueError("assemble(out=...) needs contiguous [S, nnz] tensors")
        else:
            M = torch.empty((S, self.nnz), dtype=F64, device=self.device)
            K = torch.empty((S, self.nnz), dtype=F64, device=self.device)
        check(self.lib.mlmcp_assemble(self.ctx, S, ptr(sigma), int(sigma_stride), ptr(sigma_index),
                                      ptr(nu), int(nu_stride), ptr(nu_index), ptr(M), ptr(K),
                                      stream_handle(stream)), "mlmcp_assemble")
        return M, K

    # ------------------------------------------------------------ K2-K4, K6
    def set_region_grid(self, rg) -> bool:
        """Register a fe.RegionGrid (region-linear operator on the tile path)."""
        if rg is None:
            check(self.lib.mlmcp_ctx_set_region_grid(self.ctx, 0, None, None, None),
                  "mlmcp_ctx_set_region_grid")
            self.region_grid = None
            return False
        code = np.ascontiguousarray(rg.code, dtype=np.uint32)
        mw = np.ascontiguousarray(rg.mw, dtype=np.float64)
        kw = np.ascontiguousarray(rg.kw, dtype=np.float64)
        check(self.lib.mlmcp_ctx_set_region_grid(self.ctx, int(rg.n_regions), np_ptr(code),
                                                 np_ptr(mw), np_ptr(kw)),
              "mlmcp_ctx_set_region_grid")
        self.region_grid = rg
        return True

    def propagate(self, tasks: np.ndarray, M, K, profile, omega: float, rtol: float,
                  max_it: int, xbuf, qoi=None, iters=None, status=None, active=None,
                  stream=None, tasks_dev: torch.Tensor | None = None, elapsed=None, xss=None,
                  rp=None):
        n = len(tasks)
        if n == 0:
            return None
        S = M.shape[0]
        td = tasks_dev if tasks_dev is not None else tasks_to_device(tasks, self.device)
        ws = self.workspace(n, S, stream)
        launch_on = stream
        cur = None
        if self.band_low_priority and self.propagate_path(
                n, S, xss is not None, rp is not None) == _lib.PATH_BAND:
            # calls in flight on two (high-priority) streams: the band launch
            # goes to a low-priority stream paired with the caller's, so that
            # the OTHER call's preparation kernels are dispatched to the SMs the
            # band clusters leave idle ahead of this launch's pending clusters
            cur = stream if stream is not None else torch.cuda.current_stream()
            launch_on = self._band_stream(cur)
            launch_on.wait_stream(cur)
        check(self.lib.mlmcp_propagate(self.ctx, n, ptr(td), S, ptr(M), ptr(K), ptr(rp), ptr(profile),
                                       float(omega), float(rtol), int(max_it), ptr(xss),
                                       ptr(xbuf), ptr(qoi),
                                       ptr(iters), ptr(status), ptr(active), ptr(elapsed), ptr(ws),
                                       0 if ws is None else ws.numel(), stream_handle(launch_on)),
              "mlmcp_propagate")
        if cur is not None:
            cur.wait_stream(launch_on)
        return td

    def _band_stream(self, cur):
        st = self._band_streams.get(cur.cuda_stream)
        if st is None:
            lo, _ = torch.cuda.Stream.priority_range()
            st = torch.cuda.Stream(device=self.device, priority=lo)
            self._band_streams[cur.cuda_stream] = st
        return st

    # ------------------------------------------------------------ K5
    def parareal_coarse(self, S, k, m, M, K, profile, omega, dt_c, t0, slice_k0, slice_steps,
                        rtol, max_it, U, F, C, iters, status, active, stream=None, elapsed=None,
                        xss=None, rp=None):
        ws = self.workspace(S, S, stream)
        check(self.lib.mlmcp_parareal_coarse(
            self.ctx, S, k, m, ptr(M), ptr(K), ptr(rp), ptr(profile), float(omega), float(dt_c), float(t0),
            ptr(slice_k0), ptr(slice_steps), float(rtol), int(max_it), ptr(U), ptr(F), ptr(C),
            ptr(iters), ptr(status), ptr(active), ptr(elapsed), ptr(xss), ptr(ws),
            0 if ws is None else ws.numel(), stream_handle(stream)), "mlmcp_parareal_coarse")

    # ------------------------------------------------------------ fused launch
    def run_fused(self, M, K, profile, omega, rtol, max_it, arrays, batch, S_pr, m, k_max,
                  stream=None, grid_ctas: int = 0):
        """mlmcp_run_fused with ctypes ``_lib.TaskArrays`` / ``_lib.PararealBatch``."""
        nbytes = int(self.lib.mlmcp_fused_workspace_bytes(S_pr, m, k_max))
        key = stream.cuda_stream if stream is not None else torch.cuda.current_stream().cuda_stream
        ws = self._fused_ws.get(key)
        if ws is None or ws.numel() < nbytes:
            ws = torch.empty(nbytes, dtype=torch.uint8, device=self.device)
            self._fused_ws[key] = ws
        check(self.lib.mlmcp_run_fused(self.ctx, M.shape[0], ptr(M), ptr(K), ptr(profile),
                                       float(omega), float(rtol), int(max_it),
                                       ctypes.byref(arrays), ctypes.byref(batch), int(grid_ctas),
                                       ptr(ws), ws.numel(), stream_handle(stream)),
              "mlmcp_run_fused")

    # ------------------------------------------------------------ predictor
    def periodic_state(self, sample_idx: torch.Tensor, dts: torch.Tensor, M, K, profile,
                       omega: float, rtol: float = 1e-8, max_it: int = 500, stream=None,
                       rp=None):
        """X [n, 2, N]: periodic steady states of the implicit-Euler iteration
        for (sample_idx[i], dts[i]) (initial-guess predictor)."""
        n = len(sample_idx)
        X = torch.empty((n, 2, self.n_rows), dtype=F64, device=self.device)
        if n:
            nbytes = int(self.lib.mlmcp_periodic_workspace_bytes(self.ctx, n))
            ws = None
            if nbytes:     # streaming path: grid-wide COCG in a workspace
                ws = torch.empty(nbytes, dtype=torch.uint8, device=self.device)
            check(self.lib.mlmcp_periodic_state(self.ctx, n, ptr(sample_idx), ptr(dts),
                                                M.shape[0], ptr(M), ptr(K), ptr(rp), ptr(profile),
                                                float(omega), float(rtol), int(max_it), ptr(X),
                                                None, ptr(ws), nbytes, stream_handle(stream)),
                  "mlmcp_periodic_state")
        return X

    def parareal_defect(self, S, k, m, k_max, U, F, tol, active, k_used, defects, stream=None):
        check(self.lib.mlmcp_parareal_defect(self.ctx, S, k, m, k_max, ptr(U), ptr(F), float(tol),
                                             ptr(active), ptr(k_used), ptr(defects),
                                             stream_handle(stream)), "mlmcp_parareal_defect")

    def parareal_finalize(self, S, m, U, F, k_used, stream=None):
        check(self.lib.mlmcp_parareal_finalize(self.ctx, S, m, ptr(U), ptr(F), ptr(k_used),
                                               stream_handle(stream)), "mlmcp_parareal_finalize")

    def parareal_delta(self, S, k, m, U, D, mode: int, active, stream=None):
        """mode 0: D = U (snapshot before the coarse sweep of iteration k);
        mode 1: D = U - D (after it), slices k-1 .. m-1 of the active samples."""
        check(self.lib.mlmcp_parareal_delta(self.ctx, S, k, m, ptr(U), ptr(D), int(mode),
                                            ptr(active), stream_handle(stream)),
              "mlmcp_parareal_delta")

    def propagate_path(self, n_tasks: int, S: int, with_ss: bool, with_rp: bool,
                       correction: bool = False) -> int:
        """_lib.PATH_* of an mlmcp_propagate batch of this shape."""
        return int(self.lib.mlmcp_propagate_path(self.ctx, int(n_tasks), int(S), int(with_ss),
                                                 int(with_rp), int(correction)))

    def energy(self, sample_idx: torch.Tensor, x_off: torch.Tensor, xbuf, K, stream=None):
        out = torch.empty(len(sample_idx), dtype=F64, device=self.device)
        check(self.lib.mlmcp_energy(self.ctx, len(sample_idx), ptr(sample_idx), ptr(x_off),
                                    ptr(xbuf), ptr(K), ptr(out), stream_handle(stream)),
              "mlmcp_energy")
        return out


def kl_sigma(xi: torch.Tensor, basis: torch.Tensor, log_sigma0: float, scale: float,
             stream=None) -> torch.Tensor:
    lib = _lib.load()
    S, modes = xi.shape
    E = basis.shape[1]
    out = torch.empty((S, E), dtype=F64, device=xi.device)
    check(lib.mlmcp_kl_sigma(S, E, modes, ptr(xi), ptr(basis), float(log_sigma0), float(scale),
                             ptr(out), stream_handle(stream)), "mlmcp_kl_sigma")
    return out


def region_params(params: torch.Tensor, R: int, mask: torch.Tensor | None, sigma_out=None,
                  rp_out=None, stream=None):
    """mlmcp_region_params: masked sigma [S, R] and/or (sigma, nu) pairs
    [S, R, 2] from drawn parameters [S, 2R] (nu first, sigma second)."""
    lib = _lib.load()
    S = params.shape[0]
    check(lib.mlmcp_region_params(S, int(R), ptr(params), ptr(mask), ptr(sigma_out), ptr(rp_out),
                                  stream_handle(stream)), "mlmcp_region_params")


def level_reduce(q_l: torch.Tensor, q_lm1: torch.Tensor | None, stream=None) -> torch.Tensor:
    """K7: [sum Y, sum Y^2, mean, var] of Y = q_l - q_lm1 (fixed order)."""
    lib = _lib.load()
    out = torch.empty(4, dtype=F64, device=q_l.device)
    check(lib.mlmcp_level_reduce(len(q_l), ptr(q_l), ptr(q_lm1), ptr(out), stream_handle(stream)),
          "mlmcp_level_reduce")
    return out
