"""ctypes binding of libmlmcp.so (include/mlmcp.h).

The library is built in-tree (``make`` or ``__graft_entry__.build()``) and
loaded from this package directory.  There is no fallback: if the shared
object is missing or a GPU is absent, every device entry point raises.

Error mapping:
  MLMCP_EINVAL -> ValueError, MLMCP_ENOMEM -> MemoryError,
  MLMCP_ECUDA  -> RuntimeError.  Per-task solver failures are mapped by the
  callers to SingularSystemError (timeint.py:25-30) or PropagatorError
  (parareal.py:37-43).
"""

from __future__ import annotations

import ctypes
import os
import threading

import numpy as np

LIB_NAME = "libmlmcp.so"
# MLMCP_LIB selects another in-tree build (e.g. libmlmcp_checked.so, the
# device-side-checked build of scripts/checked_suite.sh)
LIB_PATH = os.environ.get("MLMCP_LIB") or os.path.join(os.path.dirname(os.path.abspath(__file__)),
                                                       LIB_NAME)

EINVAL = -22
ECUDA = -5
ENOMEM = -12

ST_OK, ST_NOCONV, ST_BREAKDOWN, ST_NONFINITE, ST_SINGULAR, ST_UNSUPPORTED = 0, 1, 2, 3, 4, 5
STATUS_NAMES = {ST_NOCONV: "PCG did not converge within max_it",
                ST_BREAKDOWN: "PCG breakdown (operator not SPD)",
                ST_NONFINITE: "non-finite residual",
                ST_SINGULAR: "(M + dt K) is singular",
                ST_UNSUPPORTED: "task flag not supported on this path"}
STATUS_INTS = 4

QOI_NONE, QOI_FINAL_ENERGY, QOI_SUM_ENERGY, QOI_ELECTRICAL, QOI_JOULE = 0, 1, 2, 3, 4
TASK_NO_EXTRAPOLATION = 1
TASK_CORRECTION = 2
PATH_DIRECT, PATH_SMALL, PATH_CLUSTER, PATH_BAND, PATH_COOP, PATH_TILE, PATH_ELL = range(7)
ABI_VERSION = 11
DIRECT_MAX_ROWS = 4

# mlmcp_task (96 bytes, natural alignment)
TASK_DTYPE = np.dtype([
    ("sample", np.int32), ("n_steps", np.int32), ("k0", np.int64), ("dt", np.float64),
    ("t_base", np.float64), ("x_in", np.int64), ("x_out", np.int64), ("traj", np.int64),
    ("qoi_slot", np.int32), ("qoi_mode", np.int32), ("qoi_from", np.int64),
    ("group", np.int32), ("slot", np.int32), ("tag", np.int32), ("flags", np.int32),
    ("qoi_index", np.int32), ("ss_slot", np.int32),
], align=True)
assert TASK_DTYPE.itemsize == 96



class TaskArrays(ctypes.Structure):
    """mlmcp_task_arrays (include/mlmcp.h)."""
    _fields_ = [("n_seq", ctypes.c_int), ("seq_tasks_d", ctypes.c_void_p),
                ("xss_d", ctypes.c_void_p), ("xbuf_d", ctypes.c_void_p),
                ("qoi_d", ctypes.c_void_p), ("iters_d", ctypes.c_void_p),
                ("status_d", ctypes.c_void_p), ("active_d", ctypes.c_void_p),
                ("elapsed_ns_d", ctypes.c_void_p)]


class PararealBatch(ctypes.Structure):
    """mlmcp_parareal_batch (include/mlmcp.h)."""
    _fields_ = [("S", ctypes.c_int), ("row0", ctypes.c_int), ("m", ctypes.c_int),
                ("k_max", ctypes.c_int), ("tol", ctypes.c_double), ("dt_c", ctypes.c_double),
                ("t0", ctypes.c_double), ("slice_k0_d", ctypes.c_void_p),
                ("slice_steps_d", ctypes.c_void_p), ("fine_tasks_d", ctypes.c_void_p),
                ("u_off", ctypes.c_int64), ("c_tmp_off", ctypes.c_int64),
                ("C_d", ctypes.c_void_p), ("coarse_slot", ctypes.c_int),
                ("coarse_ss", ctypes.c_int), ("k_used_d", ctypes.c_void_p),
                ("defects_d", ctypes.c_void_p)]


# every symbol include/mlmcp.h declares (checked by tests/test_abi.py)
EXPORTS = (
    "mlmcp_abi_version", "mlmcp_last_error", "mlmcp_launch_count",
    "mlmcp_ctx_create", "mlmcp_ctx_destroy", "mlmcp_ctx_info", "mlmcp_ctx_set_assembly",
    "mlmcp_ctx_set_path", "mlmcp_ctx_set_region_grid", "mlmcp_region_params",
    "mlmcp_stream_timing", "mlmcp_assemble", "mlmcp_kl_sigma", "mlmcp_workspace_bytes",
    "mlmcp_propagate", "mlmcp_periodic_workspace_bytes", "mlmcp_periodic_state", "mlmcp_parareal_coarse", "mlmcp_parareal_defect",
    "mlmcp_parareal_finalize", "mlmcp_parareal_delta", "mlmcp_propagate_path", "mlmcp_energy", "mlmcp_level_reduce", "mlmcp_draw_uniform",
    "mlmcp_draw_uniform_host", "mlmcp_fused_workspace_bytes", "mlmcp_run_fused",
)

_lock = threading.Lock()
_lib = None

P = ctypes.c_void_p
I32 = ctypes.c_int32
I64 = ctypes.c_int64
F64 = ctypes.c_double
SZ = ctypes.c_size_t

_SIGS = {
    "mlmcp_abi_version": (ctypes.c_int, []),
    "mlmcp_last_error": (ctypes.c_char_p, []),
    "mlmcp_launch_count": (ctypes.c_uint64, []),
    "mlmcp_ctx_create": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, ctypes.c_int, P, P,
                                        ctypes.POINTER(P)]),
    "mlmcp_ctx_destroy": (ctypes.c_int, [P]),
    "mlmcp_stream_timing": (ctypes.c_int, [P, ctypes.c_int, ctypes.POINTER(F64),
                                           ctypes.POINTER(I64)]),
    "mlmcp_ctx_info": (ctypes.c_int, [P, ctypes.POINTER(ctypes.c_int),
                                      ctypes.POINTER(ctypes.c_int)]),
    "mlmcp_ctx_set_assembly": (ctypes.c_int, [P, ctypes.c_int, ctypes.c_int, P, P, P, P]),
    "mlmcp_ctx_set_path": (ctypes.c_int, [P, ctypes.c_int]),
    "mlmcp_assemble": (ctypes.c_int, [P, ctypes.c_int, P, I64, P, P, I64, P, P, P, P]),
    "mlmcp_kl_sigma": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, ctypes.c_int, P, P, F64, F64,
                                      P, P]),
    "mlmcp_workspace_bytes": (SZ, [P, ctypes.c_int, ctypes.c_int]),
    "mlmcp_propagate": (ctypes.c_int, [P, ctypes.c_int, P, ctypes.c_int, P, P, P, P, F64, F64,
                                       ctypes.c_int, P, P, P, P, P, P, P, P, SZ, P]),
    "mlmcp_ctx_set_region_grid": (ctypes.c_int, [P, ctypes.c_int, P, P, P]),
    "mlmcp_region_params": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, P, P, P, P, P]),
    "mlmcp_periodic_workspace_bytes": (SZ, [P, ctypes.c_int]),
    "mlmcp_periodic_state": (ctypes.c_int, [P, ctypes.c_int, P, P, ctypes.c_int, P, P, P, P, F64,
                                            F64, ctypes.c_int, P, P, P, SZ, P]),
    "mlmcp_parareal_coarse": (ctypes.c_int, [P, ctypes.c_int, ctypes.c_int, ctypes.c_int, P, P,
                                             P, P, F64, F64, F64, P, P, F64, ctypes.c_int, P, P,
                                             P, P, P, P, P, P, P, SZ, P]),
    "mlmcp_parareal_defect": (ctypes.c_int, [P, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                             ctypes.c_int, P, P, F64, P, P, P, P]),
    "mlmcp_parareal_finalize": (ctypes.c_int, [P, ctypes.c_int, ctypes.c_int, P, P, P, P]),
    "mlmcp_parareal_delta": (ctypes.c_int, [P, ctypes.c_int, ctypes.c_int, ctypes.c_int, P, P,
                                            ctypes.c_int, P, P]),
    "mlmcp_propagate_path": (ctypes.c_int, [P, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                            ctypes.c_int, ctypes.c_int]),
    "mlmcp_fused_workspace_bytes": (SZ, [ctypes.c_int, ctypes.c_int, ctypes.c_int]),
    "mlmcp_run_fused": (ctypes.c_int, [P, ctypes.c_int, P, P, P, F64, F64, ctypes.c_int, P, P,
                                       ctypes.c_int, P, SZ, P]),
    "mlmcp_draw_uniform": (ctypes.c_int, [ctypes.c_uint64, ctypes.c_uint64, I64, ctypes.c_int,
                                          ctypes.c_int, P, P, P, P]),
    "mlmcp_draw_uniform_host": (ctypes.c_int, [ctypes.c_uint64, ctypes.c_uint64, I64,
                                               ctypes.c_int, ctypes.c_int, P, P, P]),
    "mlmcp_energy": (ctypes.c_int, [P, ctypes.c_int, P, P, P, P, P, P]),
    "mlmcp_level_reduce": (ctypes.c_int, [ctypes.c_int, P, P, P, P]),
}


class LibraryMissingError(RuntimeError):
    pass


def load(path: str = LIB_PATH):
    """Load libmlmcp.so (once) and bind signatures.  Raises if absent."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(path):
            raise LibraryMissingError(
                f"{path} not found: build it with `make` or __graft_entry__.build(); "
                "there is no CPU fallback")
        lib = ctypes.CDLL(path)
        for name, (res, args) in _SIGS.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        if lib.mlmcp_abi_version() != ABI_VERSION:
            raise LibraryMissingError(f"{path} has ABI {lib.mlmcp_abi_version()}, expected "
                                      f"{ABI_VERSION}: rebuild it")
        _lib = lib
        return lib


def last_error() -> str:
    return load().mlmcp_last_error().decode(errors="replace")


def check(rc: int, what: str):
    if rc == 0:
        return
    msg = f"{what}: {last_error()}"
    if rc == EINVAL:
        raise ValueError(msg)
    if rc == ENOMEM:
        raise MemoryError(msg)
    raise RuntimeError(f"{msg} (code {rc})")


def launch_count() -> int:
    return int(load().mlmcp_launch_count())


def ptr(t) -> ctypes.c_void_p | None:
    """Device pointer of a torch tensor (None for None)."""
    if t is None:
        return None
    return ctypes.c_void_p(t.data_ptr())


def np_ptr(a: np.ndarray) -> ctypes.c_void_p:
    return a.ctypes.data_as(ctypes.c_void_p)
