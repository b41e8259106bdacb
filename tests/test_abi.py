"""CPU: libmlmcp.so loads, exports every symbol include/mlmcp.h declares, the
task struct layout matches the header, and host-side validation in the C ABI
rejects bad inputs (no kernel launches: no GPU needed)."""

import ctypes
import os
import re

import numpy as np
import pytest

from conftest import ROOT
from paper_2507_19246_b200 import _lib


def header_functions():
    src = open(os.path.join(ROOT, "include", "mlmcp.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(mlmcp_[a-z_0-9]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    lib = _lib.load()
    names = header_functions()
    assert len(names) >= 15
    for n in names:
        assert hasattr(lib, n), n
    assert sorted(_lib.EXPORTS) == names


def test_abi_version_and_counters():
    lib = _lib.load()
    assert lib.mlmcp_abi_version() == _lib.ABI_VERSION == 11
    assert _lib.launch_count() >= 0


def test_task_struct_layout_matches_header():
    src = open(os.path.join(ROOT, "include", "mlmcp.h")).read()
    body = src[src.index("typedef struct mlmcp_task {"):src.index("} mlmcp_task;")]
    fields = re.findall(r"(int32_t|int64_t|double)\s+(\w+);", body)
    assert [f for _, f in fields] == list(_lib.TASK_DTYPE.names)
    size = {"int32_t": 4, "int64_t": 8, "double": 8}
    for (ty, name) in fields:
        assert _lib.TASK_DTYPE.fields[name][0].itemsize == size[ty]
    assert _lib.TASK_DTYPE.itemsize == 96
    assert "96 bytes" in src


def create(row_ptr, col):
    lib = _lib.load()
    h = ctypes.c_void_p()
    rp = np.asarray(row_ptr, dtype=np.int32)
    cl = np.asarray(col, dtype=np.int32)
    rc = lib.mlmcp_ctx_create(0, len(rp) - 1, len(cl), _lib.np_ptr(rp), _lib.np_ptr(cl),
                              ctypes.byref(h))
    return rc, h


@pytest.mark.parametrize("row_ptr,col,msg", [
    ([0, 1, 1], [0], "empty"),                       # row without entries
    ([0, 2, 3], [1, 0, 1], "sorted"),                # unsorted columns
    ([0, 1, 2], [1, 0], "diagonal"),                 # no diagonal
    ([0, 1, 2], [0, 5], "range"),                    # column out of range
    ([0, 9] + [9], list(range(9)), "at most 8"),     # too wide a row
])
def test_ctx_create_validates_pattern(row_ptr, col, msg):
    rc, _ = create(row_ptr, col)
    assert rc == _lib.EINVAL
    assert msg in _lib.last_error()


def test_error_mapping():
    with pytest.raises(ValueError):
        _lib.check(_lib.EINVAL, "x")
    with pytest.raises(MemoryError):
        _lib.check(_lib.ENOMEM, "x")
    with pytest.raises(RuntimeError):
        _lib.check(_lib.ECUDA, "x")


def test_device_entry_points_refuse_without_gpu():
    """No CPU fallback: the engine raises when CUDA is absent."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2507_19246_b200.engine import require_cuda
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        require_cuda()


def test_missing_library_raises(tmp_path):
    with pytest.raises(_lib.LibraryMissingError):
        _lib.load.__wrapped__(str(tmp_path / "nope.so")) if hasattr(_lib.load, "__wrapped__") \
            else _load_fresh(str(tmp_path / "nope.so"))


def _load_fresh(path):
    saved = _lib._lib
    _lib._lib = None
    try:
        return _lib.load(path)
    finally:
        _lib._lib = saved


@pytest.mark.parametrize("name,cls", [("mlmcp_task_arrays", "TaskArrays"),
                                      ("mlmcp_parareal_batch", "PararealBatch")])
def test_batch_struct_layout_matches_header(name, cls):
    src = open(os.path.join(ROOT, "include", "mlmcp.h")).read()
    body = src[src.index("typedef struct %s {" % name):src.index("} %s;" % name)]
    body = re.sub(r"/\*.*?\*/", "", body, flags=re.S)
    fields = re.findall(r"(\w+)\s*;", body)
    st = getattr(_lib, cls)
    assert [f[0] for f in st._fields_] == fields
