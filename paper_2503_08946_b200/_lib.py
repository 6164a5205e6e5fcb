"""ctypes binding of libgespmm.so (the C-ABI declared in include/gespmm.h).

The library is built in-tree by ``_build.build()``.  There is no fallback: if
the shared library is missing or fails to load, importing the compute API
raises, so a GPU run can never silently take a CPU or library path.
"""
from __future__ import annotations

import ctypes
import os

from .errors import Error, ErrorKind

PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("GESPMM_LIB") or os.path.join(PKG, "libgespmm.so")

OK, CSR_INVALID, OUT_OF_BOUNDS, INVALID_ARG, CUDA_ERROR, NCCL_ERROR, NOT_SUPPORTED = range(7)
REDUCE = {"sum": 0, "max": 1, "min": 2, "mean": 3}
SEGMENT_LEN = 256  # GESPMM_SEGMENT_LEN

# Every symbol include/gespmm.h declares (checked by tests/test_capi.py).
EXPORTS = [
    "gespmm_version", "gespmm_status_string", "gespmm_last_error", "gespmm_validate_csr",
    "gespmm_validate_csr_device", "gespmm_csr_spmm", "gespmm_csr_spmm_host",
    "gespmm_plan_create", "gespmm_plan_execute", "gespmm_plan_execute_rows", "gespmm_plan_destroy",
    "gespmm_plan_execute_peers", "gespmm_ipc_get_handle", "gespmm_ipc_open_handle", "gespmm_ipc_close_handle", "gespmm_plan_get_info",
    "gespmm_variant_name", "gespmm_set_variant_override", "gespmm_set_panel_override",
    "gespmm_panel_width", "gespmm_set_schedule_override", "gespmm_set_tile_work_override", "gespmm_partition_rows",
    "gespmm_rmat_csr", "gespmm_uniform_fill", "gespmm_coo_to_csr", "gespmm_csr_transpose",
    "gespmm_comm_get_unique_id", "gespmm_comm_init", "gespmm_comm_destroy", "gespmm_sharded_spmm",
    "gespmm_sharded_spmm_chunked", "gespmm_sharded_spmm_ex", "gespmm_comm_wait",
    "gespmm_plan_last_variant",
]

_i64 = ctypes.c_int64
_int = ctypes.c_int
_vp = ctypes.c_void_p


class ShardOpts(ctypes.Structure):
    """gespmm_shard_opts_t"""
    _fields_ = [("b_panels", ctypes.c_int), ("b_panel_ws", ctypes.c_void_p), ("c_chunks", ctypes.c_int),
                ("timeout_ms", ctypes.c_int64)]


class PlanInfo(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int64) for n in (
        "M", "nnz", "n_items", "n_tiles", "n_long_rows", "n_segments", "segment_len",
        "tile_work", "kernel_launches_per_execute")]


_lib = None


def load():
    """Loads libgespmm.so (raises if it is not built -- no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is not built; run `python -c 'import __graft_entry__ as g; g.build()'` "
            "(the B200 path has no CPU fallback)")
    L = ctypes.CDLL(LIB_PATH)
    sig = {
        "gespmm_version": ([], _int),
        "gespmm_status_string": ([_int], ctypes.c_char_p),
        "gespmm_last_error": ([], ctypes.c_char_p),
        "gespmm_validate_csr": ([_i64, _i64, _i64, _vp, _i64, _vp, _i64], _int),
        "gespmm_validate_csr_device": ([_i64, _i64, _i64, _vp, _vp, _vp], _int),
        "gespmm_csr_spmm": ([_i64, _i64, _i64, _i64, _vp, _vp, _vp, _vp, _i64, _vp, _i64, _int,
                             _int, _vp], _int),
        "gespmm_csr_spmm_host": ([_i64, _i64, _i64, _i64, _vp, _vp, _vp, _vp, _i64, _vp, _i64,
                                  _int, _int, _vp], _int),
        "gespmm_plan_create": ([ctypes.POINTER(_vp), _i64, _i64, _i64, _vp, _vp, _int, _vp], _int),
        "gespmm_plan_execute": ([_vp, _i64, _vp, _vp, _vp, _vp, _i64, _vp, _i64, _int, _int, _vp],
                                _int),
        "gespmm_plan_execute_rows": ([_vp, _i64, _i64, _i64, _vp, _vp, _vp, _vp, _i64, _vp, _i64,
                                      _int, _int, _vp], _int),
        "gespmm_plan_destroy": ([_vp], _int),
        "gespmm_plan_execute_peers": ([_vp, _i64, _vp, _vp, _vp, _vp, _i64, _vp, _i64, _int, _int, _vp, _int,
                                       _i64, _vp], _int),
        "gespmm_ipc_get_handle": ([_vp, ctypes.c_char_p, ctypes.POINTER(_i64)], _int),
        "gespmm_ipc_open_handle": ([ctypes.c_char_p, ctypes.POINTER(_vp)], _int),
        "gespmm_ipc_close_handle": ([_vp], _int),
        "gespmm_plan_get_info": ([_vp, ctypes.POINTER(PlanInfo)], _int),
        "gespmm_variant_name": ([_i64, _vp, _i64, _vp, _i64, _int], ctypes.c_char_p),
        "gespmm_set_variant_override": ([ctypes.c_char_p], _int),
        "gespmm_set_panel_override": ([_i64], _int),
        "gespmm_plan_last_variant": ([_vp], ctypes.c_char_p),
        "gespmm_panel_width": ([_i64, _i64], _i64),
        "gespmm_set_schedule_override": ([_int], _int),
        "gespmm_set_tile_work_override": ([ctypes.c_int32], _int),
        "gespmm_partition_rows": ([_i64, _vp, _int, _vp], _int),
        "gespmm_rmat_csr": ([_int, _i64, ctypes.c_double, ctypes.c_double, ctypes.c_double,
                             ctypes.c_uint64, _vp, _vp, _vp, ctypes.POINTER(_i64), _vp], _int),
        "gespmm_coo_to_csr": ([_i64, _i64, _vp, _vp, _vp, _vp, _vp, _vp, _vp], _int),
        "gespmm_csr_transpose": ([_i64, _i64, _i64, _vp, _vp, _vp, _vp, _vp, _vp, _vp], _int),
        "gespmm_uniform_fill": ([_vp, _i64, ctypes.c_float, ctypes.c_float, ctypes.c_uint64, _vp], _int),
        "gespmm_comm_get_unique_id": ([ctypes.c_char_p], _int),
        "gespmm_comm_init": ([ctypes.POINTER(_vp), _int, ctypes.c_char_p, _int], _int),
        "gespmm_comm_destroy": ([_vp], _int),
        "gespmm_sharded_spmm": ([_vp, _int, _int, _int, _vp, _i64, _i64, _i64, _i64, _vp, _vp,
                                 _vp, _vp, _i64, _vp, _i64, _int, _int, _vp, _i64, _vp, _vp],
                                _int),
        "gespmm_sharded_spmm_chunked": ([_vp, _int, _int, _int, _vp, _i64, _i64, _i64, _i64, _vp, _vp,
                                         _vp, _vp, _i64, _vp, _i64, _int, _int, _vp, _i64, _vp, _int,
                                         _vp], _int),
        "gespmm_sharded_spmm_ex": ([_vp, _int, _int, _int, _vp, _i64, _i64, _i64, _i64, _vp, _vp,
                                    _vp, _vp, _i64, _vp, _i64, _int, _int, _vp, _i64, _vp,
                                    ctypes.POINTER(ShardOpts), _vp], _int),
        "gespmm_comm_wait": ([_vp, _vp, _i64], _int),
    }
    for name, (args, res) in sig.items():
        f = getattr(L, name)
        f.argtypes = args
        f.restype = res
    _lib = L
    return L


_KIND = {
    CSR_INVALID: ErrorKind.CsrInvalid,
    OUT_OF_BOUNDS: ErrorKind.OutOfBounds,
    INVALID_ARG: ErrorKind.InvalidArgument,
    CUDA_ERROR: ErrorKind.Cuda,
    NCCL_ERROR: ErrorKind.Nccl,
    NOT_SUPPORTED: ErrorKind.UnsupportedConstruct,
}


def check(status: int) -> None:
    """Raises the reference-style Error for a non-OK status."""
    if status == OK:
        return
    L = load()
    detail = L.gespmm_last_error().decode() or L.gespmm_status_string(status).decode()
    kind = _KIND.get(status, ErrorKind.Cuda)
    prefix = kind.label + ": "
    raise Error(kind, detail[len(prefix):] if detail.startswith(prefix) else detail)
