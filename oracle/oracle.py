"""CPU oracle wrappers -- TEST INFRASTRUCTURE ONLY.

Only tests/, ``__graft_entry__.smoke()`` and the ``cpu_baseline`` /
``--impl reference`` legs of ``bench.py`` may import this module.  The product
path (``paper_2503_08946_b200``) never imports it.

* ``liboracle.so`` (oracle/gespmm_oracle.c): the C restatement of the
  reference algorithm -- an fp64 restatement of the reference interpreter's
  arithmetic, and the fp32 twin that defines the B200 path's bit-exact
  semantics.
* ``_ref/libgespmm_ref.so`` (oracle/ref_replay.cpp + the reference's own
  library compiled in place): the unmodified reference interpreter
  (``raceset::run``, /root/reference/proj/src/oracle.cpp:699-736) with log
  replay to recover C.  Present only when ``make -C oracle ref`` ran where the
  reference tree exists (it then travels to the GPU box prebuilt).
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "liboracle.so")
REF_LIB_PATH = os.path.join(HERE, "_ref", "libgespmm_ref.so")

SUM, MAX, MIN, MEAN = 0, 1, 2, 3
OPS = {"sum": SUM, "max": MAX, "min": MIN, "mean": MEAN}

_i64 = ctypes.c_int64
_ptr = ctypes.c_void_p

_lib = None
_ref = None


def build(ref: bool = True) -> None:
    subprocess.run(["make", "-s", "-C", HERE, "all"], check=True)
    if ref:
        subprocess.run(["make", "-s", "-C", HERE, "ref"], check=True)


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build(ref=False)
        L = ctypes.CDLL(LIB_PATH)
        L.oracle_validate_csr.argtypes = [_i64, _i64, _i64, _ptr, _i64, _ptr, _i64]
        L.oracle_validate_csr.restype = ctypes.c_int
        L.oracle_spmm_ref_f64.argtypes = [_i64, _i64, _ptr, _ptr, _ptr, _ptr, _i64, _ptr, _i64,
                                          ctypes.c_int]
        L.oracle_spmm_ref_f64.restype = None
        L.oracle_spmm_absbound_f64.argtypes = [_i64, _i64, _ptr, _ptr, _ptr, _ptr, _i64, _ptr,
                                               _i64, ctypes.c_int]
        L.oracle_spmm_absbound_f64.restype = None
        L.oracle_spmm_ref64_op.argtypes = [_i64, _i64, _ptr, _ptr, _ptr, _ptr, _i64, _ptr, _ptr,
                                           ctypes.c_int, ctypes.c_int]
        L.oracle_spmm_ref64_op.restype = None
        L.oracle_spmm_f32.argtypes = [_i64, _i64, _ptr, _ptr, _ptr, _ptr, _i64, _ptr, _i64,
                                      ctypes.c_int, ctypes.c_int, _i64, ctypes.c_int]
        L.oracle_spmm_f32.restype = ctypes.c_int
        L.oracle_num_threads.restype = ctypes.c_int
        _lib = L
    return _lib


def ref_available() -> bool:
    return os.path.exists(REF_LIB_PATH)


def ref_lib():
    global _ref
    if _ref is None:
        if not ref_available():
            raise RuntimeError("oracle/_ref/libgespmm_ref.so not built (make -C oracle ref)")
        L = ctypes.CDLL(REF_LIB_PATH)
        L.ref_last_error.restype = ctypes.c_char_p
        L.ref_run_instance_text.argtypes = [ctypes.c_char_p, _ptr, _i64, _ptr, _ptr]
        L.ref_run_instance_text.restype = ctypes.c_int
        L.ref_spmm_csr.argtypes = [_i64, _i64, _ptr, _ptr, _ptr, _ptr, _i64, _ptr, ctypes.c_int,
                                   _i64, _ptr, _ptr]
        L.ref_spmm_csr.restype = ctypes.c_int
        _ref = L
    return _ref


def _p(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def _c(a, dtype):
    return np.ascontiguousarray(a, dtype=dtype)


def validate_csr(M, K, rowptr, colind, vals_len=None) -> int:
    rowptr = _c(rowptr, np.int32)
    colind = _c(colind, np.int32)
    vals_len = len(colind) if vals_len is None else vals_len
    return lib().oracle_validate_csr(M, K, len(rowptr), _p(rowptr), len(colind), _p(colind),
                                     vals_len)


def spmm_ref_f64(rowptr, colind, vals, B, C0=None, nthreads: int = 0) -> np.ndarray:
    """fp64 restatement of the reference interpreter: C = C0 + A*B, ascending p,
    unfused (reference oracle.cpp:593-613, gespmm_alg2.mir:51-59)."""
    rowptr = _c(rowptr, np.int32)
    colind = _c(colind, np.int32)
    vals = _c(vals, np.float64)
    B = _c(B, np.float64)
    M, N = len(rowptr) - 1, B.shape[1]
    C = np.zeros((M, N), np.float64) if C0 is None else _c(C0, np.float64).copy()
    lib().oracle_spmm_ref_f64(M, N, _p(rowptr), _p(colind), _p(vals), _p(B), N, _p(C), N,
                              nthreads)
    return C


def spmm_ref64_op(rowptr, colind, vals, B, op="sum", nthreads: int = 0):
    """The reference restatement for every reduce op in fp64 on fp32 inputs
    (oracle_spmm_ref64_op): returns (value f64 [M, N], bound f64 [M, N]) with
    bound = sum_p |val*B| (mean: / deg), the north star's tolerance scale."""
    rowptr = _c(rowptr, np.int32)
    colind = _c(colind, np.int32)
    vals = _c(vals, np.float32)
    B = _c(B, np.float32)
    M, N = len(rowptr) - 1, B.shape[1]
    out = np.zeros((M, N), np.float64)
    bound = np.zeros((M, N), np.float64)
    lib().oracle_spmm_ref64_op(M, N, _p(rowptr), _p(colind), _p(vals), _p(B), N, _p(out),
                               _p(bound), OPS[op] if isinstance(op, str) else int(op), nthreads)
    return out, bound


def ref64_error_ratio(got, ref, bound, op="sum"):
    """North-star parity of a GPU result against the fp64 reference
    restatement: sum/mean -> max |got - ref| / (1e-5 * max(|ref|, bound))
    (<= 1 passes); max/min -> the number of cells where got != (float32)ref
    (0 passes: bit-exact up to the sign of zero)."""
    got = np.asarray(got)
    if op in ("max", "min"):
        return int(np.count_nonzero(got.astype(np.float32) != ref.astype(np.float32)))
    scale = np.maximum(np.abs(ref), bound)
    err = np.abs(got.astype(np.float64) - ref)
    with np.errstate(invalid="ignore", divide="ignore"):
        r = np.where(scale > 0, err / (1e-5 * scale), np.where(err > 0, np.inf, 0.0))
    return float(r.max()) if r.size else 0.0


def spmm_absbound(rowptr, colind, vals, B, nthreads: int = 0) -> np.ndarray:
    rowptr = _c(rowptr, np.int32)
    colind = _c(colind, np.int32)
    vals = _c(vals, np.float32)
    B = _c(B, np.float32)
    M, N = len(rowptr) - 1, B.shape[1]
    out = np.zeros((M, N), np.float64)
    lib().oracle_spmm_absbound_f64(M, N, _p(rowptr), _p(colind), _p(vals), _p(B), N, _p(out),
                                   N, nthreads)
    return out


def spmm_f32(rowptr, colind, vals, B, op="sum", accumulate=False, C0=None, seg_len: int = 0,
             nthreads: int = 0) -> np.ndarray:
    """The fp32 twin (normative semantics of the B200 path)."""
    rowptr = _c(rowptr, np.int32)
    colind = _c(colind, np.int32)
    vals = _c(vals, np.float32)
    B = _c(B, np.float32)
    M, N = len(rowptr) - 1, B.shape[1]
    if accumulate:
        C = _c(C0, np.float32).copy()
    else:
        C = np.zeros((M, N), np.float32)
    rc = lib().oracle_spmm_f32(M, N, _p(rowptr), _p(colind), _p(vals), _p(B), N, _p(C), N,
                               OPS[op] if isinstance(op, str) else int(op), int(bool(accumulate)),
                               int(seg_len), nthreads)
    if rc != 0:
        raise ValueError(f"oracle_spmm_f32 rc={rc}")
    return C


def num_threads() -> int:
    return lib().oracle_num_threads()


def ref_run_instance_text(text: str):
    """Run the reference interpreter on .inst text; returns (C float64 array, log_len)."""
    L = ref_lib()
    cap = 1 << 22
    out = np.zeros(cap, np.float64)
    n = ctypes.c_int64(0)
    logn = ctypes.c_int64(0)
    rc = L.ref_run_instance_text(text.encode(), _p(out), cap, ctypes.byref(n), ctypes.byref(logn))
    if rc != 0:
        raise RuntimeError(f"reference run failed rc={rc}: {L.ref_last_error().decode()}")
    return out[: n.value].copy(), logn.value


def ref_spmm_csr(rowptr, colind, vals, B, nthreads: int = 1, want_c: bool = True,
                 C0=None, step_limit: int = 1 << 40):
    """Reference interpreter SpMM over a CSR; returns (C or None, seconds, log_entries)."""
    L = ref_lib()
    rowptr = _c(rowptr, np.int32)
    colind = _c(colind, np.int32)
    vals = _c(vals, np.float32)
    B = _c(B, np.float32)
    M, N = len(rowptr) - 1, B.shape[1]
    C = None
    if want_c:
        C = np.zeros((M, N), np.float64) if C0 is None else _c(C0, np.float64).copy()
    secs = ctypes.c_double(0)
    logn = ctypes.c_int64(0)
    rc = L.ref_spmm_csr(M, N, _p(rowptr), _p(colind), _p(vals), _p(B), N,
                        _p(C) if C is not None else None, nthreads, step_limit,
                        ctypes.byref(secs), ctypes.byref(logn))
    if rc != 0:
        raise RuntimeError(f"reference spmm failed rc={rc}: {L.ref_last_error().decode()}")
    return C, secs.value, logn.value
