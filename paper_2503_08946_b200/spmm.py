"""Public SpMM API on torch CUDA tensors (PyTorch = device memory + streams only;
all compute is libgespmm.so's sm_100a kernels through the C-ABI).

    C = csr_spmm(rowptr, colind, vals, B, reduce="sum")            # one-shot
    plan = Plan(rowptr, colind, K)                                   # reusable
    plan.execute(vals, B, reduce="max", out=C)                       # async

Reference surface this mirrors: the kernel
``@gespmm_alg2(%rowPtr, %colInd, %val, %B, %C, %M, %N, %K)``
(/root/reference/proj/fixtures/gespmm_alg2.mir:5) run through
``raceset::run`` (src/oracle.cpp:699-736), with the CSR contract of
``validate_instance`` (src/oracle.cpp:291-316).  ``accumulate=True`` is the
reference kernel's read-modify-write of C (gespmm_alg2.mir:55-59); the
default writes C = A (op) B.
"""
from __future__ import annotations

import ctypes

import numpy as np

from . import _lib
from .errors import Error, ErrorKind

_L = _lib.load()  # no library, no API (no CPU fallback)


def _torch():
    import torch

    return torch


def _stream_handle(stream, device):
    torch = _torch()
    if stream is None:
        stream = torch.cuda.current_stream(device)
    return ctypes.c_void_p(stream.cuda_stream)


def _reduce_code(reduce) -> int:
    if isinstance(reduce, int):
        return reduce
    try:
        return _lib.REDUCE[reduce]
    except KeyError:
        raise Error(ErrorKind.InvalidArgument, f"unknown reduce op {reduce!r}") from None


def _check_csr_tensors(rowptr, colind, vals):
    torch = _torch()
    for name, t, dt in (("rowptr", rowptr, torch.int32), ("colind", colind, torch.int32)):
        if t.dtype != dt or not t.is_cuda or not t.is_contiguous():
            raise Error(ErrorKind.InvalidArgument, f"{name} must be a contiguous int32 CUDA tensor")
    if vals is not None and (vals.dtype != torch.float32 or not vals.is_cuda or
                             not vals.is_contiguous()):
        raise Error(ErrorKind.InvalidArgument, "vals must be a contiguous float32 CUDA tensor")
    if vals is not None and vals.numel() != colind.numel():
        raise Error(ErrorKind.CsrInvalid, "colInd and val lengths differ")


def _check_dense(name, t):
    torch = _torch()
    if t.dtype != torch.float32 or not t.is_cuda or t.dim() != 2 or t.stride(1) != 1:
        raise Error(ErrorKind.InvalidArgument,
                    f"{name} must be a 2-D float32 CUDA tensor with unit column stride")


class Plan:
    """The nnz-balanced work decomposition of one sparsity structure
    (gespmm_plan_create).  Reusable for any vals / B / N / reduce op."""

    def __init__(self, rowptr, colind, K: int, validate: bool = True, stream=None):
        _check_csr_tensors(rowptr, colind, None)
        self.M = rowptr.numel() - 1
        self.K = int(K)
        self.nnz = colind.numel()
        self.rowptr = rowptr
        self.colind = colind
        self.device = rowptr.device
        h = ctypes.c_void_p()
        # the plan is built on (and remembers) the device its rowptr lives on
        with _torch().cuda.device(self.device):
            _lib.check(_L.gespmm_plan_create(ctypes.byref(h), self.M, self.K, self.nnz,
                                             rowptr.data_ptr(), colind.data_ptr(),
                                             1 if validate else 0,
                                             _stream_handle(stream, self.device)))
        self._h = h

    def last_variant(self) -> str:
        """The kernel variant this plan's last execute launched ("" before any),
        e.g. "vec4_lpr32_cwm1_ring" (gespmm_plan_last_variant)."""
        return _L.gespmm_plan_last_variant(self._h).decode()

    def info(self) -> dict:
        inf = _lib.PlanInfo()
        _lib.check(_L.gespmm_plan_get_info(self._h, ctypes.byref(inf)))
        return {n: getattr(inf, n) for n, _ in _lib.PlanInfo._fields_}

    def execute(self, vals, B, reduce="sum", out=None, accumulate: bool = False, stream=None):
        torch = _torch()
        _check_csr_tensors(self.rowptr, self.colind, vals)
        _check_dense("B", B)
        if B.shape[0] != self.K:
            raise Error(ErrorKind.InvalidArgument, f"B has {B.shape[0]} rows, expected K={self.K}")
        N = B.shape[1]
        if out is None:
            if accumulate:
                raise Error(ErrorKind.InvalidArgument, "accumulate=True needs out (C0)")
            out = torch.empty((self.M, N), dtype=torch.float32, device=B.device)
        _check_dense("out", out)
        if tuple(out.shape) != (self.M, N):
            raise Error(ErrorKind.InvalidArgument, f"out must be {(self.M, N)}")
        _lib.check(_L.gespmm_plan_execute(
            self._h, N, self.rowptr.data_ptr(), self.colind.data_ptr(), vals.data_ptr(),
            B.data_ptr(), B.stride(0), out.data_ptr(), out.stride(0), _reduce_code(reduce),
            1 if accumulate else 0, _stream_handle(stream, B.device)))
        return out

    def execute_rows(self, vals, B, row_begin: int, row_end: int, out, reduce="sum",
                     accumulate: bool = False, stream=None):
        """One row chunk of execute (gespmm_plan_execute_rows): after chunks
        [0, r1), [r1, r2), ..., [r_j, r_j+1) ran in order on one stream, C rows
        < r_j+1 are final.  All chunks together equal execute() bit for bit."""
        _check_csr_tensors(self.rowptr, self.colind, vals)
        _check_dense("B", B)
        _check_dense("out", out)
        N = B.shape[1]
        if B.shape[0] != self.K or tuple(out.shape) != (self.M, N):
            raise Error(ErrorKind.InvalidArgument, "B must be K x N and out M x N")
        _lib.check(_L.gespmm_plan_execute_rows(
            self._h, int(row_begin), int(row_end), N, self.rowptr.data_ptr(), self.colind.data_ptr(),
            vals.data_ptr(), B.data_ptr(), B.stride(0), out.data_ptr(), out.stride(0),
            _reduce_code(reduce), 1 if accumulate else 0, _stream_handle(stream, B.device)))
        return out

    def execute_peers(self, vals, B, out, peers, peer_row0: int, reduce="sum", accumulate: bool = False,
                      stream=None):
        """execute() with the fused C all-gather (gespmm_plan_execute_peers):
        every C row also goes to each device pointer in `peers` (full-C
        buffers with out's leading dimension) at row peer_row0 + local row."""
        _check_csr_tensors(self.rowptr, self.colind, vals)
        _check_dense("B", B)
        _check_dense("out", out)
        N = B.shape[1]
        if B.shape[0] != self.K or tuple(out.shape) != (self.M, N):
            raise Error(ErrorKind.InvalidArgument, "B must be K x N and out M x N")
        arr = (ctypes.c_void_p * max(1, len(peers)))(*[int(p) for p in peers])
        _lib.check(_L.gespmm_plan_execute_peers(
            self._h, N, self.rowptr.data_ptr(), self.colind.data_ptr(), vals.data_ptr(), B.data_ptr(),
            B.stride(0), out.data_ptr(), out.stride(0), _reduce_code(reduce), 1 if accumulate else 0, arr,
            len(peers), int(peer_row0), _stream_handle(stream, B.device)))
        return out

    def close(self):
        if getattr(self, "_h", None):
            _L.gespmm_plan_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def csr_spmm(rowptr, colind, vals, B, reduce="sum", out=None, accumulate: bool = False,
             stream=None):
    """One-shot C = A (reduce) B on CUDA tensors (gespmm_csr_spmm): validates the
    CSR on the device, plans, launches."""
    torch = _torch()
    _check_csr_tensors(rowptr, colind, vals)
    _check_dense("B", B)
    M, K, N = rowptr.numel() - 1, B.shape[0], B.shape[1]
    if out is None:
        if accumulate:
            raise Error(ErrorKind.InvalidArgument, "accumulate=True needs out (C0)")
        out = torch.empty((M, N), dtype=torch.float32, device=B.device)
    _check_dense("out", out)
    with torch.cuda.device(B.device):
        _lib.check(_L.gespmm_csr_spmm(M, K, N, colind.numel(), rowptr.data_ptr(), colind.data_ptr(),
                                      vals.data_ptr(), B.data_ptr(), B.stride(0), out.data_ptr(),
                                      out.stride(0), _reduce_code(reduce), 1 if accumulate else 0,
                                      _stream_handle(stream, B.device)))
    return out


def _np(a, dt):
    return np.ascontiguousarray(a, dtype=dt)


def csr_spmm_host(rowptr, colind, vals, B, reduce="sum", C0=None, out=None):
    """One-shot SpMM on HOST (numpy or pinned torch CPU) buffers through
    gespmm_csr_spmm_host: H2D, device validation, plan, kernel, D2H."""
    torch = _torch()

    def ptr(a):
        if isinstance(a, torch.Tensor):
            return a.data_ptr()
        return a.ctypes.data

    if not isinstance(rowptr, torch.Tensor):
        rowptr = _np(rowptr, np.int32)
        colind = _np(colind, np.int32)
        vals = _np(vals, np.float32)
        B = _np(B, np.float32)
    M = rowptr.shape[0] - 1
    K, N = B.shape
    accumulate = C0 is not None
    if out is None:
        # pinned by default: a device-to-host copy into pageable memory blocks
        # the issuing thread, which would serialize the pipelined chunks
        pinned = torch.empty((M, N), dtype=torch.float32, pin_memory=torch.cuda.is_available())
        out = pinned if isinstance(B, torch.Tensor) else pinned.numpy()
    if accumulate:
        if isinstance(out, torch.Tensor):
            out.copy_(torch.as_tensor(C0))
        else:
            out[...] = C0
    _lib.check(_L.gespmm_csr_spmm_host(M, K, N, colind.shape[0], ptr(rowptr), ptr(colind),
                                       ptr(vals), ptr(B), N, ptr(out), N, _reduce_code(reduce),
                                       1 if accumulate else 0, None))
    return out


def validate_csr(M: int, K: int, rowptr, colind, vals_len=None) -> None:
    """Host CSR validation with the reference's rules (raises Error(CsrInvalid))."""
    rp = _np(rowptr, np.int32)
    ci = _np(colind, np.int32)
    n = ci.shape[0] if vals_len is None else int(vals_len)
    _lib.check(_L.gespmm_validate_csr(M, K, rp.shape[0], rp.ctypes.data, ci.shape[0],
                                      ci.ctypes.data, n))


def validate_csr_device(rowptr, colind, K: int, stream=None) -> None:
    _check_csr_tensors(rowptr, colind, None)
    _lib.check(_L.gespmm_validate_csr_device(rowptr.numel() - 1, K, colind.numel(),
                                             rowptr.data_ptr(), colind.data_ptr(),
                                             _stream_handle(stream, rowptr.device)))


def partition_rows(rowptr, parts: int) -> np.ndarray:
    """nnz(+rows)-balanced contiguous row blocks for `parts` ranks (host)."""
    rp = _np(rowptr, np.int32)
    bounds = np.zeros(parts + 1, np.int64)
    _lib.check(_L.gespmm_partition_rows(rp.shape[0] - 1, rp.ctypes.data, parts,
                                        bounds.ctypes.data))
    return bounds


def variant_name(N: int, B=None, out=None, reduce="sum") -> str:
    bp = B.data_ptr() if B is not None else 0
    cp = out.data_ptr() if out is not None else 0
    ldb = B.stride(0) if B is not None else N
    ldc = out.stride(0) if out is not None else N
    return _L.gespmm_variant_name(N, bp, ldb, cp, ldc, _reduce_code(reduce)).decode()


def set_variant_override(name: str = "") -> None:
    _lib.check(_L.gespmm_set_variant_override(name.encode()))


def coo_to_csr(rows, cols, vals, M: int, stream=None):
    """COO (torch CUDA int32 rows/cols, float32 vals) -> (rowptr, colind, vals)
    CSR on the GPU (gespmm_coo_to_csr): stable by row, duplicates kept."""
    torch = _torch()
    nnz = rows.numel()
    rowptr = torch.empty(M + 1, dtype=torch.int32, device=rows.device)
    colind = torch.empty(max(nnz, 1), dtype=torch.int32, device=rows.device)
    v = torch.empty(max(nnz, 1), dtype=torch.float32, device=rows.device)
    _lib.check(_L.gespmm_coo_to_csr(M, nnz, rows.data_ptr(), cols.data_ptr(), vals.data_ptr(), rowptr.data_ptr(),
                                    colind.data_ptr(), v.data_ptr(), _stream_handle(stream, rows.device)))
    return rowptr, colind[:nnz], v[:nnz]


def csr_transpose(rowptr, colind, vals, K: int, stream=None):
    """CSR of A (M x K) -> CSR of A^T (K x M) on the GPU (gespmm_csr_transpose);
    row j of A^T lists column j's nonzeros in ascending row order."""
    torch = _torch()
    M = rowptr.numel() - 1
    nnz = colind.numel()
    t_rp = torch.empty(K + 1, dtype=torch.int32, device=rowptr.device)
    t_ci = torch.empty(max(nnz, 1), dtype=torch.int32, device=rowptr.device)
    t_v = torch.empty(max(nnz, 1), dtype=torch.float32, device=rowptr.device)
    _lib.check(_L.gespmm_csr_transpose(M, K, nnz, rowptr.data_ptr(), colind.data_ptr(), vals.data_ptr(),
                                       t_rp.data_ptr(), t_ci.data_ptr(), t_v.data_ptr(),
                                       _stream_handle(stream, rowptr.device)))
    return t_rp, t_ci[:nnz], t_v[:nnz]


def ipc_handle(t) -> tuple:
    """(64-byte CUDA IPC handle of the allocation holding tensor t, byte offset
    of t in it) -- for the fused all-gather's peer buffers."""
    h = ctypes.create_string_buffer(64)
    off = ctypes.c_int64(0)
    _lib.check(_L.gespmm_ipc_get_handle(ctypes.c_void_p(t.data_ptr()), h, ctypes.byref(off)))
    return bytes(h.raw), int(off.value)


def ipc_open(handle: bytes) -> int:
    """Maps a peer's allocation (CUDA IPC); returns its base device address."""
    p = ctypes.c_void_p()
    _lib.check(_L.gespmm_ipc_open_handle(handle, ctypes.byref(p)))
    return int(p.value)


def ipc_close(base: int) -> None:
    _lib.check(_L.gespmm_ipc_close_handle(ctypes.c_void_p(base)))


def panel_width(K: int, N: int) -> int:
    """Columns per kernel launch gespmm_plan_execute uses for K x N."""
    return int(_L.gespmm_panel_width(int(K), int(N)))


def set_schedule_override(mode: int = -1) -> None:
    """Item distribution: -1 automatic, 0 static warp striding, 1 dynamic counter."""
    _lib.check(_L.gespmm_set_schedule_override(int(mode)))


def set_tile_work_override(units: int = 0) -> None:
    """Tile size (work units) of plans built afterwards: 0 = automatic; results
    never depend on it.  Test/tuning knob (gespmm_set_tile_work_override)."""
    _lib.check(_L.gespmm_set_tile_work_override(int(units)))


def set_panel_override(cols: int = -1) -> None:
    """Column-panel width: -1 heuristic, 0 never split, > 0 forced width."""
    _lib.check(_L.gespmm_set_panel_override(int(cols)))
