"""The reference's instance interface, mirrored on top of the B200 path.

Reference: ``ConcreteInstance`` (/root/reference/proj/include/raceset/oracle.hpp:17-35),
``parse_instance`` / ``load_instance_file`` (src/oracle.cpp:223-289),
``validate_instance`` (src/oracle.cpp:291-316) and ``run(inst, f)``
(src/oracle.cpp:699-736) executing fixtures/gespmm_alg2.mir.

``run(inst)`` here computes the SpMM the reference kernel computes on that
instance -- on the GPU, through the C-ABI -- and returns C (the reference
returns only its access log and discards C, src/oracle.cpp:735).  With
``reference_launch=True`` (default) it keeps the kernel's launch semantics:

* rows i < min(M, grid.x) are computed (``%i = bid.x; icmp lt %i, %M``,
  gespmm_alg2.mir:7, :13-14); other rows keep their initial C;
* columns j < min(N, grid.y * block.x) (mir:8-12, :44-45);
* C is read-modified-written: C = C0 + A*B (mir:55-59);
* the kernel's shared arrays hold 4 entries (mir:5), so a launch with
  block.x > 4 over a row with more than 4 nonzeros raises OutOfBounds exactly
  as the interpreter does (src/oracle.cpp:673-677).
"""
from __future__ import annotations

import dataclasses
from typing import Dict, List, Optional

import numpy as np

from .errors import Error, ErrorKind

_FLOAT_KINDS = ("f32", "f64")
_INT_KINDS = ("i32", "i64")


@dataclasses.dataclass
class ArrayData:
    elem: str = "i32"
    ints: List[int] = dataclasses.field(default_factory=list)
    floats: List[float] = dataclasses.field(default_factory=list)

    def size(self) -> int:
        return len(self.floats) if self.elem in _FLOAT_KINDS else len(self.ints)


@dataclasses.dataclass
class CsrSpec:
    row_ptr: str = ""
    col_ind: str = ""
    val: str = ""
    cols: int = 0


@dataclasses.dataclass
class ConcreteInstance:
    name: str = ""
    params: Dict[str, int] = dataclasses.field(default_factory=dict)
    arrays: Dict[str, ArrayData] = dataclasses.field(default_factory=dict)
    grid: List[int] = dataclasses.field(default_factory=lambda: [1, 1, 1])
    block: List[int] = dataclasses.field(default_factory=lambda: [1, 1, 1])
    csr: Optional[CsrSpec] = None


def parse_instance(text: str) -> ConcreteInstance:
    """Same grammar and errors as the reference parser (src/oracle.cpp:223-281):
    keywords instance/params/grid/block/array/csr, '#' comments, commas are
    whitespace; validates the CSR triple at the end."""
    inst = ConcreteInstance()
    for lineno, raw in enumerate(text.splitlines(), start=1):
        raw = raw.split("#", 1)[0].replace(",", " ")
        tok = raw.split()
        if not tok:
            continue
        kw = tok[0]
        try:
            if kw == "instance":
                if len(tok) < 2:
                    raise Error(ErrorKind.SyntaxError, "instance name", lineno, 1)
                inst.name = tok[1]
            elif kw == "params":
                for t in tok[1:]:
                    if "=" not in t:
                        raise Error(ErrorKind.SyntaxError, "name=value, got " + t, lineno, 1)
                    k, v = t.split("=", 1)
                    inst.params[k] = int(v)
            elif kw in ("grid", "block"):
                if len(tok) != 4:
                    raise Error(ErrorKind.SyntaxError, "three extents", lineno, 1)
                ext = [int(x) for x in tok[1:4]]
                if any(e < 1 for e in ext):
                    raise Error(ErrorKind.SyntaxError, "extents must be >= 1", lineno, 1)
                if kw == "grid":
                    inst.grid = ext
                else:
                    inst.block = ext
            elif kw == "array":
                if len(tok) < 4 or tok[3] != "=":
                    raise Error(ErrorKind.SyntaxError, "array <name> <elem> = values", lineno, 1)
                elem = tok[2]
                if elem not in _FLOAT_KINDS + _INT_KINDS:
                    raise Error(ErrorKind.SyntaxError, "element type, got " + elem, lineno, 1)
                a = ArrayData(elem=elem)
                if elem in _FLOAT_KINDS:
                    a.floats = [float(x) for x in tok[4:]]
                else:
                    a.ints = [int(x) for x in tok[4:]]
                inst.arrays[tok[1]] = a
            elif kw == "csr":
                if len(tok) != 5 or not tok[4].startswith("cols="):
                    raise Error(ErrorKind.SyntaxError, "csr <rowPtr> <colInd> <val> cols=<n>",
                                lineno, 1)
                inst.csr = CsrSpec(tok[1], tok[2], tok[3], int(tok[4][5:]))
            else:
                raise Error(ErrorKind.SyntaxError, "unknown keyword " + kw, lineno, 1)
        except ValueError as e:  # std::stoll / std::stod failures
            raise Error(ErrorKind.SyntaxError, str(e), lineno, 1) from None
    validate_instance(inst)
    return inst


def load_instance_file(path: str) -> ConcreteInstance:
    try:
        with open(path) as f:
            text = f.read()
    except OSError:
        raise Error(ErrorKind.Io, "cannot open " + path) from None
    return parse_instance(text)


def validate_instance(inst: ConcreteInstance) -> None:
    """The reference's CSR rules (src/oracle.cpp:291-316), same order, same
    messages; raises Error(CsrInvalid)."""
    if inst.csr is None:
        return
    c = inst.csr

    def need(n):
        if n not in inst.arrays:
            raise Error(ErrorKind.CsrInvalid, "missing array " + n)
        return inst.arrays[n]

    rp, ci, vl = need(c.row_ptr), need(c.col_ind), need(c.val)
    if not rp.ints or rp.ints[0] != 0:
        raise Error(ErrorKind.CsrInvalid, c.row_ptr + "[0] must be 0")
    r = np.asarray(rp.ints, dtype=np.int64)
    if np.any(r[1:] < r[:-1]):
        raise Error(ErrorKind.CsrInvalid, c.row_ptr + " must be nondecreasing")
    if int(r[-1]) != ci.size():
        raise Error(ErrorKind.CsrInvalid, c.row_ptr + " end differs from nnz of " + c.col_ind)
    if ci.size() != vl.size():
        raise Error(ErrorKind.CsrInvalid, c.col_ind + " and " + c.val + " lengths differ")
    col = np.asarray(ci.ints, dtype=np.int64)
    if col.size and (col.min() < 0 or col.max() >= c.cols):
        raise Error(ErrorKind.CsrInvalid, f"{c.col_ind} entry out of [0,{c.cols})")


def _floats(inst, name):
    a = inst.arrays.get(name)
    if a is None:
        raise Error(ErrorKind.Io, "instance does not define array " + name)
    vals = a.floats if a.floats or not a.ints else [float(v) for v in a.ints]
    return np.asarray(vals, dtype=np.float64)


def _param(inst, name):
    if name not in inst.params:
        raise Error(ErrorKind.Io, "instance does not set parameter " + name)
    return int(inst.params[name])


def run(inst: ConcreteInstance, reduce: str = "sum", reference_launch: bool = True,
        device="cuda") -> np.ndarray:
    """Computes the gespmm_alg2 SpMM of `inst` on the B200 path; returns C
    (float32, M x N).  See the module docstring for the launch semantics."""
    import torch

    from .spmm import Plan

    validate_instance(inst)
    M, N, K = _param(inst, "M"), _param(inst, "N"), _param(inst, "K")
    if "rowPtr" not in inst.arrays or "colInd" not in inst.arrays:
        raise Error(ErrorKind.Io, "instance does not define array rowPtr/colInd")
    rowptr = np.asarray(inst.arrays["rowPtr"].ints, dtype=np.int64)
    colind = np.asarray(inst.arrays["colInd"].ints, dtype=np.int64)
    vals = _floats(inst, "val").astype(np.float32)
    B = _floats(inst, "B").astype(np.float32)
    C0 = _floats(inst, "C").astype(np.float32)
    if B.size < K * N or C0.size < M * N or rowptr.size < M + 1:
        raise Error(ErrorKind.OutOfBounds, "instance arrays smaller than M/N/K imply")
    if colind.size and (colind.min() < 0 or colind.max() >= K):
        raise Error(ErrorKind.OutOfBounds, f"B[{int(colind.max()) * N}] outside size {K * N}")
    C = C0[: M * N].reshape(M, N).copy()
    if reference_launch:
        if inst.grid[2] != 1 or inst.block[1] != 1 or inst.block[2] != 1:
            raise Error(ErrorKind.UnsupportedConstruct,
                        "gespmm_alg2 launch must have grid.z == block.y == block.z == 1")
        rows = min(M, inst.grid[0])
        cols = min(N, inst.grid[1] * inst.block[0])
        accumulate = True
        if inst.block[0] > 4:  # shared extent [4 x i32] (gespmm_alg2.mir:5)
            deg = np.diff(rowptr[: rows + 1])
            if deg.size and deg.max() > 4:
                raise Error(ErrorKind.OutOfBounds, "sm_k[4] outside size 4")
    else:
        rows, cols, accumulate = M, N, False
    if rows == 0 or cols == 0:
        return C
    dev = torch.device(device)
    rp = torch.as_tensor(rowptr[: rows + 1].astype(np.int32), device=dev)
    nnz = int(rowptr[rows])
    ci = torch.as_tensor(colind[:nnz].astype(np.int32), device=dev)
    vv = torch.as_tensor(vals[:nnz], device=dev)
    Bt = torch.as_tensor(B[: K * N].reshape(K, N)[:, :cols].copy(), device=dev)
    out = torch.as_tensor(C[:rows, :cols].copy(), device=dev)
    plan = Plan(rp, ci, K)
    plan.execute(vv, Bt, reduce=reduce, out=out, accumulate=accumulate)
    C[:rows, :cols] = out.cpu().numpy()
    return C
