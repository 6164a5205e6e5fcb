"""CSR file I/O around the hot path.

* ``.inst`` -- the reference's instance format (parser in ``instance.py``,
  reference src/oracle.cpp:223-289); ``format_instance`` writes it back and
  ``csr_instance`` wraps a CSR x B problem as a ``gespmm_alg2`` instance, so
  large synthetic problems can be handed to the reference interpreter.
* Binary CSR cache (``save_csr`` / ``load_csr``): the graphs of configs 3-5
  take seconds to generate; the cache stores rowptr/colind/vals raw,
  little-endian, 4 KiB-aligned (np.memmap-able, read straight into pinned
  memory or onto the GPU), with a CRC32 per array checked on load.
* Matrix Market coordinate files (``read_matrix_market`` /
  ``write_matrix_market``): real / integer / pattern, general / symmetric /
  skew-symmetric, 1-based; entries keep their file order within a row
  (stable sort by row), duplicates are kept -- like the reference's CSR
  contract, which allows unsorted and repeated columns.
"""
from __future__ import annotations

import io
import json
import os
import struct
import zlib
from typing import Optional, Tuple

import numpy as np

from .errors import Error, ErrorKind
from .instance import ArrayData, ConcreteInstance, CsrSpec, validate_instance

MAGIC = b"GESPMMCSR\x00\x01\x00"  # 12 bytes: name, NUL, format version 1
_ALIGN = 4096


# ---- .inst writer -----------------------------------------------------------

def _fmt_float(x: float) -> str:
    r = repr(float(x))
    return r[:-2] if r.endswith(".0") else r  # "3" not "3.0": the reference prints integers bare


def format_instance(inst: ConcreteInstance) -> str:
    """Text the reference parser (src/oracle.cpp:223-281) reads back into the
    same instance (round trip: parse_instance(format_instance(i)) == i)."""
    out = io.StringIO()
    if inst.name:
        out.write(f"instance {inst.name}\n")
    if inst.params:
        out.write("params " + " ".join(f"{k}={v}" for k, v in inst.params.items()) + "\n")
    out.write("grid {} {} {}\n".format(*inst.grid))
    out.write("block {} {} {}\n".format(*inst.block))
    for name, a in inst.arrays.items():
        vals = a.floats if a.elem in ("f32", "f64") else a.ints
        body = " ".join(_fmt_float(v) for v in vals) if a.elem in ("f32", "f64") else " ".join(
            str(int(v)) for v in vals)
        out.write(f"array {name} {a.elem} = {body}\n")
    if inst.csr is not None:
        c = inst.csr
        out.write(f"csr {c.row_ptr} {c.col_ind} {c.val} cols={c.cols}\n")
    return out.getvalue()


def csr_instance(rowptr, colind, vals, B, C0=None, name: str = "gespmm_csr") -> ConcreteInstance:
    """A ``gespmm_alg2`` instance (kernel params M, N, K, A_S; arrays rowPtr,
    colInd, val, B, C; the reference fixtures' layout, fixtures/gespmm_small.inst)
    with the full launch: grid (M, ceil(N/4), 1) x block (4, 1, 1)."""
    rowptr = np.asarray(rowptr, np.int64)
    B = np.asarray(B, np.float32)
    M = len(rowptr) - 1
    K, N = B.shape
    C = np.zeros((M, N), np.float32) if C0 is None else np.asarray(C0, np.float32)
    inst = ConcreteInstance(
        name=name, params={"M": M, "N": N, "K": K, "A_S": int(rowptr[-1])},
        arrays={"rowPtr": ArrayData("i32", ints=rowptr.tolist()),
                "colInd": ArrayData("i32", ints=np.asarray(colind, np.int64).tolist()),
                "val": ArrayData("f32", floats=np.asarray(vals, np.float64).tolist()),
                "B": ArrayData("f32", floats=B.astype(np.float64).ravel().tolist()),
                "C": ArrayData("f32", floats=C.astype(np.float64).ravel().tolist())},
        grid=[max(M, 1), max((N + 3) // 4, 1), 1], block=[4, 1, 1],
        csr=CsrSpec("rowPtr", "colInd", "val", K))
    validate_instance(inst)
    return inst


# ---- binary CSR cache -------------------------------------------------------

def _pad(n: int) -> int:
    return (n + _ALIGN - 1) // _ALIGN * _ALIGN


def save_csr(path: str, rowptr, colind, vals, M: int, K: int, meta: Optional[dict] = None) -> None:
    """Writes the binary CSR cache (arrays may be numpy or torch, any device)."""
    def host(a, dt):
        if hasattr(a, "detach"):
            a = a.detach().cpu().numpy()
        return np.ascontiguousarray(np.asarray(a), dtype=dt)

    rp, ci, vv = host(rowptr, "<i4"), host(colind, "<i4"), host(vals, "<f4")
    nnz = ci.shape[0]
    if rp.shape[0] != M + 1 or vv.shape[0] != nnz or int(rp[-1]) != nnz:
        raise Error(ErrorKind.CsrInvalid, "invalid csr: save_csr shape mismatch")
    arrays = [("rowptr", rp), ("colind", ci), ("vals", vv)]
    hdr = {"M": int(M), "K": int(K), "nnz": int(nnz), "meta": meta or {}, "arrays": []}
    off = _ALIGN
    for name, a in arrays:
        hdr["arrays"].append({"name": name, "dtype": a.dtype.str, "offset": off, "count": int(a.size),
                              "crc32": zlib.crc32(memoryview(a).cast("B")) & 0xFFFFFFFF})
        off += _pad(a.nbytes)
    js = json.dumps(hdr).encode()
    if len(MAGIC) + 8 + len(js) > _ALIGN:
        raise Error(ErrorKind.InvalidArgument, "save_csr: metadata too large")
    tmp = path + ".tmp"
    with open(tmp, "wb") as f:
        f.write(MAGIC + struct.pack("<Q", len(js)) + js)
        for (name, a), d in zip(arrays, hdr["arrays"]):
            f.seek(d["offset"])
            f.write(memoryview(a).cast("B"))
        f.truncate(off)
    os.replace(tmp, path)  # atomic: a half-written cache is never visible


def load_csr(path: str, verify: bool = True, mmap: bool = True):
    """Reads the cache -> (rowptr int32[M+1], colind int32[nnz], vals f32[nnz],
    M, K, meta); numpy memmaps when mmap=True.  Raises Error(Io) on a bad
    file and Error(CsrInvalid) when a CRC32 does not match."""
    try:
        with open(path, "rb") as f:
            head = f.read(_ALIGN)
    except OSError:
        raise Error(ErrorKind.Io, "cannot open " + path) from None
    if not head.startswith(MAGIC):
        raise Error(ErrorKind.Io, f"{path}: not a gespmm CSR cache")
    (n,) = struct.unpack_from("<Q", head, len(MAGIC))
    hdr = json.loads(head[len(MAGIC) + 8:len(MAGIC) + 8 + n])
    out = {}
    for d in hdr["arrays"]:
        if mmap:
            a = np.memmap(path, dtype=np.dtype(d["dtype"]), mode="r", offset=d["offset"], shape=(d["count"],))
        else:
            a = np.fromfile(path, dtype=np.dtype(d["dtype"]), count=d["count"], offset=d["offset"])
        if verify and (zlib.crc32(memoryview(np.ascontiguousarray(a)).cast("B")) & 0xFFFFFFFF) != d["crc32"]:
            raise Error(ErrorKind.CsrInvalid, f"{path}: {d['name']} checksum mismatch")
        out[d["name"]] = a
    return out["rowptr"], out["colind"], out["vals"], hdr["M"], hdr["K"], hdr.get("meta", {})


def cached_csr(path: str, make, device=None):
    """Loads ``path`` if present, else builds it with ``make()`` -> Csr (numpy or
    torch) and saves it.  Returns a workloads.Csr of torch tensors on
    ``device`` (or numpy arrays when device is None)."""
    from .workloads import Csr

    if not os.path.exists(path):
        c = make()
        save_csr(path, c.rowptr, c.colind, c.vals, c.M, c.K)
    rp, ci, vv, M, K, _ = load_csr(path)
    if device is None:
        return Csr(np.asarray(rp), np.asarray(ci), np.asarray(vv), M, K)
    import torch

    t = lambda a: torch.from_numpy(np.array(a)).to(device)  # noqa: E731  (copy: memmaps are read-only)
    return Csr(t(rp), t(ci), t(vv), M, K)


# ---- Matrix Market ------------------------------------------------------------

def read_matrix_market(path_or_text: str, text: bool = False) -> Tuple[np.ndarray, np.ndarray, np.ndarray, int, int]:
    """Matrix Market coordinate file -> (rowptr, colind, vals, M, K), int32/f32.
    Symmetric / skew-symmetric files are expanded (mirror entries follow the
    stored ones); pattern files get value 1."""
    if text:
        lines = path_or_text.splitlines()
    else:
        try:
            with open(path_or_text) as f:
                lines = f.read().splitlines()
        except OSError:
            raise Error(ErrorKind.Io, "cannot open " + path_or_text) from None
    if not lines or not lines[0].lower().startswith("%%matrixmarket"):
        raise Error(ErrorKind.SyntaxError, "missing %%MatrixMarket banner", 1, 1)
    ban = lines[0].lower().split()
    if len(ban) < 5 or ban[1] != "matrix" or ban[2] != "coordinate":
        raise Error(ErrorKind.SyntaxError, "only 'matrix coordinate' files are supported", 1, 1)
    field, sym = ban[3], ban[4]
    if field not in ("real", "integer", "pattern", "double"):
        raise Error(ErrorKind.SyntaxError, "unsupported field " + field, 1, 1)
    if sym not in ("general", "symmetric", "skew-symmetric"):
        raise Error(ErrorKind.SyntaxError, "unsupported symmetry " + sym, 1, 1)
    i = 1
    while i < len(lines) and (not lines[i].strip() or lines[i].lstrip().startswith("%")):
        i += 1
    try:
        M, K, nz = (int(x) for x in lines[i].split()[:3])
    except (ValueError, IndexError):
        raise Error(ErrorKind.SyntaxError, "size line 'rows cols entries'", i + 1, 1) from None
    body = "\n".join(ln for ln in lines[i + 1:] if ln.strip() and not ln.lstrip().startswith("%"))
    ncol = 2 if field == "pattern" else 3
    data = np.loadtxt(io.StringIO(body), ndmin=2) if body else np.zeros((0, ncol))
    if data.shape[0] != nz or (nz and data.shape[1] < ncol):
        raise Error(ErrorKind.SyntaxError, f"expected {nz} entries with {ncol} fields", i + 2, 1)
    r = data[:, 0].astype(np.int64) - 1 if nz else np.zeros(0, np.int64)
    c = data[:, 1].astype(np.int64) - 1 if nz else np.zeros(0, np.int64)
    v = data[:, 2].astype(np.float32) if (nz and field != "pattern") else np.ones(nz, np.float32)
    if nz and (r.min() < 0 or r.max() >= M or c.min() < 0 or c.max() >= K):
        raise Error(ErrorKind.OutOfBounds, "entry index outside the declared size")
    if sym != "general":
        off = r != c
        r, c, v = (np.concatenate([r, c[off]]), np.concatenate([c, r[off]]),
                   np.concatenate([v, (-v[off] if sym == "skew-symmetric" else v[off])]))
    order = np.argsort(r, kind="stable")
    counts = np.bincount(r, minlength=M)
    rowptr = np.zeros(M + 1, np.int64)
    rowptr[1:] = np.cumsum(counts)
    return rowptr.astype(np.int32), c[order].astype(np.int32), v[order].astype(np.float32), M, K


def write_matrix_market(path: str, rowptr, colind, vals, M: int, K: int, comment: str = "") -> None:
    """CSR -> Matrix Market 'coordinate real general' (1-based, row order);
    values printed with 9 significant digits (fp32 round-trips exactly)."""
    rp = np.asarray(rowptr, np.int64)
    ci = np.asarray(colind, np.int64)
    vv = np.asarray(vals, np.float32)
    rows = np.repeat(np.arange(M, dtype=np.int64), np.diff(rp))
    with open(path, "w") as f:
        f.write("%%MatrixMarket matrix coordinate real general\n")
        for ln in comment.splitlines():
            f.write("% " + ln + "\n")
        f.write(f"{M} {K} {ci.size}\n")
        np.savetxt(f, np.column_stack([rows + 1, ci + 1, vv.astype(np.float64)]), fmt="%d %d %.9g")
