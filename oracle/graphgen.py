"""TEST INFRASTRUCTURE ONLY -- numpy restatement of the native synthetic-input
generator (paper_2503_08946_b200/csrc/gespmm_graphgen.cu),
used by tests/ to check gespmm_rmat_csr / gespmm_uniform_fill bit for bit.

Philox4x32-10 follows Salmon, Moraes, Dror, Shaw, "Parallel random numbers: as
easy as 1, 2, 3" (SC'11), Random123's philox4x32 round and Weyl key schedule;
pinned by the published Random123 known-answer vectors (tests/test_graphgen.py).
The R-MAT recursion is Graph500's (no vertex permutation), as SURVEY.md 8(d)
specifies for configs 2/4/5.
"""
from __future__ import annotations

import numpy as np

M0, M1 = np.uint64(0xD2511F53), np.uint64(0xCD9E8D57)
W0, W1 = np.uint32(0x9E3779B9), np.uint32(0xBB67AE85)
MASK32 = np.uint64(0xFFFFFFFF)


def philox4x32_10(c0, c1, c2, c3, k0, k1):
    """Vectorized Philox4x32-10: uint32 arrays (broadcast) -> 4 uint32 arrays."""
    c = [np.asarray(x, dtype=np.uint32) for x in (c0, c1, c2, c3)]
    c = np.broadcast_arrays(*c)
    c = [x.copy() for x in c]
    k0 = np.uint32(k0)
    k1 = np.uint32(k1)
    for _ in range(10):
        p0 = M0 * c[0].astype(np.uint64)
        p1 = M1 * c[2].astype(np.uint64)
        h0 = (p0 >> np.uint64(32)).astype(np.uint32)
        l0 = (p0 & MASK32).astype(np.uint32)
        h1 = (p1 >> np.uint64(32)).astype(np.uint32)
        l1 = (p1 & MASK32).astype(np.uint32)
        c = [h1 ^ c[1] ^ k0, l1, h0 ^ c[3] ^ k1, l0]
        with np.errstate(over="ignore"):
            k0 = np.uint32((int(k0) + int(W0)) & 0xFFFFFFFF)
            k1 = np.uint32((int(k1) + int(W1)) & 0xFFFFFFFF)
    return c


def _thr(p: float) -> int:
    x = p * 4294967296.0
    return int(min(x, 4294967295.0))


def rmat_keys(scale: int, edges: int, a: float, b: float, c: float, seed: int) -> np.ndarray:
    """gespmm_graphgen.cu k_rmat_keys: key = row << scale | col per edge (uint64)."""
    ta, tab, tabc = _thr(a), _thr(a + b), _thr(a + b + c)
    e = np.arange(edges, dtype=np.uint64)
    e_lo = (e & MASK32).astype(np.uint32)
    e_hi = (e >> np.uint64(32)).astype(np.uint32)
    s0, s1 = seed & 0xFFFFFFFF, (seed >> 32) & 0xFFFFFFFF
    row = np.zeros(edges, np.uint64)
    col = np.zeros(edges, np.uint64)
    for l0 in range(0, scale, 4):
        r = philox4x32_10(e_lo, e_hi, np.uint32(l0), np.uint32(0x52414D54), s0, s1)
        for k in range(4):
            lv = l0 + k
            if lv >= scale:
                break
            u = r[k].astype(np.uint64)
            rb = (u >= tab).astype(np.uint64)
            cb = (((u >= ta) & (u < tab)) | (u >= tabc)).astype(np.uint64)
            row |= rb << np.uint64(lv)
            col |= cb << np.uint64(lv)
    return (row << np.uint64(scale)) | col


def uniform(n: int, lo: float, hi: float, seed: int) -> np.ndarray:
    """gespmm_graphgen.cu k_uniform_vals: lo + (hi - lo) * u, u = (x >> 8) / 2^24 (fp32)."""
    i = np.arange(n, dtype=np.uint64)
    r = philox4x32_10((i & MASK32).astype(np.uint32), (i >> np.uint64(32)).astype(np.uint32),
                      np.uint32(0x56414C53), np.uint32(0), seed & 0xFFFFFFFF, (seed >> 32) & 0xFFFFFFFF)
    u = (r[0] >> np.uint32(8)).astype(np.float32) * np.float32(1.0 / 16777216.0)
    return (np.float32(lo) + np.float32(hi - lo) * u).astype(np.float32)


def rmat_csr(scale: int, edges: int, a=0.57, b=0.19, c=0.19, seed=3):
    """gespmm_rmat_csr restated: keys -> sort -> unique -> (rowptr, colind, vals)."""
    keys = np.unique(rmat_keys(scale, edges, a, b, c, seed))
    n = 1 << scale
    rows = (keys >> np.uint64(scale)).astype(np.int64)
    colind = (keys & np.uint64(n - 1)).astype(np.int32)
    rowptr = np.zeros(n + 1, np.int64)
    np.add.at(rowptr, rows + 1, 1)
    rowptr = np.cumsum(rowptr).astype(np.int32)
    vals_seed = ((seed & 0xFFFFFFFF) ^ 0x5EED) | (seed >> 32 << 32)
    vals = uniform(len(keys), -1.0, 1.0, vals_seed)
    return rowptr, colind, vals
