"""Synthetic CSR workloads for the BASELINE.json configs.

All matrices are fp32 values / int32 indices, seeded and reproducible:

* ``uniform_csr``  -- Bernoulli(density) pattern (config 1: 4096^2, 1%, seed 1).
* ``rmat_csr``     -- Graph500 R-MAT (a, b, c, d) = (.57, .19, .19, .05), edges
  deduplicated and sorted into CSR (configs 2, 4, 5).  Runs on any torch device;
  on a B200 the 16M-edge scale-20 graph takes well under a second.
* ``reddit_like_csr`` -- power-law degree sequence with the Reddit graph's shape
  (233K rows, ~115M nnz, mean degree ~492) for config 3.

Values and B are U(-1, 1).  These generators are the "step before the path"
(SURVEY.md section 8 row f3); the hot path itself is paper_2503_08946_b200.spmm.
"""
from __future__ import annotations

import dataclasses

import numpy as np


@dataclasses.dataclass
class Csr:
    rowptr: "np.ndarray | object"  # int32 [M+1] (numpy or torch)
    colind: "np.ndarray | object"  # int32 [nnz]
    vals: "np.ndarray | object"    # float32 [nnz]
    M: int
    K: int

    @property
    def nnz(self) -> int:
        return int(self.colind.shape[0])


def uniform_csr(M: int, K: int, density: float, seed: int = 1) -> Csr:
    """Bernoulli(density) sparsity, vals ~ U(-1,1) fp32 (numpy, host)."""
    rng = np.random.default_rng(seed)
    rowptr = np.zeros(M + 1, np.int64)
    cols = []
    for r0 in range(0, M, 1024):
        r1 = min(M, r0 + 1024)
        mask = rng.random((r1 - r0, K)) < density
        rowptr[r0 + 1:r1 + 1] = mask.sum(1)
        cols.append(np.nonzero(mask)[1])
    rowptr = np.cumsum(rowptr).astype(np.int32)
    colind = (np.concatenate(cols) if cols else np.zeros(0, np.int64)).astype(np.int32)
    vals = rng.uniform(-1.0, 1.0, colind.shape[0]).astype(np.float32)
    return Csr(rowptr, colind, vals, M, K)


def dense(K: int, N: int, seed: int = 2) -> np.ndarray:
    rng = np.random.default_rng(seed)
    return rng.uniform(-1.0, 1.0, (K, N)).astype(np.float32)


def rmat_csr(scale: int, edges: int, seed: int = 3, device="cpu", a=0.57, b=0.19, c=0.19,
             chunk: int = 1 << 26):
    """Graph500 R-MAT on a torch device -> deduplicated, row-sorted CSR (torch tensors).

    Each edge picks one quadrant per level with probabilities (a, b, c, d); the
    row bit is set in quadrants c/d, the column bit in b/d.  Duplicates are
    removed (torch.unique on row*2^scale+col), which also sorts by (row, col).
    """
    import torch

    dev = torch.device(device)
    g = torch.Generator(device=dev)
    g.manual_seed(seed)
    n = 1 << scale
    keys = []
    for e0 in range(0, edges, chunk):
        m = min(chunk, edges - e0)
        row = torch.zeros(m, dtype=torch.int64, device=dev)
        col = torch.zeros(m, dtype=torch.int64, device=dev)
        for bit in range(scale):
            r = torch.rand(m, generator=g, device=dev)
            rbit = r >= (a + b)
            cbit = ((r >= a) & (r < a + b)) | (r >= (a + b + c))
            row |= rbit.to(torch.int64) << bit
            col |= cbit.to(torch.int64) << bit
        keys.append(row * n + col)
        del row, col
    key = torch.unique(torch.cat(keys))
    del keys
    rows = key // n
    colind = (key % n).to(torch.int32)
    counts = torch.bincount(rows, minlength=n)
    rowptr = torch.zeros(n + 1, dtype=torch.int64, device=dev)
    rowptr[1:] = torch.cumsum(counts, 0)
    rowptr = rowptr.to(torch.int32)
    del key, rows, counts
    vals = torch.rand(colind.shape[0], generator=g, device=dev) * 2.0 - 1.0
    return Csr(rowptr, colind, vals.to(torch.float32), n, n)


def reddit_like_csr(M: int = 232_965, nnz_target: int = 114_615_892, seed: int = 5,
                    device="cpu", alpha: float = 2.2, max_deg: int = 21_657):
    """Reddit-shaped graph (BASELINE configs[2]): M = 232,965 rows, ~114.6 M
    nonzeros (mean degree ~492), Pareto(alpha) degrees capped at Reddit's max
    degree 21,657; columns uniform per row, deduplicated (torch tensors).

    The degree scale is bisected so that the EXPECTED number of unique
    columns, sum_i M(1 - (1 - 1/M)^deg_i), equals nnz_target: the post-dedup
    nnz lands within ~0.1% of the target."""
    import torch

    dev = torch.device(device)
    gh = torch.Generator()
    gh.manual_seed(seed)
    u = torch.rand(M, generator=gh, dtype=torch.float64)
    w = (1.0 - u).pow(-1.0 / (alpha - 1.0))
    lo, hi = 1e-3, 1e9
    for _ in range(80):
        s = (lo * hi) ** 0.5
        d = torch.clamp((w * s).round(), 1, max_deg)
        uniq = float((M * (1.0 - (1.0 - 1.0 / M) ** d)).sum())
        if uniq < nnz_target:
            lo = s
        else:
            hi = s
    deg = torch.clamp((w * hi).round(), 1, max_deg).to(torch.int64).to(dev)
    g = torch.Generator(device=dev)
    g.manual_seed(seed)
    nnz = int(deg.sum())
    rows = torch.repeat_interleave(torch.arange(M, device=dev), deg)
    cols = torch.randint(0, M, (nnz,), generator=g, device=dev)
    key = torch.unique(rows * M + cols)
    del rows, cols
    rows = key // M
    colind = (key % M).to(torch.int32)
    counts = torch.bincount(rows, minlength=M)
    rowptr = torch.zeros(M + 1, dtype=torch.int64, device=dev)
    rowptr[1:] = torch.cumsum(counts, 0)
    vals = torch.rand(colind.shape[0], generator=g, device=dev) * 2.0 - 1.0
    return Csr(rowptr.to(torch.int32), colind, vals.to(torch.float32), M, M)


def dense_torch(K: int, N: int, seed: int = 2, device="cpu"):
    import torch

    g = torch.Generator(device=torch.device(device))
    g.manual_seed(seed)
    return torch.rand(K, N, generator=g, device=device) * 2.0 - 1.0


def csr_stats(rowptr) -> dict:
    rp = np.asarray(rowptr, dtype=np.int64)
    deg = np.diff(rp)
    return {"M": int(len(rp) - 1), "nnz": int(rp[-1]), "empty_rows": int((deg == 0).sum()),
            "max_row": int(deg.max()) if len(deg) else 0,
            "mean_row": float(deg.mean()) if len(deg) else 0.0}
