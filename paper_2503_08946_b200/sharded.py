"""Row-block sharding over torch.distributed.

The hot path shards naturally: C row i depends only on CSR row i and B.  Each
rank owns a contiguous, nnz-balanced row block (``partition``), keeps its C
slab, and the ONE exchange is the broadcast of B from the root (NCCL over
NVLink 5 / NVSwitch on B200s; gloo in the CPU tests).  The optional C
all-gather moves the uneven slabs with one broadcast per owner.

Per-row reduction order and the long-row segmentation depend only on the row
itself, so results are bit-identical for any world size (tested).

The C++ hosts' equivalent is ``gespmm_sharded_spmm`` in the C-ABI, which
issues the same NCCL calls itself.
"""
from __future__ import annotations

from typing import Callable, Optional

import numpy as np


def partition(rowptr_host, world: int) -> np.ndarray:
    """bounds[0..world]: contiguous row blocks balancing nnz + rows (C-ABI
    gespmm_partition_rows; rows never span ranks)."""
    from .spmm import partition_rows

    return partition_rows(np.asarray(rowptr_host), world)


def local_block(rowptr, colind, vals, bounds, rank: int):
    """Slices this rank's row block out of a full CSR (numpy or torch); the
    local rowptr is rebased to 0."""
    a, b = int(bounds[rank]), int(bounds[rank + 1])
    p0, p1 = int(rowptr[a]), int(rowptr[b])
    rp = rowptr[a:b + 1] - p0
    if hasattr(rp, "contiguous"):
        return rp.contiguous(), colind[p0:p1].contiguous(), vals[p0:p1].contiguous()
    return np.ascontiguousarray(rp), colind[p0:p1].copy(), vals[p0:p1].copy()


def broadcast_B(B, root: int = 0, group=None):
    """The path's only exchange: B from the root, in place."""
    import torch.distributed as dist

    dist.broadcast(B, src=root, group=group)
    return B


def gather_C(C_local, bounds, group=None):
    """All ranks receive the full C (rows bounds[-1] x N) -- one broadcast per
    slab owner, since slabs are uneven."""
    import torch
    import torch.distributed as dist

    rank = dist.get_rank(group)
    world = dist.get_world_size(group)
    N = C_local.shape[1]
    M = int(bounds[-1])
    full = torch.empty((M, N), dtype=C_local.dtype, device=C_local.device)
    for w in range(world):
        a, b = int(bounds[w]), int(bounds[w + 1])
        if b <= a:
            continue
        if w == rank:
            full[a:b].copy_(C_local)
        buf = full[a:b]
        dist.broadcast(buf, src=w, group=group)
    return full


class ShardedSpMM:
    """Per-rank driver: owns the rank's row block and its cached Plan.

    ``compute`` defaults to the B200 path (Plan.execute); it is injectable so
    the host-side sharding logic can be exercised with CPU tensors.
    """

    def __init__(self, rowptr_local, colind_local, K: int, bounds, root: int = 0,
                 group=None, compute: Optional[Callable] = None):
        self.rowptr = rowptr_local
        self.colind = colind_local
        self.K = int(K)
        self.bounds = np.asarray(bounds)
        self.root = root
        self.group = group
        self._compute = compute
        self._plan = None
        if compute is None:
            from .spmm import Plan

            self._plan = Plan(rowptr_local, colind_local, K)

    def __call__(self, vals_local, B, reduce: str = "sum", gather: bool = False,
                 broadcast: bool = True):
        if broadcast:
            broadcast_B(B, self.root, self.group)
        if self._compute is not None:
            C = self._compute(self.rowptr, self.colind, vals_local, B, reduce)
        else:
            C = self._plan.execute(vals_local, B, reduce)
        if gather:
            return gather_C(C, self.bounds, self.group)
        return C
