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
    local rowptr is rebased to 0.  The slab is copied into its own storage:
    a view starting at an arbitrary nonzero p0 is 16-byte aligned only when
    p0 % 4 == 0, and unaligned colind/vals take the kernel's 4-byte staging
    path (and the view would keep the full CSR alive)."""
    a, b = int(bounds[rank]), int(bounds[rank + 1])
    p0, p1 = int(rowptr[a]), int(rowptr[b])
    rp = rowptr[a:b + 1] - p0
    if hasattr(rp, "contiguous"):
        return rp.contiguous(), colind[p0:p1].clone(), vals[p0:p1].clone()
    return np.ascontiguousarray(rp), colind[p0:p1].copy(), vals[p0:p1].copy()


def broadcast_B(B, root: int = 0, group=None):
    """The path's only exchange: B from the root, in place."""
    import torch.distributed as dist

    dist.broadcast(B, src=root, group=group)
    return B


def panel_bounds(N: int, panels: int):
    """Column panels [c0, c1) of B for the overlapped broadcast: `panels`
    near-equal widths, multiples of 32 columns where N allows (one warp row
    per panel row), never empty."""
    panels = max(1, min(int(panels), -(-N // 32)))  # at most one panel per 32 columns
    step = -(-N // panels)
    if N >= 32:
        step = -(-step // 32) * 32
    out, c0 = [], 0
    while c0 < N:
        out.append((c0, min(N, c0 + step)))
        c0 += step
    return out


def broadcast_B_overlapped(compute_panel, B, panels: int, root: int = 0, group=None, cuda_streams=None,
                           packed=None):
    """The B broadcast overlapped with the compute.

    B (K x N, row-major) is cut into column panels; the root packs panel p
    into a contiguous K x w buffer (NCCL moves contiguous bytes), panel p is
    broadcast on the comm stream while panel p-1 computes, and
    ``compute_panel(p, Bp, c0, c1)`` runs on the compute stream as soon as
    panel p has landed (C[:, c0:c1] from the K x w panel, ldb = w).  Time is
    max(broadcast, compute) + one panel of the other, instead of their sum.
    Each column's reduction does not depend on which other columns share its
    launch, so results are bit-identical to the unpanelled path (tested).

    ``packed``: optional list of preallocated K x w panel buffers (reused
    across calls).  Non-root ranks' B is not written (the panels hold the
    broadcast data).  ``cuda_streams`` = (compute, comm) torch streams on
    GPUs; None runs the same schedule synchronously (gloo/CPU).  Returns the
    list of panel buffers."""
    import torch
    import torch.distributed as dist

    rank = dist.get_rank(group)
    K, N = B.shape
    pb = panel_bounds(N, panels)
    if packed is None:
        packed = [torch.empty((K, c1 - c0), dtype=B.dtype, device=B.device) for c0, c1 in pb]
    if cuda_streams is None:
        for p, (c0, c1) in enumerate(pb):
            if rank == root:
                packed[p].copy_(B[:, c0:c1])
            dist.broadcast(packed[p], src=root, group=group)
            compute_panel(p, packed[p], c0, c1)
        return packed
    comp, comm = cuda_streams
    comm.wait_stream(comp)  # B and the panel buffers are ready on the compute stream
    for p, (c0, c1) in enumerate(pb):
        with torch.cuda.stream(comm):
            if rank == root:
                packed[p].copy_(B[:, c0:c1])
            dist.broadcast(packed[p], src=root, group=group)
            ev = torch.cuda.Event()
            ev.record(comm)
        comp.wait_event(ev)
        with torch.cuda.stream(comp):
            compute_panel(p, packed[p], c0, c1)
    return packed


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


def chunk_bounds(bounds, world: int, chunks: int):
    """Row chunks of every rank's slab, computable by all ranks from the
    partition alone: chunk j of rank w is rows [lo, hi) of the GLOBAL matrix,
    equal row counts."""
    out = []
    for w in range(world):
        a, b = int(bounds[w]), int(bounds[w + 1])
        out.append([(a + (b - a) * j // chunks, a + (b - a) * (j + 1) // chunks) for j in range(chunks)])
    return out


def gather_C_overlapped(compute_chunk, full, bounds, chunks: int, group=None, cuda_streams=None):
    """Compute-overlapped C all-gather.  For j = 0..chunks-1
    every rank computes chunk j of its slab (``compute_chunk(j, lo, hi)``, rows
    of the global matrix, written into ``full``), then every rank's chunk j is
    broadcast by its owner while chunk j+1 is computed.  All ranks post the
    broadcasts in the same (j, owner) order.  ``cuda_streams`` = (compute,
    comm) torch streams on GPUs; None runs the same schedule synchronously
    (gloo/CPU)."""
    import torch
    import torch.distributed as dist

    rank = dist.get_rank(group)
    world = dist.get_world_size(group)
    cb = chunk_bounds(bounds, world, chunks)
    for j in range(chunks):
        lo, hi = cb[rank][j]
        compute_chunk(j, lo, hi)
        if cuda_streams is None:
            for w in range(world):
                a, b = cb[w][j]
                if b > a:
                    dist.broadcast(full[a:b], src=w, group=group)
            continue
        comp, comm = cuda_streams
        ev = torch.cuda.Event()
        ev.record(comp)
        with torch.cuda.stream(comm):
            comm.wait_event(ev)  # this rank's chunk j is final (execute_rows contract)
            for w in range(world):
                a, b = cb[w][j]
                if b > a:
                    dist.broadcast(full[a:b], src=w, group=group)
    if cuda_streams is not None:
        cuda_streams[0].wait_stream(cuda_streams[1])
    return full


class ShardedSpMM:
    """Per-rank driver: owns the rank's row block and its cached Plan.

    ``compute`` / ``compute_rows`` default to the B200 path (Plan.execute /
    Plan.execute_rows); they are injectable so the host-side sharding logic
    can be exercised with CPU tensors (gloo).
    """

    def __init__(self, rowptr_local, colind_local, K: int, bounds, root: int = 0,
                 group=None, compute: Optional[Callable] = None,
                 compute_rows: Optional[Callable] = None):
        self.rowptr = rowptr_local
        self.colind = colind_local
        self.K = int(K)
        self.bounds = np.asarray(bounds)
        self.root = root
        self.group = group
        self._compute = compute
        self._compute_rows = compute_rows
        self._comm_stream = None
        self._plan = None
        if compute is None and compute_rows is None:
            from .spmm import Plan

            self._plan = Plan(rowptr_local, colind_local, K)

    def __call__(self, vals_local, B, reduce: str = "sum", gather=False,
                 broadcast: bool = True, chunks: int = 1, b_panels: int = 1):
        """gather=True: C all-gather after the compute (one broadcast per slab
        owner), overlapped with it when chunks > 1 (gather_C_overlapped);
        gather="peer": FUSED into the kernel -- every C row is stored straight
        into every rank's full-C buffer over NVLink (CUDA IPC), no collective
        (gespmm_plan_execute_peers).
        b_panels > 1 (with broadcast): the B broadcast is cut into column
        panels overlapped with the compute (broadcast_B_overlapped); the
        result is this rank's C slab (gathered afterwards if asked)."""
        if broadcast and b_panels > 1 and gather != "peer":
            C = self._compute_panelled(vals_local, B, reduce, b_panels)
            return gather_C(C, self.bounds, self.group) if gather else C
        if broadcast:
            broadcast_B(B, self.root, self.group)
        if gather == "peer":
            return self._gather_peer(vals_local, B, reduce)
        if gather and chunks > 1 and (self._plan is not None or self._compute_rows is not None):
            return self._gather_overlapped(vals_local, B, reduce, chunks)
        if self._compute is not None:
            C = self._compute(self.rowptr, self.colind, vals_local, B, reduce)
        else:
            C = self._plan.execute(vals_local, B, reduce)
        if gather:
            return gather_C(C, self.bounds, self.group)
        return C

    def _compute_panelled(self, vals_local, B, reduce, panels):
        import torch

        M = self.rowptr.shape[0] - 1
        N = B.shape[1]
        if self._compute is not None:  # injected (CPU tests): one call per panel
            C = torch.empty((M, N), dtype=torch.float32, device=B.device)

            def panel(p, Bp, c0, c1):
                C[:, c0:c1] = self._compute(self.rowptr, self.colind, vals_local, Bp, reduce)
            broadcast_B_overlapped(panel, B, panels, self.root, self.group)
            return C
        C = torch.empty((M, N), dtype=torch.float32, device=B.device)
        comp = torch.cuda.current_stream(B.device)
        if self._comm_stream is None:
            self._comm_stream = torch.cuda.Stream(device=B.device)

        def panel(p, Bp, c0, c1):
            self._plan.execute(vals_local, Bp, reduce, out=C[:, c0:c1], stream=comp)
        packed = getattr(self, "_packed", None)
        want = [(B.shape[0], c1 - c0) for c0, c1 in panel_bounds(N, panels)]
        if packed is None or [tuple(t.shape) for t in packed] != want or packed[0].device != B.device:
            packed = None
        self._packed = broadcast_B_overlapped(panel, B, panels, self.root, self.group,
                                              cuda_streams=(comp, self._comm_stream), packed=packed)
        return C

    def _gather_overlapped(self, vals_local, B, reduce, chunks):
        import torch
        import torch.distributed as dist

        rank = dist.get_rank(self.group)
        M = int(self.bounds[-1])
        a = int(self.bounds[rank])
        N = B.shape[1]
        full = torch.empty((M, N), dtype=torch.float32, device=B.device)
        slab = full[a:int(self.bounds[rank + 1])]  # this rank's C rows, ldc = N

        if self._compute_rows is not None:  # injected (CPU tests): rows [lo, hi) only
            def chunk(j, lo, hi):
                slab[lo - a:hi - a] = self._compute_rows(self.rowptr, self.colind, vals_local, B, reduce,
                                                         lo - a, hi - a)
            return gather_C_overlapped(chunk, full, self.bounds, chunks, self.group)

        comp = torch.cuda.current_stream(B.device)
        if self._comm_stream is None:
            self._comm_stream = torch.cuda.Stream(device=B.device)

        def chunk(j, lo, hi):
            self._plan.execute_rows(vals_local, B, lo - a, hi - a, out=slab, reduce=reduce,
                                    stream=comp)

        return gather_C_overlapped(chunk, full, self.bounds, chunks, self.group,
                                   cuda_streams=(comp, self._comm_stream))

    def _gather_peer(self, vals_local, B, reduce):
        """Fused all-gather: each rank's full-C buffer is opened by every other
        rank (CUDA IPC handles exchanged over the process group); the kernel's
        epilogue writes each finished row to all of them.  A barrier after the
        local stream drains makes every peer's rows visible."""
        import torch
        import torch.distributed as dist

        from .spmm import ipc_close, ipc_handle, ipc_open

        rank = dist.get_rank(self.group)
        world = dist.get_world_size(self.group)
        if world > 8:
            raise ValueError("fused all-gather: at most 8 ranks (one node)")
        M = int(self.bounds[-1])
        a, b = int(self.bounds[rank]), int(self.bounds[rank + 1])
        N = B.shape[1]
        full = torch.empty((M, N), dtype=torch.float32, device=B.device)
        h, off = ipc_handle(full)
        allh = [None] * world
        dist.all_gather_object(allh, (h, off), group=self.group)
        opened, peers = [], []
        for w, (hw, ow) in enumerate(allh):
            if w != rank:  # this rank's rows reach `full` as the kernel's own output (slab)
                base = ipc_open(hw)
                opened.append(base)
                peers.append(base + ow)
        slab = full[a:b]
        self._plan.execute_peers(vals_local, B, slab, peers, a, reduce=reduce)
        torch.cuda.current_stream(B.device).synchronize()
        dist.barrier(group=self.group)  # every rank's rows have landed in every buffer
        for base in opened:
            ipc_close(base)
        return full
