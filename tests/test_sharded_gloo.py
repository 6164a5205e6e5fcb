"""Multi-rank host logic of the row-sharded path on CPU (gloo, world size 2 and
4): partition, B broadcast from the root (the only exchange; whole, or in
column panels overlapped with the compute), per-rank slabs,
uneven C all-gather -- and the result is bit-identical to the single-process
computation (the per-rank compute here is the oracle's fp32 twin, the same
semantics the GPU path is bit-exact to)."""
import os
import socket
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _make(seed=5):
    rng = np.random.default_rng(seed)
    M, K, N = 3000, 800, 32
    deg = np.minimum((rng.pareto(1.2, M) * 4).astype(np.int64), 2000)
    deg[rng.random(M) < 0.3] = 0
    rowptr = np.concatenate([[0], np.cumsum(deg)]).astype(np.int32)
    colind = rng.integers(0, K, int(rowptr[-1])).astype(np.int32)
    vals = rng.uniform(-1, 1, colind.size).astype(np.float32)
    B = rng.uniform(-1, 1, (K, N)).astype(np.float32)
    return rowptr, colind, vals, B


def _worker(rank, world, port, q):
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch
    import torch.distributed as dist

    from oracle import oracle as O
    from paper_2503_08946_b200 import sharded as S

    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        rowptr, colind, vals, B_full = _make()
        bounds = S.partition(rowptr, world)
        rp, ci, vv = S.local_block(rowptr, colind, vals, bounds, rank)
        B = torch.from_numpy(B_full.copy()) if rank == 0 else torch.zeros(B_full.shape)

        def twin(rp_, ci_, vv_, B_, op):
            return torch.from_numpy(O.spmm_f32(rp_, ci_, vv_, B_.numpy(), op, seg_len=256))

        def twin_rows(rp_, ci_, vv_, B_, op, r0, r1):  # rows [r0, r1) of the local block only
            p0, p1 = int(rp_[r0]), int(rp_[r1])
            return torch.from_numpy(O.spmm_f32(rp_[r0:r1 + 1] - p0, ci_[p0:p1], vv_[p0:p1], B_.numpy(), op,
                                               seg_len=256))

        sh = S.ShardedSpMM(rp, ci, B_full.shape[0], bounds, root=0, compute=twin)
        shc = S.ShardedSpMM(rp, ci, B_full.shape[0], bounds, root=0, compute_rows=twin_rows)
        out = {}
        for op in ("sum", "max", "mean"):
            C = sh(vv, B, op, gather=True)
            out[op] = C.numpy()
            Cc = shc(vv, B, op, gather=True, chunks=3, broadcast=False)  # overlapped all-gather
            assert np.array_equal(Cc.numpy(), out[op]), op
        assert np.array_equal(B.numpy(), B_full)  # broadcast reached every rank
        # B broadcast in column panels overlapped with the compute (f4): B96 is
        # only on the root; 3 panels of 32 columns, bit-identical to one launch
        B96_full = np.random.default_rng(11).uniform(-1, 1, (B_full.shape[0], 96)).astype(np.float32)
        for op in ("sum", "max"):
            B96 = torch.from_numpy(B96_full.copy()) if rank == 0 else torch.zeros(B96_full.shape)
            Cp = sh(vv, B96, op, gather=True, b_panels=3)
            out[op + "96"] = Cp.numpy()
        q.put((rank, out, bounds.tolist()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_sharded_gloo_bit_identical(world, oracle_mod):
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = [q.get(timeout=240) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    rowptr, colind, vals, B = _make()
    for op in ("sum", "max", "mean"):
        want = oracle_mod.spmm_f32(rowptr, colind, vals, B, op, seg_len=256)
        for rank, out, bounds in results:
            np.testing.assert_array_equal(out[op], want)
        if op in ("sum", "max"):
            B96 = np.random.default_rng(11).uniform(-1, 1, (B.shape[0], 96)).astype(np.float32)
            want96 = oracle_mod.spmm_f32(rowptr, colind, vals, B96, op, seg_len=256)
            for rank, out, bounds in results:
                np.testing.assert_array_equal(out[op + "96"], want96)
    b = results[0][2]
    assert b[0] == 0 and b[-1] == len(rowptr) - 1 and all(x <= y for x, y in zip(b, b[1:]))


@pytest.mark.parametrize("N,panels,want", [(128, 4, [(0, 32), (32, 64), (64, 96), (96, 128)]),
                                           (128, 3, [(0, 64), (64, 128)]),
                                           (80, 2, [(0, 64), (64, 80)]), (80, 4, [(0, 32), (32, 64), (64, 80)]),
                                           (16, 4, [(0, 16)]), (100, 1, [(0, 100)]), (256, 99, None)])
def test_panel_bounds(N, panels, want):
    """Column panels of the overlapped B broadcast: cover [0, N) in order, no
    empty panel, widths multiples of 32 except the last (one warp row each)."""
    from paper_2503_08946_b200.sharded import panel_bounds

    pb = panel_bounds(N, panels)
    if want is not None:
        assert pb == want
    assert pb[0][0] == 0 and pb[-1][1] == N
    assert all(a < b for a, b in pb) and all(pb[i][1] == pb[i + 1][0] for i in range(len(pb) - 1))
    assert all((b - a) % 32 == 0 for a, b in pb[:-1])
    assert len(pb) <= max(1, panels)
