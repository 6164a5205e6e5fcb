"""GPU parity of the TMA gather4 ring (gespmm_kernel.cuh "TMA ring"): the
128-column ring tile fed by `cp.async.bulk.tensor.2d.tile::gather4` with the
plan's L2 hot set regrouping each batch hot-first.  The fold order is every
other variant's, so the results must be bit-identical to the fp32 twin
(oracle/gespmm_oracle.c) -- for every op, with and without a hot set (none /
part of the columns / all of them: mixed, all-hot and all-cold groups), with
split long rows, accumulate, partial column blocks (N not a multiple of 128:
the tensor map zero-fills the missing columns), strided B, and through the
pipelined host entry point (chunk launches, no hot set).
"""
import numpy as np
import pytest

from test_gpu_parity import SEG, gpu_spmm, powerlaw_csr, random_csr, to_dev

pytestmark = pytest.mark.gpu


@pytest.fixture
def tma_on():
    from paper_2503_08946_b200.spmm import set_tma_override

    def force(hot_rows=-1):
        set_tma_override(1, hot_rows)

    yield force
    set_tma_override(-1, -1)


def _plan_variant(plan):
    return plan.last_variant()


@pytest.mark.parametrize("hot_rows", [-1, 0, 40, 100000])
@pytest.mark.parametrize("op", ["sum", "max", "min", "mean"])
@pytest.mark.parametrize("N", [128, 200, 384])
def test_tma_ring_bit_exact(cuda, oracle_mod, tma_on, op, N, hot_rows):
    """N=128: one column block; 384: three (tensor column coordinates 0 / 128
    / 256); 200: the ring tile forced at a partial second block (72 of 128
    columns: the tensor map zero-fills the rest, never stored)."""
    from paper_2503_08946_b200.spmm import set_variant_override

    tma_on(hot_rows)
    rng = np.random.default_rng(900 + N)
    M, K = 700, 300
    rowptr, colind, vals = random_csr(rng, M, K, 0.05, long_rows=[(5, 1000), (6, 257), (699, 2600)],
                                      dup=True, empty_frac=0.3)
    B = rng.uniform(-1, 1, (K, N)).astype(np.float32)
    if N % 128:
        set_variant_override("vec4_lpr32_cwm1_ring")
    try:
        got, plan = gpu_spmm(cuda, rowptr, colind, vals, B, op)
    finally:
        set_variant_override("")
    want = oracle_mod.spmm_f32(rowptr, colind, vals, B, op, seg_len=SEG)
    np.testing.assert_array_equal(got, want)
    assert _plan_variant(plan) == "vec4_lpr32_cwm1_ring_tma"


@pytest.mark.parametrize("op", ["sum", "max"])
def test_tma_ring_accumulate_and_powerlaw(cuda, oracle_mod, tma_on, op):
    tma_on(2000)
    rng = np.random.default_rng(77)
    M, K, N = 20_000, 9_000, 128
    rowptr, colind, vals = powerlaw_csr(rng, M, K, 20, long_rows=[(3, 5000), (10_000, 777)])
    B = rng.uniform(-1, 1, (K, N)).astype(np.float32)
    C0 = rng.uniform(-1, 1, (M, N)).astype(np.float32)
    got, plan = gpu_spmm(cuda, rowptr, colind, vals, B, op, C0=C0)
    want = oracle_mod.spmm_f32(rowptr, colind, vals, B, op, accumulate=True, C0=C0, seg_len=SEG)
    np.testing.assert_array_equal(got, want)
    assert _plan_variant(plan) == "vec4_lpr32_cwm1_ring_tma"


def test_tma_ring_strided_b_and_repeat(cuda, oracle_mod, tma_on):
    """B as a column view of a wider matrix (ldb = 192), executed twice on
    one plan (the hot set is built once, kept with the plan)."""
    import torch

    from paper_2503_08946_b200.spmm import Plan

    tma_on(64)
    rng = np.random.default_rng(5)
    M, K, N = 3000, 2000, 128
    rowptr, colind, vals = random_csr(rng, M, K, 0.01, long_rows=[(7, 1500)])
    Bw = rng.uniform(-1, 1, (K, 192)).astype(np.float32)
    rp, ci, vv, Bt = to_dev(cuda, rowptr, colind, vals, Bw)
    plan = Plan(rp, ci, K)
    want = oracle_mod.spmm_f32(rowptr, colind, vals, np.ascontiguousarray(Bw[:, 32:160]), "sum", seg_len=SEG)
    for _ in range(2):
        out = plan.execute(vv, Bt[:, 32:160], reduce="sum")
        torch.cuda.synchronize()
        np.testing.assert_array_equal(out.cpu().numpy(), want)
    assert plan.last_variant() == "vec4_lpr32_cwm1_ring_tma"


def test_tma_ring_through_host_pipeline(cuda, oracle_mod, tma_on):
    """The pipelined host entry point (chunk launches over item ranges) with
    the TMA ring forced: no hot set there, same bits."""
    from paper_2503_08946_b200.spmm import csr_spmm_host

    tma_on()
    rng = np.random.default_rng(41)
    M, K, N = 40_000, 6_000, 128  # C = 20 MB -> row chunks
    long_rows = [(i * M // 3 + d, 300 + 97 * d) for i in range(1, 3) for d in (-1, 0, 1)]
    rowptr, colind, vals = powerlaw_csr(rng, M, K, 12, long_rows)
    B = rng.uniform(-1, 1, (K, N)).astype(np.float32)
    got = csr_spmm_host(rowptr, colind, vals, B, "sum")
    want = oracle_mod.spmm_f32(rowptr, colind, vals, B, "sum", seg_len=SEG)
    np.testing.assert_array_equal(got, want)


def test_tma_auto_mode_selection(cuda):
    """Automatic mode: the TMA ring only where B's 128-column slab exceeds the
    L2 budget (80 MB: K > 163,840 rows; below 327,680 rows 64-column panels
    run instead), on persistent plans."""
    import torch

    from paper_2503_08946_b200.spmm import Plan, set_tma_override

    set_tma_override(-1, -1)
    for K, want in [(4096, "vec4_lpr32_cwm1_ring"), (400_000, "vec4_lpr32_cwm1_ring_tma")]:
        rowptr = np.arange(0, 2 * 64 + 1, 2, dtype=np.int32)  # 64 rows x 2 nonzeros
        colind = np.array([0, K - 1] * 64, dtype=np.int32)
        vals = np.ones(128, np.float32)
        rp, ci, vv = to_dev(cuda, rowptr, colind, vals)
        B = torch.ones((K, 128), dtype=torch.float32, device=cuda)
        plan = Plan(rp, ci, K)
        out = plan.execute(vv, B, reduce="sum")
        torch.cuda.synchronize()
        assert float(out.min()) == 2.0 and float(out.max()) == 2.0
        assert plan.last_variant() == want
