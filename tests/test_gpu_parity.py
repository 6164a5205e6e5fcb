"""GPU parity: the sm_100a path (through the C-ABI) against the oracle.

Bar (BASELINE.json north star): sum/mean within 1e-5 norm-wise of the fp64
reference; and -- stronger -- bit-identical to the fp32 twin
(oracle/gespmm_oracle.c) for every op, every kernel variant, split and
unsplit rows.
"""
import os

import numpy as np
import pytest

from conftest import golden_cases, load_golden

pytestmark = pytest.mark.gpu

SEG = 256
OPS = ["sum", "max", "min", "mean"]
VARIANTS = ["vec1_lpr32_cwm1", "vec1_lpr32_cwm2", "vec2_lpr32_cwm1", "vec2_lpr32_cwm2",
            "vec4_lpr32_cwm1", "vec4_lpr32_cwm2", "pair_vec1", "pair_vec2", "pair_vec4",
            "vec2_lpr32_cwm1_ring", "vec4_lpr32_cwm1_ring"]


def to_dev(cuda, *arrs):
    import torch

    return [torch.as_tensor(np.ascontiguousarray(a), device=cuda) for a in arrs]


def random_csr(rng, M, K, density, long_rows=(), dup=False, empty_frac=0.0):
    rows = []
    for i in range(M):
        d = rng.binomial(K, density)
        if rng.random() < empty_frac:
            d = 0
        for (r, dd) in long_rows:
            if r == i:
                d = dd
        c = rng.integers(0, K, d) if (dup or d > K) else np.sort(rng.choice(K, d, replace=False))
        rows.append(c)
    rowptr = np.concatenate([[0], np.cumsum([len(r) for r in rows])]).astype(np.int32)
    colind = np.concatenate(rows).astype(np.int32) if rows else np.zeros(0, np.int32)
    vals = rng.uniform(-1, 1, colind.size).astype(np.float32)
    return rowptr, colind, vals


def gpu_spmm(cuda, rowptr, colind, vals, B, op, C0=None, K=None):
    import torch

    from paper_2503_08946_b200.spmm import Plan

    rp, ci, vv, Bt = to_dev(cuda, rowptr, colind, vals, B)
    K = B.shape[0] if K is None else K
    plan = Plan(rp, ci, K)
    if C0 is not None:
        out = torch.as_tensor(C0.copy(), device=cuda)
        plan.execute(vv, Bt, reduce=op, out=out, accumulate=True)
    else:
        out = plan.execute(vv, Bt, reduce=op)
    torch.cuda.synchronize()
    return out.cpu().numpy(), plan


@pytest.mark.parametrize("name", golden_cases())
def test_golden_instances_via_reference_interface(cuda, name):
    """run(inst) with the reference's launch semantics vs the reference's own C."""
    from paper_2503_08946_b200 import instance as I

    g = load_golden(name)
    M, N, K = g["M"], g["N"], g["K"]
    inst = I.ConcreteInstance(
        name=name, params={"M": M, "N": N, "K": K, "A_S": len(g["colind"])},
        arrays={"rowPtr": I.ArrayData("i32", ints=g["rowptr"]),
                "colInd": I.ArrayData("i32", ints=g["colind"]),
                "val": I.ArrayData("f32", floats=g["vals"]),
                "B": I.ArrayData("f32", floats=g["B"]),
                "C": I.ArrayData("f32", floats=g["C0"])},
        grid=g["grid"], block=g["block"], csr=I.CsrSpec("rowPtr", "colInd", "val", K))
    C = I.run(inst).astype(np.float64)
    ref = np.asarray(g["C"], np.float64).reshape(M, N)
    C0 = np.abs(np.asarray(g["C0"], np.float64).reshape(M, N))
    rp = np.asarray(g["rowptr"], np.int64)
    ci = np.asarray(g["colind"], np.int64)
    v = np.abs(np.asarray(g["vals"], np.float64))
    Bm = np.abs(np.asarray(g["B"], np.float64).reshape(K, N))
    bound = np.zeros((M, N))
    for i in range(M):
        for p in range(rp[i], rp[i + 1]):
            bound[i] += v[p] * Bm[ci[p]]
    tol = 1e-5 * np.maximum(np.abs(ref), bound + C0) + 1e-30
    assert np.all(np.abs(C - ref) <= tol), np.abs(C - ref).max()
    if name.startswith("ref_"):
        np.testing.assert_array_equal(C, ref)  # integer-valued shipped instances: exact


@pytest.mark.parametrize("op", OPS)
@pytest.mark.parametrize("N", [1, 4, 12, 16, 32, 64, 100, 128, 256, 264, 512])
def test_bit_exact_vs_twin(cuda, oracle_mod, op, N):
    rng = np.random.default_rng(100 + N)
    M, K = 700, 300
    rowptr, colind, vals = random_csr(rng, M, K, 0.05, long_rows=[(5, 1000), (6, 257), (699, 2600)],
                                      dup=True, empty_frac=0.3)
    B = rng.uniform(-1, 1, (K, N)).astype(np.float32)
    got, _ = gpu_spmm(cuda, rowptr, colind, vals, B, op)
    want = oracle_mod.spmm_f32(rowptr, colind, vals, B, op, seg_len=SEG)
    np.testing.assert_array_equal(got, want)


@pytest.mark.parametrize("op", OPS)
def test_accumulate_bit_exact(cuda, oracle_mod, op):
    rng = np.random.default_rng(7)
    M, K, N = 500, 400, 64
    rowptr, colind, vals = random_csr(rng, M, K, 0.03, long_rows=[(3, 900)], empty_frac=0.2)
    B = rng.uniform(-1, 1, (K, N)).astype(np.float32)
    C0 = rng.uniform(-1, 1, (M, N)).astype(np.float32)
    got, _ = gpu_spmm(cuda, rowptr, colind, vals, B, op, C0=C0)
    want = oracle_mod.spmm_f32(rowptr, colind, vals, B, op, accumulate=True, C0=C0, seg_len=SEG)
    np.testing.assert_array_equal(got, want)


@pytest.mark.parametrize("mode", [0, 1])
@pytest.mark.parametrize("N", [16, 64, 128, 200])
@pytest.mark.parametrize("op", ["sum", "max", "mean"])
def test_schedules_bit_exact(cuda, oracle_mod, op, N, mode):
    """Static warp striding and the dynamic item counter give the twin's bits
    (incl. long rows spanning many segments, empty rows, accumulate)."""
    from paper_2503_08946_b200 import spmm

    rng = np.random.default_rng(120 + N)
    M, K = 3_000, 900
    rowptr, colind, vals = powerlaw_csr(rng, M, K, 9, [(1, 5_000), (2, 257), (2_999, 700)])
    B = rng.uniform(-1, 1, (K, N)).astype(np.float32)
    C0 = rng.uniform(-1, 1, (M, N)).astype(np.float32)
    spmm.set_schedule_override(mode)
    try:
        got, _ = gpu_spmm(cuda, rowptr, colind, vals, B, op)
        got2, _ = gpu_spmm(cuda, rowptr, colind, vals, B, op)  # counters re-armed per launch
        got_acc, _ = gpu_spmm(cuda, rowptr, colind, vals, B, op, C0=C0)
    finally:
        spmm.set_schedule_override(-1)
    want = oracle_mod.spmm_f32(rowptr, colind, vals, B, op, seg_len=SEG)
    np.testing.assert_array_equal(got, want)
    np.testing.assert_array_equal(got2, want)
    np.testing.assert_array_equal(
        got_acc, oracle_mod.spmm_f32(rowptr, colind, vals, B, op, accumulate=True, C0=C0, seg_len=SEG))


@pytest.mark.parametrize("N,panel", [(256, 64), (100, 32), (200, 64), (64, 16)])
@pytest.mark.parametrize("op", OPS)
def test_column_panels_bit_exact(cuda, oracle_mod, op, N, panel):
    """Column panels (one launch per panel) give the same bits as one launch."""
    from paper_2503_08946_b200 import spmm

    rng = np.random.default_rng(31 + N)
    M, K = 600, 350
    rowptr, colind, vals = random_csr(rng, M, K, 0.04, long_rows=[(7, 1300), (8, 257)], empty_frac=0.3)
    B = rng.uniform(-1, 1, (K, N)).astype(np.float32)
    C0 = rng.uniform(-1, 1, (M, N)).astype(np.float32)
    spmm.set_panel_override(panel)
    try:
        got, _ = gpu_spmm(cuda, rowptr, colind, vals, B, op)
        got_acc, _ = gpu_spmm(cuda, rowptr, colind, vals, B, op, C0=C0)
    finally:
        spmm.set_panel_override(-1)
    np.testing.assert_array_equal(got, oracle_mod.spmm_f32(rowptr, colind, vals, B, op, seg_len=SEG))
    np.testing.assert_array_equal(
        got_acc, oracle_mod.spmm_f32(rowptr, colind, vals, B, op, accumulate=True, C0=C0, seg_len=SEG))


@pytest.mark.parametrize("tile_work", [0, 256])
@pytest.mark.parametrize("variant", VARIANTS)
@pytest.mark.parametrize("op", ["sum", "max", "min"])
def test_every_variant_bit_exact(cuda, oracle_mod, variant, op, tile_work):
    """Every kernel variant, at the automatic tile size (small here) and the
    largest (up to 128 rows per tile)."""
    from paper_2503_08946_b200 import spmm

    rng = np.random.default_rng(11)
    M, K, N = 900, 500, 96
    rowptr, colind, vals = random_csr(rng, M, K, 0.04, long_rows=[(10, 3000)], empty_frac=0.4)
    B = rng.uniform(-1, 1, (K, N)).astype(np.float32)
    spmm.set_variant_override(variant)
    spmm.set_tile_work_override(tile_work)
    try:
        got, plan = gpu_spmm(cuda, rowptr, colind, vals, B, op)
        if tile_work:
            assert plan.info()["tile_work"] == tile_work
        # the variant that really ran (N=96 is a multiple of every VEC; the
        # ring needs 16-byte B rows, so it may fall back to the register path)
        ran = plan.last_variant()
        assert ran == variant or (variant.endswith("_ring") and ran == variant[:-5]), ran
    finally:
        spmm.set_variant_override("")
        spmm.set_tile_work_override(0)
    want = oracle_mod.spmm_f32(rowptr, colind, vals, B, op, seg_len=SEG)
    np.testing.assert_array_equal(got, want)


def test_max_min_special_values(cuda, oracle_mod):
    """NaN first/later messages, +-0, +-inf: max/min bit-exact by construction."""
    rng = np.random.default_rng(5)
    M, K, N = 300, 64, 32
    rowptr, colind, vals = random_csr(rng, M, K, 0.2, long_rows=[(1, 600), (2, 700)])
    vals[::7] = np.nan
    vals[1::11] = 0.0
    vals[2::13] = -0.0
    vals[3::17] = np.inf
    B = rng.uniform(-1, 1, (K, N)).astype(np.float32)
    B[::5] = -0.0
    B[1::9] = -np.inf
    for op in ("max", "min", "sum", "mean"):
        got, _ = gpu_spmm(cuda, rowptr, colind, vals, B, op)
        want = oracle_mod.spmm_f32(rowptr, colind, vals, B, op, seg_len=SEG)
        # NaN payloads are not part of the contract (the GPU's canonical NaN is
        # 0x7fffffff, x86's 0x7fc00000): NaN positions must match, every other
        # value bit for bit (including the sign of zero and infinities).
        nan = np.isnan(want)
        np.testing.assert_array_equal(np.isnan(got), nan)
        np.testing.assert_array_equal(got[~nan].view(np.uint32), want[~nan].view(np.uint32))


@pytest.mark.parametrize("N", [1, 5, 16, 32, 64, 100, 128, 256])
@pytest.mark.parametrize("accumulate", [False, True])
def test_max_min_maximum_number_all_bits(cuda, oracle_mod, N, accumulate):
    """max/min = maximumNumber/minimumNumber (FMNMX): every bit equal to the
    twin, NaNs included (an all-NaN row is the canonical 0x7fffffff on both
    sides), across every kernel variant N selects, long rows and accumulate."""
    rng = np.random.default_rng(100 + N)
    M, K = 400, 96
    rowptr, colind, vals = random_csr(rng, M, K, 0.1, long_rows=[(1, 900), (2, 300)], empty_frac=0.1)
    vals[::7] = np.nan
    vals[1::11] = 0.0
    vals[2::13] = -0.0
    vals[3::17] = np.inf
    B = rng.uniform(-1, 1, (K, N)).astype(np.float32)
    B[::5] = -0.0
    B[1::9] = -np.inf
    B[2::10] = 0.0
    # rows whose messages are all NaN / all +-0
    for r, v in ((3, np.nan), (4, 0.0), (5, -0.0)):
        vals[rowptr[r]:rowptr[r + 1]] = v
    C0 = rng.uniform(-1, 1, (M, N)).astype(np.float32) if accumulate else None
    if accumulate:
        C0[::6] = np.nan
        C0[1::8] = -0.0
    for op in ("max", "min"):
        got, _ = gpu_spmm(cuda, rowptr, colind, vals, B, op, C0=C0)
        want = oracle_mod.spmm_f32(rowptr, colind, vals, B, op, accumulate=accumulate, C0=C0, seg_len=SEG)
        np.testing.assert_array_equal(got.view(np.uint32), want.view(np.uint32))


def test_tile_work_is_automatic_and_result_free(cuda, oracle_mod):
    """Small matrices get small tiles (more items than warp slots), large ones
    256; every tile size gives the same bits."""
    from paper_2503_08946_b200 import spmm

    rng = np.random.default_rng(21)
    rowptr, colind, vals = random_csr(rng, 3000, 800, 0.02, long_rows=[(5, 900)], empty_frac=0.3)
    B = rng.uniform(-1, 1, (800, 48)).astype(np.float32)
    want = oracle_mod.spmm_f32(rowptr, colind, vals, B, "sum", seg_len=SEG)
    got, plan = gpu_spmm(cuda, rowptr, colind, vals, B, "sum")
    assert plan.info()["tile_work"] == 16
    np.testing.assert_array_equal(got, want)
    for tw in (2, 5, 64, 200, 256):
        spmm.set_tile_work_override(tw)
        try:
            got, plan = gpu_spmm(cuda, rowptr, colind, vals, B, "sum")
        finally:
            spmm.set_tile_work_override(0)
        assert plan.info()["tile_work"] == tw
        np.testing.assert_array_equal(got, want)
    with pytest.raises(Exception):
        spmm.set_tile_work_override(300)


def test_segmented_max_equals_unsegmented(cuda, oracle_mod):
    """Max/min are independent of the long-row split (proved in DESIGN.md)."""
    rng = np.random.default_rng(9)
    rowptr, colind, vals = random_csr(rng, 50, 4000, 0.01, long_rows=[(0, 3999), (7, 513)])
    B = rng.uniform(-1, 1, (4000, 64)).astype(np.float32)
    for op in ("max", "min"):
        got, _ = gpu_spmm(cuda, rowptr, colind, vals, B, op)
        want = oracle_mod.spmm_f32(rowptr, colind, vals, B, op, seg_len=0)
        np.testing.assert_array_equal(got, want)


def test_empty_and_degenerate(cuda, oracle_mod):
    import torch

    from paper_2503_08946_b200.spmm import csr_spmm

    # nnz = 0
    rowptr = np.zeros(11, np.int32)
    colind = np.zeros(0, np.int32)
    vals = np.zeros(0, np.float32)
    B = np.ones((5, 8), np.float32)
    for op in OPS:
        got, _ = gpu_spmm(cuda, rowptr, colind, vals, B, op)
        np.testing.assert_array_equal(got, np.zeros((10, 8), np.float32))
    # M = 0
    rp, ci, vv, Bt = to_dev(cuda, np.zeros(1, np.int32), colind, vals, B)
    out = csr_spmm(rp, ci, vv, Bt)
    assert tuple(out.shape) == (0, 8)
    # single dense row
    rowptr = np.array([0, 5], np.int32)
    colind = np.arange(5, dtype=np.int32)
    vals = np.arange(1, 6, dtype=np.float32)
    got, _ = gpu_spmm(cuda, rowptr, colind, vals, B, "sum")
    np.testing.assert_array_equal(got, np.full((1, 8), 15.0, np.float32))
    torch.cuda.synchronize()


def test_misaligned_views_bit_exact(cuda, oracle_mod):
    """Offset (non-16B-aligned) colind/vals/B/C force the scalar staging and
    VEC=1 paths."""
    import torch

    from paper_2503_08946_b200.spmm import Plan

    rng = np.random.default_rng(21)
    M, K, N = 400, 300, 64
    rowptr, colind, vals = random_csr(rng, M, K, 0.05, long_rows=[(4, 800)])
    B = rng.uniform(-1, 1, (K, N)).astype(np.float32)
    ci_big = torch.zeros(colind.size + 1, dtype=torch.int32, device=cuda)
    ci_big[1:] = torch.as_tensor(colind, device=cuda)
    v_big = torch.zeros(vals.size + 1, dtype=torch.float32, device=cuda)
    v_big[1:] = torch.as_tensor(vals, device=cuda)
    B_big = torch.zeros(K * N + 1, dtype=torch.float32, device=cuda)
    B_big[1:] = torch.as_tensor(B.ravel(), device=cuda)
    Bt = B_big[1:].view(K, N)
    C_big = torch.zeros(M * N + 1, dtype=torch.float32, device=cuda)
    out = C_big[1:].view(M, N)
    rp = torch.as_tensor(rowptr, device=cuda)
    plan = Plan(rp, ci_big[1:], K)
    plan.execute(v_big[1:], Bt, reduce="sum", out=out)
    torch.cuda.synchronize()
    want = oracle_mod.spmm_f32(rowptr, colind, vals, B, "sum", seg_len=SEG)
    np.testing.assert_array_equal(out.cpu().numpy(), want)


def test_strided_B_and_C(cuda, oracle_mod):
    import torch

    from paper_2503_08946_b200.spmm import Plan

    rng = np.random.default_rng(3)
    M, K, N = 300, 200, 64
    rowptr, colind, vals = random_csr(rng, M, K, 0.05)
    Bw = rng.uniform(-1, 1, (K, N + 8)).astype(np.float32)
    rp, ci, vv = to_dev(cuda, rowptr, colind, vals)
    Bt = torch.as_tensor(Bw, device=cuda)[:, :N]
    outw = torch.full((M, N + 4), 7.0, device=cuda)
    plan = Plan(rp, ci, K)
    plan.execute(vv, Bt, reduce="sum", out=outw[:, :N])
    torch.cuda.synchronize()
    want = oracle_mod.spmm_f32(rowptr, colind, vals, np.ascontiguousarray(Bw[:, :N]), "sum",
                               seg_len=SEG)
    np.testing.assert_array_equal(outw[:, :N].cpu().numpy(), want)
    assert torch.all(outw[:, N:] == 7.0)


def test_invalid_csr_raises_like_reference(cuda):
    from paper_2503_08946_b200 import Error, ErrorKind
    from paper_2503_08946_b200.spmm import csr_spmm

    B = np.ones((2, 4), np.float32)
    bad = [  # (rowptr, colind, message) -- reference src/oracle.cpp:302-315 wording
        (np.array([0, 2, 1], np.int32), np.array([0, 0], np.int32), "nondecreasing"),
        (np.array([1, 2, 2], np.int32), np.array([0, 0], np.int32), "[0] must be 0"),
        (np.array([0, 1, 3], np.int32), np.array([0, 1], np.int32), "end differs"),
        (np.array([0, 1, 2], np.int32), np.array([0, 2], np.int32), "out of [0,2)"),
        # a 2^30-long first row: more work items than the one-shot plan's
        # device-side bound (build_plan_async) -- the emit stops at the bound
        # and the launch aborts on the error bits; no out-of-bounds write
        (np.array([0, 1 << 30, 2], np.int32), np.array([0, 0], np.int32), "nondecreasing"),
    ]
    for rowptr, colind, msg in bad:
        rp, ci, vv, Bt = to_dev(cuda, rowptr, colind, np.ones(colind.size, np.float32), B)
        with pytest.raises(Error) as ei:
            csr_spmm(rp, ci, vv, Bt)
        assert ei.value.kind == ErrorKind.CsrInvalid
        assert msg in str(ei.value)


def test_host_entry_point(cuda, oracle_mod):
    from paper_2503_08946_b200.spmm import csr_spmm_host

    rng = np.random.default_rng(4)
    M, K, N = 1000, 800, 32
    rowptr, colind, vals = random_csr(rng, M, K, 0.02, long_rows=[(2, 700)])
    B = rng.uniform(-1, 1, (K, N)).astype(np.float32)
    got = csr_spmm_host(rowptr, colind, vals, B, "mean")
    want = oracle_mod.spmm_f32(rowptr, colind, vals, B, "mean", seg_len=SEG)
    np.testing.assert_array_equal(got, want)
    C0 = rng.uniform(-1, 1, (M, N)).astype(np.float32)
    got = csr_spmm_host(rowptr, colind, vals, B, "sum", C0=C0)
    want = oracle_mod.spmm_f32(rowptr, colind, vals, B, "sum", accumulate=True, C0=C0, seg_len=SEG)
    np.testing.assert_array_equal(got, want)


def powerlaw_csr(rng, M, K, mean_deg, long_rows=()):
    """Vectorized: heavy-tailed degrees (many empty rows), unsorted columns with
    duplicates, plus the given (row, degree) long rows."""
    deg = np.minimum((rng.pareto(1.5, M) * mean_deg / 2).astype(np.int64), 4000)
    deg[rng.random(M) < 0.3] = 0
    for r, d in long_rows:
        deg[r] = d
    rowptr = np.concatenate([[0], np.cumsum(deg)]).astype(np.int32)
    colind = rng.integers(0, K, int(rowptr[-1])).astype(np.int32)
    vals = rng.uniform(-1, 1, colind.size).astype(np.float32)
    return rowptr, colind, vals


@pytest.mark.parametrize("op", ["sum", "max", "mean"])
def test_host_entry_point_pipelined_chunks(cuda, oracle_mod, op):
    """gespmm_csr_spmm_host at a size where it pipelines row chunks (C >= 16 MB:
    B first, colind/vals per chunk, C rows back per chunk), long rows and
    tiles straddling the chunk boundaries; bit-exact to the twin."""
    from paper_2503_08946_b200.spmm import csr_spmm_host

    rng = np.random.default_rng(40)
    M, K, N = 150_000, 20_000, 64  # C = 38 MB -> 4 chunks
    long_rows = [(i * M // 4 + d, 300 + 97 * d) for i in range(1, 4) for d in (-2, -1, 0, 1)]
    rowptr, colind, vals = powerlaw_csr(rng, M, K, 12, long_rows)
    B = rng.uniform(-1, 1, (K, N)).astype(np.float32)
    got = csr_spmm_host(rowptr, colind, vals, B, op)
    want = oracle_mod.spmm_f32(rowptr, colind, vals, B, op, seg_len=SEG)
    np.testing.assert_array_equal(got, want)
    C0 = rng.uniform(-1, 1, (M, N)).astype(np.float32)
    got = csr_spmm_host(rowptr, colind, vals, B, op, C0=C0)
    want = oracle_mod.spmm_f32(rowptr, colind, vals, B, op, accumulate=True, C0=C0, seg_len=SEG)
    np.testing.assert_array_equal(got, want)


def test_host_entry_point_pipelined_invalid_colind(cuda, oracle_mod):
    """An out-of-range column in a late chunk: CsrInvalid with the reference's
    message, no launch touches it (no sticky CUDA error), the next call works."""
    from paper_2503_08946_b200.errors import Error, ErrorKind
    from paper_2503_08946_b200.spmm import csr_spmm_host

    rng = np.random.default_rng(41)
    M, K, N = 150_000, 20_000, 64
    rowptr, colind, vals = powerlaw_csr(rng, M, K, 12)
    B = rng.uniform(-1, 1, (K, N)).astype(np.float32)
    bad = colind.copy()
    bad[int(rowptr[-1]) * 3 // 4] = K + 5
    with pytest.raises(Error) as ei:
        csr_spmm_host(rowptr, bad, vals, B, "sum")
    assert ei.value.kind == ErrorKind.CsrInvalid
    assert f"colInd entry out of [0,{K})" in str(ei.value)
    got = csr_spmm_host(rowptr, colind, vals, B, "sum")
    np.testing.assert_array_equal(got, oracle_mod.spmm_f32(rowptr, colind, vals, B, "sum", seg_len=SEG))


@pytest.mark.parametrize("badval", [-1, -(2**31), 7_000_000])
def test_host_entry_point_single_chunk_invalid_colind(cuda, oracle_mod, badval):
    """Small M (one chunk, no item range): a negative or huge column is caught
    by the on-device check and the launch returns without gathering through it
    (with 32-bit offsets a negative column would wrap ~16 GB past B) -- a clean
    CsrInvalid, no sticky CUDA error, and the next call works."""
    import torch

    from paper_2503_08946_b200.errors import Error, ErrorKind
    from paper_2503_08946_b200.spmm import csr_spmm_host

    rng = np.random.default_rng(43)
    M, K, N = 300, 200, 128
    rowptr, colind, vals = random_csr(rng, M, K, 0.05, long_rows=[(7, 700)])
    B = rng.uniform(-1, 1, (K, N)).astype(np.float32)
    for pos in (0, int(rowptr[-1]) // 2, int(rowptr[-1]) - 1):
        bad = colind.copy()
        bad[pos] = badval
        with pytest.raises(Error) as ei:
            csr_spmm_host(rowptr, bad, vals, B, "sum")
        assert ei.value.kind == ErrorKind.CsrInvalid
        torch.cuda.synchronize()  # no sticky error from an out-of-bounds gather
    got = csr_spmm_host(rowptr, colind, vals, B, "sum")
    np.testing.assert_array_equal(got, oracle_mod.spmm_f32(rowptr, colind, vals, B, "sum", seg_len=SEG))


@pytest.mark.parametrize("op", ["sum", "min"])
def test_host_entry_point_front_loaded_chunks(cuda, oracle_mod, op):
    """Nonzeros piled into the first rows (as in R-MAT): the host pipeline runs
    its item-aligned chunks out of row order (fewest nonzeros first); results
    bit-exact, with and without accumulate, and an invalid column in the chunk
    that runs first or last is reported the same way."""
    from paper_2503_08946_b200.errors import Error, ErrorKind
    from paper_2503_08946_b200.spmm import csr_spmm_host

    rng = np.random.default_rng(42)
    M, K, N = 150_000, 30_000, 64
    deg = np.where(np.arange(M) < M // 10, rng.integers(50, 400, M), rng.integers(0, 4, M))
    rowptr = np.concatenate([[0], np.cumsum(deg)]).astype(np.int32)
    colind = rng.integers(0, K, int(rowptr[-1])).astype(np.int32)
    vals = rng.uniform(-1, 1, colind.size).astype(np.float32)
    B = rng.uniform(-1, 1, (K, N)).astype(np.float32)
    got = csr_spmm_host(rowptr, colind, vals, B, op)
    np.testing.assert_array_equal(got, oracle_mod.spmm_f32(rowptr, colind, vals, B, op, seg_len=SEG))
    C0 = rng.uniform(-1, 1, (M, N)).astype(np.float32)
    got = csr_spmm_host(rowptr, colind, vals, B, op, C0=C0)
    np.testing.assert_array_equal(
        got, oracle_mod.spmm_f32(rowptr, colind, vals, B, op, accumulate=True, C0=C0, seg_len=SEG))
    for pos in (int(rowptr[M // 20]), int(rowptr[-1]) - 3):  # heavy chunk (runs last) / light one (first)
        bad = colind.copy()
        bad[pos] = -7
        with pytest.raises(Error) as ei:
            csr_spmm_host(rowptr, bad, vals, B, op)
        assert ei.value.kind == ErrorKind.CsrInvalid
    got = csr_spmm_host(rowptr, colind, vals, B, op)
    np.testing.assert_array_equal(got, oracle_mod.spmm_f32(rowptr, colind, vals, B, op, seg_len=SEG))


@pytest.mark.parametrize("rule", ["equal_rows", "equal_bytes"])
@pytest.mark.parametrize("chunks", [7, 64])
def test_host_entry_point_chunk_rules(cuda, oracle_mod, monkeypatch, rule, chunks):
    """Chunk boundaries by equal rows (default) and by equal PCIe bytes
    (GESPMM_HOST_EQUAL_BYTES), up to the 64-chunk cap: a few
    very long rows hold most of the bytes, so several byte targets fall inside
    one row and collapse to empty chunks after item alignment.  Bit-exact to the
    twin with and without accumulate; an invalid column is still caught."""
    from paper_2503_08946_b200.errors import Error, ErrorKind
    from paper_2503_08946_b200.spmm import csr_spmm_host

    monkeypatch.setenv("GESPMM_HOST_CHUNKS", str(chunks))
    if rule == "equal_bytes":
        monkeypatch.setenv("GESPMM_HOST_EQUAL_BYTES", "1")
    rng = np.random.default_rng(44)
    M, K, N = 60_000, 20_000, 32
    long_rows = [(5, 150_000), (6, 90_000), (M // 2, 60_000), (M - 1, 40_000)]
    rowptr, colind, vals = powerlaw_csr(rng, M, K, 6, long_rows)
    B = rng.uniform(-1, 1, (K, N)).astype(np.float32)
    for op in ("sum", "max"):
        got = csr_spmm_host(rowptr, colind, vals, B, op)
        np.testing.assert_array_equal(got, oracle_mod.spmm_f32(rowptr, colind, vals, B, op, seg_len=SEG))
    C0 = rng.uniform(-1, 1, (M, N)).astype(np.float32)
    got = csr_spmm_host(rowptr, colind, vals, B, "mean", C0=C0)
    np.testing.assert_array_equal(
        got, oracle_mod.spmm_f32(rowptr, colind, vals, B, "mean", accumulate=True, C0=C0, seg_len=SEG))
    bad = colind.copy()
    bad[int(rowptr[M // 2]) + 7] = K
    with pytest.raises(Error) as ei:
        csr_spmm_host(rowptr, bad, vals, B, "sum")
    assert ei.value.kind == ErrorKind.CsrInvalid


def test_host_entry_point_never_gathers_through_stale_entries(cuda, oracle_mod):
    """Chunks run out of row order, so the 16-byte staging granule before a
    chunk's first item can hold entries of a chunk not yet transferred (here:
    stale columns of a previous call with K = 20 M).  The kernel zeroes the
    staged head before its item: no gather leaves B, results stay exact.
    (Best effort: a stale gather only faults when it lands on unmapped
    memory; the build without the head zeroing passed this test too.)"""
    from paper_2503_08946_b200.spmm import csr_spmm_host

    rng = np.random.default_rng(43)
    Kbig = 20_000_000
    rp1 = np.linspace(0, 3_000_000, 4001).astype(np.int32)
    ci1 = rng.integers(Kbig // 2, Kbig, 3_000_000).astype(np.int32)
    v1 = np.ones(ci1.size, np.float32)
    B1 = np.ones((Kbig, 1), np.float32)
    csr_spmm_host(rp1, ci1, v1, B1, "sum")  # leaves large columns in the workspace
    M, K, N = 150_000, 30_000, 64
    deg = np.where(np.arange(M) < M // 10, rng.integers(20, 200, M), rng.integers(0, 3, M))
    deg[rng.random(M) < 0.3] += 1  # ragged chunk starts (not 4-aligned)
    rowptr = np.concatenate([[0], np.cumsum(deg)]).astype(np.int32)
    colind = rng.integers(0, K, int(rowptr[-1])).astype(np.int32)
    vals = rng.uniform(-1, 1, colind.size).astype(np.float32)
    B = rng.uniform(-1, 1, (K, N)).astype(np.float32)
    for op in ("sum", "max"):
        got = csr_spmm_host(rowptr, colind, vals, B, op)
        np.testing.assert_array_equal(got, oracle_mod.spmm_f32(rowptr, colind, vals, B, op, seg_len=SEG))


def test_deterministic_and_shard_invariant(cuda, oracle_mod):
    """Same bits run-to-run, and row-sharded computation (the multi-GPU path's
    per-rank work) reproduces the unsharded result bit for bit."""
    import torch

    from paper_2503_08946_b200 import workloads as W
    from paper_2503_08946_b200.spmm import Plan, partition_rows

    csr = W.rmat_csr(14, 200_000, seed=3, device=cuda)
    M, K, N = csr.M, csr.K, 64
    B = W.dense_torch(K, N, seed=2, device=cuda)
    plan = Plan(csr.rowptr, csr.colind, K)
    c1 = plan.execute(csr.vals, B, "sum").clone()
    c2 = plan.execute(csr.vals, B, "sum").clone()
    assert torch.equal(c1, c2)
    rp_h = csr.rowptr.cpu().numpy()
    for parts in (2, 4, 8):
        bounds = partition_rows(rp_h, parts)
        full = torch.empty_like(c1)
        for r in range(parts):
            a, b = int(bounds[r]), int(bounds[r + 1])
            p0, p1 = int(rp_h[a]), int(rp_h[b])
            rp = (csr.rowptr[a:b + 1] - p0).contiguous()
            sp = Plan(rp, csr.colind[p0:p1].contiguous(), K)
            sp.execute(csr.vals[p0:p1].contiguous(), B, "sum", out=full[a:b])
        torch.cuda.synchronize()
        assert torch.equal(full, c1)
    want = oracle_mod.spmm_f32(rp_h, csr.colind.cpu().numpy(), csr.vals.cpu().numpy(),
                               B.cpu().numpy(), "sum", seg_len=SEG)
    np.testing.assert_array_equal(c1.cpu().numpy(), want)


@pytest.mark.parametrize("op", ["sum", "max"])
def test_config2_full_size_bit_exact(cuda, oracle_mod, op):
    """BASELINE config 2 (R-MAT scale 20, 16M edges, N=64) at full size: GPU
    equals the twin bit for bit (the twin runs on all host cores)."""
    import torch

    from paper_2503_08946_b200 import workloads as W
    from paper_2503_08946_b200.spmm import Plan

    csr = W.rmat_csr(20, 16 * 2**20, seed=3, device=cuda)
    B = W.dense_torch(csr.K, 64, seed=2, device=cuda)
    plan = Plan(csr.rowptr, csr.colind, csr.K)
    got = plan.execute(csr.vals, B, op)
    torch.cuda.synchronize()
    want = oracle_mod.spmm_f32(csr.rowptr.cpu().numpy(), csr.colind.cpu().numpy(),
                               csr.vals.cpu().numpy(), B.cpu().numpy(), op, seg_len=SEG)
    np.testing.assert_array_equal(got.cpu().numpy(), want)


@pytest.mark.parametrize("workload,op", [("config4", "sum"), ("config4", "mean"), ("config5", "sum"),
                                         ("config3-256", "sum")])
def test_full_size_whole_matrix_bit_exact(cuda, oracle_mod, workload, op):
    """Every cell, not a sample: the headline configuration (config 5: R-MAT
    2^24, 1.02 B nonzeros, N=128 -- 2.1 G output cells), config 4 and config 3
    at N=256 (column panels), exactly as bench.py generates them, against the
    fp32 twin on all host cores (~30 GB of host memory for config 5)."""
    import sys

    import torch

    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import bench
    from paper_2503_08946_b200.spmm import Plan

    spec = bench.workload_spec(workload)
    csr, B = bench.make_workload(spec, cuda, "torch")
    plan = Plan(csr.rowptr, csr.colind, csr.K)
    got = plan.execute(csr.vals, B, op)
    torch.cuda.synchronize()
    got_h = got.cpu().numpy()
    del got
    args = [t.cpu().numpy() for t in (csr.rowptr, csr.colind, csr.vals, B)]
    del csr, B, plan
    torch.cuda.empty_cache()
    want = oracle_mod.spmm_f32(*args, op, seg_len=SEG)
    neq = int(np.count_nonzero(got_h.view(np.uint32) != want.view(np.uint32)))
    assert neq == 0, f"{workload} {op}: {neq} of {want.size} cells differ from the twin"


def sampled_rows_bit_exact(oracle_mod, csr, B, C, op, n_random=3000, seed=0, tag=""):
    """Checks C on a sample of rows (the 16 longest rows, random rows, the first
    and last rows) without moving the full B to the host: each sampled row's
    result depends only on its own nonzeros and the B rows they name, so the
    sub-problem uses a compacted B.  Two checks per row:
      * bit for bit against the fp32 twin (oracle_spmm_f32);
      * against the fp64 reference restatement (oracle_spmm_ref64_op: the
        reference interpreter's ascending, unfused fp64 sum,
        gespmm_alg2.mir:38-59, oracle.cpp:593-613): sum/mean within the north
        star's 1e-5 norm-wise bound |gpu - ref| <= 1e-5 max(|ref|, sum|v b|),
        max/min equal to (float) ref exactly.
    Returns (rows, nnz, ratio) -- ratio = max |gpu-ref| / (1e-5 scale) for
    sum/mean, mismatching cells for max/min."""
    import torch

    from conftest import record_parity

    rp = csr.rowptr.long()
    deg = (rp[1:] - rp[:-1])
    M = csr.M
    g = torch.Generator(device="cpu")
    g.manual_seed(seed)
    rows = torch.cat([torch.topk(deg, min(16, M)).indices.cpu(), torch.randint(0, M, (n_random,), generator=g),
                      torch.tensor([0, M - 1])]).unique().to(rp.device)
    sdeg = deg[rows]
    srp = torch.zeros(rows.numel() + 1, dtype=torch.int64, device=rp.device)
    srp[1:] = torch.cumsum(sdeg, 0)
    pos = torch.repeat_interleave(rp[rows], sdeg) + (
        torch.arange(int(srp[-1]), device=rp.device) - torch.repeat_interleave(srp[:-1], sdeg))
    cols = csr.colind.long()[pos]
    ucols, inv = torch.unique(cols, return_inverse=True)
    srp_h, inv_h, v_h, B_h = (srp.int().cpu().numpy(), inv.int().cpu().numpy(), csr.vals[pos].cpu().numpy(),
                              B[ucols].cpu().numpy())
    got = C[rows].cpu().numpy()
    want = oracle_mod.spmm_f32(srp_h, inv_h, v_h, B_h, op, seg_len=SEG)
    np.testing.assert_array_equal(got, want)
    ref, bound = oracle_mod.spmm_ref64_op(srp_h, inv_h, v_h, B_h, op)
    ratio = oracle_mod.ref64_error_ratio(got, ref, bound, op)
    record_parity("sampled_rows_vs_ref64", workload=tag, op=op, N=int(B.shape[1]), rows=int(rows.numel()),
                  nnz=int(srp[-1]), max_row_nnz=int(sdeg.max()), ratio=ratio,
                  metric="max|gpu-ref64|/(1e-5*max(|ref|,sum|vb|))" if op in ("sum", "mean")
                  else "cells != (float)ref64")
    if op in ("sum", "mean"):
        assert ratio <= 1.0, f"{tag} {op}: error {ratio:.3g} x the 1e-5 norm-wise bound"
    else:
        assert ratio == 0, f"{tag} {op}: {ratio} cells differ from (float) of the fp64 reference"
    return int(rows.numel()), int(srp[-1]), ratio


@pytest.mark.parametrize("workload,N", [("config2", 64), ("config4", 64), ("config4", 128), ("config4", 256),
                                        ("config5", 128), ("config3", 16), ("config3", 32), ("config3", 64),
                                        ("config3", 128), ("config3", 256)])
def test_full_size_configs_sampled_bit_exact(cuda, oracle_mod, workload, N):
    """BASELINE configs 2-5 at full size (R-MAT scale 20/16M with N=64, scale
    22/64M with N=64/128/256, scale 24/2^30 edges with N=128, Reddit-like
    114.6M nnz over config 3's whole N sweep 16-256: the paired-lane kernel,
    the 16-gather fast batch, column panels) on one GPU: every op bit-exact to
    the twin AND within the north-star bound of the fp64 reference (max/min
    exact) on sampled rows incl. the 16 longest rows (up to ~10^5 nonzeros)."""
    import torch

    from paper_2503_08946_b200 import workloads as W
    from paper_2503_08946_b200.spmm import Plan

    if workload == "config3":
        csr = W.reddit_like_csr(device=cuda)
    else:
        scale, edges = {"config2": (20, 16 * 2**20), "config4": (22, 64 * 2**20),
                        "config5": (24, 2**30)}[workload]
        csr = W.rmat_csr_gpu(scale, edges, seed=3, device=cuda)
    B = W.dense_gpu(csr.K, N, seed=2, device=cuda)
    plan = Plan(csr.rowptr, csr.colind, csr.K)
    C = torch.empty((csr.M, N), dtype=torch.float32, device=cuda)
    for op in OPS:
        plan.execute(csr.vals, B, op, out=C)
        torch.cuda.synchronize()
        sampled_rows_bit_exact(oracle_mod, csr, B, C, op, n_random=2000 if workload == "config5" else 3000,
                               tag=f"{workload}-N{N}")


def test_reference_side_cpp_adapter(cuda, tmp_path):
    """The C++ binding a raceset maintainer adds (examples/raceset_adapter.cpp,
    linked against the reference's own library) computes the shipped instance
    through libgespmm.so; matches the reference interpreter's full-launch C."""
    import os
    import subprocess

    from test_instance import golden_inst_text

    exe = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "examples",
                       "raceset_adapter")
    if not os.path.exists(exe):
        pytest.skip("examples/raceset_adapter not built (reference tree absent at build time)")
    for name in ("ref_gespmm_small_full.json", "rnd_ragged_c0.json"):
        g = load_golden(name)
        inst = tmp_path / (name + ".inst")
        inst.write_text(golden_inst_text(g, "adapter"))
        out = subprocess.run([exe, str(inst)], capture_output=True, text=True, timeout=120)
        assert out.returncode == 0, out.stderr
        got = np.array([float(x) for x in out.stdout.split()], np.float64)
        ref = np.asarray(g["C"], np.float64)
        # the north star's norm-wise bound: 1e-5 max(|ref|, |C0| + sum_p |v b|)
        M, N, K = g["M"], g["N"], g["K"]
        rp = np.asarray(g["rowptr"], np.int64)
        ci = np.asarray(g["colind"], np.int64)
        v = np.abs(np.asarray(g["vals"], np.float64))
        Bm = np.abs(np.asarray(g["B"], np.float64).reshape(K, N))
        bound = np.abs(np.asarray(g["C0"], np.float64).reshape(M, N)).copy()
        for i in range(M):
            for p in range(rp[i], rp[i + 1]):
                bound[i] += v[p] * Bm[ci[p]]
        tol = 1e-5 * np.maximum(np.abs(ref), bound.reshape(-1))
        assert np.all(np.abs(got - ref) <= tol), np.abs(got - ref).max()


@pytest.mark.parametrize("mode", [-1, 1])
@pytest.mark.parametrize("op", ["sum", "max", "mean"])
def test_execute_rows_chunks_equal_execute(cuda, oracle_mod, op, mode):
    """gespmm_plan_execute_rows: consecutive row chunks on one stream equal one
    execute bit for bit, and after chunk j every row < r_j+1 is already final
    (the contract the overlapped all-gather relies on)."""
    import torch

    from paper_2503_08946_b200.spmm import Plan

    rng = np.random.default_rng(50)
    M, K, N = 30_000, 5_000, 64
    long_rows = [(7_000, 2_000), (7_001, 300), (15_000, 257), (29_999, 900)]
    rowptr, colind, vals = powerlaw_csr(rng, M, K, 10, long_rows)
    B = rng.uniform(-1, 1, (K, N)).astype(np.float32)
    rp, ci, vv, Bt = to_dev(cuda, rowptr, colind, vals, B)
    plan = Plan(rp, ci, K)
    want = oracle_mod.spmm_f32(rowptr, colind, vals, B, op, seg_len=SEG)
    cuts = [0, 1, 6_999, 7_000, 7_001, 7_002, 12_345, 15_000, 29_998, M]
    out = torch.full((M, N), float("nan"), device=cuda)
    from paper_2503_08946_b200 import spmm

    spmm.set_schedule_override(mode)  # 1: the dynamic item counter inside row ranges too
    try:
        for j in range(len(cuts) - 1):
            plan.execute_rows(vv, Bt, cuts[j], cuts[j + 1], out=out, reduce=op)
            torch.cuda.synchronize()
            done = out[:cuts[j + 1]].cpu().numpy()
            np.testing.assert_array_equal(done, want[:cuts[j + 1]])
    finally:
        spmm.set_schedule_override(-1)
    np.testing.assert_array_equal(out.cpu().numpy(), want)


def test_overlapped_allgather_nccl_single_rank(cuda, oracle_mod):
    """ShardedSpMM(chunks=4, gather=True) over NCCL (world 1 on the one GPU):
    execute_rows on the compute stream, broadcasts on a comm stream."""
    import socket

    import torch
    import torch.distributed as dist

    from paper_2503_08946_b200 import sharded as S

    rng = np.random.default_rng(51)
    M, K, N = 20_000, 3_000, 64
    rowptr, colind, vals = powerlaw_csr(rng, M, K, 10, [(5_000, 1_500)])
    B = rng.uniform(-1, 1, (K, N)).astype(np.float32)
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1,
                            device_id=cuda)
    try:
        rp, ci, vv, Bt = to_dev(cuda, rowptr, colind, vals, B)
        bounds = S.partition(rowptr, 1)
        sh = S.ShardedSpMM(rp, ci, K, bounds)
        for op in ("sum", "min"):
            C = sh(vv, Bt, op, gather=True, chunks=4)
            torch.cuda.synchronize()
            np.testing.assert_array_equal(C.cpu().numpy(),
                                          oracle_mod.spmm_f32(rowptr, colind, vals, B, op, seg_len=SEG))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("chunks", [1, 3])
def test_capi_sharded_spmm_single_rank(cuda, oracle_mod, chunks):
    """gespmm_sharded_spmm[_chunked] through the C-ABI (NCCL resolved by dlopen,
    world 1 on the one GPU): B broadcast, local slab, C all-gather (overlapped
    with the computation when chunks > 1) -- bit-exact to the twin."""
    import ctypes

    import torch

    from paper_2503_08946_b200 import _lib

    L = _lib.load()
    rng = np.random.default_rng(60)
    M, K, N = 12_000, 2_000, 64
    rowptr, colind, vals = powerlaw_csr(rng, M, K, 10, [(3_000, 1_200)])
    B = rng.uniform(-1, 1, (K, N)).astype(np.float32)
    rp, ci, vv, Bt = to_dev(cuda, rowptr, colind, vals, B)
    uid = ctypes.create_string_buffer(128)
    _lib.check(L.gespmm_comm_get_unique_id(uid))
    comm = ctypes.c_void_p()
    _lib.check(L.gespmm_comm_init(ctypes.byref(comm), 1, uid, 0))
    try:
        C = torch.empty((M, N), device=cuda)
        Cf = torch.full((M, N), float("nan"), device=cuda)
        bounds = (ctypes.c_int64 * 2)(0, M)
        s = torch.cuda.current_stream(cuda).cuda_stream
        _lib.check(L.gespmm_sharded_spmm_chunked(
            comm, 1, 0, 0, None, M, K, N, int(rowptr[-1]), rp.data_ptr(), ci.data_ptr(), vv.data_ptr(),
            Bt.data_ptr(), N, C.data_ptr(), N, 0, 0, Cf.data_ptr(), N, bounds, chunks, s))
        torch.cuda.synchronize()
        want = oracle_mod.spmm_f32(rowptr, colind, vals, B, "sum", seg_len=SEG)
        np.testing.assert_array_equal(C.cpu().numpy(), want)
        np.testing.assert_array_equal(Cf.cpu().numpy(), want)
    finally:
        L.gespmm_comm_destroy(comm)


@pytest.mark.parametrize("panels,gather", [(2, False), (3, True), (4, True)])
def test_capi_sharded_spmm_ex_panelled_broadcast(cuda, oracle_mod, panels, gather):
    """gespmm_sharded_spmm_ex with the B broadcast in column panels overlapped
    with the compute (world 1 over NCCL on the one GPU), with and
    without a caller workspace, bounded error-polled wait: bit-exact to the
    twin for N = 128 (4 x 32 panels) and a ragged N = 80."""
    import ctypes

    import torch

    from paper_2503_08946_b200 import _lib

    L = _lib.load()
    rng = np.random.default_rng(61)
    M, K = 9_000, 1_500
    rowptr, colind, vals = powerlaw_csr(rng, M, K, 10, [(100, 900)])
    uid = ctypes.create_string_buffer(128)
    _lib.check(L.gespmm_comm_get_unique_id(uid))
    comm = ctypes.c_void_p()
    _lib.check(L.gespmm_comm_init(ctypes.byref(comm), 1, uid, 0))
    try:
        for N, op in ((128, "sum"), (80, "max")):
            B = rng.uniform(-1, 1, (K, N)).astype(np.float32)
            rp, ci, vv, Bt = to_dev(cuda, rowptr, colind, vals, B)
            C = torch.full((M, N), float("nan"), device=cuda)
            Cf = torch.full((M, N), float("nan"), device=cuda) if gather else None
            ws = torch.empty(K * N, device=cuda) if panels == 3 else None
            bounds = (ctypes.c_int64 * 2)(0, M)
            o = _lib.ShardOpts(panels, ws.data_ptr() if ws is not None else None, 1, 60_000)
            s = torch.cuda.current_stream(cuda).cuda_stream
            _lib.check(L.gespmm_sharded_spmm_ex(
                comm, 1, 0, 0, None, M, K, N, int(rowptr[-1]), rp.data_ptr(), ci.data_ptr(), vv.data_ptr(),
                Bt.data_ptr(), N, C.data_ptr(), N, {"sum": 0, "max": 1}[op], 0,
                Cf.data_ptr() if gather else None, N, bounds, ctypes.byref(o), s))
            torch.cuda.synchronize()
            want = oracle_mod.spmm_f32(rowptr, colind, vals, B, op, seg_len=SEG)
            np.testing.assert_array_equal(C.cpu().numpy(), want)
            if gather:
                np.testing.assert_array_equal(Cf.cpu().numpy(), want)
    finally:
        L.gespmm_comm_destroy(comm)


def test_capi_sharded_spmm_ex_validates_before_any_collective(cuda):
    """No plan passed: the temporary plan validates colind before the B
    broadcast: an out-of-range column is GESPMM_CSR_INVALID, not an
    out-of-bounds gather; the communicator stays usable."""
    import ctypes

    import torch

    from paper_2503_08946_b200 import _lib
    from paper_2503_08946_b200.errors import Error, ErrorKind

    L = _lib.load()
    rng = np.random.default_rng(62)
    M, K, N = 500, 300, 64
    rowptr, colind, vals = random_csr(rng, M, K, 0.05)
    bad = colind.copy()
    bad[len(bad) // 2] = K + 5
    B = rng.uniform(-1, 1, (K, N)).astype(np.float32)
    uid = ctypes.create_string_buffer(128)
    _lib.check(L.gespmm_comm_get_unique_id(uid))
    comm = ctypes.c_void_p()
    _lib.check(L.gespmm_comm_init(ctypes.byref(comm), 1, uid, 0))
    try:
        s = torch.cuda.current_stream(cuda).cuda_stream
        C = torch.empty((M, N), device=cuda)
        for panels in (1, 2):
            rp, ci, vv, Bt = to_dev(cuda, rowptr, bad, vals, B)
            o = _lib.ShardOpts(panels, None, 1, 60_000)
            with pytest.raises(Error) as ei:
                _lib.check(L.gespmm_sharded_spmm_ex(
                    comm, 1, 0, 0, None, M, K, N, int(rowptr[-1]), rp.data_ptr(), ci.data_ptr(), vv.data_ptr(),
                    Bt.data_ptr(), N, C.data_ptr(), N, 0, 0, None, N, None, ctypes.byref(o), s))
            assert ei.value.kind == ErrorKind.CsrInvalid
        torch.cuda.synchronize()
        ci = torch.as_tensor(colind, device=cuda)
        _lib.check(L.gespmm_sharded_spmm_ex(
            comm, 1, 0, 0, None, M, K, N, int(rowptr[-1]), rp.data_ptr(), ci.data_ptr(), vv.data_ptr(),
            Bt.data_ptr(), N, C.data_ptr(), N, 0, 0, None, N, None, ctypes.byref(o), s))
        torch.cuda.synchronize()
    finally:
        L.gespmm_comm_destroy(comm)


def test_comm_wait_timeout_aborts_instead_of_hanging(cuda):
    """gespmm_comm_wait polls ncclCommGetAsyncError while the stream runs; a
    wait past its bound (here: a stream held by a ~1 s spin kernel, standing in
    for a collective whose peer died) aborts the communicator and returns
    GESPMM_NCCL_ERROR; destroying the aborted comm is a no-op; a short wait on
    an idle stream is OK."""
    import ctypes

    import torch

    from paper_2503_08946_b200 import _lib

    L = _lib.load()
    uid = ctypes.create_string_buffer(128)
    _lib.check(L.gespmm_comm_get_unique_id(uid))
    comm = ctypes.c_void_p()
    _lib.check(L.gespmm_comm_init(ctypes.byref(comm), 1, uid, 0))
    stream = torch.cuda.Stream(device=cuda)
    assert L.gespmm_comm_wait(comm, stream.cuda_stream, 1000) == 0
    with torch.cuda.stream(stream):
        torch.cuda._sleep(2_000_000_000)  # ~1 s of GPU clock cycles
    rc = L.gespmm_comm_wait(comm, stream.cuda_stream, 50)
    assert rc == 5, rc  # GESPMM_NCCL_ERROR
    assert b"timed out" in L.gespmm_last_error()
    stream.synchronize()
    assert L.gespmm_comm_wait(comm, stream.cuda_stream, 50) == 5  # aborted: stays an error
    assert L.gespmm_comm_destroy(comm) == 0


@pytest.mark.parametrize("args", [("20000", "5000", "128", "24", "4"), ("30000", "7000", "80", "16", "3"),
                                  ("5000", "3000", "32", "8", "1")])
def test_cpp_host_sharded_path(cuda, args):
    """examples/sharded_host: a plain C++ host (no Python in the process) runs
    the multi-GPU path through the C-ABI -- one NCCL rank per visible GPU,
    per-rank validation + agreement, column-panelled B broadcast overlapped
    with the compute, C all-gather, bounded wait -- and checks rank 0's full
    C against a host fp64 sum under the north-star bound."""
    import os
    import subprocess

    exe = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "examples", "sharded_host")
    if not os.path.exists(exe):
        pytest.skip("examples/sharded_host not built")
    r = subprocess.run([exe, *args], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "sharded_host ok" in r.stdout, r.stdout


@pytest.mark.parametrize("op", OPS)
def test_64bit_b_offsets(cuda, oracle_mod, op):
    """K * ldb > 2^32: the kernel's 64-bit B-row addressing path (staged 32-bit
    offsets would overflow).  B is a strided view (ldb ~ 7.2 M floats) into a
    17 GB buffer; only its K x N window is written."""
    import torch

    from paper_2503_08946_b200.spmm import Plan

    rng = np.random.default_rng(70)
    M, K, N = 3_000, 600, 64
    ldb = (2**32) // (K - 1) + 64  # (K-1) * ldb > 2^32
    rowptr, colind, vals = powerlaw_csr(rng, M, K, 8, [(100, 700)])
    B = rng.uniform(-1, 1, (K, N)).astype(np.float32)
    big = torch.empty((K - 1) * ldb + N, dtype=torch.float32, device=cuda)
    Bv = big.as_strided((K, N), (ldb, 1))
    Bv.copy_(torch.from_numpy(B))
    rp, ci, vv, _ = to_dev(cuda, rowptr, colind, vals, B[:1])
    plan = Plan(rp, ci, K)
    got = plan.execute(vv, Bv, op)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(got.cpu().numpy(), oracle_mod.spmm_f32(rowptr, colind, vals, B, op, seg_len=SEG))
    del big, Bv


@pytest.mark.parametrize("op", ["sum", "max"])
def test_max_nnz_near_int32_limit(cuda, oracle_mod, op):
    """The largest nnz the int32 CSR contract admits (2^31 - 2048): 1024 rows of
    ~2.1 M nonzeros (8,191 segments each), N=4.  Exercises every position /
    segment / partial-slot computation at its upper range; sampled rows
    (incl. first/last) bit-exact to the twin."""
    import torch

    from paper_2503_08946_b200 import workloads as W
    from paper_2503_08946_b200.spmm import Plan

    M, K, N = 1024, 4096, 4
    nnz = 2**31 - 2048
    per = nnz // M
    rowptr = torch.arange(M + 1, dtype=torch.int64, device=cuda) * per
    rowptr[-1] = nnz
    rowptr = rowptr.to(torch.int32)
    pos = torch.arange(nnz, dtype=torch.int32, device=cuda)
    colind = (pos * 7 + (pos >> 12)) % K
    vals = ((pos % 13) - 6).to(torch.float32) * 0.125
    del pos
    csr = W.Csr(rowptr, colind, vals, M, K)
    B = W.dense_gpu(K, N, seed=4, device=cuda)
    plan = Plan(rowptr, colind, K)
    C = plan.execute(vals, B, op)
    torch.cuda.synchronize()
    sampled_rows_bit_exact(oracle_mod, csr, B, C, op, n_random=3)
    del csr, colind, vals, plan
    torch.cuda.empty_cache()


@pytest.mark.parametrize("N,op", [(64, "sum"), (32, "max"), (256, "mean"), (16, "sum")])
def test_fused_peer_stores(cuda, oracle_mod, N, op):
    """gespmm_plan_execute_peers: every row also lands in each peer buffer at
    row peer_row0 + local row (one GPU: the peers are two other buffers);
    N=16 sum (a paired-lane shape) and N=256 (column panels) included."""
    import torch

    from paper_2503_08946_b200.spmm import Plan

    rng = np.random.default_rng(80 + N)
    M, K = 5_000, 1_500
    rowptr, colind, vals = powerlaw_csr(rng, M, K, 9, [(10, 1_300), (4_999, 300)])
    B = rng.uniform(-1, 1, (K, N)).astype(np.float32)
    rp, ci, vv, Bt = to_dev(cuda, rowptr, colind, vals, B)
    plan = Plan(rp, ci, K)
    C = torch.empty((M, N), device=cuda)
    row0 = 777
    fulls = [torch.full((M + 1_000, N), float("nan"), device=cuda) for _ in range(2)]
    plan.execute_peers(vv, Bt, C, [f.data_ptr() for f in fulls], row0, reduce=op)
    torch.cuda.synchronize()
    want = oracle_mod.spmm_f32(rowptr, colind, vals, B, op, seg_len=SEG)
    np.testing.assert_array_equal(C.cpu().numpy(), want)
    for f in fulls:
        np.testing.assert_array_equal(f[row0:row0 + M].cpu().numpy(), want)
        assert torch.isnan(f[:row0]).all() and torch.isnan(f[row0 + M:]).all()


def _peer_worker(rank, world, port, q):
    import os
    import sys

    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch
    import torch.distributed as dist

    from paper_2503_08946_b200 import sharded as S

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        rng = np.random.default_rng(90)
        M, K, N = 20_000, 3_000, 64
        rowptr, colind, vals = powerlaw_csr(rng, M, K, 9, [(9_999, 2_000), (10_000, 500)])
        B = rng.uniform(-1, 1, (K, N)).astype(np.float32)
        bounds = S.partition(rowptr, world)
        rp, ci, vv = S.local_block(rowptr, colind, vals, bounds, rank)
        dev = torch.device("cuda", 0)
        sh = S.ShardedSpMM(torch.as_tensor(rp, device=dev), torch.as_tensor(ci, device=dev), K, bounds)
        Bt = torch.as_tensor(B, device=dev)
        full = sh(torch.as_tensor(vv, device=dev), Bt, "sum", gather="peer", broadcast=False)
        q.put((rank, full.cpu().numpy()))
    finally:
        dist.destroy_process_group()


def test_fused_peer_allgather_two_processes(cuda, oracle_mod):
    """ShardedSpMM(gather="peer") with two ranks on the one GPU: CUDA IPC
    handles exchanged over the process group, each rank's kernel writes its
    rows into both ranks' full-C buffers; both equal the twin."""
    import socket

    import torch.multiprocessing as mp

    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_peer_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    out = dict(q.get(timeout=300) for _ in ps)
    for p in ps:
        p.join(timeout=60)
    rng = np.random.default_rng(90)
    M, K, N = 20_000, 3_000, 64
    rowptr, colind, vals = powerlaw_csr(rng, M, K, 9, [(9_999, 2_000), (10_000, 500)])
    B = rng.uniform(-1, 1, (K, N)).astype(np.float32)
    want = oracle_mod.spmm_f32(rowptr, colind, vals, B, "sum", seg_len=SEG)
    np.testing.assert_array_equal(out[0], want)
    np.testing.assert_array_equal(out[1], want)


@pytest.mark.parametrize("op", ["sum", "max"])
def test_execute_under_cuda_graph_capture(cuda, oracle_mod, op):
    """plan.execute is capturable into a CUDA graph (after one warm-up call
    sized the workspace): replays with new vals/B contents in the same buffers
    give the twin's bits -- launch-bound small SpMMs (config 1) replay without
    per-call host overhead."""
    import torch

    from paper_2503_08946_b200 import spmm
    from paper_2503_08946_b200.spmm import Plan

    rng = np.random.default_rng(140)
    M, K, N = 4096, 4096, 32
    rowptr, colind, vals = powerlaw_csr(rng, M, K, 20, [(17, 900)])
    rp, ci = to_dev(cuda, rowptr, colind)
    vv = torch.empty(colind.size, dtype=torch.float32, device=cuda)
    Bt = torch.empty((K, N), dtype=torch.float32, device=cuda)
    C = torch.empty((M, N), dtype=torch.float32, device=cuda)
    plan = Plan(rp, ci, K)
    for mode in (-1, 1):  # static striding (small plan) and the dynamic counter (memset node)
        spmm.set_schedule_override(mode)
        try:
            s = torch.cuda.Stream(device=cuda)
            with torch.cuda.stream(s):
                plan.execute(vv, Bt, op, out=C, stream=s)  # warm-up: workspace, attributes
            torch.cuda.synchronize()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=s):
                plan.execute(vv, Bt, op, out=C, stream=s)
            for rep in range(3):
                v = rng.uniform(-1, 1, colind.size).astype(np.float32)
                B = rng.uniform(-1, 1, (K, N)).astype(np.float32)
                vv.copy_(torch.from_numpy(v))
                Bt.copy_(torch.from_numpy(B))
                g.replay()
                torch.cuda.synchronize()
                np.testing.assert_array_equal(C.cpu().numpy(),
                                              oracle_mod.spmm_f32(rowptr, colind, v, B, op, seg_len=SEG))
        finally:
            spmm.set_schedule_override(-1)
