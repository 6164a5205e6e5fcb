"""Randomized parity sweep (seeded, deterministic): shapes, densities, long
rows, empty rows, duplicate/unsorted columns, odd N, strided/misaligned B and
C, accumulate, every reduce op, both item schedules, forced column panels and
forced kernel variants, the cached-plan and the one-shot entry points -- GPU
bit-exact to the fp32 twin in every case."""
import os

import numpy as np
import pytest

SEG = 256
VARIANTS = ["", "vec1_lpr32_cwm1", "vec1_lpr32_cwm2", "vec2_lpr32_cwm1", "vec2_lpr32_cwm2", "vec4_lpr32_cwm1",
            "vec4_lpr32_cwm2", "pair_vec1", "pair_vec2", "pair_vec4", "vec2_lpr32_cwm1_ring",
            "vec4_lpr32_cwm1_ring"]


def rand_csr(rng, M, K, mean_deg):
    deg = np.minimum((rng.pareto(1.3, M) * mean_deg / 2).astype(np.int64), 6000)
    deg[rng.random(M) < rng.uniform(0, 0.6)] = 0
    if M > 3 and rng.random() < 0.7:
        deg[rng.integers(0, M)] = int(rng.integers(257, 3000))  # a long row (several segments)
    rowptr = np.concatenate([[0], np.cumsum(deg)]).astype(np.int32)
    colind = rng.integers(0, K, int(rowptr[-1])).astype(np.int32)
    vals = rng.uniform(-2, 2, colind.size).astype(np.float32)
    if colind.size and rng.random() < 0.3:
        vals[rng.integers(0, colind.size, max(1, colind.size // 50))] = 0.0  # exact zeros (+-0 messages)
    return rowptr, colind, vals


CASES = list(range(int(os.environ.get("GESPMM_FUZZ_CASES", "200"))))


@pytest.mark.gpu
@pytest.mark.parametrize("case", CASES)
def test_fuzz_bit_exact(cuda, oracle_mod, case):
    import torch

    from paper_2503_08946_b200 import spmm
    from paper_2503_08946_b200.spmm import Plan

    rng = np.random.default_rng(1000 + case)
    M = int(rng.integers(1, 3000))
    K = int(rng.integers(1, 2500))
    N = int(rng.choice([1, 2, 3, 4, 7, 8, 16, 17, 31, 32, 33, 48, 64, 65, 96, 100, 128, 129, 200, 256, 300]))
    op = ["sum", "max", "min", "mean"][case % 4]
    rowptr, colind, vals = rand_csr(rng, M, K, float(rng.uniform(1, 40)))
    B = rng.uniform(-1, 1, (K, N)).astype(np.float32)
    special = rng.random() < 0.15  # NaN / inf / -0 operands
    if special and vals.size:
        vals[rng.integers(0, vals.size, max(1, vals.size // 40))] = np.nan
        vals[rng.integers(0, vals.size, max(1, vals.size // 40))] = -0.0
        B.ravel()[rng.integers(0, B.size, max(1, B.size // 30))] = np.inf
        B.ravel()[rng.integers(0, B.size, max(1, B.size // 30))] = -0.0
    accumulate = rng.random() < 0.3
    C0 = rng.uniform(-1, 1, (M, N)).astype(np.float32) if accumulate else None
    # strided / offset views of B and C
    ldb = N + int(rng.choice([0, 0, 1, 3, 4, 16]))
    ldc = N + int(rng.choice([0, 0, 2, 4, 8]))
    boff = int(rng.choice([0, 0, 1, 2, 4]))
    coff = int(rng.choice([0, 0, 1, 4]))
    Bbig = torch.zeros(K * ldb + boff + 8, dtype=torch.float32, device=cuda)
    Bt = Bbig[boff:boff + K * ldb].view(K, ldb)[:, :N]
    Bt.copy_(torch.from_numpy(B))
    Cbig = torch.full((M * ldc + coff + 8,), float("nan"), dtype=torch.float32, device=cuda)
    Ct = Cbig[coff:coff + M * ldc].view(M, ldc)[:, :N]
    if accumulate:
        Ct.copy_(torch.from_numpy(C0))
    rp = torch.as_tensor(rowptr, device=cuda)
    ci = torch.as_tensor(colind, device=cuda)
    vv = torch.as_tensor(vals, device=cuda)
    variant = VARIANTS[case % len(VARIANTS)]
    spmm.set_variant_override(variant)
    spmm.set_schedule_override(int(rng.integers(-1, 2)))
    spmm.set_panel_override(int(rng.choice([-1, -1, 0, 32, 64])))
    tw = int(rng.choice([0, 0, 2, 13, 32, 256]))
    spmm.set_tile_work_override(tw)
    # every third case through the one-shot entry point (gespmm_csr_spmm: the
    # plan built on the device with a-priori item bounds, one trailing sync)
    oneshot = case % 3 == 2
    try:
        if oneshot:
            spmm.csr_spmm(rp, ci, vv, Bt, op, out=Ct, accumulate=accumulate)
        else:
            plan = Plan(rp, ci, K)
            plan.execute(vv, Bt, op, out=Ct, accumulate=accumulate)
        torch.cuda.synchronize()
    finally:
        spmm.set_variant_override("")
        spmm.set_schedule_override(-1)
        spmm.set_panel_override(-1)
        spmm.set_tile_work_override(0)
    want = oracle_mod.spmm_f32(rowptr, colind, vals, B, op, accumulate=accumulate, C0=C0, seg_len=SEG)
    got = Ct.cpu().numpy()
    np.testing.assert_array_equal(got, want, err_msg=f"case {case}: M={M} K={K} N={N} op={op} variant={variant} "
                                                     f"tw={tw} oneshot={oneshot}")
    if op in ("max", "min"):  # maximumNumber: every bit, NaNs included
        np.testing.assert_array_equal(got.view(np.uint32), want.view(np.uint32), err_msg=f"case {case} bits")
    # nothing outside the C view was written
    full = Cbig.cpu().numpy()
    mask = np.ones(full.size, bool)
    idx = coff + (np.arange(M)[:, None] * ldc + np.arange(N)[None, :]).ravel()
    mask[idx] = False
    assert np.isnan(full[mask]).all(), f"case {case}: wrote outside C"
