"""CPU tier: the fp32 twin (the normative semantics the GPU is bit-exact to)
checked against a pure-Python restatement on small cases, plus the algebraic
properties DESIGN.md relies on (order/segmentation invariance of max/min, mean =
sum/deg, accumulate = the reference's C read-modify-write order)."""
import math
from fractions import Fraction

import numpy as np
import pytest

SEG = 256


def assert_same_bits(got, want):
    """Bit-exact, except NaN payload/sign bits (not part of the contract)."""
    nan = np.isnan(want)
    np.testing.assert_array_equal(np.isnan(got), nan)
    np.testing.assert_array_equal(got[~nan].view(np.uint32), want[~nan].view(np.uint32))


def fma32(a, b, c):
    """Correctly rounded fp32 fused multiply-add (math.fma is Python >= 3.13):
    exact rational a*b + c, rounded to the nearest fp32, ties to even."""
    a, b, c = float(a), float(b), float(c)
    if not all(map(math.isfinite, (a, b, c))):
        return np.float32(a * b + c)  # inf/nan propagate identically
    exact = Fraction(a) * Fraction(b) + Fraction(c)
    x = np.float32(float(exact))
    if not math.isfinite(float(x)):
        return x
    cands = [x, np.nextafter(x, np.float32(np.inf)), np.nextafter(x, np.float32(-np.inf))]
    cands = [y for y in cands if math.isfinite(float(y))]
    return min(cands, key=lambda y: (abs(Fraction(float(y)) - exact), int(np.float32(y).view(np.uint32)) & 1))


CANON_NAN = np.array([0x7FFFFFFF], np.uint32).view(np.float32)[0]


def pick(op, a, b):
    """IEEE 754-2019 maximumNumber / minimumNumber as the B200's FMNMX computes
    them: NaN operands ignored, NaN+NaN -> canonical NaN, -0 < +0."""
    if np.isnan(a):
        return CANON_NAN if np.isnan(b) else b
    if np.isnan(b):
        return a
    if a == b:  # +-0 tie (equal non-zeros are identical)
        return b if bool(np.signbit(a)) == (op == "max") else a
    return (a if a > b else b) if op == "max" else (a if a < b else b)


def py_twin(rowptr, colind, vals, B, op, accumulate=False, C0=None, seg=0):
    """Pure-Python fp32 restatement (np.float32 scalars, fma32 above)."""
    f32 = np.float32
    M, N = len(rowptr) - 1, B.shape[1]
    C = np.zeros((M, N), np.float32) if C0 is None else C0.astype(np.float32).copy()
    for i in range(M):
        rs, re = int(rowptr[i]), int(rowptr[i + 1])
        deg = re - rs
        segs = [(rs, re)] if (seg <= 0 or deg <= seg) else [(s, min(s + seg, re)) for s in range(rs, re, seg)]
        for j in range(N):
            c0 = f32(C[i, j]) if accumulate else f32(0)
            if op in ("sum", "mean"):
                acc_total = None
                for k, (a, b) in enumerate(segs):
                    # two chains: even offsets from the segment start (seeded with
                    # C0 or +0) and odd offsets (seeded with -0.0); value = A + B
                    ca = c0 if (k == 0 and accumulate and op == "sum") else f32(0)
                    cb = f32(-0.0)
                    for p in range(a, b):
                        if (p - a) % 2 == 0:
                            ca = fma32(vals[p], B[colind[p], j], ca)
                        else:
                            cb = fma32(vals[p], B[colind[p], j], cb)
                    acc = f32(ca + cb)
                    acc_total = acc if acc_total is None else f32(acc_total + acc)
                if acc_total is None:
                    acc_total = c0 if (accumulate and op == "sum") else f32(0)
                if op == "mean":
                    r = f32(acc_total / f32(deg)) if deg else f32(0)
                    C[i, j] = f32(c0 + r) if accumulate else r
                else:
                    C[i, j] = acc_total
            else:
                if deg == 0:
                    C[i, j] = c0 if accumulate else f32(0)
                    continue
                acc = c0 if accumulate else CANON_NAN
                for p in range(rs, re):  # order-free: segments do not matter
                    acc = pick(op, acc, f32(vals[p] * B[colind[p], j]))
                C[i, j] = acc
    return C


def rand_case(seed, M=40, K=30, N=5, long_deg=0, special=False):
    rng = np.random.default_rng(seed)
    deg = rng.integers(0, 8, M)
    deg[rng.random(M) < 0.25] = 0
    if long_deg:
        deg[3] = long_deg
    rowptr = np.concatenate([[0], np.cumsum(deg)]).astype(np.int32)
    colind = rng.integers(0, K, int(rowptr[-1])).astype(np.int32)
    vals = rng.uniform(-1, 1, colind.size).astype(np.float32)
    B = rng.uniform(-1, 1, (K, N)).astype(np.float32)
    if special:
        vals[::5] = np.nan
        vals[1::7] = -0.0
        B[::3] = -0.0
        B[1::4] = np.inf
    C0 = rng.uniform(-1, 1, (M, N)).astype(np.float32)
    return rowptr, colind, vals, B, C0


@pytest.mark.parametrize("op", ["sum", "max", "min", "mean"])
@pytest.mark.parametrize("accumulate", [False, True])
@pytest.mark.parametrize("special", [False, True])
def test_twin_matches_python_restatement(oracle_mod, op, accumulate, special):
    rowptr, colind, vals, B, C0 = rand_case(1, long_deg=40, special=special)
    for seg in (0, 16):
        want = py_twin(rowptr, colind, vals, B, op, accumulate, C0 if accumulate else None, seg)
        got = oracle_mod.spmm_f32(rowptr, colind, vals, B, op, accumulate=accumulate,
                                  C0=C0 if accumulate else None, seg_len=seg)
        assert_same_bits(got, want)


@pytest.mark.parametrize("op", ["max", "min"])
@pytest.mark.parametrize("seg", [1, 3, 16, 256])
def test_max_min_independent_of_segmentation(oracle_mod, op, seg):
    for special in (False, True):
        rowptr, colind, vals, B, C0 = rand_case(7, M=60, K=50, N=9, long_deg=700, special=special)
        for acc in (False, True):
            a = oracle_mod.spmm_f32(rowptr, colind, vals, B, op, accumulate=acc, C0=C0, seg_len=0)
            b = oracle_mod.spmm_f32(rowptr, colind, vals, B, op, accumulate=acc, C0=C0, seg_len=seg)
            assert_same_bits(b, a)


def test_mean_is_sum_over_degree(oracle_mod):
    rowptr, colind, vals, B, _ = rand_case(3, long_deg=600)
    s = oracle_mod.spmm_f32(rowptr, colind, vals, B, "sum", seg_len=SEG)
    m = oracle_mod.spmm_f32(rowptr, colind, vals, B, "mean", seg_len=SEG)
    deg = np.diff(rowptr).astype(np.float32)[:, None]
    want = np.where(deg > 0, s / np.where(deg > 0, deg, 1), 0).astype(np.float32)
    np.testing.assert_array_equal(m, want)


def test_accumulate_sum_seeds_chain_a_with_c0(oracle_mod):
    """accumulate=1 seeds chain A (even offsets) with C0, the reference's
    c = C0; c = c + v*b order restricted to that chain."""
    rowptr = np.array([0, 3], np.int32)
    colind = np.array([0, 1, 2], np.int32)
    vals = np.array([1e8, 1.0, -1e8], np.float32)
    B = np.ones((3, 1), np.float32)
    C0 = np.array([[1.0]], np.float32)
    got = oracle_mod.spmm_f32(rowptr, colind, vals, B, "sum", accumulate=True, C0=C0)
    f = np.float32
    chain_a = f(f(f(1) + f(1e8)) + f(-1e8))  # C0, then positions 0 and 2
    chain_b = f(f(-0.0) + f(1.0))             # position 1
    assert got[0, 0] == f(chain_a + chain_b)


def test_sign_of_zero_preserved_by_the_minus_zero_seed(oracle_mod):
    """Chain B starts at -0.0, so a one-nonzero row returns exactly fma(v, b, +0)
    and an accumulate of C0 = -0 over an empty row returns -0."""
    B = np.array([[-0.0], [2.0]], np.float32)
    got = oracle_mod.spmm_f32(np.array([0, 1], np.int32), np.array([0], np.int32),
                              np.array([3.0], np.float32), B, "sum")
    assert got[0, 0] == 0.0 and not np.signbit(got[0, 0])  # 3 * -0 + (+0) = +0
    C0 = np.array([[-0.0]], np.float32)
    got = oracle_mod.spmm_f32(np.array([0, 0], np.int32), np.zeros(0, np.int32),
                              np.zeros(0, np.float32), B, "sum", accumulate=True, C0=C0)
    assert np.signbit(got[0, 0])


def test_empty_rows_give_zero(oracle_mod):
    rowptr = np.array([0, 0, 0], np.int32)
    B = np.ones((3, 4), np.float32)
    for op in ("sum", "max", "min", "mean"):
        got = oracle_mod.spmm_f32(rowptr, np.zeros(0, np.int32), np.zeros(0, np.float32), B, op)
        np.testing.assert_array_equal(got, np.zeros((2, 4), np.float32))


def _bits(x):
    return np.asarray(x, np.float32).view(np.uint32)


def test_max_min_are_maximum_number(oracle_mod):
    """max/min = IEEE 754-2019 maximumNumber/minimumNumber over the messages:
    NaN messages ignored, all-NaN -> canonical NaN, -0 < +0, order-free."""
    B = np.array([[1.0], [-0.0], [np.nan], [0.0]], np.float32)
    one = np.float32(1.0)
    cases = [  # (columns of the row's messages (vals all 1), max, min)
        ([1, 3], 0.0, -0.0), ([3, 1], 0.0, -0.0),           # +-0 either order
        ([2, 0], 1.0, 1.0), ([0, 2], 1.0, 1.0),             # NaN first or last: ignored
        ([2, 2], CANON_NAN, CANON_NAN), ([2], CANON_NAN, CANON_NAN),
        ([1], -0.0, -0.0), ([1, 2, 3, 0], 1.0, -0.0),
    ]
    for cols, want_max, want_min in cases:
        rowptr = np.array([0, len(cols)], np.int32)
        colind = np.array(cols, np.int32)
        vals = np.full(len(cols), one, np.float32)
        for op, want in (("max", want_max), ("min", want_min)):
            got = oracle_mod.spmm_f32(rowptr, colind, vals, B, op)
            assert _bits(got[0, 0]) == _bits(want), (cols, op, got[0, 0], want)
            assert _bits(got[0, 0]) == _bits(py_twin(rowptr, colind, vals, B, op)[0, 0])


@pytest.mark.parametrize("op", ["max", "min"])
def test_max_min_independent_of_order(oracle_mod, op):
    """Permuting each row's nonzeros changes nothing, bit for bit (NaN included)."""
    rng = np.random.default_rng(11)
    rowptr, colind, vals, B, C0 = rand_case(5, M=50, K=40, N=7, long_deg=300, special=True)
    a = oracle_mod.spmm_f32(rowptr, colind, vals, B, op, accumulate=True, C0=C0, seg_len=16)
    for i in range(len(rowptr) - 1):
        rs, re = rowptr[i], rowptr[i + 1]
        perm = rs + rng.permutation(re - rs)
        colind[rs:re], vals[rs:re] = colind[perm].copy(), vals[perm].copy()
    b = oracle_mod.spmm_f32(rowptr, colind, vals, B, op, accumulate=True, C0=C0, seg_len=0)
    np.testing.assert_array_equal(_bits(a), _bits(b))
