"""Pins the CPU oracle (oracle/gespmm_oracle.c) against golden vectors produced
by the reference interpreter itself (tests/golden/make_golden.py), and -- when
oracle/_ref is built -- re-runs the reference live on the same inputs."""
import hashlib

import numpy as np
import pytest

from conftest import golden_cases, load_golden


def arrays(g):
    M, N, K = g["M"], g["N"], g["K"]
    rowptr = np.asarray(g["rowptr"], np.int32)
    colind = np.asarray(g["colind"], np.int32)
    vals = np.asarray(g["vals"], np.float64)
    B = np.asarray(g["B"], np.float64).reshape(K, N)
    C0 = np.asarray(g["C0"], np.float64).reshape(M, N)
    C = np.asarray(g["C"], np.float64).reshape(M, N)
    return M, N, K, rowptr, colind, vals, B, C0, C


def launch_rows_cols(g):
    M, N = g["M"], g["N"]
    return min(M, g["grid"][0]), min(N, g["grid"][1] * g["block"][0])


@pytest.mark.parametrize("name", golden_cases())
def test_f64_restatement_equals_reference_bitwise(oracle_mod, name):
    g = load_golden(name)
    M, N, K, rowptr, colind, vals, B, C0, C = arrays(g)
    rows, cols = launch_rows_cols(g)
    got = C0.copy()
    rp = rowptr[: rows + 1]
    got[:rows, :cols] = oracle_mod.spmm_ref_f64(rp, colind, vals, B[:, :cols], C0[:rows, :cols])
    np.testing.assert_array_equal(got, C)  # bit-exact fp64


@pytest.mark.parametrize("name", golden_cases())
@pytest.mark.parametrize("seg_len", [0, 256, 7])
def test_f32_twin_within_north_star_tolerance(oracle_mod, name, seg_len):
    # sum: |twin - ref64| <= 1e-5 * max(|ref64|, sum_p |val*B|)  (north star, norm-wise)
    g = load_golden(name)
    M, N, K, rowptr, colind, vals, B, C0, C = arrays(g)
    rows, cols = launch_rows_cols(g)
    rp = rowptr[: rows + 1]
    twin = oracle_mod.spmm_f32(rp, colind, vals.astype(np.float32), B[:, :cols].astype(np.float32),
                               "sum", accumulate=True, C0=C0[:rows, :cols].astype(np.float32),
                               seg_len=seg_len)
    bound = oracle_mod.spmm_absbound(rp, colind, vals.astype(np.float32),
                                     B[:, :cols].astype(np.float32))
    ref = C[:rows, :cols]
    scale = np.maximum(np.abs(ref), bound + np.abs(C0[:rows, :cols]))
    assert np.all(np.abs(twin.astype(np.float64) - ref) <= 1e-5 * scale + 1e-30)


def test_shipped_goldens_match_survey_appendix_a():
    # SURVEY.md Appendix A, produced by the reference interpreter
    small = load_golden("ref_gespmm_small_full.json")
    assert small["C"] == [19, 22, 25, 28, 67, 74, 81, 88, 45, 50, 55, 60, 6, 12, 18, 24]
    assert small["log_len"] == 176
    shipped = load_golden("ref_gespmm_small_shipped.json")
    assert shipped["C"][8:] == [0] * 8 and shipped["log_len"] == 112
    assert load_golden("ref_gespmm_nnz2_shipped.json")["log_len"] == 64


def test_config1_checksum(oracle_mod):
    from paper_2503_08946_b200 import workloads as W

    g = load_golden("config1_checksum.json")
    csr = W.uniform_csr(4096, 4096, 0.01, seed=1)
    B = W.dense(4096, 32, seed=2)
    assert csr.nnz == g["nnz"]
    assert hashlib.sha256(csr.rowptr.tobytes()).hexdigest() == g["rowptr_sha256"]
    assert hashlib.sha256(csr.colind.tobytes()).hexdigest() == g["colind_sha256"]
    C = oracle_mod.spmm_ref_f64(csr.rowptr, csr.colind, csr.vals.astype(np.float64),
                                B.astype(np.float64))
    assert hashlib.sha256(C.tobytes()).hexdigest() == g["c_f64_sha256"]
    np.testing.assert_array_equal(C.sum(1), np.asarray(g["row_sums"]))


@pytest.mark.parametrize("name", ["rnd_ragged_c0.json", "rnd_unsorted_dup.json",
                                  "ref_gespmm_small_shipped.json"])
def test_live_reference_rerun(oracle_mod, name):
    """Re-run the unmodified reference interpreter (oracle/_ref) on the golden
    inputs: the committed vectors are still what the reference computes."""
    if not oracle_mod.ref_available():
        pytest.skip("oracle/_ref not built (reference tree absent)")
    g = load_golden(name)
    M, N, K, rowptr, colind, vals, B, C0, C = arrays(g)
    rows, cols = launch_rows_cols(g)
    got = C0.copy()
    Cr, secs, nlog = oracle_mod.ref_spmm_csr(rowptr[: rows + 1], colind,
                                             vals.astype(np.float32), B.astype(np.float32)[:, :cols],
                                             nthreads=2, C0=C0[:rows, :cols])
    got[:rows, :cols] = Cr
    np.testing.assert_array_equal(got, C)


def test_ref64_op_sum_is_the_pinned_reference(oracle_mod):
    """oracle_spmm_ref64_op (the per-op fp64 restatement the GPU parity tests
    hold every op to) computes, for sum, exactly the reference interpreter's
    C on config 1 (the golden sha256 of tests/golden/config1_checksum.json)."""
    from paper_2503_08946_b200 import workloads as W

    g = load_golden("config1_checksum.json")
    csr = W.uniform_csr(4096, 4096, 0.01, seed=1)
    B = W.dense(4096, 32, seed=2)
    C, bound = oracle_mod.spmm_ref64_op(csr.rowptr, csr.colind, csr.vals, B, "sum")
    assert hashlib.sha256(C.tobytes()).hexdigest() == g["c_f64_sha256"]
    assert np.all(bound >= np.abs(C))
    # max/min: (float) of the exact fp64 extreme product is what a correct fp32
    # max/min must produce; the fp32 twin agrees everywhere
    for op in ("max", "min"):
        ref, _ = oracle_mod.spmm_ref64_op(csr.rowptr, csr.colind, csr.vals, B, op)
        twin = oracle_mod.spmm_f32(csr.rowptr, csr.colind, csr.vals, B, op, seg_len=256)
        assert oracle_mod.ref64_error_ratio(twin, ref, None, op) == 0
    for op in ("sum", "mean"):
        ref, bound = oracle_mod.spmm_ref64_op(csr.rowptr, csr.colind, csr.vals, B, op)
        twin = oracle_mod.spmm_f32(csr.rowptr, csr.colind, csr.vals, B, op, seg_len=256)
        assert oracle_mod.ref64_error_ratio(twin, ref, bound, op) <= 1.0
