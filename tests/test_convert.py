"""GPU format conversions (COO -> CSR, CSR transpose) against numpy stable-sort
restatements, and the transpose feeding the SpMM path (A^T x B)."""
import numpy as np
import pytest

SEG = 256


def np_coo_to_csr(rows, cols, vals, M):
    order = np.argsort(rows, kind="stable")
    rowptr = np.zeros(M + 1, np.int64)
    np.add.at(rowptr, rows + 1, 1)
    return np.cumsum(rowptr).astype(np.int32), cols[order], vals[order]


@pytest.mark.gpu
@pytest.mark.parametrize("seed,M,K,nnz", [(0, 1000, 700, 20_000), (1, 1, 5, 3), (2, 50, 50, 0), (3, 4000, 3000, 200_000)])
def test_coo_to_csr_bit_exact(seed, M, K, nnz):
    import torch

    from paper_2503_08946_b200.spmm import coo_to_csr

    rng = np.random.default_rng(seed)
    rows = rng.integers(0, M, nnz).astype(np.int32)
    cols = rng.integers(0, K, nnz).astype(np.int32)
    vals = rng.uniform(-1, 1, nnz).astype(np.float32)
    d = torch.device("cuda:0")
    t = lambda a: torch.as_tensor(a, device=d)  # noqa: E731
    rp, ci, vv = coo_to_csr(t(rows), t(cols), t(vals), M)
    torch.cuda.synchronize()
    wrp, wci, wvv = np_coo_to_csr(rows, cols, vals, M)
    np.testing.assert_array_equal(rp.cpu().numpy(), wrp)
    np.testing.assert_array_equal(ci.cpu().numpy(), wci)
    np.testing.assert_array_equal(vv.cpu().numpy(), wvv)


@pytest.mark.gpu
def test_coo_to_csr_out_of_range_row():
    import torch

    from paper_2503_08946_b200.errors import Error, ErrorKind
    from paper_2503_08946_b200.spmm import coo_to_csr

    d = torch.device("cuda:0")
    rows = torch.tensor([0, 5], dtype=torch.int32, device=d)
    cols = torch.tensor([0, 1], dtype=torch.int32, device=d)
    vals = torch.tensor([1.0, 2.0], device=d)
    with pytest.raises(Error) as ei:
        coo_to_csr(rows, cols, vals, 3)
    assert ei.value.kind == ErrorKind.OutOfBounds


@pytest.mark.gpu
def test_transpose_and_spmm_of_transpose(oracle_mod):
    """A^T via the GPU transpose equals the numpy CSC of A; A^T x B on the GPU
    path equals the twin on the transposed CSR; transposing twice restores A
    up to within-row order (sorted rows are restored exactly)."""
    import torch

    from paper_2503_08946_b200 import workloads as W
    from paper_2503_08946_b200.spmm import Plan, csr_transpose

    c = W.rmat_csr(12, 30_000, seed=5)  # sorted, unique columns per row
    rp, ci, vv = c.rowptr.numpy(), c.colind.numpy(), c.vals.numpy()
    M = K = c.M
    rows = np.repeat(np.arange(M, dtype=np.int32), np.diff(rp))
    wrp, wci, wvv = np_coo_to_csr(ci, rows, vv, K)  # CSC of A = CSR of A^T, stable in row order
    d = torch.device("cuda:0")
    t = lambda a: torch.as_tensor(np.ascontiguousarray(a), device=d)  # noqa: E731
    trp, tci, tvv = csr_transpose(t(rp), t(ci), t(vv), K)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(trp.cpu().numpy(), wrp)
    np.testing.assert_array_equal(tci.cpu().numpy(), wci)
    np.testing.assert_array_equal(tvv.cpu().numpy(), wvv)
    B = np.random.default_rng(0).uniform(-1, 1, (M, 64)).astype(np.float32)
    got = Plan(trp, tci, M).execute(tvv, t(B), "sum")
    np.testing.assert_array_equal(got.cpu().numpy(), oracle_mod.spmm_f32(wrp, wci, wvv, B, "sum", seg_len=SEG))
    rrp, rci, rvv = csr_transpose(trp, tci, tvv, M)
    np.testing.assert_array_equal(rrp.cpu().numpy(), rp)
    np.testing.assert_array_equal(rci.cpu().numpy(), ci)
    np.testing.assert_array_equal(rvv.cpu().numpy(), vv)
