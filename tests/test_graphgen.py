"""Native synthetic-input generator: the numpy restatement
(oracle/graphgen.py) pinned by Random123's published Philox4x32-10 known-answer
vectors, the R-MAT structure, and the CUDA generator bit for bit against it."""
import numpy as np
import pytest

from oracle import graphgen as G

# Random123 kat_vectors, philox4x32 10 rounds: (counter, key) -> output
KAT = [
    ((0, 0, 0, 0), (0, 0), (0x6627E8D5, 0xE169C58D, 0xBC57AC4C, 0x9B00DBD8)),
    ((0xFFFFFFFF,) * 4, (0xFFFFFFFF,) * 2, (0x408F276D, 0x41C83B0E, 0xA20BC7C6, 0x6D5451FD)),
    ((0x243F6A88, 0x85A308D3, 0x13198A2E, 0x03707344), (0xA4093822, 0x299F31D0),
     (0xD16CFE09, 0x94FDCCEB, 0x5001E420, 0x24126EA1)),
]


@pytest.mark.parametrize("ctr,key,want", KAT)
def test_philox_known_answers(ctr, key, want):
    got = G.philox4x32_10(*[np.uint32(x) for x in ctr], *key)
    assert tuple(int(x) for x in got) == want


def test_rmat_structure():
    scale, edges = 12, 60_000
    rp, ci, v = G.rmat_csr(scale, edges, seed=9)
    n = 1 << scale
    assert rp.shape == (n + 1,) and rp[0] == 0 and np.all(np.diff(rp) >= 0)
    nnz = int(rp[-1])
    assert 0.8 * edges < nnz <= edges and ci.shape == (nnz,) and v.shape == (nnz,)
    assert ci.min() >= 0 and ci.max() < n
    for r in range(0, n, 97):  # rows sorted and duplicate-free
        seg = ci[rp[r]:rp[r + 1]]
        assert np.all(np.diff(seg) > 0)
    assert v.dtype == np.float32 and v.min() >= -1.0 and v.max() < 1.0
    # quadrant statistics: a row bit is set with p = c + d = 0.24 per level
    keys = G.rmat_keys(scale, edges, 0.57, 0.19, 0.19, 9)
    rowbits = np.unpackbits((keys >> np.uint64(scale)).astype(">u8").view(np.uint8)).mean() * 64 / scale
    assert abs(rowbits - 0.24) < 0.01
    # power law: the hub row 0 is the heaviest
    assert np.argmax(np.diff(rp)) == 0


def test_rmat_deterministic():
    a = G.rmat_keys(10, 1000, 0.57, 0.19, 0.19, 3)
    b = G.rmat_keys(10, 1000, 0.57, 0.19, 0.19, 3)
    c = G.rmat_keys(10, 1000, 0.57, 0.19, 0.19, 4)
    assert np.array_equal(a, b) and not np.array_equal(a, c)


@pytest.mark.gpu
@pytest.mark.parametrize("scale,edges,seed", [(12, 40_000, 3), (9, 3_000, 77), (14, 5, 1)])
def test_native_rmat_bit_exact(scale, edges, seed):
    import torch

    from paper_2503_08946_b200 import workloads as W

    csr = W.rmat_csr_gpu(scale, edges, seed=seed, device="cuda:0")
    torch.cuda.synchronize()
    rp, ci, v = G.rmat_csr(scale, edges, seed=seed)
    np.testing.assert_array_equal(csr.rowptr.cpu().numpy(), rp)
    np.testing.assert_array_equal(csr.colind.cpu().numpy(), ci)
    np.testing.assert_array_equal(csr.vals.cpu().numpy(), v)


@pytest.mark.gpu
def test_native_uniform_fill_bit_exact():
    import torch

    from paper_2503_08946_b200 import workloads as W

    B = W.dense_gpu(1000, 37, seed=11, device="cuda:0")
    torch.cuda.synchronize()
    np.testing.assert_array_equal(B.cpu().numpy().ravel(), G.uniform(1000 * 37, -1.0, 1.0, 11))


@pytest.mark.gpu
def test_native_rmat_config2_properties():
    """Full config-2 size: sorted, unique, in range, and the nnz Graph500 dedup gives."""
    import torch

    from paper_2503_08946_b200 import workloads as W

    csr = W.rmat_csr_gpu(20, 16 * 2**20, seed=3, device="cuda:0")
    rp = csr.rowptr.long()
    ci = csr.colind.long()
    assert int(rp[0]) == 0 and int(rp[-1]) == csr.nnz and bool((rp[1:] >= rp[:-1]).all())
    assert 16_000_000 < csr.nnz < 16_200_000
    rows = torch.repeat_interleave(torch.arange(csr.M, device=ci.device), rp[1:] - rp[:-1])
    key = rows * csr.M + ci
    assert bool((key[1:] > key[:-1]).all())  # sorted by (row, col), no duplicates
    assert int(ci.min()) >= 0 and int(ci.max()) < csr.M
