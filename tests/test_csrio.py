""".inst writer, binary CSR cache, Matrix Market I/O (CPU tier)."""
import os

import numpy as np
import pytest

from oracle import oracle as O
from paper_2503_08946_b200 import csrio
from paper_2503_08946_b200 import instance as I
from paper_2503_08946_b200.errors import Error, ErrorKind

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_FIXTURES = "/root/reference/proj/fixtures"


def _csr(seed=0, M=300, K=200):
    rng = np.random.default_rng(seed)
    deg = rng.integers(0, 9, M)
    deg[5] = 700  # a long row
    rowptr = np.concatenate([[0], np.cumsum(deg)]).astype(np.int32)
    colind = rng.integers(0, K, int(rowptr[-1])).astype(np.int32)  # unsorted, duplicates
    vals = rng.uniform(-1, 1, colind.size).astype(np.float32)
    return rowptr, colind, vals, M, K


def test_binary_cache_round_trip(tmp_path):
    rp, ci, vv, M, K = _csr()
    p = str(tmp_path / "g.csr")
    csrio.save_csr(p, rp, ci, vv, M, K, meta={"workload": "test"})
    assert os.path.getsize(p) % 4096 == 0
    r2, c2, v2, M2, K2, meta = csrio.load_csr(p)
    assert (M2, K2, meta) == (M, K, {"workload": "test"})
    np.testing.assert_array_equal(r2, rp)
    np.testing.assert_array_equal(c2, ci)
    np.testing.assert_array_equal(v2.view(np.uint32), vv.view(np.uint32))


def test_binary_cache_detects_corruption(tmp_path):
    rp, ci, vv, M, K = _csr(1)
    p = str(tmp_path / "g.csr")
    csrio.save_csr(p, rp, ci, vv, M, K)
    with open(p, "r+b") as f:
        f.seek(4096 * 2 + 8)  # inside colind
        b = f.read(1)
        f.seek(4096 * 2 + 8)
        f.write(bytes([b[0] ^ 0xFF]))
    with pytest.raises(Error) as ei:
        csrio.load_csr(p)
    assert ei.value.kind == ErrorKind.CsrInvalid
    with pytest.raises(Error) as ei:
        csrio.load_csr(str(tmp_path / "missing.csr"))
    assert ei.value.kind == ErrorKind.Io


def test_cached_csr_builds_once(tmp_path):
    from paper_2503_08946_b200 import workloads as W

    calls = []

    def make():
        calls.append(1)
        rp, ci, vv, M, K = _csr(2)
        return W.Csr(rp, ci, vv, M, K)

    p = str(tmp_path / "c.csr")
    a = csrio.cached_csr(p, make)
    b = csrio.cached_csr(p, make)
    assert len(calls) == 1
    np.testing.assert_array_equal(a.colind, b.colind)


def test_matrix_market_round_trip_and_spmm(tmp_path):
    rp, ci, vv, M, K = _csr(3)
    p = str(tmp_path / "g.mtx")
    csrio.write_matrix_market(p, rp, ci, vv, M, K, comment="test")
    r2, c2, v2, M2, K2 = csrio.read_matrix_market(p)
    assert (M2, K2) == (M, K)
    np.testing.assert_array_equal(r2, rp)
    np.testing.assert_array_equal(c2, ci)  # file order kept within rows, duplicates kept
    np.testing.assert_array_equal(v2, vv)  # %.9g round-trips fp32
    B = np.random.default_rng(0).uniform(-1, 1, (K, 16)).astype(np.float32)
    np.testing.assert_array_equal(O.spmm_f32(r2, c2, v2, B, "sum"), O.spmm_f32(rp, ci, vv, B, "sum"))


def test_matrix_market_symmetric_pattern():
    txt = """%%MatrixMarket matrix coordinate pattern symmetric
% a 3x3 path graph
3 3 3
1 1
2 1
3 2
"""
    rp, ci, vv, M, K = csrio.read_matrix_market(txt, text=True)
    assert (M, K) == (3, 3)
    assert rp.tolist() == [0, 2, 4, 5]
    assert ci.tolist() == [0, 1, 0, 2, 1]
    assert vv.tolist() == [1, 1, 1, 1, 1]
    skew = "%%MatrixMarket matrix coordinate real skew-symmetric\n2 2 1\n2 1 3.5\n"
    rp, ci, vv, _, _ = csrio.read_matrix_market(skew, text=True)
    assert rp.tolist() == [0, 1, 2] and ci.tolist() == [1, 0] and vv.tolist() == [-3.5, 3.5]


def test_matrix_market_errors():
    with pytest.raises(Error) as ei:
        csrio.read_matrix_market("3 3 0\n", text=True)
    assert ei.value.kind == ErrorKind.SyntaxError
    with pytest.raises(Error) as ei:
        csrio.read_matrix_market("%%MatrixMarket matrix coordinate real general\n2 2 1\n3 1 1.0\n", text=True)
    assert ei.value.kind == ErrorKind.OutOfBounds


def test_inst_writer_round_trip_on_generated_instance():
    rp, ci, vv, M, K = _csr(4, M=6, K=5)
    B = np.arange(K * 3, dtype=np.float32).reshape(K, 3)
    inst = csrio.csr_instance(rp, ci, vv, B)
    back = I.parse_instance(csrio.format_instance(inst))
    assert back == inst


@pytest.mark.skipif(not os.path.isdir(REF_FIXTURES), reason="reference fixtures absent")
@pytest.mark.parametrize("name", ["gespmm_small.inst", "gespmm_nnz4.inst", "gespmm_nnz2.inst", "polyp_n4.inst"])
def test_inst_writer_round_trips_reference_fixtures(name):
    inst = I.load_instance_file(os.path.join(REF_FIXTURES, name))
    assert I.parse_instance(csrio.format_instance(inst)) == inst


@pytest.mark.gpu
def test_files_to_gpu_path(tmp_path, oracle_mod):
    """A Matrix Market file and a binary cache feed the GPU path directly; the
    cache round trip lands on the device (cached_csr(device=...))."""
    import torch

    from paper_2503_08946_b200 import workloads as W
    from paper_2503_08946_b200.spmm import Plan

    rp, ci, vv, M, K = _csr(7, M=2000, K=700)
    B = np.random.default_rng(1).uniform(-1, 1, (K, 48)).astype(np.float32)
    mtx = str(tmp_path / "a.mtx")
    csrio.write_matrix_market(mtx, rp, ci, vv, M, K)
    r2, c2, v2, M2, K2 = csrio.read_matrix_market(mtx)
    dev = torch.device("cuda:0")
    t = lambda a: torch.as_tensor(np.ascontiguousarray(a), device=dev)  # noqa: E731
    got = Plan(t(r2), t(c2), K2).execute(t(v2), t(B), "max")
    np.testing.assert_array_equal(got.cpu().numpy(), oracle_mod.spmm_f32(rp, ci, vv, B, "max", seg_len=256))
    cache = str(tmp_path / "a.csr")
    c = csrio.cached_csr(cache, lambda: W.Csr(rp, ci, vv, M, K), device=dev)
    got = Plan(c.rowptr, c.colind, c.K).execute(c.vals, t(B), "sum")
    np.testing.assert_array_equal(got.cpu().numpy(), oracle_mod.spmm_f32(rp, ci, vv, B, "sum", seg_len=256))


@pytest.mark.gpu
def test_device_validation_matches_host_messages():
    """gespmm_validate_csr_device reports the reference's messages like the host check."""
    import torch

    from paper_2503_08946_b200 import _lib
    from paper_2503_08946_b200.errors import Error, ErrorKind

    L = _lib.load()
    dev = torch.device("cuda:0")
    cases = [
        (np.array([1, 2], np.int32), np.array([0, 1], np.int32), "rowPtr[0] must be 0"),
        (np.array([0, 2, 1], np.int32), np.array([0, 1], np.int32), "nondecreasing"),
        (np.array([0, 1, 3], np.int32), np.array([0, 1], np.int32), "rowPtr end differs"),
        (np.array([0, 1, 2], np.int32), np.array([0, 9], np.int32), "colInd entry out of [0,5)"),
    ]
    for rp, ci, msg in cases:
        M = len(rp) - 1
        trp, tci = torch.as_tensor(rp, device=dev), torch.as_tensor(ci, device=dev)
        st = L.gespmm_validate_csr_device(M, 5, len(ci), trp.data_ptr(), tci.data_ptr(), None)
        with pytest.raises(Error) as ei:
            _lib.check(st)
        assert ei.value.kind == ErrorKind.CsrInvalid and msg in str(ei.value), (msg, str(ei.value))
    good_rp = torch.as_tensor(np.array([0, 1, 2], np.int32), device=dev)
    good_ci = torch.as_tensor(np.array([0, 4], np.int32), device=dev)
    assert L.gespmm_validate_csr_device(2, 5, 2, good_rp.data_ptr(), good_ci.data_ptr(), None) == 0
