"""CPU tier: libgespmm.so loads, exports every symbol include/gespmm.h declares,
and its host-only entry points (validation, partitioning, variant choice)
behave like the reference contract.  No compute calls (no GPU here)."""
import ctypes
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def L():
    from paper_2503_08946_b200 import _build, _lib

    _build.build()
    return _lib.load()


def header_functions():
    text = open(os.path.join(ROOT, "include", "gespmm.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(gespmm_[a-z_]+)\s*\(", text)))


def test_exports_every_declared_symbol(L):
    from paper_2503_08946_b200 import _lib

    declared = header_functions()
    assert len(declared) >= 18
    for name in declared:
        assert hasattr(L, name), f"libgespmm.so does not export {name}"
    assert sorted(_lib.EXPORTS) == declared


def test_library_is_sm100a(L):
    from paper_2503_08946_b200 import _lib

    out = os.popen(f"/usr/local/cuda/bin/cuobjdump --list-elf {_lib.LIB_PATH}").read()
    assert "sm_100a" in out


def test_version_and_status_strings(L):
    assert L.gespmm_version() == 1
    assert L.gespmm_status_string(1) == b"invalid csr"
    assert L.gespmm_status_string(2) == b"out of bounds"


def _validate(L, M, K, rowptr, colind, vals_len=None):
    rp = np.ascontiguousarray(rowptr, np.int32)
    ci = np.ascontiguousarray(colind, np.int32)
    n = len(ci) if vals_len is None else vals_len
    st = L.gespmm_validate_csr(M, K, len(rp), rp.ctypes.data, len(ci), ci.ctypes.data, n)
    return st, L.gespmm_last_error().decode()


def test_host_validation_matches_reference_rules(L):
    # reference test_oracle.cpp:94-110: rowPtr 0 2 1 is rejected as CsrInvalid
    st, msg = _validate(L, 2, 2, [0, 2, 1], [0, 0])
    assert st == 1 and "nondecreasing" in msg
    assert _validate(L, 2, 2, [1, 2, 2], [0, 0])[0] == 1
    st, msg = _validate(L, 2, 2, [0, 1, 3], [0, 1])
    assert st == 1 and "end differs" in msg
    st, msg = _validate(L, 2, 2, [0, 1, 2], [0, 1], vals_len=3)
    assert st == 1 and "lengths differ" in msg
    st, msg = _validate(L, 2, 2, [0, 1, 2], [0, 2])
    assert st == 1 and "out of [0,2)" in msg
    assert _validate(L, 2, 2, [0, 1, 2], [0, -1])[0] == 1
    assert _validate(L, 3, 2, [0, 1, 2], [0, 1])[0] == 1  # |rowptr| != M+1
    # the reference accepts unsorted and duplicate columns
    assert _validate(L, 2, 4, [0, 3, 4], [3, 1, 3, 0])[0] == 0
    assert _validate(L, 0, 0, [0], [])[0] == 0


def test_python_validate_raises_reference_error():
    from paper_2503_08946_b200 import Error, ErrorKind
    from paper_2503_08946_b200.spmm import validate_csr

    with pytest.raises(Error) as ei:
        validate_csr(2, 2, [0, 2, 1], [0, 0])
    assert ei.value.kind == ErrorKind.CsrInvalid
    assert str(ei.value).startswith("invalid csr: ")


def test_partition_rows_balanced_and_contiguous():
    from paper_2503_08946_b200.spmm import partition_rows

    rng = np.random.default_rng(0)
    deg = (rng.pareto(1.5, 100_000) * 3).astype(np.int64)
    rowptr = np.concatenate([[0], np.cumsum(deg)]).astype(np.int32)
    for parts in (1, 2, 4, 8):
        b = partition_rows(rowptr, parts)
        assert b[0] == 0 and b[-1] == len(deg) and np.all(np.diff(b) >= 0)
        work = [int(rowptr[b[i + 1]] - rowptr[b[i]] + b[i + 1] - b[i]) for i in range(parts)]
        total = int(rowptr[-1]) + len(deg)
        assert max(work) <= total / parts + deg.max() + 1


def test_variant_selection_by_N():
    from paper_2503_08946_b200.spmm import variant_name

    # the paired-lane kernel where 32 lanes would idle (every op)
    assert variant_name(16) == "pair_vec1"
    assert variant_name(16, reduce="mean") == "pair_vec1"
    assert variant_name(16, reduce="max") == "pair_vec1"
    assert variant_name(32) == "vec1_lpr32_cwm1"
    assert variant_name(64) == "vec2_lpr32_cwm1"
    assert variant_name(128) == "vec4_lpr32_cwm1_ring"  # the shared-memory gather ring at 512-byte rows
    assert variant_name(256) == "vec4_lpr32_cwm2"
    assert variant_name(512) == "vec4_lpr32_cwm2"
    assert variant_name(33) == "pair_vec1"  # 3 blocks of 16: 15 idle columns vs 31
    # max/min at the 32-column tile: the paired-lane kernel (profiles/r2_pairperm/)
    assert variant_name(32, reduce="min") == "pair_vec2"
    assert variant_name(32, reduce="max") == "pair_vec2"
    assert variant_name(32, reduce="mean") == "vec1_lpr32_cwm1"
    assert variant_name(64, reduce="max") == "vec2_lpr32_cwm1"
    assert variant_name(33, reduce="max") == "pair_vec1"


def test_cuda_path_fails_loudly_without_gpu():
    """No silent CPU fallback: without a device the CUDA entry points error."""
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2503_08946_b200 import _lib

    L = _lib.load()
    h = ctypes.c_void_p()
    rp = np.zeros(5, np.int32)
    st = L.gespmm_plan_create(ctypes.byref(h), 4, 4, 0, rp.ctypes.data, rp.ctypes.data, 0, None)
    assert st == 4  # GESPMM_CUDA_ERROR
    assert L.gespmm_last_error().decode()
