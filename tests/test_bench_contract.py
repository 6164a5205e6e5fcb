"""bench.py's contract pieces that need no GPU: workload specs for every
BASELINE config, the algorithmic byte model, the peak source,
and the CPU-baseline leg on a small matrix."""
import json
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


@pytest.mark.parametrize("name,N", [("config1", 32), ("config2", 64), ("config3-16", 16), ("config3-256", 256),
                                    ("config4", 128), ("config5", 128)])
def test_workload_specs(name, N):
    spec = bench.workload_spec(name)
    assert spec["N"] == N and spec["desc"]


def test_unknown_workload_rejected():
    with pytest.raises(SystemExit):
        bench.workload_spec("config9")


def test_algorithmic_bytes_config2():
    M = K = 1 << 20
    nnz, N = 16_085_882, 64
    U, G = bench.algorithmic_bytes(M, K, N, nnz)
    assert U == 4 * (M + 1) + 8 * nnz + 4 * K * N + 4 * M * N == 669_752_276
    assert G == 4 * (M + 1) + 8 * nnz + 4 * nnz * N + 4 * M * N
    assert G > U


def test_peaks_source(tmp_path, monkeypatch):
    peak, src = bench.peaks()
    assert peak > 1000 and src
    monkeypatch.setattr(bench, "ROOT", str(tmp_path))
    (tmp_path / "MEASURED_PEAKS.json").write_text(json.dumps({"hbm_gbs": 6534.5}))
    assert bench.peaks() == (6534.5, "measured (MEASURED_PEAKS.json hbm_gbs)")


def test_defaults_are_the_north_star_run():
    """No flags: BASELINE configs[4] (R-MAT 2^24, 2^30 edges, N=128) on one
    GPU; at N > 1 the same matrix row-split (strong scaling) with the
    column-panelled B broadcast; configs[1] rides along at N=1."""
    a = bench.parse_args([])
    assert a.workload == "config5" and a.scaling == "strong" and a.gpus == 1
    assert a.extra == "config2,config4" and a.generator == "torch" and a.b_panels > 1
    assert a.warmup >= 3


def test_traffic_file_covers_the_default_line():
    with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
        t = json.load(f)
    assert t["config5:sum"] > 0 and t["config2:sum"] > 0


@pytest.mark.parametrize("target", [1, 5_000, 10**9])
def test_row_sample(target):
    import numpy as np

    from paper_2503_08946_b200 import workloads as W

    c = W.rmat_csr(12, 40_000, seed=3)
    rp = c.rowptr.numpy()
    ci = c.colind.numpy()
    rows, srp, pos, s = bench.row_sample(rp, target)
    assert np.array_equal(rows, np.arange(0, c.M, s))
    assert srp[0] == 0 and srp[-1] == pos.size
    for k in range(0, rows.size, max(1, rows.size // 50)):
        r = rows[k]
        np.testing.assert_array_equal(ci[pos[srp[k]:srp[k + 1]]], ci[rp[r]:rp[r + 1]])
    if target >= c.nnz:
        assert s == 1 and pos.size == c.nnz


def test_cpu_baseline_leg_small():
    from paper_2503_08946_b200 import workloads as W

    c = W.rmat_csr(12, 20_000, seed=3)
    B = W.dense_torch(c.K, 16)
    args = (c.rowptr.numpy(), c.colind.numpy(), c.vals.numpy(), B.numpy(), 16, "sum")
    r = bench.cpu_baseline_port(*args, budget_s=0.2)
    assert r["kind"] == "port" and r["cores"] >= 1 and r["value"] > 0
    assert r["single_thread"]["cores"] == 1 and r["single_thread"]["value"] > 0
    r2 = bench.cpu_baseline_port(*args, budget_s=0.2, target_nnz=5_000)
    assert "every" in r2["sample"] and r2["value"] > 0


def test_fingerprint_identifies_the_input():
    import torch

    from paper_2503_08946_b200 import workloads as W

    spec = dict(bench.workload_spec("config2"), scale=10, edges=5_000)
    a = bench.fingerprint(*bench.make_workload(spec, torch.device("cpu"), "torch"))
    b = bench.fingerprint(*bench.make_workload(spec, torch.device("cpu"), "torch"))
    assert a == b and a["nnz"] > 0
    c = bench.fingerprint(*bench.make_workload(dict(spec, seed=4), torch.device("cpu"), "torch"))
    assert c != a
    del W


def test_ncu_metrics_file_covers_the_default_line():
    """roofline.ncu: the committed capture's DRAM throughput and L2 hit rate
    (report both beside the algorithmic fraction)."""
    import json
    import os

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    with open(os.path.join(root, "profiles", "ncu_metrics.json")) as f:
        d = json.load(f)
    m = d["config2:sum"]
    assert 0 < m["dram_throughput_pct"] < 100 and 0 < m["l2_hit_pct"] < 100
    with open(os.path.join(root, "profiles", "traffic.json")) as f:
        assert json.load(f)["config2:sum"] == m["dram_bytes"]
