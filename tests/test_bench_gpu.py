"""The driver-facing entry points on the GPU: bench.py's JSON line (both arms)
and __graft_entry__.smoke()."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def run_bench(*args, timeout=900):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                       timeout=timeout, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    return json.loads(lines[0])


@pytest.mark.gpu
def test_bench_line_contract():
    d = run_bench("--workload", "config2", "--extra", "config1", "--steps", "4", "--warmup", "3",
                  "--sustained-s", "0.2")
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "roofline", "cpu_baseline", "e2e", "clocks",
              "gpu_launches"):
        assert k in d, k
    assert d["n_gpus"] == 1 and d["steps"] == 4 and d["value"] > 0 and d["higher_is_better"] is True
    assert d["config"]["workload"].startswith("R-MAT scale 20")
    rf = d["roofline"]
    assert rf["bound"] == "hbm" and rf["unit"] == "GB/s" and 0 < rf["frac"] < 1
    assert abs(rf["frac"] - rf["achieved"] / rf["peak"]) < 1e-9
    assert d["cpu_baseline"]["kind"] == "port" and d["cpu_baseline"]["cores"] >= 1
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    assert d["gpu_launches"] >= d["steps"]
    assert d["clocks"] is None or d["clocks"]["sm_max_mhz"] > 0
    assert e["equals_device_result"] is True
    x = d["extra"]["config1"]
    assert "error" not in x, x
    assert x["clocks"] is None or x["clocks"]["sm_max_mhz"] > 0
    assert x["value"] > 0 and x["e2e"]["value"] > 0 and x["e2e"]["equals_device_result"] is True


@pytest.mark.gpu
def test_bench_reference_arm_line():
    """The reference arm reads the identical matrix (same generator and seed):
    its input fingerprint equals our arm's."""
    d = run_bench("--impl", "reference", "--workload", "config2", "--steps", "1", "--warmup", "3")
    assert d["impl"] == "reference"
    if "unavailable" in d:
        pytest.skip(d["unavailable"])
    assert d["value"] > 0 and d["cpu_baseline"]["kind"] == "reference"
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]
    ours = run_bench("--workload", "config2", "--extra", "", "--steps", "3", "--warmup", "3", "--no-cpu-baseline",
                     "--no-e2e", "--sustained-s", "0", "--no-clocks")
    assert d["config"]["input"] == ours["config"]["input"]
    assert d["config"]["sample"]["row_cap_nnz"] > 0


@pytest.mark.gpu
def test_smoke_entry_point():
    sys.path.insert(0, ROOT)
    import __graft_entry__ as g

    g.smoke()


@pytest.mark.gpu
@pytest.mark.parametrize("scaling", ["weak", "strong"])
def test_bench_two_ranks(scaling):
    """bench.py's N > 1 path, launched as the driver does (torch.distributed.run,
    127.0.0.1), with two ranks sharing the one GPU over gloo: sharding, the B
    broadcast, max-over-ranks timing, the fused peer-store C all-gather (CUDA
    IPC between the two processes) vs the NCCL-style broadcasts, e2e."""
    import socket

    with socket.socket() as s_:
        s_.bind(("127.0.0.1", 0))
        port = s_.getsockname()[1]
    env = dict(os.environ, GESPMM_BENCH_BACKEND="gloo", GESPMM_NO_PROBE="1")
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                        "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.join(ROOT, "bench.py"),
                        "--gpus", "2", "--steps", "3", "--warmup", "3", "--workload", "config1",
                        "--scaling", scaling, "--no-cpu-baseline", "--sustained-s", "0", "--no-clocks",
                        "--b-panels", "2", "--N", "64"],
                       capture_output=True, text=True, timeout=900, cwd=ROOT, env=env)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]  # rank 0 alone prints
    d = json.loads(lines[0])
    one = run_bench("--workload", "config1", "--steps", "3", "--warmup", "3", "--no-cpu-baseline",
                    "--no-e2e", "--sustained-s", "0", "--no-clocks", "--extra", "", "--N", "64")
    assert d["n_gpus"] == 2 and d["scaling"] == scaling and d["value"] > 0
    assert d["config"]["nnz"] == (2 if scaling == "weak" else 1) * one["config"]["nnz"]
    ca = d["c_allgather"]
    assert "error" not in ca, ca
    assert ca["identical"] is True and ca["fused_peer_stores_ms"] > 0 and ca["nccl_broadcasts_ms"] > 0
    assert d["e2e"]["value"] > 0 and d["config"]["b_broadcast_ms"] >= 0
    assert d["e2e"]["equals_device_result"] is True and d["e2e"]["b_panels"] == 2
    bc = d["broadcast"]  # broadcast-inclusive legs, reported beside the kernel-only time
    assert bc["identical"] is True and bc["b_panels"] == 2
    assert bc["overlapped_ms"] > 0 and bc["broadcast_then_compute_ms"] > 0
