"""A/B of the host pipeline's chunk rule (gespmm_csr_spmm_host, pinned host
buffers) on a BASELINE workload: equal-row chunks (the rule, 16 chunks) vs
equal-PCIe-byte chunks (GESPMM_HOST_EQUAL_BYTES, 64 / 32 chunks), interleaved rep by rep, wall clock per
call.  One JSON line per rule; with --timeline, one GESPMM_TRACE=3 call per
rule (device timeline on stderr).

    python tools/e2e_chunks_probe.py [--workload config5] [--reps 6] [--timeline]
"""
import argparse
import json
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import bench  # noqa: E402
from paper_2503_08946_b200.spmm import csr_spmm_host  # noqa: E402

RULES = {
    "equal_rows_16": {},
    "bytes_64": {"GESPMM_HOST_EQUAL_BYTES": "1", "GESPMM_HOST_CHUNKS": "64"},
    "bytes_32": {"GESPMM_HOST_EQUAL_BYTES": "1", "GESPMM_HOST_CHUNKS": "32"},
}


def set_rule(name):
    for k in ("GESPMM_HOST_EQUAL_BYTES", "GESPMM_HOST_CHUNKS", "GESPMM_TRACE"):
        os.environ.pop(k, None)
    os.environ.update(RULES[name])


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="config5")
    ap.add_argument("--reps", type=int, default=6)
    ap.add_argument("--timeline", action="store_true")
    a = ap.parse_args()
    dev = torch.device("cuda:0")
    spec = bench.workload_spec(a.workload)
    csr, B = bench.make_workload(spec, dev)
    N = spec["N"]
    h = [bench.pinned_like(t) for t in (csr.rowptr, csr.colind, csr.vals, B)]
    nnz = int(csr.colind.numel())
    del B
    csr = None
    torch.cuda.empty_cache()
    hC = torch.empty((h[0].numel() - 1, N), dtype=torch.float32, pin_memory=True)
    ref = None
    times = {r: [] for r in RULES}
    for r in RULES:  # warm + bit-identity across rules
        set_rule(r)
        csr_spmm_host(*h, "sum", out=hC)
        if ref is None:
            ref = hC.clone()
        elif not torch.equal(ref, hC):
            raise SystemExit(f"rule {r}: result differs")
    for _ in range(a.reps):
        for r in RULES:
            set_rule(r)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            csr_spmm_host(*h, "sum", out=hC)
            times[r].append((time.perf_counter() - t0) * 1e3)
    flops = 2.0 * nnz * N
    for r, ts in times.items():
        med = statistics.median(ts)
        print(json.dumps({"workload": a.workload, "rule": r, "env": RULES[r], "ms_median": round(med, 2),
                          "ms_min": round(min(ts), 2), "ms": [round(t, 2) for t in ts],
                          "e2e_gflops": round(flops / med / 1e6, 1), "bit_identical": True}), flush=True)
    if a.timeline:
        for r in RULES:
            set_rule(r)
            os.environ["GESPMM_TRACE"] = "3"
            print(f"[timeline] rule {r}", file=sys.stderr, flush=True)
            csr_spmm_host(*h, "sum", out=hC)
            torch.cuda.synchronize()


if __name__ == "__main__":
    main()
