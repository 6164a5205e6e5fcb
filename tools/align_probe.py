"""Kernel time with 16-byte-aligned colind/vals vs the same arrays behind a
4-byte offset (what a row-block view starting at p0 % 4 != 0 gives a rank:
the kernel's 4-byte staging path).  CUDA events, L2 flushed between steps,
interleaved; results bit-identical.  One JSON line per workload.

    python tools/align_probe.py [config5 config4 config2]
"""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import bench  # noqa: E402
from paper_2503_08946_b200.spmm import Plan  # noqa: E402


def main():
    names = sys.argv[1:] or ["config5", "config4", "config2"]
    dev = torch.device("cuda:0")
    s = torch.cuda.current_stream(dev)
    flush = torch.empty(256 << 18, dtype=torch.float32, device=dev)
    for name in names:
        spec = bench.workload_spec(name)
        csr, B = bench.make_workload(spec, dev)
        nnz = csr.colind.numel()
        ci_buf = torch.empty(nnz + 1, dtype=torch.int32, device=dev)
        v_buf = torch.empty(nnz + 1, dtype=torch.float32, device=dev)
        ci_buf[1:].copy_(csr.colind)
        v_buf[1:].copy_(csr.vals)
        ci_u, v_u = ci_buf[1:], v_buf[1:]
        plan_a = Plan(csr.rowptr, csr.colind, csr.K)
        plan_u = Plan(csr.rowptr, ci_u, csr.K)
        C_a = torch.empty((csr.M, spec["N"]), dtype=torch.float32, device=dev)
        C_u = torch.empty_like(C_a)
        arms = {"aligned": (plan_a, csr.vals, C_a), "offset4": (plan_u, v_u, C_u)}
        times = {k: [] for k in arms}
        for _ in range(3):
            for k, (p, v, C) in arms.items():
                p.execute(v, B, "sum", out=C, stream=s)
        for _ in range(10):
            for k, (p, v, C) in arms.items():
                flush.zero_()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(s)
                p.execute(v, B, "sum", out=C, stream=s)
                e1.record(s)
                e1.synchronize()
                times[k].append(e0.elapsed_time(e1))
        same = bool(torch.equal(C_a, C_u))
        print(json.dumps({"workload": name, "ms_aligned": round(statistics.median(times["aligned"]), 4),
                          "ms_offset4": round(statistics.median(times["offset4"]), 4),
                          "variant": plan_a.last_variant(), "bit_identical": same}), flush=True)
        plan_a.close()
        plan_u.close()
        del csr, B, ci_buf, v_buf, C_a, C_u
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
