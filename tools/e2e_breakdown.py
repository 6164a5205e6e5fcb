"""Phase breakdown of the end-to-end host path on the config-2 workload.

Times (wall clock, synchronized) the one-shot host call and its pieces done
separately: pinned H2D of the CSR and B, device validation + plan build,
kernel, D2H of C.  Prints one JSON line.
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2503_08946_b200 import workloads as W  # noqa: E402
from paper_2503_08946_b200.spmm import Plan, csr_spmm_host  # noqa: E402


def timed(fn, reps=3):
    ts = []
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        ts.append((time.perf_counter() - t0) * 1e3)
    return min(ts), ts


def main():
    dev = torch.device("cuda:0")
    csr = W.rmat_csr(20, 16 * 2**20, seed=3, device=dev)
    B = W.dense_torch(csr.K, 64, seed=2, device=dev)
    h = {k: v.cpu().pin_memory() for k, v in
         dict(rp=csr.rowptr, ci=csr.colind, v=csr.vals, B=B).items()}
    hC = torch.empty((csr.M, 64), dtype=torch.float32).pin_memory()
    out = {}
    out["host_call_ms"] = timed(lambda: csr_spmm_host(h["rp"], h["ci"], h["v"], h["B"], "sum", out=hC))
    d = {}

    def h2d():
        for k, v in h.items():
            d[k] = v.to(dev, non_blocking=True)
    out["h2d_ms"] = timed(h2d)
    out["h2d_B_ms"] = timed(lambda: h["B"].to(dev, non_blocking=True))
    plans = []
    out["plan_ms"] = timed(lambda: plans.append(Plan(d["rp"], d["ci"], csr.K, validate=True)))
    out["plan_novalidate_ms"] = timed(lambda: plans.append(Plan(d["rp"], d["ci"], csr.K, validate=False)))
    p = plans[-1]
    C = torch.empty((csr.M, 64), device=dev)
    out["exec_ms"] = timed(lambda: p.execute(d["v"], d["B"], "sum", out=C))
    out["d2h_ms"] = timed(lambda: hC.copy_(C, non_blocking=True))
    out["alloc_700MB_ms"] = timed(lambda: torch.empty(700 << 20, dtype=torch.uint8, device=dev))
    print(json.dumps(out))


if __name__ == "__main__":
    main()
