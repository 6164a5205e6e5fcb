"""Plan-build and one-shot timings on a BASELINE workload (VERDICT r1 Next 7).

    python tools/plan_timing.py [--workload config2] [--reps 10]

Prints one JSON line: Plan() construction (fresh plan objects: device time
between events on the stream and wall time), and the one-shot
gespmm_csr_spmm (plan + kernel + trailing sync) against a cached-plan execute.
Run with GESPMM_TRACE=3 for the per-phase device timeline on stderr.
"""
import argparse
import json
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="config2")
    ap.add_argument("--reps", type=int, default=10)
    a = ap.parse_args()
    import torch

    import bench
    from paper_2503_08946_b200 import spmm

    dev = torch.device("cuda:0")
    spec = bench.workload_spec(a.workload)
    csr, B = bench.make_workload(spec, dev, "torch")
    st = torch.cuda.current_stream(dev)
    C = torch.empty((csr.M, spec["N"]), device=dev)

    def timed(fn):
        dts, wts = [], []
        for _ in range(a.reps + 1):
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            t0 = time.perf_counter()
            e0.record(st)
            fn()
            e1.record(st)
            torch.cuda.synchronize()
            wts.append((time.perf_counter() - t0) * 1e3)
            dts.append(e0.elapsed_time(e1))
        return {"device_ms": statistics.median(dts[1:]), "wall_ms": statistics.median(wts[1:])}

    plans = []
    out = {"workload": a.workload, "M": csr.M, "nnz": csr.nnz, "N": spec["N"]}
    out["plan_fresh"] = timed(lambda: plans.append(spmm.Plan(csr.rowptr, csr.colind, csr.K)))
    out["plan_fresh_novalidate"] = timed(
        lambda: plans.append(spmm.Plan(csr.rowptr, csr.colind, csr.K, validate=False)))
    p = plans[-1]
    out["execute_cached"] = timed(lambda: p.execute(csr.vals, B, "sum", out=C))
    out["csr_spmm_oneshot"] = timed(lambda: spmm.csr_spmm(csr.rowptr, csr.colind, csr.vals, B, "sum", out=C))
    out["info"] = p.info()
    print(json.dumps(out))


if __name__ == "__main__":
    main()
