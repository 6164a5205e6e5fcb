"""Experiment: gather-only probe of config 2's column stream where the H hottest
B rows are first copied (per step, after the L2 flush) into a compact region in
front of B and gathered from there.  Measures whether a freshly written hot
set raises the gather rate enough to pay for the copy."""
import ctypes
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2503_08946_b200 import workloads as W  # noqa: E402


def main():
    L = ctypes.CDLL(os.path.join(ROOT, "tools", "libgather_probe.so"))
    L.gather_probe.restype = ctypes.c_float
    L.gather_probe.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_int,
                               ctypes.c_int, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64]
    dev = torch.device("cuda:0")
    csr = W.rmat_csr_gpu(20, 16 * 2**20, seed=3, device=dev)
    K, nnz = csr.K, csr.nnz
    B = W.dense_gpu(K, 64, seed=2, device=dev)
    sink = torch.zeros(4, device=dev)
    deg = torch.bincount(csr.colind.long(), minlength=K)
    order = torch.argsort(deg, descending=True)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
    ts = []
    for _ in range(6):
        flush.zero_()
        torch.cuda.synchronize()
        ts.append(L.gather_probe(B.data_ptr(), csr.colind.data_ptr(), nnz, 8, 256, 4, 0, sink.data_ptr(), 0, 0))
    out = {"plain_flushed_ms": min(ts[1:])}
    for H in (100_000, 250_000, 400_000):
        hot = order[:H]
        newidx = torch.arange(K, device=dev) + H
        newidx[hot] = torch.arange(H, device=dev)
        idx2 = newidx[csr.colind.long()].to(torch.int32).contiguous()
        comb = torch.empty((H + K, 64), device=dev)
        comb[H:] = B
        covered = float(deg[hot].sum()) / nnz
        ts_copy, ts_probe = [], []
        for _ in range(6):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            comb[:H] = B[hot]  # the per-step hot-set build (writes the hot rows into L2)
            e1.record()
            torch.cuda.synchronize()
            ts_copy.append(e0.elapsed_time(e1))
            ts_probe.append(L.gather_probe(comb.data_ptr(), idx2.data_ptr(), nnz, 8, 256, 4, 0, sink.data_ptr(),
                                           0, 0))
        out[f"H{H}"] = {"nnz_covered": covered, "copy_ms": min(ts_copy[1:]), "probe_ms": min(ts_probe[1:]),
                        "hot_MB": H * 256 / 1e6}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
