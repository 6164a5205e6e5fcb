"""Gather ceiling for the config-2 matrix: replays its colind stream through
tools/libgather_probe.so (pure B-row gathers, N=64, L2 flushed before each
rep) at several loads-in-flight / occupancy points: register loads, 16-byte
cp.async rings and TMA bulk-copy rings (one cp.async.bulk per row, mbarrier
completion).  Prints one JSON line."""
import ctypes
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2503_08946_b200 import workloads as W  # noqa: E402


def main():
    L = ctypes.CDLL(os.path.join(ROOT, "tools", "libgather_probe.so"))
    L.gather_probe.restype = ctypes.c_float
    L.gather_probe.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int,
                               ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_void_p,
                               ctypes.c_void_p, ctypes.c_int64]
    L.gather_probe_ring.restype = ctypes.c_float
    L.gather_probe_ring.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int,
                                    ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                    ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64]
    L.gather_probe_bulk.restype = ctypes.c_float
    L.gather_probe_bulk.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_int,
                                    ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_void_p,
                                    ctypes.c_void_p, ctypes.c_int64]
    L.gather_probe_pair.restype = ctypes.c_float
    L.gather_probe_pair.argtypes = L.gather_probe.argtypes
    dev = torch.device("cuda:0")
    csr = W.rmat_csr_gpu(20, 16 * 2**20, seed=3, device=dev)
    B = W.dense_gpu(csr.K, 64, seed=2, device=dev)
    sink = torch.zeros(4, device=dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    nnz = csr.nnz
    out = {"nnz": nnz, "gather_bytes": nnz * 256, "results": []}
    streams = {"csr_order": csr.colind,
               "shuffled": csr.colind[torch.randperm(nnz, device=dev)].contiguous()}
    for name, idx in streams.items():
        for U, bps in ((8, 8), (16, 8), (8, 4), (16, 4), (8, 3)):
            ms = L.gather_probe(B.data_ptr(), idx.data_ptr(), nnz, U, 256, bps, 5, sink.data_ptr(),
                                flush.data_ptr(), flush.numel())
            out["results"].append({"stream": name, "U": U, "warps_per_sm": 8 * bps, "ms": ms,
                                   "gather_TBs": nnz * 256 / (ms * 1e-3) / 1e12 if ms > 0 else None})
        if name != "csr_order":
            continue
        for U, bps in ((8, 4), (16, 4), (32, 4)):  # U rows per warp, 16-byte loads by half-warps
            ms = L.gather_probe_pair(B.data_ptr(), idx.data_ptr(), nnz, U, 256, bps, 5, sink.data_ptr(),
                                     flush.data_ptr(), flush.numel())
            out["results"].append({"stream": name, "pair": f"U{U}", "warps_per_sm": 8 * bps, "ms": ms,
                                   "regs_per_lane_in_flight": U * 2,
                                   "gather_TBs": nnz * 256 / (ms * 1e-3) / 1e12 if ms > 0 else None})
        for U, D, bps in ((8, 2, 4), (8, 3, 4), (8, 4, 3), (16, 2, 3), (4, 4, 4), (8, 2, 3), (8, 3, 3)):
            ms = L.gather_probe_ring(B.data_ptr(), idx.data_ptr(), nnz, U, D, 256, bps, 5, sink.data_ptr(),
                                     flush.data_ptr(), flush.numel())
            out["results"].append({"stream": name, "ring": f"U{U}xD{D}", "warps_per_sm": 8 * bps, "ms": ms,
                                   "gather_TBs": nnz * 256 / (ms * 1e-3) / 1e12 if ms > 0 else None})
        # TMA bulk-copy ring: one single-lane cp.async.bulk per 256-byte row,
        # mbarrier completion (VERDICT r1 Next 4)
        for U, D, Wc, bps in ((16, 2, 8, 1), (16, 2, 8, 2), (16, 2, 8, 3), (16, 3, 8, 2), (32, 2, 4, 3),
                              (32, 2, 8, 1), (8, 4, 8, 3), (16, 2, 4, 6)):
            ms = L.gather_probe_bulk(B.data_ptr(), idx.data_ptr(), nnz, U, D, Wc, 256, bps, 5, sink.data_ptr(),
                                     flush.data_ptr(), flush.numel())
            out["results"].append({"stream": name, "bulk": f"U{U}xD{D}", "warps_per_sm": Wc * bps,
                                   "rows_in_flight_per_sm": Wc * bps * U * (D - 1), "ms": ms,
                                   "gather_TBs": nnz * 256 / (ms * 1e-3) / 1e12 if ms > 0 else None})
    print(json.dumps(out))


if __name__ == "__main__":
    main()
