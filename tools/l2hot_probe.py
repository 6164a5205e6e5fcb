"""Driver for tools/l2hot_probe.cu: B-row gather replay of a large R-MAT's
column stream with an L2 hot set of the highest-degree columns (VERDICT r1
Next 3).  Prints one JSON line per (mode, hot budget).

    python tools/l2hot_probe.py [--workload config5] [--modes 0,1,2,3,4] [--hot-mb 0,48,64,80,96]
"""
import argparse
import ctypes
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="config5")
    ap.add_argument("--modes", default="0,1,2,3,4")
    ap.add_argument("--hot-mb", default="48,64,80,96")
    ap.add_argument("--persist", default="0,max")
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--span", type=int, default=256)
    ap.add_argument("--bps", type=int, default=4)
    ap.add_argument("--panels", default="", help="row widths to replay as column panels, e.g. 32,64,128")
    ap.add_argument("--panel-modes", default="0,1")
    ap.add_argument("--panel-u", type=int, default=8, help="rows in flight per warp (register replay)")
    ap.add_argument("--ldgsts", default="", help="LDGSTS ring configs vec:U:D:warps_per_sm,...")
    ap.add_argument("--bulk", default="", help="bulk-copy ring configs vec:U:D;... e.g. 2:16:2,4:8:4")
    ap.add_argument("--pinned", default="", help="pinned hot set + plain LDGSTS ring, configs U:D:warps_per_sm")
    ap.add_argument("--tma", default="", help="TMA gather4 ring configs S:G:warps_per_sm, e.g. 4:1:24,3:2:16")
    ap.add_argument("--tma-mode", type=int, default=1,
                    help="--tma with a hot set: 1 = per-gather4 hint (any hot row -> evict_last), 2 / 3 = the "
                         "stage's positions regrouped hot-first, mixed groups evict_first / evict_normal")
    ap.add_argument("--tma-sorted", action="store_true",
                    help="--tma: within each span, hot positions first (stable) -- the best case for a "
                         "per-gather4 hint (gather order may differ from fold order)")
    a = ap.parse_args()
    import bench
    from paper_2503_08946_b200 import workloads as W

    so = os.path.join(ROOT, "tools", "libl2hot_probe.so")
    L = ctypes.CDLL(so)
    L.l2hot_probe.restype = ctypes.c_float
    L.l2hot_probe.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int,
                              ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p,
                              ctypes.c_int64, ctypes.c_int64, ctypes.c_int64, ctypes.c_float]
    L.l2hot_max_persist.restype = ctypes.c_int64
    dev = torch.device("cuda:0")
    spec = bench.workload_spec(a.workload)
    csr = W.rmat_csr_gpu(spec["scale"], spec["edges"], seed=spec["seed"], device=dev)
    K = csr.K
    B = torch.rand(K, 128, device=dev)
    col = csr.colind
    deg = torch.bincount(col, minlength=K)
    order = torch.argsort(deg, descending=True)
    cum = torch.cumsum(deg[order].double(), 0) / col.numel()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    sink = torch.zeros(4, device=dev)
    maxp = int(L.l2hot_max_persist())
    print(json.dumps({"nnz": col.numel(), "K": K, "max_persisting_l2": maxp,
                      "l2": torch.cuda.get_device_properties(0).L2_cache_size}), flush=True)
    if a.tma:
        L.l2hot_probe_tma.restype = ctypes.c_float
        L.l2hot_probe_tma.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int,
                                      ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                      ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64]
        for mb in [0] + [int(x) for x in a.hot_mb.split(",")]:
            H = (mb << 20) // 512
            hotflag = torch.zeros(K, dtype=torch.bool, device=dev)
            if H:
                hotflag[order[:H]] = True
            flagged = col | (hotflag[col].to(torch.int32) << 31)
            if a.tma_sorted and H:
                n = col.numel()
                key = (torch.arange(n, device=dev, dtype=torch.int64) // a.span) * 2 + (flagged >= 0).to(torch.int64)
                perm = torch.sort(key, stable=True).indices
                del key
                flagged = flagged[perm].contiguous()
                del perm
            for cfg in a.tma.split(","):
                S_, G_, wps = (int(x) for x in cfg.split(":"))
                ms = L.l2hot_probe_tma(B.data_ptr(), K, flagged.data_ptr(), col.numel(), a.tma_mode if mb else 0,
                                       S_, G_, wps,
                                       a.span, a.reps, sink.data_ptr(), flush.data_ptr(), flush.numel())
                print(json.dumps({"tma": cfg, "mode": a.tma_mode if mb else 0, "hot_mb": mb,
                                  "sorted": bool(a.tma_sorted),
                                  "hot_share": round(float(cum[H - 1]), 4) if H else 0, "ms": round(ms, 3)}),
                      flush=True)
            del flagged
        return
    if a.pinned:
        L.l2hot_probe_pinned.restype = ctypes.c_float
        L.l2hot_probe_pinned.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p,
                                         ctypes.c_int64, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                         ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64,
                                         ctypes.POINTER(ctypes.c_float)]
        for mb in [0] + [int(x) for x in a.hot_mb.split(",")]:
            H = (mb << 20) // 512
            hot = order[:H].to(torch.int32).contiguous()
            for cfg in a.pinned.split(","):
                U, D, wps = (int(x) for x in cfg.split(":"))
                pin = ctypes.c_float(0)
                ms = L.l2hot_probe_pinned(B.data_ptr(), col.data_ptr(), col.numel(), hot.data_ptr(), H, U, D,
                                          a.span, wps, a.reps, sink.data_ptr(), flush.data_ptr(), flush.numel(),
                                          ctypes.byref(pin))
                print(json.dumps({"pinned": cfg, "hot_mb": mb, "hot_share": round(float(cum[H - 1]), 4) if H else 0,
                                  "ms_incl_pin_and_demote": round(ms, 3), "pin_ms": round(pin.value, 3)}),
                      flush=True)
        return
    if a.panels:
        L.l2hot_probe_panels.restype = ctypes.c_float
        L.l2hot_probe_panels.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_int,
                                         ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p,
                                         ctypes.c_int64, ctypes.c_int]
        L.l2hot_probe_ldgsts.restype = ctypes.c_float
        L.l2hot_probe_ldgsts.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_int,
                                         ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                         ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64]
        L.l2hot_probe_bulk.restype = ctypes.c_float
        L.l2hot_probe_bulk.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_int,
                                       ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                       ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64]
        for w in [int(x) for x in a.panels.split(",")]:
            for mb in [0] + [int(x) for x in a.hot_mb.split(",")]:
                H = (mb << 20) // (4 * w)
                hotflag = torch.zeros(K, dtype=torch.bool, device=dev)
                if H:
                    hotflag[order[:H]] = True
                share = float(cum[min(H, K) - 1]) if H else 0.0
                flagged = col | (hotflag[col].to(torch.int32) << 31)
                for mode in [int(m) for m in a.panel_modes.split(",")]:
                    if (mb == 0) != (mode == 0):
                        continue
                    if a.panel_u:
                        ms = L.l2hot_probe_panels(B.data_ptr(), flagged.data_ptr(), col.numel(), mode, w // 32,
                                                  a.span, a.bps, a.reps, sink.data_ptr(), flush.data_ptr(),
                                                  flush.numel(), a.panel_u)
                        print(json.dumps({"panel_cols": w, "panels": 128 // w, "mode": mode, "U": a.panel_u,
                                          "hot_mb": mb, "hot_rows": H, "hot_share": round(share, 4),
                                          "ms": round(ms, 3)}), flush=True)
                    for cfg in [c for c in a.ldgsts.split(",") if c]:
                        vec, U, D, wps = (int(x) for x in cfg.split(":"))
                        if 32 * vec != w:
                            continue
                        ms = L.l2hot_probe_ldgsts(B.data_ptr(), flagged.data_ptr(), col.numel(), mode, vec, U, D,
                                                  a.span, wps, a.reps, sink.data_ptr(), flush.data_ptr(),
                                                  flush.numel())
                        print(json.dumps({"ldgsts": cfg, "panel_cols": w, "mode": mode, "hot_mb": mb,
                                          "hot_share": round(share, 4), "ms": round(ms, 3)}), flush=True)
                    for cfg in [c for c in a.bulk.split(",") if c]:
                        vec, U, D = (int(x) for x in cfg.split(":"))
                        if 32 * vec != w:
                            continue
                        ms = L.l2hot_probe_bulk(B.data_ptr(), flagged.data_ptr(), col.numel(), mode, vec, U, D,
                                                a.span, 1, a.reps, sink.data_ptr(), flush.data_ptr(), flush.numel())
                        print(json.dumps({"bulk": cfg, "panel_cols": w, "mode": mode, "hot_mb": mb,
                                          "hot_share": round(share, 4), "ms": round(ms, 3)}), flush=True)
                del flagged
        return
    rowb = 512
    for mb in [0] + [int(x) for x in a.hot_mb.split(",")]:
        H = (mb << 20) // rowb
        hotflag = torch.zeros(K, dtype=torch.bool, device=dev)
        if H:
            hotflag[order[:H]] = True
        share = float(cum[H - 1]) if H else 0.0
        flagged = col | (hotflag[col].to(torch.int32) << 31)
        for mode in [int(m) for m in a.modes.split(",")]:
            if mb == 0 and mode != 0:
                continue
            if mb and mode == 0:
                continue
            Hbuf = None
            idx = flagged
            if mode == 4:
                hid = torch.full((K,), -1, dtype=torch.int64, device=dev)
                hid[order[:H]] = torch.arange(H, device=dev)
                Hbuf = B[order[:H]].contiguous()
                hc = hid[col]
                idx = torch.where(hc >= 0, (hc.to(torch.int32) | torch.tensor(-2**31, dtype=torch.int32, device=dev)), col)
                del hc
            for pers in a.persist.split(","):
                pb = maxp if pers == "max" else int(pers)
                win = H * rowb if mode == 4 else 0
                ms = L.l2hot_probe(B.data_ptr(), Hbuf.data_ptr() if Hbuf is not None else 0, idx.data_ptr(),
                                   col.numel(), mode, a.span, a.bps, a.reps, sink.data_ptr(), flush.data_ptr(),
                                   flush.numel(), pb, min(win, pb) if win else 0, 1.0)
                print(json.dumps({"mode": mode, "hot_mb": mb, "hot_rows": H, "hot_share": round(share, 4),
                                  "persist": pb, "ms": round(ms, 3)}), flush=True)
                if mode in (0,):
                    break
            del Hbuf, idx
            torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
