"""Generates the golden fixtures under tests/golden/ from the REFERENCE ITSELF.

Run in the build container (needs /root/reference and oracle/_ref built):

    make -C oracle all ref && python tests/golden/make_golden.py

Every C value stored here was computed by the unmodified reference interpreter
(raceset::run on /root/reference/proj/fixtures/gespmm_alg2.mir, reference
src/oracle.cpp:699-736) and recovered by log replay (oracle/ref_replay.cpp).
Nothing here is produced by this repo's own restatement; the tests then pin
oracle/gespmm_oracle.c and the B200 path against these files.

Fixtures:
  * ref_<name>_shipped.json / ref_<name>_full.json -- the three shipped CSR
    instances (proj/fixtures/gespmm_{small,nnz4,nnz2}.inst) with their own
    launch (grid 2,1,1: rows >= 2 keep C0) and with a full launch (grid M).
  * rnd_*.json -- seeded random CSR instances covering the edge cases the
    reference contract allows: empty rows, empty matrix, unsorted and duplicate
    column indices, a long row, non-multiple-of-4 N, N=1, nonzero C0
    (the kernel accumulates into C, gespmm_alg2.mir:55-59), large magnitudes
    and cancellation.
  * config1_checksum.json -- BASELINE config 1 (uniform 4096^2, 1%, N=32,
    seed 1) run through the reference interpreter on all host threads; stores
    the sha256 of the fp64 C and per-row sums (the full C is 1 MB).
"""
from __future__ import annotations

import hashlib
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import oracle as O  # noqa: E402
from paper_2503_08946_b200 import workloads as W  # noqa: E402

REF_FIX = "/root/reference/proj/fixtures"


def parse_inst_arrays(text: str) -> dict:
    """Minimal reading of the shipped .inst files (format: reference
    src/oracle.cpp:223-281) -- only to record the inputs next to the outputs."""
    out = {"arrays": {}, "params": {}}
    for raw in text.splitlines():
        line = raw.split("#", 1)[0].replace(",", " ").split()
        if not line:
            continue
        kw = line[0]
        if kw == "array":
            vals = line[4:]
            out["arrays"][line[1]] = [float(v) if line[2].startswith("f") else int(v) for v in vals]
        elif kw in ("grid", "block"):
            out[kw] = [int(v) for v in line[1:4]]
        elif kw == "params":
            for kv in line[1:]:
                k, v = kv.split("=")
                out["params"][k] = int(v)
        elif kw == "csr":
            out["csr_cols"] = int(line[4].split("=")[1])
    return out


def inst_text(name, rowptr, colind, vals, B, C0, grid, block):
    M = len(rowptr) - 1
    K, N = B.shape
    fmt = lambda a: " ".join(repr(float(x)) for x in np.ravel(a))  # noqa: E731
    fmti = lambda a: " ".join(str(int(x)) for x in np.ravel(a))  # noqa: E731
    return (f"instance {name}\nparams M={M} N={N} K={K} A_S={len(colind)}\n"
            f"grid {grid[0]}, {grid[1]}, {grid[2]}\nblock {block[0]}, {block[1]}, {block[2]}\n"
            f"array rowPtr i32 = {fmti(rowptr)}\narray colInd i32 = {fmti(colind)}\n"
            f"array val f32 = {fmt(vals)}\narray B f32 = {fmt(B)}\narray C f32 = {fmt(C0)}\n"
            f"csr rowPtr colInd val cols={K}\n")


def dump(path, obj):
    with open(path, "w") as f:
        json.dump(obj, f, indent=None, separators=(",", ":"))
        f.write("\n")


def shipped():
    for name in ("gespmm_small", "gespmm_nnz4", "gespmm_nnz2"):
        src = os.path.join(REF_FIX, name + ".inst")
        text = open(src).read()
        meta = parse_inst_arrays(text)
        p = meta["params"]
        for launch in ("shipped", "full"):
            t = text if launch == "shipped" else text.replace(
                f"grid {meta['grid'][0]}, {meta['grid'][1]}, {meta['grid'][2]}",
                f"grid {p['M']}, {meta['grid'][1]}, {meta['grid'][2]}")
            C, nlog = O.ref_run_instance_text(t)
            a = meta["arrays"]
            grid = meta["grid"] if launch == "shipped" else [p["M"]] + meta["grid"][1:]
            dump(os.path.join(HERE, f"ref_{name}_{launch}.json"), {
                "source": f"/root/reference/proj/fixtures/{name}.inst (reference interpreter run, "
                          f"{launch} launch)",
                "M": p["M"], "N": p["N"], "K": p["K"], "grid": grid, "block": meta["block"],
                "rowptr": a["rowPtr"], "colind": a["colInd"], "vals": a["val"], "B": a["B"],
                "C0": a["C"], "C": C.tolist(), "log_len": nlog,
            })
            print(name, launch, C.tolist(), nlog)


def random_case(name, seed, M, K, N, density, *, C0_nonzero=False, long_row=None,
                unsorted=False, dup=False, scale=1.0, cancel=False, empty=False):
    rng = np.random.default_rng(seed)
    if empty:
        rowptr = np.zeros(M + 1, np.int32)
        colind = np.zeros(0, np.int32)
    else:
        rows = []
        for i in range(M):
            d = rng.binomial(K, density)
            if long_row is not None and i == long_row[0]:
                d = long_row[1]
            c = rng.integers(0, K, d) if (dup or d > K) else rng.choice(K, d, replace=False)
            if not unsorted:
                c = np.sort(c)
            rows.append(c)
        rowptr = np.concatenate([[0], np.cumsum([len(r) for r in rows])]).astype(np.int32)
        colind = (np.concatenate(rows) if rows else np.zeros(0)).astype(np.int32)
    nnz = len(colind)
    vals = (rng.uniform(-1, 1, nnz) * scale).astype(np.float32)
    B = (rng.uniform(-1, 1, (K, N)) * scale).astype(np.float32)
    if cancel:
        vals[::2] = 1.0
        vals[1::2] = -1.0
    C0 = (rng.uniform(-1, 1, (M, N)) if C0_nonzero else np.zeros((M, N))).astype(np.float32)
    text = inst_text(name, rowptr, colind, vals, B, C0, [max(M, 1), (N + 3) // 4, 1], [4, 1, 1])
    t0 = time.time()
    C, nlog = O.ref_run_instance_text(text)
    dt = time.time() - t0
    dump(os.path.join(HERE, f"rnd_{name}.json"), {
        "source": f"seeded random instance (seed {seed}) run through the reference interpreter",
        "M": M, "N": N, "K": K, "grid": [max(M, 1), (N + 3) // 4, 1], "block": [4, 1, 1],
        "rowptr": rowptr.tolist(), "colind": colind.tolist(),
        "vals": [float(x) for x in vals], "B": [float(x) for x in B.ravel()],
        "C0": [float(x) for x in C0.ravel()], "C": C.tolist(), "log_len": nlog,
    })
    print(name, M, K, N, nnz, nlog, f"{dt:.2f}s")


def config1_checksum():
    csr = W.uniform_csr(4096, 4096, 0.01, seed=1)
    B = W.dense(4096, 32, seed=2)
    nth = os.cpu_count() or 1
    C, secs, nlog = O.ref_spmm_csr(csr.rowptr, csr.colind, csr.vals, B, nthreads=nth)
    digest = hashlib.sha256(np.ascontiguousarray(C, np.float64).tobytes()).hexdigest()
    dump(os.path.join(HERE, "config1_checksum.json"), {
        "source": "BASELINE config 1: uniform 4096x4096 Bernoulli(0.01) seed 1 "
                  "(workloads.uniform_csr), B = workloads.dense(4096, 32, seed 2); reference "
                  "interpreter, rows split over host threads, C recovered by log replay",
        "M": 4096, "K": 4096, "N": 32, "nnz": int(csr.nnz),
        "rowptr_sha256": hashlib.sha256(csr.rowptr.tobytes()).hexdigest(),
        "colind_sha256": hashlib.sha256(csr.colind.tobytes()).hexdigest(),
        "c_f64_sha256": digest, "row_sums": C.sum(1).tolist(), "log_len": nlog,
        "ref_seconds": secs, "ref_threads": nth,
    })
    print("config1", csr.nnz, nlog, f"{secs:.1f}s on {nth} threads", digest)


if __name__ == "__main__":
    shipped()
    random_case("uniform64", 11, 64, 64, 8, 0.1)
    random_case("ragged_c0", 12, 48, 40, 12, 0.15, C0_nonzero=True, long_row=(7, 300), dup=True)
    random_case("empty_rows", 13, 40, 33, 5, 0.02)
    random_case("empty_matrix", 14, 6, 9, 4, 0.0, empty=True)
    random_case("unsorted_dup", 15, 30, 20, 16, 0.3, unsorted=True, dup=True)
    random_case("n1", 16, 50, 50, 1, 0.2)
    random_case("bigmag", 17, 32, 32, 8, 0.25, scale=1e18)
    random_case("cancel", 18, 32, 16, 8, 0.9, cancel=True, dup=True)
    random_case("longrow", 19, 8, 2048, 8, 0.01, long_row=(3, 1500))
    if "--no-config1" not in sys.argv:
        config1_checksum()
