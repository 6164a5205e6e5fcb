"""Builds libgespmm.so in-tree with nvcc for sm_100a (no GPU needed).

    python -m paper_2503_08946_b200._build        # or __graft_entry__.build()

Every .cu under csrc/ is compiled to an object with
``-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo`` (in parallel) and
linked into ``paper_2503_08946_b200/libgespmm.so`` next to this file, so the
built library travels to the GPU box with the repo snapshot.
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
INCLUDE = os.path.join(ROOT, "include")
BUILD = os.path.join(PKG, "build")
LIB = os.path.join(PKG, "libgespmm.so")
# Experiment builds: GESPMM_BUILD_TAG=mb3 GESPMM_EXTRA_FLAGS="-DGESPMM_MINBLOCKS=3"
# -> libgespmm_mb3.so (selected at run time with GESPMM_LIB=...).
TAG = os.environ.get("GESPMM_BUILD_TAG", "")
EXTRA = os.environ.get("GESPMM_EXTRA_FLAGS", "").split()
if TAG:
    LIB = os.path.join(PKG, f"libgespmm_{TAG}.so")
    BUILD = os.path.join(PKG, f"build_{TAG}")
    # experiment knobs (incl. the wrong-result GESPMM_ABL_* ablations) compile
    # only into tagged libraries, never into the product libgespmm.so
    EXTRA = EXTRA + ["-DGESPMM_EXPERIMENT_BUILD"]
elif EXTRA:
    raise SystemExit("GESPMM_EXTRA_FLAGS needs GESPMM_BUILD_TAG (experiment builds go to libgespmm_<tag>.so)")

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O2", "-I", INCLUDE, "-I", CSRC,
         "--expt-relaxed-constexpr", "-Xptxas", "-warn-spills"]


def _sources():
    return sorted(os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith(".cu"))


def _headers():
    hs = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".h", ".cuh"))]
    hs.append(os.path.join(INCLUDE, "gespmm.h"))
    return hs


def _compile(src: str, verbose: bool) -> str:
    obj = os.path.join(BUILD, os.path.basename(src) + ".o")
    newest_dep = max(os.path.getmtime(p) for p in [src] + _headers())
    if os.path.exists(obj) and os.path.getmtime(obj) >= newest_dep:
        return obj
    cmd = [NVCC, *ARCH, *FLAGS, *EXTRA, "-c", src, "-o", obj]
    if verbose:
        cmd += ["-Xptxas", "-v"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
    if verbose and r.stderr:
        sys.stderr.write(r.stderr)
    return obj


def build(verbose: bool = False) -> str:
    os.makedirs(BUILD, exist_ok=True)
    srcs = _sources()
    with cf.ThreadPoolExecutor(max_workers=min(8, len(srcs))) as ex:
        objs = list(ex.map(lambda s: _compile(s, verbose), srcs))
    if os.path.exists(LIB) and os.path.getmtime(LIB) >= max(os.path.getmtime(o) for o in objs):
        return LIB
    cmd = [NVCC, *ARCH, "-shared", "-o", LIB, *objs, "-ldl", "-lpthread"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    return LIB


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv))
