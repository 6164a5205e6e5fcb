"""e2e diagnostics: wall time per gespmm_csr_spmm_host call on config 2
(pinned host buffers), N calls; prints per-call ms (dev helper)."""
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_2503_08946_b200 import workloads as W  # noqa: E402
from paper_2503_08946_b200.spmm import csr_spmm_host  # noqa: E402

dev = torch.device("cuda:0")
csr = W.rmat_csr_gpu(20, 16 * 2**20, seed=3, device=dev)
B = W.dense_gpu(csr.K, 64, seed=2, device=dev)
hp = lambda t: t.cpu().pin_memory()  # noqa: E731
h_rp, h_ci, h_v, h_B = hp(csr.rowptr), hp(csr.colind), hp(csr.vals), hp(B)
h_C = torch.empty((csr.M, 64), dtype=torch.float32).pin_memory()
ts = []
for i in range(int(sys.argv[1]) if len(sys.argv) > 1 else 8):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    csr_spmm_host(h_rp, h_ci, h_v, h_B, "sum", out=h_C)
    ts.append((time.perf_counter() - t0) * 1e3)
print("per-call ms:", [round(t, 2) for t in ts])
