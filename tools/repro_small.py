"""Small SpMM repro for compute-sanitizer runs: python tools/repro_small.py N [op] [variant]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from test_gpu_parity import gpu_spmm, random_csr  # noqa: E402
from oracle import oracle as O  # noqa: E402
from paper_2503_08946_b200 import spmm  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 32
op = sys.argv[2] if len(sys.argv) > 2 else "sum"
if len(sys.argv) > 3:
    spmm.set_variant_override(sys.argv[3])
rng = np.random.default_rng(100 + N)
M, K = 700, 300
rowptr, colind, vals = random_csr(rng, M, K, 0.05, long_rows=[(5, 1000), (6, 257), (699, 2600)],
                                  dup=True, empty_frac=0.3)
B = rng.uniform(-1, 1, (K, N)).astype(np.float32)
got, _ = gpu_spmm(torch.device("cuda:0"), rowptr, colind, vals, B, op)
want = O.spmm_f32(rowptr, colind, vals, B, op, seg_len=256)
print("equal", np.array_equal(got, want), "maxdiff", np.abs(got - want).max())
