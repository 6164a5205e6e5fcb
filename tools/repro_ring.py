import sys, numpy as np, torch
sys.path.insert(0, '.')
sys.path.insert(0, 'tests')
from test_gpu_parity import random_csr
from paper_2503_08946_b200.spmm import Plan
rng = np.random.default_rng(100 + 128)
M, K, N = 700, 300, 128
rowptr, colind, vals = random_csr(rng, M, K, 0.05, long_rows=[(5, 1000), (6, 257), (699, 2600)], dup=True, empty_frac=0.3)
B = rng.uniform(-1, 1, (K, N)).astype(np.float32)
d = torch.device('cuda:0')
rp, ci, vv, Bt = [torch.as_tensor(np.ascontiguousarray(a), device=d) for a in (rowptr, colind, vals, B)]
plan = Plan(rp, ci, K)
out = plan.execute(vv, Bt, sys.argv[1] if len(sys.argv) > 1 else 'sum')
torch.cuda.synchronize()
print('ok', out.sum().item())
