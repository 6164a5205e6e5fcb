# device timeline of the pipelined host entry point (GESPMM_TRACE=3) on config 2: per-chunk H2D / kernel / D2H completion times (profiles/r1_e2e_timeline.txt)
mkdir -p gpurun_out
GESPMM_TRACE=3 python -c "
import torch,sys
sys.path.insert(0,'.')
from paper_2503_08946_b200 import workloads as W
from paper_2503_08946_b200.spmm import csr_spmm_host
dev=torch.device('cuda:0')
csr=W.rmat_csr(20,16*2**20,seed=3,device=dev); B=W.dense_torch(csr.K,64,seed=2,device=dev)
h=[t.cpu().pin_memory() for t in (csr.rowptr,csr.colind,csr.vals,B)]
hC=torch.empty((csr.M,64)).pin_memory()
for i in range(3): csr_spmm_host(*h,'sum',out=hC)
" > gpurun_out/e2e_timeline.txt 2>&1
