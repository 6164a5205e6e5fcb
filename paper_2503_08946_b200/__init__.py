"""B200-native GE-SpMM hot path (arXiv 2503.08946's CSR x dense SpMM).

Layout:
  csrc/          sm_100a CUDA kernels + the C-ABI (include/gespmm.h) -> libgespmm.so
  _lib.py        ctypes binding (no fallback: the compute API needs libgespmm.so)
  spmm.py        torch-tensor API: csr_spmm, Plan, csr_spmm_host, validate_csr
  instance.py    the reference's .inst interface (parse_instance, validate_instance, run)
  sharded.py     row-block sharding over torch.distributed (B broadcast once)
  workloads.py   synthetic CSR generators for the BASELINE configs
  errors.py      Error / ErrorKind mirroring raceset::Error

Importing the package does not load CUDA code; ``spmm`` / ``instance.run``
load libgespmm.so on first use and raise if it is not built.
"""
from .errors import Error, ErrorKind  # noqa: F401

__all__ = ["Error", "ErrorKind"]
