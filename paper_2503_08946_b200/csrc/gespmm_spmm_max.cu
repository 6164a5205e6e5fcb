// Instantiates the GE-SpMM kernel family for the MAX reduce op
// (one translation unit per op so the variants compile in parallel).
#include "gespmm_kernel.cuh"

namespace gespmm {
cudaError_t launch_spmm_max(const Variant& v, const KParams& p, cudaStream_t s) {
  return kern::launch_op<GESPMM_REDUCE_MAX>(v, p, s);
}
}  // namespace gespmm
