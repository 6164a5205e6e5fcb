// Instantiates the GE-SpMM kernel family for the MEAN reduce op
// (one translation unit per op so the variants compile in parallel).
#include "gespmm_kernel.cuh"

namespace gespmm {
cudaError_t launch_spmm_mean(const Variant& v, const KParams& p, cudaStream_t s) {
  return kern::launch_op<GESPMM_REDUCE_MEAN>(v, p, s);
}
}  // namespace gespmm
