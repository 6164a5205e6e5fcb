// Instantiates the GE-SpMM kernel family for the MAX reduce op
// (one translation unit per op so the variants compile in parallel).
#include "gespmm_kernel_pair.cuh"

namespace gespmm {
cudaError_t launch_spmm_max(const Variant& v, const KParams& p, cudaStream_t s) {
  if (v.pair) return kern::launch_pair<GESPMM_REDUCE_MAX>(v, p, s);
  return kern::launch_op<GESPMM_REDUCE_MAX>(v, p, s);
}
}  // namespace gespmm
