// gespmm_convert.cu -- sparse-format conversions on the GPU, the data formats
// either side of the hot path (SURVEY.md 8 "next" rows: the callers' formats).
//
//   gespmm_coo_to_csr   COO (row, col, val) triples -> CSR; entries keep their
//                       input order within a row (stable by row), duplicates
//                       kept -- the reference CSR contract allows both
//                       (src/oracle.cpp:291-316 checks neither sortedness nor
//                       uniqueness), and the within-row order is the fold order.
//   gespmm_csr_transpose CSR of A (M x K) -> CSR of A^T (K x M); row j of A^T
//                       lists the nonzeros of column j of A in ascending row
//                       order (stable), i.e. the CSC of A.  The SpMM of A^T
//                       (e.g. a GNN backward pass) then runs on the same path.
//
// Both: a stable CUB radix sort of (key, position) pairs on the key's bits,
// a gather of the payload through the permutation, and rowptr from the sorted
// keys (first index of each key).  All on `stream`; one D2H-free pipeline
// (counts are known: nnz in = nnz out).
#include <cub/device/device_radix_sort.cuh>

#include "gespmm_internal.h"

namespace gespmm {
namespace {

__global__ void k_iota(int32_t* __restrict__ p, int64_t n) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n; i += stride)
    p[i] = static_cast<int32_t>(i);
}

// keys[p] = row of position p from a CSR rowptr (expands rows), i.e. the COO row list
__global__ void k_expand_rows(const int32_t* __restrict__ rowptr, int64_t M, int32_t* __restrict__ rows) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t r = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; r < M; r += stride)
    for (int32_t p = rowptr[r]; p < rowptr[r + 1]; ++p) rows[p] = static_cast<int32_t>(r);
}

__global__ void k_gather(const int32_t* __restrict__ perm, const int32_t* __restrict__ src_i,
                         const float* __restrict__ src_v, int64_t n, int32_t* __restrict__ dst_i,
                         float* __restrict__ dst_v) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n; i += stride) {
    const int32_t q = perm[i];
    dst_i[i] = src_i[q];
    dst_v[i] = src_v[q];
  }
}

// rowptr[k] = first i with keys[i] >= k (keys sorted), rowptr[n_rows] = n
__global__ void k_rowptr_from_sorted(const int32_t* __restrict__ keys, int64_t n, int64_t n_rows,
                                     int32_t* __restrict__ rowptr) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i <= n; i += stride) {
    const int64_t k = i < n ? keys[i] : n_rows;
    const int64_t kp = i > 0 ? keys[i - 1] : -1;
    for (int64_t q = kp + 1; q <= k; ++q) rowptr[q] = static_cast<int32_t>(i);
  }
}

__global__ void k_key_range(const int32_t* __restrict__ keys, int64_t n, int64_t lim, int* __restrict__ bad) {
  int b = 0;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n; i += stride)
    b |= (keys[i] < 0) | (keys[i] >= lim);
  if (__any_sync(0xffffffffu, b) && (threadIdx.x & 31) == 0) atomicOr(bad, 1);
}

unsigned grid_for(int64_t n) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  int64_t b = (n + 255) / 256;
  if (b > static_cast<int64_t>(sms) * 16) b = static_cast<int64_t>(sms) * 16;
  return static_cast<unsigned>(b < 1 ? 1 : b);
}

int key_bits(int64_t n_keys) {
  int b = 1;
  while ((int64_t(1) << b) < n_keys) ++b;
  return b;
}

// Stable sort of positions by key (keys[0..n) in [0, n_keys)), then the CSR:
// out_rowptr[n_keys + 1], out_idx/out_val = payload gathered in sorted order.
gespmm_status_t sort_to_csr(const int32_t* keys, const int32_t* payload_i, const float* payload_v,
                            int64_t n, int64_t n_keys, int32_t* out_rowptr, int32_t* out_idx,
                            float* out_val, cudaStream_t s) {
  int32_t *k_sorted = nullptr, *perm_in = nullptr, *perm_out = nullptr;
  void* tmp = nullptr;
  int* bad = nullptr;
  const int nn = static_cast<int>(n);
  size_t t_bytes = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, t_bytes, keys, k_sorted, perm_in, perm_out, nn, 0,
                                  key_bits(n_keys), s);
  cudaError_t e = cudaMallocAsync(&k_sorted, static_cast<size_t>(n > 0 ? n : 1) * 4, s);
  if (e == cudaSuccess) e = cudaMallocAsync(&perm_in, static_cast<size_t>(n > 0 ? n : 1) * 4, s);
  if (e == cudaSuccess) e = cudaMallocAsync(&perm_out, static_cast<size_t>(n > 0 ? n : 1) * 4, s);
  if (e == cudaSuccess) e = cudaMallocAsync(&tmp, t_bytes + 256, s);
  if (e == cudaSuccess) e = cudaMallocAsync(&bad, sizeof(int), s);
  int h_bad = 0;
  if (e == cudaSuccess) {
    cudaMemsetAsync(bad, 0, sizeof(int), s);
    if (n > 0) k_key_range<<<grid_for(n), 256, 0, s>>>(keys, n, n_keys, bad);
    e = cudaMemcpyAsync(&h_bad, bad, sizeof(int), cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  }
  if (e == cudaSuccess && !h_bad) {
    if (n > 0) {
      k_iota<<<grid_for(n), 256, 0, s>>>(perm_in, n);
      size_t tb = t_bytes;
      cub::DeviceRadixSort::SortPairs(tmp, tb, keys, k_sorted, perm_in, perm_out, nn, 0, key_bits(n_keys), s);
      k_gather<<<grid_for(n), 256, 0, s>>>(perm_out, payload_i, payload_v, n, out_idx, out_val);
    }
    k_rowptr_from_sorted<<<grid_for(n + 1), 256, 0, s>>>(k_sorted, n, n_keys, out_rowptr);
    e = cudaGetLastError();
  }
  for (void* p : {static_cast<void*>(k_sorted), static_cast<void*>(perm_in), static_cast<void*>(perm_out), tmp,
                  static_cast<void*>(bad)})
    if (p) cudaFreeAsync(p, s);
  if (e != cudaSuccess) return cuda_fail(e, "sparse conversion");
  if (h_bad) return fail(GESPMM_OUT_OF_BOUNDS, "out of bounds: an index lies outside the matrix shape");
  return GESPMM_OK;
}

}  // namespace
}  // namespace gespmm

using namespace gespmm;

extern "C" {

gespmm_status_t gespmm_coo_to_csr(int64_t M, int64_t nnz, const int32_t* rows, const int32_t* cols,
                                  const float* vals, int32_t* rowptr, int32_t* colind, float* vals_out,
                                  void* stream) {
  if (M < 0 || nnz < 0 || !rowptr || (nnz > 0 && (!rows || !cols || !vals || !colind || !vals_out)))
    return fail(GESPMM_INVALID_ARG, "invalid argument: coo_to_csr");
  if (nnz > (int64_t(1) << 31) - 1024 || M > (int64_t(1) << 31) - 2)
    return fail(GESPMM_INVALID_ARG, "invalid argument: M and nnz must fit int32 indexing");
  return sort_to_csr(rows, cols, vals, nnz, M, rowptr, colind, vals_out, reinterpret_cast<cudaStream_t>(stream));
}

gespmm_status_t gespmm_csr_transpose(int64_t M, int64_t K, int64_t nnz, const int32_t* rowptr,
                                     const int32_t* colind, const float* vals, int32_t* t_rowptr,
                                     int32_t* t_colind, float* t_vals, void* stream) {
  if (M < 0 || K < 0 || nnz < 0 || !t_rowptr || (M > 0 && !rowptr) ||
      (nnz > 0 && (!colind || !vals || !t_colind || !t_vals)))
    return fail(GESPMM_INVALID_ARG, "invalid argument: csr_transpose");
  if (nnz > (int64_t(1) << 31) - 1024 || K > (int64_t(1) << 31) - 2)
    return fail(GESPMM_INVALID_ARG, "invalid argument: K and nnz must fit int32 indexing");
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  int32_t* rows = nullptr;
  cudaError_t e = cudaMallocAsync(&rows, static_cast<size_t>(nnz > 0 ? nnz : 1) * 4, s);
  if (e != cudaSuccess) return cuda_fail(e, "csr_transpose rows");
  if (M > 0) k_expand_rows<<<grid_for(M), 256, 0, s>>>(rowptr, M, rows);
  // sort the (col -> row) pairs by col, stably: row j of A^T lists rows ascending
  const gespmm_status_t st = sort_to_csr(colind, rows, vals, nnz, K, t_rowptr, t_colind, t_vals, s);
  cudaFreeAsync(rows, s);
  return st;
}

}  // extern "C"
