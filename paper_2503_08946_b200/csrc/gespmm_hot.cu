// gespmm_hot.cu -- the L2 hot set of B rows for products whose B is many
// times larger than L2 (DESIGN.md 5.2 "Hot set"; R-MAT configs 4/5).
//
// Each nonzero gathers one B row (gespmm_alg2.mir:51-53).  With B >> L2 the
// row stream misses L2 unless it names a popular column; under LRU the cold
// misses also evict the popular rows.  The hot set is the H most-referenced
// columns (H x row bytes ~ the L2 budget): the kernel gathers their rows with
// an L2 evict_last policy and every other row with evict_first, so cold rows
// stream through without displacing the hot ones.  Only cache policies
// change -- never an address or an arithmetic step -- so results are
// bit-identical with or without it.
//
// Built on the device with no host synchronization (graph-capturable after
// the first call), once per plan and hot-set size:
//   k_coldeg    column degrees (one atomic per nonzero)
//   k_deghist   a 4096-bucket histogram of the degrees (shared-memory
//               privatized; bucket = degree below 2048, then 32-wide bins)
//   k_threshold one block: the smallest bucket b* whose suffix count fits H
//   k_hotbits   bit c of the bitmap = bucket(deg[c]) >= b* (one ballot per
//               32 columns, no atomics)
#include "gespmm_internal.h"

namespace gespmm {
namespace {

constexpr int kBuckets = 4096;

__device__ __forceinline__ int deg_bucket(int d) {
  if (d < 2048) return d;
  const int b = 2048 + ((d - 2048) >> 5);
  return b < kBuckets ? b : kBuckets - 1;
}

__global__ void k_coldeg(const int* __restrict__ colind, int64_t nnz, int K, int* __restrict__ deg) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t p = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; p < nnz; p += stride) {
    const int c = __ldcs(colind + p);
    if (static_cast<unsigned>(c) < static_cast<unsigned>(K)) atomicAdd(deg + c, 1);
  }
}

__global__ void k_deghist(const int* __restrict__ deg, int K, unsigned* __restrict__ hist) {
  __shared__ unsigned h[kBuckets];
  for (int i = threadIdx.x; i < kBuckets; i += blockDim.x) h[i] = 0;
  __syncthreads();
  const int stride = gridDim.x * blockDim.x;
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < K; c += stride) {
    const int d = deg[c];
    if (d > 0) atomicAdd(&h[deg_bucket(d)], 1u);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < kBuckets; i += blockDim.x)
    if (h[i]) atomicAdd(hist + i, h[i]);
}

// One block of 1024 threads (4 buckets each): b* = the smallest bucket b >= 1
// with sum_{b' >= b} hist[b'] <= H (unreferenced columns, bucket 0, are cold;
// b* = kBuckets when nothing fits).
__global__ void k_threshold(const unsigned* __restrict__ hist, int64_t H, int* __restrict__ out) {
  constexpr int kPer = kBuckets / 1024;
  __shared__ unsigned long long part[1024];
  const int t = threadIdx.x;
  if (t == 0) *out = kBuckets;  // the only block: ordered before the atomicMin below
  unsigned long long mine = 0;
  for (int k = 0; k < kPer; ++k) mine += hist[t * kPer + k];
  part[t] = mine;
  __syncthreads();
  for (int off = 1; off < 1024; off <<= 1) {  // inclusive suffix sum over the threads
    const unsigned long long v = t + off < 1024 ? part[t + off] : 0ULL;
    __syncthreads();
    part[t] += v;
    __syncthreads();
  }
  unsigned long long suf = part[t];  // sum of buckets >= t*kPer
  for (int k = 0; k < kPer; ++k) {
    const int b = t * kPer + k;
    if (b >= 1 && suf <= static_cast<unsigned long long>(H)) {
      atomicMin(out, b);
      break;
    }
    suf -= hist[b];
  }
}

__global__ void k_hotbits(const int* __restrict__ deg, int K, const int* __restrict__ thr,
                          uint32_t* __restrict__ bits) {
  const int b = *thr;
  const int nw = (K + 31) >> 5;
  const int lane = threadIdx.x & 31;
  const int wstride = (gridDim.x * blockDim.x) >> 5;
  for (int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; w < nw; w += wstride) {
    const int c = (w << 5) + lane;
    const int d = c < K ? deg[c] : 0;
    const unsigned m = __ballot_sync(0xffffffffu, d > 0 && deg_bucket(d) >= b);
    if (lane == 0) bits[w] = m;
  }
}

}  // namespace

cudaError_t build_hot_bits(gespmm_plan_s* plan, const int* colind, int64_t H, cudaStream_t s) {
  const int64_t K = plan->K;
  const int64_t words = (K + 31) / 32;
  cudaError_t e = cudaSuccess;
  if (!plan->hot_bits || plan->hot_words < words) {
    if (plan->hot_bits) cudaFree(plan->hot_bits);
    plan->hot_bits = nullptr;
    plan->hot_words = 0;
    e = cudaMallocAsync(&plan->hot_bits, static_cast<size_t>(words > 0 ? words : 1) * 4, s);
    if (e != cudaSuccess) return e;
    plan->hot_words = words;
  }
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  char* tmp = nullptr;
  const size_t deg_bytes = (static_cast<size_t>(K) * 4 + 255) & ~size_t(255);
  e = cudaMallocAsync(&tmp, deg_bytes + kBuckets * 4 + 256, s);
  if (e != cudaSuccess) return e;
  int* deg = reinterpret_cast<int*>(tmp);
  unsigned* hist = reinterpret_cast<unsigned*>(tmp + deg_bytes);
  int* thr = reinterpret_cast<int*>(tmp + deg_bytes + kBuckets * 4);
  cudaMemsetAsync(tmp, 0, deg_bytes + kBuckets * 4 + 256, s);
  const int64_t nnz = plan->nnz;
  if (nnz > 0) {
    int64_t blocks = (nnz + 255) / 256;
    if (blocks > 8 * sms) blocks = 8 * sms;
    k_coldeg<<<static_cast<unsigned>(blocks), 256, 0, s>>>(colind, nnz, static_cast<int>(K), deg);
  }
  if (K > 0) {
    int64_t blocks = (K + 255) / 256;
    if (blocks > 2 * sms) blocks = 2 * sms;
    k_deghist<<<static_cast<unsigned>(blocks), 256, 0, s>>>(deg, static_cast<int>(K), hist);
    k_threshold<<<1, 1024, 0, s>>>(hist, H, thr);
    int64_t wb = (words * 32 + 255) / 256;
    if (wb > 8 * sms) wb = 8 * sms;
    k_hotbits<<<static_cast<unsigned>(wb), 256, 0, s>>>(deg, static_cast<int>(K), thr, plan->hot_bits);
  }
  e = cudaGetLastError();
  cudaFreeAsync(tmp, s);
  plan->hot_key = H;
  return e;
}

}  // namespace gespmm
