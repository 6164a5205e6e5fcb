// gespmm_graphgen.cu -- synthetic CSR generation on the GPU (SURVEY.md 8 row f3:
// "GPU R-MAT/uniform generation, sort, dedup" -- the step before the hot path).
//
// R-MAT (Graph500 quadrant recursion, no vertex permutation, as SURVEY 8(d)):
// edge e picks one quadrant per level l < scale with probabilities (a, b, c, d):
// u < a -> (0,0); u < a+b -> (0,1); u < a+b+c -> (1,0); else (1,1), setting
// row/col bit l.  The uniforms are Philox4x32-10 outputs keyed by the seed
// and counted by (edge, level group): the graph depends only on (scale, edges,
// a, b, c, seed) -- never on the grid or the device.
//
// Pipeline (all on `stream`, temporaries stream-ordered):
//   k_rmat_keys   edge -> key = row << scale | col            (HBM write, 8 B/edge)
//   CUB radix sort on the low 2*scale bits                    (sorted by (row, col))
//   CUB unique    -> nnz unique keys (dedup)
//   k_csr_from_keys: colind = key & mask; rowptr by row-boundary scatter
//   k_uniform_vals: vals[p] = 2u - 1, u = Philox(p) (fp32, U[-1, 1))
// One D2H of the unique count is the only host sync.
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_select.cuh>

#include "gespmm_internal.h"

namespace gespmm {
namespace {

struct U4 {
  uint32_t x, y, z, w;
};

// Philox4x32-10 (Salmon et al., SC'11): counter (c0..c3), key (k0, k1).
__host__ __device__ __forceinline__ U4 philox(U4 c, uint32_t k0, uint32_t k1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint64_t p0 = static_cast<uint64_t>(0xD2511F53u) * c.x;
    const uint64_t p1 = static_cast<uint64_t>(0xCD9E8D57u) * c.z;
    const uint32_t h0 = static_cast<uint32_t>(p0 >> 32), l0 = static_cast<uint32_t>(p0);
    const uint32_t h1 = static_cast<uint32_t>(p1 >> 32), l1 = static_cast<uint32_t>(p1);
    c = U4{h1 ^ c.y ^ k0, l1, h0 ^ c.w ^ k1, l0};
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  return c;
}

// Probability thresholds as 32-bit fixed point: u32 < t  <=>  u < t / 2^32.
struct Thr {
  uint32_t a, ab, abc;
};

__global__ void k_rmat_keys(int64_t edges, int scale, Thr t, uint32_t s0, uint32_t s1,
                            uint64_t* __restrict__ keys) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < edges; e += stride) {
    uint64_t row = 0, col = 0;
    for (int l0 = 0; l0 < scale; l0 += 4) {
      const U4 r = philox(U4{static_cast<uint32_t>(e), static_cast<uint32_t>(e >> 32),
                             static_cast<uint32_t>(l0), 0x52414D54u /* "RMAT" */},
                          s0, s1);
      const uint32_t u[4] = {r.x, r.y, r.z, r.w};
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int l = l0 + k;
        if (l >= scale) break;
        const uint64_t rb = u[k] >= t.ab;                           // quadrants c, d
        const uint64_t cb = (u[k] >= t.a && u[k] < t.ab) || u[k] >= t.abc;  // b, d
        row |= rb << l;
        col |= cb << l;
      }
    }
    keys[e] = (row << scale) | col;
  }
}

// keys sorted and unique: colind[i] = col(key[i]); rowptr[r] = first i with row >= r.
__global__ void k_csr_from_keys(const uint64_t* __restrict__ keys, int64_t nnz, int scale,
                                int64_t n_rows, int32_t* __restrict__ rowptr,
                                int32_t* __restrict__ colind) {
  const uint64_t mask = (uint64_t(1) << scale) - 1;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i <= nnz; i += stride) {
    const int64_t r = i < nnz ? static_cast<int64_t>(keys[i] >> scale) : n_rows;
    const int64_t rp = i > 0 ? static_cast<int64_t>(keys[i - 1] >> scale) : -1;
    for (int64_t q = rp + 1; q <= r; ++q) rowptr[q] = static_cast<int32_t>(i);
    if (i < nnz) colind[i] = static_cast<int32_t>(keys[i] & mask);
  }
}

__global__ void k_uniform_vals(int64_t n, uint32_t s0, uint32_t s1, float lo, float hi,
                               float* __restrict__ out) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n; i += stride) {
    const U4 r = philox(U4{static_cast<uint32_t>(i), static_cast<uint32_t>(i >> 32), 0x56414C53u /* "VALS" */, 0},
                        s0, s1);
    const float u = static_cast<float>(r.x >> 8) * (1.0f / 16777216.0f);  // [0, 1), 24 bits
    out[i] = lo + (hi - lo) * u;
  }
}

unsigned grid_for(int64_t n, int threads = 256) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  int64_t b = (n + threads - 1) / threads;
  const int64_t cap = static_cast<int64_t>(sms) * 16;
  if (b > cap) b = cap;
  return static_cast<unsigned>(b < 1 ? 1 : b);
}

}  // namespace
}  // namespace gespmm

using namespace gespmm;

extern "C" {

gespmm_status_t gespmm_rmat_csr(int32_t scale, int64_t edges, double a, double b, double c,
                                uint64_t seed, int32_t* rowptr, int32_t* colind, float* vals,
                                int64_t* nnz_out, void* stream) {
  if (scale < 1 || scale > 30 || edges < 0 || !nnz_out || !rowptr || (edges > 0 && (!colind || !vals)))
    return fail(GESPMM_INVALID_ARG, "invalid argument: rmat needs 1 <= scale <= 30, edges >= 0, buffers");
  if (edges > (int64_t(1) << 31) - 1024)
    return fail(GESPMM_INVALID_ARG, "invalid argument: rmat edges must fit int32 positions");
  if (!(a >= 0 && b >= 0 && c >= 0 && a + b + c <= 1.0))
    return fail(GESPMM_INVALID_ARG, "invalid argument: rmat probabilities");
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const int64_t n_rows = int64_t(1) << scale;
  auto thr = [](double p) {
    const double x = p * 4294967296.0;
    return static_cast<uint32_t>(x >= 4294967295.0 ? 4294967295.0 : x);
  };
  const Thr t{thr(a), thr(a + b), thr(a + b + c)};
  const uint32_t s0 = static_cast<uint32_t>(seed), s1 = static_cast<uint32_t>(seed >> 32);
  *nnz_out = 0;
  if (edges == 0) {
    cudaError_t e = cudaMemsetAsync(rowptr, 0, static_cast<size_t>(n_rows + 1) * 4, s);
    return e == cudaSuccess ? GESPMM_OK : cuda_fail(e, "rmat rowptr");
  }
  const int n = static_cast<int>(edges);
  uint64_t *k0 = nullptr, *k1 = nullptr;
  int64_t* d_cnt = nullptr;
  void* tmp = nullptr;
  size_t t_sort = 0, t_uniq = 0;
  cub::DeviceRadixSort::SortKeys(nullptr, t_sort, k0, k1, n, 0, 2 * scale, s);
  cub::DeviceSelect::Unique(nullptr, t_uniq, k1, k0, d_cnt, n, s);
  const size_t t_bytes = t_sort > t_uniq ? t_sort : t_uniq;
  cudaError_t e = cudaMallocAsync(&k0, static_cast<size_t>(n) * 8, s);
  if (e == cudaSuccess) e = cudaMallocAsync(&k1, static_cast<size_t>(n) * 8, s);
  if (e == cudaSuccess) e = cudaMallocAsync(&tmp, t_bytes + 256, s);
  if (e == cudaSuccess) e = cudaMallocAsync(&d_cnt, sizeof(int64_t), s);
  int64_t nnz = 0;
  if (e == cudaSuccess) {
    k_rmat_keys<<<grid_for(edges), 256, 0, s>>>(edges, scale, t, s0, s1, k0);
    size_t tb = t_bytes;
    cub::DeviceRadixSort::SortKeys(tmp, tb, k0, k1, n, 0, 2 * scale, s);
    tb = t_bytes;
    cub::DeviceSelect::Unique(tmp, tb, k1, k0, d_cnt, n, s);
    e = cudaMemcpyAsync(&nnz, d_cnt, sizeof(int64_t), cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  }
  if (e == cudaSuccess) {
    k_csr_from_keys<<<grid_for(nnz + 1), 256, 0, s>>>(k0, nnz, scale, n_rows, rowptr, colind);
    k_uniform_vals<<<grid_for(nnz), 256, 0, s>>>(nnz, s0 ^ 0x5EEDu, s1, -1.0f, 1.0f, vals);
    e = cudaGetLastError();
  }
  if (k0) cudaFreeAsync(k0, s);
  if (k1) cudaFreeAsync(k1, s);
  if (tmp) cudaFreeAsync(tmp, s);
  if (d_cnt) cudaFreeAsync(d_cnt, s);
  if (e != cudaSuccess) return cuda_fail(e, "rmat generation");
  *nnz_out = nnz;
  return GESPMM_OK;
}

gespmm_status_t gespmm_uniform_fill(float* out, int64_t n, float lo, float hi, uint64_t seed,
                                    void* stream) {
  if (n < 0 || (n > 0 && !out)) return fail(GESPMM_INVALID_ARG, "invalid argument: uniform fill");
  if (n == 0) return GESPMM_OK;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  k_uniform_vals<<<grid_for(n), 256, 0, s>>>(n, static_cast<uint32_t>(seed),
                                             static_cast<uint32_t>(seed >> 32), lo, hi, out);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? GESPMM_OK : cuda_fail(e, "uniform fill");
}

}  // extern "C"
