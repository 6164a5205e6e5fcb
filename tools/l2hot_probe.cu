// l2hot_probe.cu -- how much of the large-R-MAT DRAM traffic an L2 hot set
// can remove (VERDICT r1 "Next" 3).
//
// Replays a column stream (a CSR's colind) as 512-byte B-row gathers (N=128
// fp32, one 16-byte LDG per lane), the SpMM's order: each warp walks
// contiguous spans of `span` positions, U rows in flight.  Nothing else is
// read or written, so the time and DRAM bytes isolate the B gathers.
//
// idx entries carry a hot flag in bit 31 (set by the caller from the column
// degrees).  Modes:
//   0  plain loads (no cache hint)
//   1  hot rows L2::evict_last, cold rows L2::evict_first (per-lane policy select)
//   2  hot rows evict_last, cold rows evict_normal
//   3  hot rows normal, cold rows evict_first
//   4  hot rows from a compact copy (hot index in the low bits), cold rows
//      plain -- with an access-policy window on the copy set by the caller
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>

// GESPMM_PROBE_SUSTAINED=1: report the mean of the second half of the reps
// (back-to-back runs under sustained power/clock state) instead of the best.
struct RepStat {
  int reps;
  float best = 1e30f;
  double tail = 0;
  int ntail = 0;
  explicit RepStat(int r) : reps(r) {}
  void add(int r, float ms) {
    if (r >= 1 && ms < best) best = ms;
    if (r > reps / 2) tail += ms, ++ntail;
  }
  float result() const {
    const char* e = std::getenv("GESPMM_PROBE_SUSTAINED");
    return (e && *e == '1' && ntail) ? static_cast<float>(tail / ntail) : best;
  }
};

template <int VEC>
struct VT;
template <>
struct VT<1> { using T = float; };
template <>
struct VT<2> { using T = float2; };
template <>
struct VT<4> { using T = float4; };

__device__ __forceinline__ void ldh(float& d, const float* p, uint64_t pol) {
  asm volatile("ld.global.nc.L2::cache_hint.f32 %0, [%1], %2;" : "=f"(d) : "l"(p), "l"(pol));
}
__device__ __forceinline__ void ldh(float2& d, const float* p, uint64_t pol) {
  asm volatile("ld.global.nc.L2::cache_hint.v2.f32 {%0, %1}, [%2], %3;" : "=f"(d.x), "=f"(d.y) : "l"(p), "l"(pol));
}
__device__ __forceinline__ void ldh(float4& d, const float* p, uint64_t pol) {
  asm volatile("ld.global.nc.L2::cache_hint.v4.f32 {%0, %1, %2, %3}, [%4], %5;"
               : "=f"(d.x), "=f"(d.y), "=f"(d.z), "=f"(d.w) : "l"(p), "l"(pol));
}
__device__ __forceinline__ float sum(float v) { return v; }
__device__ __forceinline__ float sum(float2 v) { return v.x + v.y; }
__device__ __forceinline__ float sum(float4 v) { return v.x + v.y + v.z + v.w; }

// Row-width generic form: each row gathers 32*VEC floats at column offset
// `col0` of a 128-wide B (one column panel of a panelled execution).
template <int U, int MODE, int VEC>
__global__ void __launch_bounds__(256, U * VEC <= 32 ? 4 : U * VEC <= 64 ? 2 : 1)
    probe_w(const float* __restrict__ B, const int* __restrict__ idx, int64_t nidx, int span, int col0,
            float* sink) {
  using T = typename VT<VEC>::T;
  const int lane = threadIdx.x & 31;
  const int64_t warp = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  uint64_t pl, pf, pn;
  asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pl));
  asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pf));
  asm("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(pn));
  float a0 = 0.f;
  for (int64_t s0 = warp * span; s0 < nidx; s0 += nw * span) {
    const int64_t s1 = s0 + span < nidx ? s0 + span : nidx;
    for (int64_t base = s0; base < s1; base += U) {
      const int my = (lane < U && base + lane < s1) ? __ldg(idx + base + lane) : 0;
      T v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int e = __shfl_sync(0xffffffffu, my, u);
        const bool hot = e < 0;
        const uint32_t r = static_cast<uint32_t>(e) & 0x7fffffffu;
        const float* src = B + static_cast<int64_t>(r) * 128 + col0 + VEC * lane;
        const uint64_t pol = MODE == 0 ? pn : MODE == 1 ? (hot ? pl : pf) : MODE == 2 ? (hot ? pl : pn) : (hot ? pn : pf);
        ldh(v[u], src, pol);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) a0 += sum(v[u]);
    }
  }
  if (a0 == 1234.5f) sink[0] = a0;
}

// Panelled replay: 128 / (32*vec) passes over idx, one per column panel
// (same stream order per pass); returns the best total of `reps` (ms).
// Bulk-copy ring: each warp owns D slots of U rows in shared memory; batch k
// is fetched by U lanes issuing one cp.async.bulk (global -> shared, the row's
// 32*VEC floats) each, completion tracked by the slot's mbarrier (expect_tx
// armed by lane 0 first); rows are read back with one LDS per lane per row.
// No registers hold in-flight rows, one instruction moves a whole row.
template <int U, int D, int VEC, int MODE>
__global__ void __launch_bounds__(256, 1)
    probe_bulk(const float* __restrict__ B, const int* __restrict__ idx, int64_t nidx, int span, int col0,
               float* sink) {
  extern __shared__ __align__(128) unsigned char smraw[];
  constexpr int RB = 128 * VEC;  // row bytes
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  unsigned char* ring = smraw + wib * (D * U * RB);
  __shared__ __align__(8) unsigned long long bar[8][D];
  const int64_t warp = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  uint64_t pl, pf;
  asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pl));
  asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pf));
  if (lane < D) {
    const uint32_t b = static_cast<uint32_t>(__cvta_generic_to_shared(&bar[wib][lane]));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b));
  }
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncwarp();
  uint32_t phase = 0;  // bit d: parity of slot d
  float a0 = 0.f;
  for (int64_t s0 = warp * span; s0 < nidx; s0 += nw * span) {
    const int64_t s1 = s0 + span < nidx ? s0 + span : nidx;
    const int nb = static_cast<int>((s1 - s0 + U - 1) / U);
    auto issue = [&](int k) {
      if (k >= nb) return;
      const int d = k % D;
      const uint32_t b = static_cast<uint32_t>(__cvta_generic_to_shared(&bar[wib][d]));
      const int64_t p = s0 + static_cast<int64_t>(k) * U + lane;
      const int nrow = static_cast<int>(s1 - (s0 + static_cast<int64_t>(k) * U) < U ? s1 - (s0 + static_cast<int64_t>(k) * U) : U);
      if (lane == 0)
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(nrow * RB) : "memory");
      __syncwarp();
      if (lane < nrow) {
        const int e = __ldg(idx + p);
        const bool hot = e < 0;
        const uint32_t r = static_cast<uint32_t>(e) & 0x7fffffffu;
        const float* src = B + static_cast<int64_t>(r) * 128 + col0;
        const uint32_t dst = static_cast<uint32_t>(__cvta_generic_to_shared(ring + (d * U + lane) * RB));
        if (MODE == 1) {
          const uint64_t pol = hot ? pl : pf;
          asm volatile(
              "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(dst),
              "l"(src), "n"(RB), "r"(b), "l"(pol)
              : "memory");
        } else {
          asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
                       "l"(src), "n"(RB), "r"(b)
                       : "memory");
        }
      }
    };
    for (int k = 0; k < D - 1; ++k) issue(k);
    for (int k = 0; k < nb; ++k) {
      issue(k + D - 1);
      const int d = k % D;
      const uint32_t b = static_cast<uint32_t>(__cvta_generic_to_shared(&bar[wib][d]));
      const uint32_t par = (phase >> d) & 1u;
      uint32_t done = 0;
      while (!done)
        asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                     : "=r"(done) : "r"(b), "r"(par) : "memory");
      phase ^= 1u << d;
      const int nrow = static_cast<int>(s1 - (s0 + static_cast<int64_t>(k) * U) < U ? s1 - (s0 + static_cast<int64_t>(k) * U) : U);
#pragma unroll 4
      for (int u = 0; u < nrow; ++u) {
        const float* row = reinterpret_cast<const float*>(ring + (d * U + u) * RB);
        if (VEC == 4) {
          const float4 v = reinterpret_cast<const float4*>(row)[lane];
          a0 += v.x + v.y + v.z + v.w;
        } else if (VEC == 2) {
          const float2 v = reinterpret_cast<const float2*>(row)[lane];
          a0 += v.x + v.y;
        } else {
          a0 += row[lane];
        }
      }
      __syncwarp();  // slot d is refilled by issue(k + D)
    }
  }
  if (a0 == 1234.5f) sink[0] = a0;
}

extern "C" float l2hot_probe_bulk(const float* B, const int* idx, int64_t nidx, int mode, int vec, int U, int D,
                                  int span, int blocks_per_sm, int reps, float* sink, void* flush, int64_t flush_bytes) {
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int smem = 8 * D * U * 128 * vec;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e30f;
  const int grid = sms * blocks_per_sm;
  const int w = 32 * vec;
#define KB(UU, DD, VV, MM) probe_bulk<UU, DD, VV, MM>
#define SETA(UU, DD, VV, MM) cudaFuncSetAttribute(KB(UU, DD, VV, MM), cudaFuncAttributeMaxDynamicSharedMemorySize, smem)
#define RUN(UU, DD, VV, MM) KB(UU, DD, VV, MM)<<<grid, 256, smem>>>(B, idx, nidx, span, c0, sink)
#define ALL(X, MM)                                                          \
  if (vec == 2 && U == 16 && D == 2) X(16, 2, 2, MM);                      \
  else if (vec == 2 && U == 16 && D == 4) X(16, 4, 2, MM);                 \
  else if (vec == 2 && U == 32 && D == 2) X(32, 2, 2, MM);                 \
  else if (vec == 4 && U == 8 && D == 4) X(8, 4, 4, MM);                   \
  else if (vec == 4 && U == 16 && D == 2) X(16, 2, 4, MM);                 \
  else if (vec == 4 && U == 8 && D == 2) X(8, 2, 4, MM);                   \
  else if (vec == 1 && U == 32 && D == 2) X(32, 2, 1, MM);                 \
  else X(8, 2, 2, MM);
  if (mode == 1) { ALL(SETA, 1) } else { ALL(SETA, 0) }
  for (int r = 0; r < reps + 1; ++r) {
    cudaDeviceSynchronize();
    if (flush) cudaMemsetAsync(flush, r & 0xff, flush_bytes);
    cudaEventRecord(e0);
    for (int c0 = 0; c0 < 128; c0 += w) {
      if (mode == 1) { ALL(RUN, 1) } else { ALL(RUN, 0) }
    }
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    if (r >= 1 && ms < best) best = ms;
  }
#undef ALL
#undef RUN
#undef SETA
#undef KB
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  const cudaError_t err = cudaGetLastError();
  return err == cudaSuccess ? best : -static_cast<float>(err);
}

extern "C" float l2hot_probe_panels(const float* B, const int* idx, int64_t nidx, int mode, int vec, int span,
                                    int blocks_per_sm, int reps, float* sink, void* flush, int64_t flush_bytes,
                                    int U) {
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e30f;
  const int grid = sms * blocks_per_sm;
  const int w = 32 * vec;
  for (int r = 0; r < reps + 1; ++r) {
    cudaDeviceSynchronize();
    if (flush) cudaMemsetAsync(flush, r & 0xff, flush_bytes);
    cudaEventRecord(e0);
    for (int c0 = 0; c0 < 128; c0 += w) {
#define L(M, V)                                                                       \
  (U == 16 ? probe_w<16, M, V><<<grid, 256>>>(B, idx, nidx, span, c0, sink)          \
           : U == 32 ? probe_w<32, M, V><<<grid, 256>>>(B, idx, nidx, span, c0, sink) \
                     : probe_w<8, M, V><<<grid, 256>>>(B, idx, nidx, span, c0, sink))
#define LV(M) (vec == 1 ? L(M, 1) : vec == 2 ? L(M, 2) : L(M, 4))
      switch (mode) {
        case 1: LV(1); break;
        case 2: LV(2); break;
        case 3: LV(3); break;
        default: LV(0); break;
      }
#undef LV
#undef L
    }
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    if (r >= 1 && ms < best) best = ms;
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  const cudaError_t err = cudaGetLastError();
  return err == cudaSuccess ? best : -static_cast<float>(err);
}

template <int U, int MODE>
__global__ void __launch_bounds__(256, 4)
    probe_hot(const float* __restrict__ B, const float* __restrict__ H, const int* __restrict__ idx,
              int64_t nidx, int span, float* sink) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  uint64_t pl, pf;
  asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pl));
  asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pf));
  uint64_t pn;
  asm("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(pn));
  float a0 = 0.f, a1 = 0.f;
  for (int64_t s0 = warp * span; s0 < nidx; s0 += nw * span) {
    const int64_t s1 = s0 + span < nidx ? s0 + span : nidx;
    for (int64_t base = s0; base < s1; base += U) {
      const int my = (lane < U && base + lane < s1) ? __ldg(idx + base + lane) : 0;
      float4 v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int e = __shfl_sync(0xffffffffu, my, u);
        const bool hot = e < 0;
        const uint32_t r = static_cast<uint32_t>(e) & 0x7fffffffu;
        if (MODE == 0) {
          v[u] = __ldg(reinterpret_cast<const float4*>(B + static_cast<int64_t>(r) * 128) + lane);
        } else if (MODE == 4) {
          const float* src = (hot ? H : B) + static_cast<int64_t>(r) * 128;
          v[u] = __ldg(reinterpret_cast<const float4*>(src) + lane);
        } else {
          const uint64_t pol = MODE == 1 ? (hot ? pl : pf) : MODE == 2 ? (hot ? pl : pn) : (hot ? pn : pf);
          const float* src = B + static_cast<int64_t>(r) * 128 + 4 * lane;
          asm volatile("ld.global.nc.L2::cache_hint.v4.f32 {%0, %1, %2, %3}, [%4], %5;"
                       : "=f"(v[u].x), "=f"(v[u].y), "=f"(v[u].z), "=f"(v[u].w)
                       : "l"(src), "l"(pol));
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        a0 += v[u].x + v[u].z;
        a1 += v[u].y + v[u].w;
      }
    }
  }
  if (a0 == 1234.5f) sink[0] = a1;
}

// Returns the best of `reps` timed runs (ms), L2 flushed before each; -1 on error.
// persist_bytes >= 0: cudaLimitPersistingL2CacheSize is set to it first;
// win_bytes > 0 (mode 4): an access-policy window [H, H + win_bytes) persisting.
extern "C" float l2hot_probe(const float* B, const float* H, const int* idx, int64_t nidx, int mode,
                             int span, int blocks_per_sm, int reps, float* sink, void* flush,
                             int64_t flush_bytes, int64_t persist_bytes, int64_t win_bytes, float hit_ratio) {
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (persist_bytes >= 0) cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, static_cast<size_t>(persist_bytes));
  cudaStream_t s = 0;
  cudaStreamCreate(&s);
  if (win_bytes > 0) {
    cudaStreamAttrValue a = {};
    a.accessPolicyWindow.base_ptr = const_cast<float*>(H);
    a.accessPolicyWindow.num_bytes = static_cast<size_t>(win_bytes);
    a.accessPolicyWindow.hitRatio = hit_ratio;
    a.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
    a.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
    cudaStreamSetAttribute(s, cudaStreamAttributeAccessPolicyWindow, &a);
  }
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e30f;
  const int grid = sms * blocks_per_sm;
  for (int r = 0; r < reps + 1; ++r) {
    cudaStreamSynchronize(s);
    cudaCtxResetPersistingL2Cache();  // no hot lines carried over from the previous rep
    if (flush) cudaMemsetAsync(flush, r & 0xff, flush_bytes, s);
    cudaEventRecord(e0, s);
    switch (mode) {
      case 1: probe_hot<8, 1><<<grid, 256, 0, s>>>(B, H, idx, nidx, span, sink); break;
      case 2: probe_hot<8, 2><<<grid, 256, 0, s>>>(B, H, idx, nidx, span, sink); break;
      case 3: probe_hot<8, 3><<<grid, 256, 0, s>>>(B, H, idx, nidx, span, sink); break;
      case 4: probe_hot<8, 4><<<grid, 256, 0, s>>>(B, H, idx, nidx, span, sink); break;
      default: probe_hot<8, 0><<<grid, 256, 0, s>>>(B, H, idx, nidx, span, sink); break;
    }
    cudaEventRecord(e1, s);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    if (r >= 1 && ms < best) best = ms;
  }
  if (win_bytes > 0) {
    cudaStreamAttrValue a = {};
    a.accessPolicyWindow.num_bytes = 0;
    cudaStreamSetAttribute(s, cudaStreamAttributeAccessPolicyWindow, &a);
    cudaCtxResetPersistingL2Cache();
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaStreamDestroy(s);
  const cudaError_t err = cudaGetLastError();
  return err == cudaSuccess ? best : -static_cast<float>(err);
}

extern "C" int64_t l2hot_max_persist(void) {
  int dev = 0, v = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&v, cudaDevAttrMaxPersistingL2CacheSize, dev);
  return v;
}

// LDGSTS ring: D slots of U rows per warp in shared memory, rows copied with
// 16-byte cp.async (a row of 32*VEC floats takes 8*VEC lanes; 32/(8*VEC) rows
// per warp instruction), one commit group per slot, read back with one LDS per
// lane per row.  MODE 1: cp.async.L2::cache_hint with evict_last (hot rows) /
// evict_first (cold rows).
template <int U, int D, int VEC, int MODE>
__global__ void __launch_bounds__(256, 1)
    probe_ldgsts(const float* __restrict__ B, const int* __restrict__ idx, int64_t nidx, int span, int col0,
                 float* sink) {
  extern __shared__ __align__(128) unsigned char smraw[];
  constexpr int RB = 128 * VEC;          // row bytes
  constexpr int LPR = RB / 16;           // lanes per row
  constexpr int RPI = 32 / LPR;          // rows per warp instruction
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  unsigned char* ring = smraw + wib * (D * U * RB);
  const int64_t warp = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  uint64_t pl, pf;
  asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pl));
  asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pf));
  const int sub = lane / LPR, chunk = lane % LPR;
  float a0 = 0.f;
  for (int64_t s0 = warp * span; s0 < nidx; s0 += nw * span) {
    const int64_t s1 = s0 + span < nidx ? s0 + span : nidx;
    const int nb = static_cast<int>((s1 - s0 + U - 1) / U);
    auto issue = [&](int k) {
      if (k < nb) {
        const int d = k % D;
        const int64_t p0 = s0 + static_cast<int64_t>(k) * U;
        const int my = (lane < U && p0 + lane < s1) ? __ldg(idx + p0 + lane) : 0;
#pragma unroll
        for (int u = 0; u < U; u += RPI) {
          const int e = __shfl_sync(0xffffffffu, my, u + sub);
          const bool hot = e < 0;
          const uint32_t r = static_cast<uint32_t>(e) & 0x7fffffffu;
          const float* src = B + static_cast<int64_t>(r) * 128 + col0 + 4 * chunk;
          const uint32_t dst =
              static_cast<uint32_t>(__cvta_generic_to_shared(ring + (d * U + u + sub) * RB + 16 * chunk));
          if (MODE == 1) {
            const uint64_t pol = hot ? pl : pf;
            asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2;" ::"r"(dst), "l"(src),
                         "l"(pol) : "memory");
          } else if (MODE == 2) {  // the .ca form (L1 + L2) with the hint
            const uint64_t pol = hot ? pl : pf;
            asm volatile("cp.async.ca.shared.global.L2::cache_hint [%0], [%1], 16, %2;" ::"r"(dst), "l"(src),
                         "l"(pol) : "memory");
          } else {
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
          }
        }
      }
      asm volatile("cp.async.commit_group;" ::: "memory");
    };
    for (int k = 0; k < D - 1; ++k) issue(k);
    for (int k = 0; k < nb; ++k) {
      issue(k + D - 1);
      asm volatile("cp.async.wait_group %0;" ::"n"(D - 1) : "memory");
      __syncwarp();
      const int d = k % D;
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const float* row = reinterpret_cast<const float*>(ring + (d * U + u) * RB);
        if (VEC == 4) {
          const float4 v = reinterpret_cast<const float4*>(row)[lane];
          a0 += v.x + v.y + v.z + v.w;
        } else if (VEC == 2) {
          const float2 v = reinterpret_cast<const float2*>(row)[lane];
          a0 += v.x + v.y;
        } else {
          a0 += row[lane];
        }
      }
      __syncwarp();
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
  }
  if (a0 == 1234.5f) sink[0] = a0;
}

extern "C" float l2hot_probe_ldgsts(const float* B, const int* idx, int64_t nidx, int mode, int vec, int U, int D,
                                    int span, int warps_per_sm, int reps, float* sink, void* flush,
                                    int64_t flush_bytes) {
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int smem = 8 * D * U * 128 * vec;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  RepStat st(reps);
  const int grid = sms * (warps_per_sm / 8);
  const int w = 32 * vec;
#define KB(UU, DD, VV, MM) probe_ldgsts<UU, DD, VV, MM>
#define SETA(UU, DD, VV, MM) cudaFuncSetAttribute(KB(UU, DD, VV, MM), cudaFuncAttributeMaxDynamicSharedMemorySize, smem)
#define RUN(UU, DD, VV, MM) KB(UU, DD, VV, MM)<<<grid, 256, smem>>>(B, idx, nidx, span, c0, sink)
#define ALL(X, MM)                                          \
  if (vec == 2 && U == 8 && D == 4) X(8, 4, 2, MM);        \
  else if (vec == 2 && U == 8 && D == 3) X(8, 3, 2, MM);   \
  else if (vec == 2 && U == 16 && D == 2) X(16, 2, 2, MM); \
  else if (vec == 4 && U == 4 && D == 4) X(4, 4, 4, MM);   \
  else if (vec == 4 && U == 8 && D == 2) X(8, 2, 4, MM);   \
  else if (vec == 4 && U == 4 && D == 6) X(4, 6, 4, MM);   \
  else if (vec == 4 && U == 4 && D == 2) X(4, 2, 4, MM);   \
  else X(8, 2, 2, MM);
  if (mode == 1) { ALL(SETA, 1) } else if (mode == 2) { ALL(SETA, 2) } else { ALL(SETA, 0) }
  for (int r = 0; r < reps + 1; ++r) {
    cudaDeviceSynchronize();
    if (flush) cudaMemsetAsync(flush, r & 0xff, flush_bytes);
    cudaEventRecord(e0);
    for (int c0 = 0; c0 < 128; c0 += w) {
      if (mode == 1) { ALL(RUN, 1) } else if (mode == 2) { ALL(RUN, 2) } else { ALL(RUN, 0) }
    }
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    st.add(r, ms);
  }
#undef ALL
#undef RUN
#undef SETA
#undef KB
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  const cudaError_t err = cudaGetLastError();
  return err == cudaSuccess ? st.result() : -static_cast<float>(err);
}

// Hot rows pinned ahead of a plain (hint-free) LDGSTS ring: one pass puts every
// line of the hot rows in L2 with evict_last priority (prefetch with a
// policy), the ring runs, then a pass demotes them to evict_normal (so the
// next launch's L2 flush really flushes them).
__global__ void pin_rows(const float* __restrict__ B, const int* __restrict__ rows, int64_t n, int demote) {
  uint64_t pl;
  asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pl));
  const int64_t lines = n * 4;  // 512-byte rows = 4 lines
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < lines;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const float* a = B + static_cast<int64_t>(rows[i >> 2]) * 128 + (i & 3) * 32;
    if (demote) asm volatile("applypriority.global.L2::evict_normal [%0], 128;" ::"l"(a) : "memory");
    else asm volatile("prefetch.global.L2::evict_last [%0];" ::"l"(a) : "memory");
  }
}

extern "C" float l2hot_probe_pinned(const float* B, const int* idx, int64_t nidx, const int* hot_rows, int64_t nhot,
                                    int U, int D, int span, int warps_per_sm, int reps, float* sink, void* flush,
                                    int64_t flush_bytes, float* pin_ms) {
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int smem = 8 * D * U * 512;
  const int grid = sms * (warps_per_sm / 8);
  auto k = (U == 8 && D == 2) ? probe_ldgsts<8, 2, 4, 0> : probe_ldgsts<4, 4, 4, 0>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaEvent_t e0, e1, e2;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventCreate(&e2);
  float best = 1e30f, bpin = 0;
  for (int r = 0; r < reps + 1; ++r) {
    cudaDeviceSynchronize();
    if (flush) cudaMemsetAsync(flush, r & 0xff, flush_bytes);
    cudaEventRecord(e0);
    if (nhot > 0) pin_rows<<<sms * 4, 256>>>(B, hot_rows, nhot, 0);
    cudaEventRecord(e1);
    k<<<grid, 256, smem>>>(B, idx, nidx, span, 0, sink);
    if (nhot > 0) pin_rows<<<sms * 4, 256>>>(B, hot_rows, nhot, 1);
    cudaEventRecord(e2);
    cudaEventSynchronize(e2);
    float ms = 0, p = 0;
    cudaEventElapsedTime(&ms, e0, e2);
    cudaEventElapsedTime(&p, e0, e1);
    if (r >= 1 && ms < best) {
      best = ms;
      bpin = p;
    }
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaEventDestroy(e2);
  if (pin_ms) *pin_ms = bpin;
  const cudaError_t err = cudaGetLastError();
  return err == cudaSuccess ? best : -static_cast<float>(err);
}

// TMA gather4 ring (round 2): B rows (512 B, N = 128) fetched four at a time
// by one elected lane with cp.async.bulk.tensor.2d.tile::gather4 into a
// per-warp shared-memory ring (S stages x G gather4 = 4G rows per stage),
// mbarrier completion.  MODE 1: the gather4 carries an L2 cache hint --
// evict_last when any of its 4 rows is hot, evict_first otherwise.
#include <cuda.h>
#include <cudaTypedefs.h>

template <int S, int G, int MODE>
__global__ void __launch_bounds__(256, 1) probe_tma(const __grid_constant__ CUtensorMap tm, const int* __restrict__ idx,
                                                  int64_t nidx, int span, float* sink) {
  extern __shared__ __align__(128) unsigned char smraw[];
  constexpr int RB = 512, STAGE = G * 4 * RB;
  __shared__ __align__(8) uint64_t bar[8][S];
  __shared__ __align__(16) int scratch[8][4 * G];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  unsigned char* ring = smraw + wib * S * STAGE;
  const int64_t warp = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  uint64_t pl, pf, pn;
  asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pl));
  asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pf));
  asm("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(pn));
  if (lane < S) {
    const uint32_t b = static_cast<uint32_t>(__cvta_generic_to_shared(&bar[wib][lane]));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b));
  }
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncwarp();
  uint32_t phase = 0;
  float a0 = 0.f;
  constexpr int PER = 4 * G;
  for (int64_t s0 = warp * span; s0 < nidx; s0 += nw * span) {
    const int64_t s1 = s0 + span < nidx ? s0 + span : nidx;
    const int nb = static_cast<int>((s1 - s0) / PER);  // whole stages only (the tail is skipped: a probe)
    auto issue = [&](int k) {
      if (MODE >= 2 || k >= nb || lane != 0) return;  // grouped modes: issue_grouped
      const int d = k % S;
      const uint32_t b = static_cast<uint32_t>(__cvta_generic_to_shared(&bar[wib][d]));
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(STAGE) : "memory");
      const int* ip = idx + s0 + static_cast<int64_t>(k) * PER;
#pragma unroll
      for (int g = 0; g < G; ++g) {
        const int e0 = __ldg(ip + 4 * g), e1 = __ldg(ip + 4 * g + 1), e2 = __ldg(ip + 4 * g + 2),
                  e3 = __ldg(ip + 4 * g + 3);
        const uint32_t dst = static_cast<uint32_t>(__cvta_generic_to_shared(ring + d * STAGE + g * 4 * RB));
        const int r0 = e0 & 0x7fffffff, r1 = e1 & 0x7fffffff, r2 = e2 & 0x7fffffff, r3 = e3 & 0x7fffffff;
        if (MODE == 1) {
          const uint64_t pol = (e0 | e1 | e2 | e3) < 0 ? pl : pf;
          asm volatile(
              "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes.L2::cache_hint"
              " [%0], [%1, {%2, %3, %4, %5, %6}], [%7], %8;" ::"r"(dst),
              "l"(reinterpret_cast<uint64_t>(&tm)), "r"(0), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(b), "l"(pol)
              : "memory");
        } else {
          asm volatile(
              "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes"
              " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(dst),
              "l"(reinterpret_cast<uint64_t>(&tm)), "r"(0), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(b)
              : "memory");
        }
      }
    };
    // window grouping (what a kernel can do): the stage's PER positions
    // regrouped hot-first into its gather4s -- lanes < PER each take one
    // position, a ballot gives each its slot, the row indices go through a
    // per-warp scratch to the issuing lane; the consumer would read slot
    // sigma(u) for position u.  All-hot group: evict_last; all-cold:
    // evict_first; mixed: evict_first (MODE 2) / evict_normal (MODE 3).
    auto issue_grouped = [&](int k) {
      if (k >= nb) return;
      const int d = k % S;
      const int* ip = idx + s0 + static_cast<int64_t>(k) * PER;
      const int e = lane < PER ? __ldg(ip + lane) : 0;
      const unsigned hm = __ballot_sync(0xffffffffu, lane < PER && e < 0);
      const int nh = __popc(hm);
      const unsigned lt = (1u << lane) - 1u;
      const int slot = (e < 0) ? __popc(hm & lt) : nh + __popc(~hm & lt & ((1u << PER) - 1u));
      if (lane < PER) scratch[wib][slot] = e & 0x7fffffff;
      __syncwarp();
      if (lane == 0) {
        const uint32_t b = static_cast<uint32_t>(__cvta_generic_to_shared(&bar[wib][d]));
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(STAGE) : "memory");
#pragma unroll
        for (int g = 0; g < G; ++g) {
          const int4 rr = *reinterpret_cast<const int4*>(&scratch[wib][4 * g]);
          const uint32_t dst = static_cast<uint32_t>(__cvta_generic_to_shared(ring + d * STAGE + g * 4 * RB));
          const int hot_in = min(max(nh - 4 * g, 0), 4);
          // MODE 4: the grouping alone (every group evict_normal) -- its cost
          const uint64_t pol =
              MODE == 4 ? pn : hot_in == 4 ? pl : hot_in == 0 ? pf : (MODE == 2 ? pf : pn);
          asm volatile(
              "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes.L2::cache_hint"
              " [%0], [%1, {%2, %3, %4, %5, %6}], [%7], %8;" ::"r"(dst),
              "l"(reinterpret_cast<uint64_t>(&tm)), "r"(0), "r"(rr.x), "r"(rr.y), "r"(rr.z), "r"(rr.w), "r"(b),
              "l"(pol)
              : "memory");
        }
      }
      __syncwarp();
    };
    if (MODE >= 2) {
      for (int k = 0; k < S - 1; ++k) issue_grouped(k);
    }
    for (int k = 0; k < S - 1; ++k) issue(k);
    for (int k = 0; k < nb; ++k) {
      if (MODE >= 2) issue_grouped(k + S - 1);
      else issue(k + S - 1);
      const int d = k % S;
      const uint32_t b = static_cast<uint32_t>(__cvta_generic_to_shared(&bar[wib][d]));
      const uint32_t par = (phase >> d) & 1u;
      uint32_t done = 0;
      while (!done)
        asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                     : "=r"(done) : "r"(b), "r"(par) : "memory");
      phase ^= 1u << d;
#pragma unroll
      for (int u = 0; u < PER; ++u) {
        const float4 v = reinterpret_cast<const float4*>(ring + d * STAGE + u * RB)[lane];
        a0 += v.x + v.y + v.z + v.w;
      }
      __syncwarp();
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
  }
  if (a0 == 1234.5f) sink[0] = a0;
}

extern "C" float l2hot_probe_tma(const float* B, int64_t K, const int* idx, int64_t nidx, int mode, int S, int G,
                                 int warps_per_sm, int span, int reps, float* sink, void* flush, int64_t flush_bytes) {
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", reinterpret_cast<void**>(&encode), cudaEnableDefault, &q) !=
          cudaSuccess || !encode)
    return -1.f;
  CUtensorMap tm;
  cuuint64_t dims[2] = {128, static_cast<cuuint64_t>(K)};
  cuuint64_t strides[1] = {128 * 4};
  cuuint32_t box[2] = {128, 1};
  cuuint32_t es[2] = {1, 1};
  if (encode(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(B), dims, strides, box, es,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return -3.f;
  const int smem = 8 * S * G * 4 * 512;
  const int grid = sms * (warps_per_sm / 8);
#define TMA_ALL(X)                                   \
  if (S == 4 && G == 1) { X(4, 1) }                  \
  else if (S == 3 && G == 2) { X(3, 2) }             \
  else if (S == 2 && G == 2) { X(2, 2) }             \
  else if (S == 6 && G == 1) { X(6, 1) }             \
  else if (S == 2 && G == 4) { X(2, 4) }             \
  else if (S == 3 && G == 4) { X(3, 4) }             \
  else return -2.f;
#define TMA_SET(a, b)                                                                                        \
  cudaFuncSetAttribute(probe_tma<a, b, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);              \
  cudaFuncSetAttribute(probe_tma<a, b, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);              \
  cudaFuncSetAttribute(probe_tma<a, b, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);              \
  cudaFuncSetAttribute(probe_tma<a, b, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);              \
  cudaFuncSetAttribute(probe_tma<a, b, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
#define TMA_RUN(a, b)                                                                              \
  if (mode == 1) probe_tma<a, b, 1><<<grid, 256, smem>>>(tm, idx, nidx, span, sink);              \
  else if (mode == 2) probe_tma<a, b, 2><<<grid, 256, smem>>>(tm, idx, nidx, span, sink);         \
  else if (mode == 3) probe_tma<a, b, 3><<<grid, 256, smem>>>(tm, idx, nidx, span, sink);         \
  else if (mode == 4) probe_tma<a, b, 4><<<grid, 256, smem>>>(tm, idx, nidx, span, sink);         \
  else probe_tma<a, b, 0><<<grid, 256, smem>>>(tm, idx, nidx, span, sink);
  TMA_ALL(TMA_SET)
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  RepStat st(reps);
  for (int r = 0; r < reps + 1; ++r) {
    cudaDeviceSynchronize();
    if (flush) cudaMemsetAsync(flush, r & 0xff, flush_bytes);
    cudaEventRecord(e0);
    TMA_ALL(TMA_RUN)
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    st.add(r, ms);
  }
#undef TMA_ALL
#undef TMA_SET
#undef TMA_RUN
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  const cudaError_t err = cudaGetLastError();
  return err == cudaSuccess ? st.result() : -static_cast<float>(err);
}
