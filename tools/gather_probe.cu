// gather_probe.cu -- the gather-only ceiling for a given column stream.
//
// Replays idx[] (e.g. a CSR's colind) as 256-byte B-row gathers (N = 64 fp32)
// in the SpMM's order: each warp walks contiguous spans of `span` positions in
// batches of U loads in flight, warps grid-stride over spans.  Nothing else is
// read or written (no colind staging, no C), so the time is a lower bound for
// any kernel that gathers the same rows in the same order.
//
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -shared -Xcompiler -fPIC
//          -o tools/libgather_probe.so tools/gather_probe.cu
#include <cuda_runtime.h>

#include <cstdint>

template <int U>
__global__ void __launch_bounds__(256) probe(const float* __restrict__ B, const int* __restrict__ idx,
                                             int64_t nidx, int span, float* sink) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  float a0 = 0.f, a1 = 0.f;
  for (int64_t s0 = warp * span; s0 < nidx; s0 += nw * span) {
    const int64_t s1 = s0 + span < nidx ? s0 + span : nidx;
    for (int64_t base = s0; base < s1; base += U) {
      const int my = (lane < U && base + lane < s1) ? __ldg(idx + base + lane) : 0;
      float2 v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int r = __shfl_sync(0xffffffffu, my, u);
        v[u] = __ldg(reinterpret_cast<const float2*>(B + static_cast<int64_t>(r) * 64) + lane);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        a0 += v[u].x;
        a1 += v[u].y;
      }
    }
  }
  if (a0 == 1234.5f) sink[0] = a1;
}

// Paired variant: half-warps gather different rows with 16-byte loads (two
// 256-byte rows per warp instruction), U rows in flight per warp with the same
// registers as the 8-byte-per-lane variant -- separates a per-request limit
// from a per-byte one.
template <int U>
__global__ void __launch_bounds__(256) probe_pair(const float* __restrict__ B, const int* __restrict__ idx,
                                                  int64_t nidx, int span, float* sink) {
  const int lane = threadIdx.x & 31;
  const int half = lane >> 4;
  const int64_t warp = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  float a0 = 0.f, a1 = 0.f;
  for (int64_t s0 = warp * span; s0 < nidx; s0 += nw * span) {
    const int64_t s1 = s0 + span < nidx ? s0 + span : nidx;
    for (int64_t base = s0; base < s1; base += U) {
      const int my = (lane < U && base + lane < s1) ? __ldg(idx + base + lane) : 0;
      float4 v[U / 2];
#pragma unroll
      for (int u = 0; u < U / 2; ++u) {
        const int r = __shfl_sync(0xffffffffu, my, 2 * u + half);
        v[u] = __ldg(reinterpret_cast<const float4*>(B + static_cast<int64_t>(r) * 64) + (lane & 15));
      }
#pragma unroll
      for (int u = 0; u < U / 2; ++u) {
        a0 += v[u].x + v[u].z;
        a1 += v[u].y + v[u].w;
      }
    }
  }
  if (a0 == 1234.5f) sink[0] = a1;
}

extern "C" float gather_probe_pair(const float* B, const int* idx, int64_t nidx, int U, int span,
                                   int blocks_per_sm, int reps, float* sink, void* flush, int64_t flush_bytes) {
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e30f;
  for (int r = 0; r < reps + 2; ++r) {
    if (flush) cudaMemsetAsync(flush, r & 0xff, flush_bytes);
    cudaEventRecord(e0);
    const int grid = sms * blocks_per_sm;
    if (U == 16) probe_pair<16><<<grid, 256>>>(B, idx, nidx, span, sink);
    else if (U == 32) probe_pair<32><<<grid, 256>>>(B, idx, nidx, span, sink);
    else probe_pair<8><<<grid, 256>>>(B, idx, nidx, span, sink);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    if (r >= 2 && ms < best) best = ms;
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  return cudaGetLastError() == cudaSuccess ? best : -1.f;
}

// Ring variant: B rows land in a per-warp shared-memory ring with cp.async
// (16 B per lane, a half-warp per 256-byte row), D batches of U rows in
// flight, no registers held by in-flight data; consumed with 8-byte LDS.
template <int U, int D>
__global__ void __launch_bounds__(256) probe_ring(const float* __restrict__ B, const int* __restrict__ idx,
                                                  int64_t nidx, int span, float* sink) {
  extern __shared__ float4 sm[];
  const int lane = threadIdx.x & 31;
  float4* ring = sm + (threadIdx.x >> 5) * (D * U * 16);
  const int64_t warp = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  float a0 = 0.f, a1 = 0.f;
  for (int64_t s0 = warp * span; s0 < nidx; s0 += nw * span) {
    const int64_t s1 = s0 + span < nidx ? s0 + span : nidx;
    const int nb = static_cast<int>((s1 - s0 + U - 1) / U);
    auto load_idx = [&](int k) {
      const int64_t p = s0 + static_cast<int64_t>(k) * U + lane;
      return (k < nb && lane < U && p < s1) ? __ldg(idx + p) : 0;
    };
    auto issue = [&](int k, int my) {
      if (k < nb) {
        float4* slot = ring + (k % D) * U * 16;
#pragma unroll
        for (int u = 0; u < U; u += 2) {
          const int r = __shfl_sync(0xffffffffu, my, u + (lane >> 4));
          const float* src = B + static_cast<int64_t>(r) * 64 + (lane & 15) * 4;
          const uint32_t dst = static_cast<uint32_t>(__cvta_generic_to_shared(slot + (u + (lane >> 4)) * 16 + (lane & 15)));
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
        }
      }
      asm volatile("cp.async.commit_group;" ::: "memory");
    };
    int nxt = load_idx(0);
    for (int k = 0; k < D - 1; ++k) {
      const int my = nxt;
      nxt = load_idx(k + 1);
      issue(k, my);
    }
    for (int k = 0; k < nb; ++k) {
      const int my = nxt;
      nxt = load_idx(k + D);
      issue(k + D - 1, my);
      asm volatile("cp.async.wait_group %0;" ::"n"(D - 1) : "memory");
      __syncwarp();
      const float4* slot = ring + (k % D) * U * 16;
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const float2 v = reinterpret_cast<const float2*>(slot + u * 16)[lane];
        a0 += v.x;
        a1 += v.y;
      }
      __syncwarp();
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
  }
  if (a0 == 1234.5f) sink[0] = a1;
}

extern "C" float gather_probe_ring(const float* B, const int* idx, int64_t nidx, int U, int D, int span,
                                   int blocks_per_sm, int reps, float* sink, void* flush, int64_t flush_bytes) {
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int smem = 8 * D * U * 256;
  auto set = [&](auto k) { cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem); };
  set(probe_ring<8, 2>); set(probe_ring<8, 3>); set(probe_ring<8, 4>); set(probe_ring<16, 2>); set(probe_ring<4, 4>);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e30f;
  for (int r = 0; r < reps + 2; ++r) {
    if (flush) cudaMemsetAsync(flush, r & 0xff, flush_bytes);
    cudaEventRecord(e0);
    const int grid = sms * blocks_per_sm;
    if (U == 8 && D == 2) probe_ring<8, 2><<<grid, 256, smem>>>(B, idx, nidx, span, sink);
    else if (U == 8 && D == 3) probe_ring<8, 3><<<grid, 256, smem>>>(B, idx, nidx, span, sink);
    else if (U == 8 && D == 4) probe_ring<8, 4><<<grid, 256, smem>>>(B, idx, nidx, span, sink);
    else if (U == 16 && D == 2) probe_ring<16, 2><<<grid, 256, smem>>>(B, idx, nidx, span, sink);
    else probe_ring<4, 4><<<grid, 256, smem>>>(B, idx, nidx, span, sink);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    if (r >= 2 && ms < best) best = ms;
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  return cudaGetLastError() == cudaSuccess ? best : -1.f;
}

extern "C" float gather_probe(const float* B, const int* idx, int64_t nidx, int U, int span,
                              int blocks_per_sm, int reps, float* sink, void* flush, int64_t flush_bytes) {
  if (reps == 0) {  // one timed run, no warm-up (the caller prepared the cache state)
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    const int grid = sms * blocks_per_sm;
    if (U == 8) probe<8><<<grid, 256>>>(B, idx, nidx, span, sink);
    else if (U == 16) probe<16><<<grid, 256>>>(B, idx, nidx, span, sink);
    else probe<4><<<grid, 256>>>(B, idx, nidx, span, sink);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    return cudaGetLastError() == cudaSuccess ? ms : -1.f;
  }
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e30f;
  for (int r = 0; r < reps + 2; ++r) {
    if (flush) cudaMemsetAsync(flush, r & 0xff, flush_bytes);
    cudaEventRecord(e0);
    const int grid = sms * blocks_per_sm;
    if (U == 8) probe<8><<<grid, 256>>>(B, idx, nidx, span, sink);
    else if (U == 16) probe<16><<<grid, 256>>>(B, idx, nidx, span, sink);
    else probe<4><<<grid, 256>>>(B, idx, nidx, span, sink);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    if (r >= 2 && ms < best) best = ms;
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  return cudaGetLastError() == cudaSuccess ? best : -1.f;
}

// Bulk-copy ring (VERDICT r1 Next 4): each B row (256 B) moves with ONE
// single-lane cp.async.bulk (the TMA engine's non-tensor bulk copy) into a
// per-warp shared-memory ring, completion counted on a per-slot mbarrier
// (complete_tx::bytes) and awaited with mbarrier.try_wait.parity; lane u
// issues row u of a batch, so one warp instruction puts U rows in flight with
// no registers holding them.  D slots of U rows, W warps per CTA; consumed
// with one 8-byte LDS per lane per row.
template <int U, int D, int W>
__global__ void __launch_bounds__(W * 32) probe_bulk(const float* __restrict__ B, const int* __restrict__ idx,
                                                     int64_t nidx, int span, float* sink) {
  static_assert(U <= 32, "one lane per row");
  extern __shared__ __align__(128) unsigned char smraw[];
  __shared__ __align__(8) uint64_t bar[W][D];
  constexpr int RB = 256;
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  unsigned char* ring = smraw + wib * (D * U * RB);
  const int64_t warp = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  if (lane < D) {
    const uint32_t b = static_cast<uint32_t>(__cvta_generic_to_shared(&bar[wib][lane]));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b));
  }
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncwarp();
  uint32_t phase = 0;  // bit d: parity of slot d
  float a0 = 0.f, a1 = 0.f;
  for (int64_t s0 = warp * span; s0 < nidx; s0 += nw * span) {
    const int64_t s1 = s0 + span < nidx ? s0 + span : nidx;
    const int nb = static_cast<int>((s1 - s0 + U - 1) / U);
    auto rows_in = [&](int k) {
      const int64_t r = s1 - (s0 + static_cast<int64_t>(k) * U);
      return static_cast<int>(r < U ? r : U);
    };
    auto issue = [&](int k) {
      if (k >= nb) return;
      const int d = k % D;
      const uint32_t b = static_cast<uint32_t>(__cvta_generic_to_shared(&bar[wib][d]));
      const int nrow = rows_in(k);
      if (lane == 0)
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(nrow * RB) : "memory");
      __syncwarp();
      if (lane < nrow) {
        const int r = __ldg(idx + s0 + static_cast<int64_t>(k) * U + lane);
        const float* src = B + static_cast<int64_t>(r) * 64;
        const uint32_t dst = static_cast<uint32_t>(__cvta_generic_to_shared(ring + (d * U + lane) * RB));
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
                     "l"(src), "n"(RB), "r"(b)
                     : "memory");
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
      const int nrow = rows_in(k);
#pragma unroll 8
      for (int u = 0; u < nrow; ++u) {
        const float2 v = reinterpret_cast<const float2*>(ring + (d * U + u) * RB)[lane];
        a0 += v.x;
        a1 += v.y;
      }
      __syncwarp();  // slot d is refilled by issue(k + D)
    }
  }
  if (a0 == 1234.5f) sink[0] = a1;
}

// configs (U, D, warps per CTA); blocks_per_sm CTAs per SM
extern "C" float gather_probe_bulk(const float* B, const int* idx, int64_t nidx, int U, int D, int W, int span,
                                   int blocks_per_sm, int reps, float* sink, void* flush, int64_t flush_bytes) {
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int smem = W * D * U * 256;
#define GP_ALL(X)                                  \
  if (U == 16 && D == 2 && W == 8) X(16, 2, 8);    \
  else if (U == 16 && D == 3 && W == 8) X(16, 3, 8); \
  else if (U == 32 && D == 2 && W == 4) X(32, 2, 4); \
  else if (U == 8 && D == 4 && W == 8) X(8, 4, 8); \
  else if (U == 16 && D == 2 && W == 4) X(16, 2, 4); \
  else if (U == 32 && D == 2 && W == 8) X(32, 2, 8); \
  else return -2.f;
#define GP_SET(a, b, c) cudaFuncSetAttribute(probe_bulk<a, b, c>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem)
#define GP_RUN(a, b, c) probe_bulk<a, b, c><<<sms * blocks_per_sm, (c) * 32, smem>>>(B, idx, nidx, span, sink)
  GP_ALL(GP_SET)
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e30f;
  for (int r = 0; r < reps + 2; ++r) {
    if (flush) cudaMemsetAsync(flush, r & 0xff, flush_bytes);
    cudaEventRecord(e0);
    GP_ALL(GP_RUN)
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    if (r >= 2 && ms < best) best = ms;
  }
#undef GP_ALL
#undef GP_SET
#undef GP_RUN
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  const cudaError_t err = cudaGetLastError();
  return err == cudaSuccess ? best : -static_cast<float>(err);
}
