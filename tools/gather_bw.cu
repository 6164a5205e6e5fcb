// gather_bw.cu -- microbenchmark: the B200 ceiling for the SpMM's B-row gathers.
//
// Random rows of a [R x N] fp32 table (N = 64 -> 256-byte rows, the config-2
// gather unit) are fetched by
//   (a) LDG:  each warp keeps U independent 256-byte row loads in flight
//             (the register-based mechanism of gespmm_kernel.cuh), and
//   (b) TMA:  cp.async.bulk.tensor.2d.tile::gather4 -- 4 rows per instruction
//             into a per-warp shared-memory ring tracked by mbarriers; the warp
//             then reads its slice back (as the SpMM consumer would).
// Table sizes: L2-resident (16 MB) and HBM-sized (1 GB).  Prints one JSON line.
//
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/gather_bw tools/gather_bw.cu
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <cstdio>
#include <cstdlib>
#include <random>
#include <vector>

#define CK(x)                                                                   \
  do {                                                                          \
    cudaError_t e_ = (x);                                                       \
    if (e_ != cudaSuccess) {                                                    \
      fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); \
      exit(1);                                                                  \
    }                                                                           \
  } while (0)

constexpr int N = 64;

template <int U>
__global__ void __launch_bounds__(256) ldg_gather(const float* __restrict__ B, const int* __restrict__ idx,
                                                  int64_t nidx, float* sink) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  float a0 = 0.f, a1 = 0.f;
  for (int64_t base = warp * U; base + U <= nidx; base += nw * U) {
    const int my = (lane < U) ? __ldg(idx + base + lane) : 0;
    float2 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int r = __shfl_sync(0xffffffffu, my, u);
      v[u] = __ldg(reinterpret_cast<const float2*>(B + static_cast<int64_t>(r) * N) + lane);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      a0 += v[u].x;
      a1 += v[u].y;
    }
  }
  if (a0 == 1234.5f) sink[0] = a1;
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(static_cast<uint32_t>(__cvta_generic_to_shared(bar))),
               "r"(count));
}
__device__ __forceinline__ void mbar_expect(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(
                   static_cast<uint32_t>(__cvta_generic_to_shared(bar))),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  const uint32_t a = static_cast<uint32_t>(__cvta_generic_to_shared(bar));
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n}\n" ::"r"(a),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_gather4(void* dst, const CUtensorMap* tm, int col, int r0, int r1, int r2,
                                            int r3, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(static_cast<uint32_t>(__cvta_generic_to_shared(dst))),
      "l"(reinterpret_cast<uint64_t>(tm)), "r"(col), "r"(r0), "r"(r1), "r"(r2), "r"(r3),
      "r"(static_cast<uint32_t>(__cvta_generic_to_shared(bar)))
      : "memory");
}

// Per warp: S stages x G gather4 ops (4 rows of 256 B each) in a ring.
template <int WPB, int S, int G>
__global__ void __launch_bounds__(WPB * 32) tma_gather(const __grid_constant__ CUtensorMap tm,
                                                      const int* __restrict__ idx, int64_t nidx, float* sink) {
  extern __shared__ __align__(1024) unsigned char smem[];
  constexpr int STAGE_BYTES = G * 4 * N * 4;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  unsigned char* ring = smem + warp * S * STAGE_BYTES;
  __shared__ __align__(8) uint64_t bars[WPB][S];
  if (lane == 0)
    for (int s = 0; s < S; ++s) mbar_init(&bars[warp][s], 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncwarp();
  const int64_t gw = (static_cast<int64_t>(blockIdx.x) * WPB + warp);
  const int64_t nw = static_cast<int64_t>(gridDim.x) * WPB;
  constexpr int PER = G * 4;  // rows per stage
  const int64_t nsteps = nidx / PER;
  auto issue = [&](int64_t step, int s) {
    if (lane == 0) {
      mbar_expect(&bars[warp][s], STAGE_BYTES);
      const int* ip = idx + step * PER;
#pragma unroll
      for (int g = 0; g < G; ++g)
        tma_gather4(ring + s * STAGE_BYTES + g * 4 * N * 4, &tm, 0, __ldg(ip + 4 * g), __ldg(ip + 4 * g + 1),
                    __ldg(ip + 4 * g + 2), __ldg(ip + 4 * g + 3), &bars[warp][s]);
    }
  };
  float a0 = 0.f, a1 = 0.f;
  int64_t k = 0;
  // prologue
  for (int s = 0; s < S; ++s)
    if (gw + (k + s) * nw < nsteps) issue(gw + (k + s) * nw, s);
  uint32_t phase = 0;
  for (;; k += S) {
    bool any = false;
    for (int s = 0; s < S; ++s) {
      const int64_t step = gw + (k + s) * nw;
      if (step >= nsteps) break;
      any = true;
      mbar_wait(&bars[warp][s], phase);
      const float2* rows = reinterpret_cast<const float2*>(ring + s * STAGE_BYTES);
#pragma unroll
      for (int r = 0; r < PER; ++r) {
        float2 v = rows[r * (N / 2) + lane];
        a0 += v.x;
        a1 += v.y;
      }
      __syncwarp();
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      const int64_t nstep = gw + (k + s + S) * nw;
      if (nstep < nsteps) issue(nstep, s);
    }
    phase ^= 1;
    if (!any) break;
  }
  if (a0 == 1234.5f) sink[0] = a1;
}

int main() {
  int dev = 0, sms = 0;
  CK(cudaGetDevice(&dev));
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", reinterpret_cast<void**>(&encode), cudaEnableDefault, &q));
  const int64_t nidx = int64_t(1) << 24;  // 16M gathers x 256 B = 4.3 GB per pass
  float* sink;
  CK(cudaMalloc(&sink, 16));
  int* d_idx;
  CK(cudaMalloc(&d_idx, nidx * 4));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  printf("{\"sms\": %d, \"results\": [", sms);
  bool first = true;
  for (int64_t R : {int64_t(1) << 16, int64_t(1) << 20, int64_t(1) << 22}) {
    float* B;
    CK(cudaMalloc(&B, R * N * 4));
    CK(cudaMemset(B, 0, R * N * 4));
    std::vector<int> h(nidx);
    std::mt19937_64 rng(R);
    for (auto& x : h) x = static_cast<int>(rng() % R);
    CK(cudaMemcpy(d_idx, h.data(), nidx * 4, cudaMemcpyHostToDevice));
    CUtensorMap tm;
    cuuint64_t dims[2] = {N, static_cast<cuuint64_t>(R)};
    cuuint64_t strides[1] = {N * 4};
    cuuint32_t box[2] = {N, 1};
    cuuint32_t es[2] = {1, 1};
    CUresult cr = encode(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, B, dims, strides, box, es,
                         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                         CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (cr != CUDA_SUCCESS) {
      fprintf(stderr, "encode failed %d\n", cr);
      return 1;
    }
    auto timeit = [&](auto launch) {
      for (int w = 0; w < 2; ++w) launch();
      CK(cudaDeviceSynchronize());
      float best = 1e30f;
      for (int r = 0; r < 5; ++r) {
        CK(cudaEventRecord(e0));
        launch();
        CK(cudaEventRecord(e1));
        CK(cudaEventSynchronize(e1));
        float ms;
        CK(cudaEventElapsedTime(&ms, e0, e1));
        best = ms < best ? ms : best;
      }
      CK(cudaGetLastError());
      return static_cast<double>(nidx) * N * 4 / (best * 1e-3) / 1e9;
    };
    auto report = [&](const char* name, double gbs) {
      printf("%s{\"table_mb\": %lld, \"mech\": \"%s\", \"gbs\": %.1f}", first ? "" : ", ",
             static_cast<long long>(R * N * 4 >> 20), name, gbs);
      first = false;
      fflush(stdout);
    };
    report("ldg_u8_occ64", timeit([&] { ldg_gather<8><<<sms * 8, 256>>>(B, d_idx, nidx, sink); }));
    report("ldg_u16_occ64", timeit([&] { ldg_gather<16><<<sms * 8, 256>>>(B, d_idx, nidx, sink); }));
    {
      constexpr int WPB = 4, S = 4, G = 2;  // 8 KB/stage, 32 KB/warp, 128 KB/CTA
      const int sm = WPB * S * G * 4 * N * 4;
      CK(cudaFuncSetAttribute(tma_gather<WPB, S, G>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm));
      report("tma_g4_w4_s4_g2", timeit([&] { tma_gather<WPB, S, G><<<sms, WPB * 32, sm>>>(tm, d_idx, nidx, sink); }));
    }
    {
      constexpr int WPB = 8, S = 3, G = 2;  // 8 KB/stage, 24 KB/warp, 192 KB/CTA
      const int sm = WPB * S * G * 4 * N * 4;
      CK(cudaFuncSetAttribute(tma_gather<WPB, S, G>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm));
      report("tma_g4_w8_s3_g2", timeit([&] { tma_gather<WPB, S, G><<<sms, WPB * 32, sm>>>(tm, d_idx, nidx, sink); }));
    }
    {
      constexpr int WPB = 16, S = 2, G = 1;  // 4 KB/stage, 8 KB/warp, 128 KB/CTA
      const int sm = WPB * S * G * 4 * N * 4;
      CK(cudaFuncSetAttribute(tma_gather<WPB, S, G>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm));
      report("tma_g4_w16_s2_g1", timeit([&] { tma_gather<WPB, S, G><<<sms, WPB * 32, sm>>>(tm, d_idx, nidx, sink); }));
    }
    CK(cudaFree(B));
  }
  printf("]}\n");
  return 0;
}
