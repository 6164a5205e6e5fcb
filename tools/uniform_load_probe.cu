// uniform_load_probe.cu -- L1 data-pipe cost of a warp-uniform (broadcast)
// read of staged (col, val) entries: shared LDS.32/64/128 vs L1-resident
// global LDG.128/256.  Each warp reads a small per-warp window repeatedly
// (every lane the same address), 32 warps/SM; the time per warp instruction
// per SM gives the pipe's cycles per instruction.
//
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/uniform_load_probe tools/uniform_load_probe.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

template <int MODE>
__global__ void __launch_bounds__(256, 4) probe(const int* __restrict__ g, int iters, int* sink) {
  __shared__ __align__(32) int s[8][256];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = lane; i < 256; i += 32) s[warp][i] = i;
  __syncwarp();
  // per-warp global window of 1 KB (L1 resident after the first pass)
  const int* gw = g + (static_cast<int64_t>(blockIdx.x) * 8 + warp) * 256;
  const uint32_t sa = static_cast<uint32_t>(__cvta_generic_to_shared(&s[warp][0]));
  int acc = 0;
  for (int it = 0; it < iters; ++it) {
    const int o = (it * 8) & 255;  // 32-byte steps through the window
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int oo = (o + 32 * k) & 255;
      if (MODE == 0) {  // LDS.32 broadcast
        int x;
        asm volatile("ld.shared.s32 %0, [%1];" : "=r"(x) : "r"(sa + 4u * oo));
        acc += x;
      } else if (MODE == 1) {  // LDS.64 broadcast
        int x, y;
        asm volatile("ld.shared.v2.s32 {%0, %1}, [%2];" : "=r"(x), "=r"(y) : "r"(sa + 4u * oo));
        acc += x ^ y;
      } else if (MODE == 2) {  // LDS.128 broadcast
        int x, y, z, w;
        asm volatile("ld.shared.v4.s32 {%0, %1, %2, %3}, [%4];" : "=r"(x), "=r"(y), "=r"(z), "=r"(w) : "r"(sa + 4u * oo));
        acc += x ^ y ^ z ^ w;
      } else if (MODE == 3) {  // LDG.128 uniform (L1)
        int x, y, z, w;
        asm volatile("ld.global.nc.v4.s32 {%0, %1, %2, %3}, [%4];" : "=r"(x), "=r"(y), "=r"(z), "=r"(w) : "l"(gw + oo));
        acc += x ^ y ^ z ^ w;
      } else if (MODE == 4) {  // LDG.256 uniform (L1)
        int a[8];
        asm volatile("ld.global.nc.v8.s32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
                     : "=r"(a[0]), "=r"(a[1]), "=r"(a[2]), "=r"(a[3]), "=r"(a[4]), "=r"(a[5]), "=r"(a[6]), "=r"(a[7])
                     : "l"(gw + oo));
        acc += a[0] ^ a[1] ^ a[2] ^ a[3] ^ a[4] ^ a[5] ^ a[6] ^ a[7];
      } else if (MODE == 5) {  // LDS.128, the two half-warps at different addresses
        int x, y, z, w;
        asm volatile("ld.shared.v4.s32 {%0, %1, %2, %3}, [%4];" : "=r"(x), "=r"(y), "=r"(z), "=r"(w) : "r"(sa + 4u * oo + 16u * (lane >> 4)));
        acc += x ^ y ^ z ^ w;
      } else if (MODE == 6) {  // LDG.128, half-warps at different 16-B granules of one line
        int x, y, z, w;
        asm volatile("ld.global.nc.v4.s32 {%0, %1, %2, %3}, [%4];" : "=r"(x), "=r"(y), "=r"(z), "=r"(w) : "l"(gw + oo + 4 * (lane >> 4)));
        acc += x ^ y ^ z ^ w;
      } else if (MODE == 7) {  // LDG.32 uniform
        int x;
        asm volatile("ld.global.nc.s32 %0, [%1];" : "=r"(x) : "l"(gw + oo));
        acc += x;
      }
    }
  }
  if (acc == 0x12345678) sink[0] = acc;
}

template <int MODE>
float run(const int* g, int blocks, int iters, int* sink) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  probe<MODE><<<blocks, 256>>>(g, 4, sink);
  cudaEventRecord(a);
  probe<MODE><<<blocks, 256>>>(g, iters, sink);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  return ms;
}

int main() {
  int sms = 0, clk = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const int blocks = sms * 4, iters = 20000;
  int *g, *sink;
  cudaMalloc(&g, static_cast<size_t>(blocks) * 8 * 256 * 4 + 64);
  cudaMemset(g, 1, static_cast<size_t>(blocks) * 8 * 256 * 4 + 64);
  cudaMalloc(&sink, 4);
  const double instr_per_sm = 4.0 * 8 * iters * 8;  // CTAs/SM x warps x iters x 8 loads
  const char* names[] = {"LDS.32 bcast", "LDS.64 bcast", "LDS.128 bcast", "LDG.128 uniform",
                         "LDG.256 uniform", "LDS.128 2-addr", "LDG.128 2-addr", "LDG.32 uniform"};
  float ms[8];
  ms[0] = run<0>(g, blocks, iters, sink);
  ms[1] = run<1>(g, blocks, iters, sink);
  ms[2] = run<2>(g, blocks, iters, sink);
  ms[3] = run<3>(g, blocks, iters, sink);
  ms[4] = run<4>(g, blocks, iters, sink);
  ms[5] = run<5>(g, blocks, iters, sink);
  ms[6] = run<6>(g, blocks, iters, sink);
  ms[7] = run<7>(g, blocks, iters, sink);
  for (int m = 0; m < 8; ++m) {
    const double cyc = ms[m] * 1e-3 * clk * 1e3;  // at the max clock
    std::printf("{\"mode\": \"%s\", \"ms\": %.3f, \"cycles_per_warp_instr_per_sm\": %.3f}\n", names[m], ms[m],
                cyc / instr_per_sm);
  }
  std::printf("{\"err\": \"%s\"}\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
