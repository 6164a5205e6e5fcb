#include <cstdio>
#include <cstdint>
__global__ void k(const float* a, const float* b, const float* c, float* o2, float* o3, float* n2, int n) {
  int i = threadIdx.x + blockIdx.x * blockDim.x;
  if (i >= n) return;
  float r2, r3, rn;
  asm("max.f32 %0, %1, %2;" : "=f"(r2) : "f"(a[i]), "f"(b[i]));
  asm("max.f32 %0, %1, %2, %3;" : "=f"(r3) : "f"(a[i]), "f"(b[i]), "f"(c[i]));
  asm("min.f32 %0, %1, %2;" : "=f"(rn) : "f"(a[i]), "f"(b[i]));
  o2[i] = r2; o3[i] = r3; n2[i] = rn;
}
int main() {
  const int n = 16;
  uint32_t A[n] = {0x80000000u, 0x00000000u, 0x7fc00000u, 0x3f800000u, 0x7fc00001u, 0xffc00000u, 0x7f800001u, 0x80000000u,
                   0x00000000u, 0xff800000u, 0x7fc00000u, 0x80000000u, 0x3f800000u, 0x7fa00000u, 0, 0};
  uint32_t B[n] = {0x00000000u, 0x80000000u, 0x3f800000u, 0x7fc00000u, 0x7fc00002u, 0xffc00000u, 0x3f800000u, 0x80000000u,
                   0x00000000u, 0x7fc00000u, 0x80000000u, 0x7fc00000u, 0x7fa00000u, 0x7fa00000u, 0, 0};
  uint32_t C[n] = {0x80000000u, 0x80000000u, 0x7fc00000u, 0x7fc00000u, 0x7fc00000u, 0x7fc00000u, 0x7fc00000u, 0x00000000u,
                   0x80000000u, 0x7fc00000u, 0x7fc00000u, 0x7fc00000u, 0x7fc00000u, 0x7fa00000u, 0, 0};
  float *d; cudaMalloc(&d, 6 * n * 4);
  cudaMemcpy(d, A, n*4, cudaMemcpyHostToDevice); cudaMemcpy(d+n, B, n*4, cudaMemcpyHostToDevice); cudaMemcpy(d+2*n, C, n*4, cudaMemcpyHostToDevice);
  k<<<1, 32>>>(d, d+n, d+2*n, d+3*n, d+4*n, d+5*n, n);
  uint32_t O[3*n]; cudaMemcpy(O, d+3*n, 3*n*4, cudaMemcpyDeviceToHost);
  printf("err %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  for (int i = 0; i < 14; ++i) printf("a=%08x b=%08x c=%08x  max2=%08x max3=%08x min2=%08x\n", A[i], B[i], C[i], O[i], O[n+i], O[2*n+i]);
}
