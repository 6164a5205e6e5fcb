// gespmm_semiring.cuh -- the generalized reduce semiring as compile-time
// functors (BASELINE.json north star item (3)).
//
// The reference kernel has the SUM semiring only:
//   %prod = mul %vv, %b ; %c1 = add %c0, %prod     (gespmm_alg2.mir:54-58)
// evaluated in fp64 with separate roundings (reference src/oracle.cpp:599-604).
// The B200 path computes fp32 in the same per-cell order (p ascending) with an
// explicit FMA; MAX/MIN/MEAN are the north star's extension.  The host twin in
// oracle/gespmm_oracle.c spells out the same expressions, so results are
// bit-identical by construction:
//
//   SUM : acc = fma(v, b, acc)           seed 0 (accumulate: C0)
//   MEAN: SUM from 0, finalize acc/deg   (accumulate: C0 + acc/deg)
//   MAX : m = v*b (rounded, unfused); acc = first ? m : (m > acc ? m : acc)
//   MIN : same with <
//   later long-row segments start from the identity (0 / -inf / +inf) and are
//   combined left to right: SUM/MEAN acc + part, MAX/MIN better(part, acc).
#pragma once

#include <cuda_runtime.h>
#include <math_constants.h>

#include <cstdint>

#include "gespmm.h"

namespace gespmm {

// Blackwell packed fp32 FMA (FFMA2): two independent round-to-nearest FMAs
// a_i = fma(v, b_i, a_i) in one instruction -- bit-identical to two __fmaf_rn.
__device__ __forceinline__ void fma2_rn(float& a0, float& a1, float v, float b0, float b1) {
  uint64_t acc, bb, vv;
  asm("mov.b64 %0, {%1, %2};" : "=l"(acc) : "f"(a0), "f"(a1));
  asm("mov.b64 %0, {%1, %2};" : "=l"(bb) : "f"(b0), "f"(b1));
  asm("mov.b64 %0, {%1, %1};" : "=l"(vv) : "f"(v));
  asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(acc) : "l"(vv), "l"(bb));
  asm("mov.b64 {%0, %1}, %2;" : "=f"(a0), "=f"(a1) : "l"(acc));
}

template <gespmm_reduce_t OP>
struct Semiring;

template <>
struct Semiring<GESPMM_REDUCE_SUM> {
  static constexpr bool kSeedC0 = true;   // accumulate: the chain starts at C0
  static constexpr bool kFirstMsg = false;
  static constexpr bool kFma2 = true;     // update() is a plain FMA: pairs -> FFMA2
  __device__ __forceinline__ static float zero() { return 0.0f; }
  __device__ __forceinline__ static float identity() { return 0.0f; }
  __device__ __forceinline__ static float update(float acc, float v, float b, bool) {
    return __fmaf_rn(v, b, acc);
  }
  __device__ __forceinline__ static float combine(float acc, float part) {
    return __fadd_rn(acc, part);
  }
  __device__ __forceinline__ static float finalize(float acc, int, bool, float) { return acc; }
};

template <>
struct Semiring<GESPMM_REDUCE_MEAN> {
  static constexpr bool kSeedC0 = false;  // C0 is added after the division
  static constexpr bool kFirstMsg = false;
  static constexpr bool kFma2 = true;
  __device__ __forceinline__ static float zero() { return 0.0f; }
  __device__ __forceinline__ static float identity() { return 0.0f; }
  __device__ __forceinline__ static float update(float acc, float v, float b, bool) {
    return __fmaf_rn(v, b, acc);
  }
  __device__ __forceinline__ static float combine(float acc, float part) {
    return __fadd_rn(acc, part);
  }
  __device__ __forceinline__ static float finalize(float acc, int deg, bool accumulate, float c0) {
    float r = deg ? __fdiv_rn(acc, static_cast<float>(deg)) : 0.0f;
    return accumulate ? __fadd_rn(c0, r) : r;
  }
};

template <>
struct Semiring<GESPMM_REDUCE_MAX> {
  static constexpr bool kSeedC0 = true;
  static constexpr bool kFirstMsg = true;  // acc starts at the first message
  static constexpr bool kFma2 = false;
  __device__ __forceinline__ static float zero() { return 0.0f; }
  __device__ __forceinline__ static float identity() { return -CUDART_INF_F; }
  __device__ __forceinline__ static float better(float m, float acc) { return (m > acc) ? m : acc; }
  __device__ __forceinline__ static float update(float acc, float v, float b, bool first) {
    const float m = __fmul_rn(v, b);
    return first ? m : better(m, acc);
  }
  __device__ __forceinline__ static float combine(float acc, float part) {
    return better(part, acc);
  }
  __device__ __forceinline__ static float finalize(float acc, int deg, bool accumulate, float) {
    return (deg == 0 && !accumulate) ? 0.0f : acc;
  }
};

template <>
struct Semiring<GESPMM_REDUCE_MIN> {
  static constexpr bool kSeedC0 = true;
  static constexpr bool kFirstMsg = true;
  static constexpr bool kFma2 = false;
  __device__ __forceinline__ static float zero() { return 0.0f; }
  __device__ __forceinline__ static float identity() { return CUDART_INF_F; }
  __device__ __forceinline__ static float better(float m, float acc) { return (m < acc) ? m : acc; }
  __device__ __forceinline__ static float update(float acc, float v, float b, bool first) {
    const float m = __fmul_rn(v, b);
    return first ? m : better(m, acc);
  }
  __device__ __forceinline__ static float combine(float acc, float part) {
    return better(part, acc);
  }
  __device__ __forceinline__ static float finalize(float acc, int deg, bool accumulate, float) {
    return (deg == 0 && !accumulate) ? 0.0f : acc;
  }
};

}  // namespace gespmm
