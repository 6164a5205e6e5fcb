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
//   MAX : m = v*b (rounded, unfused); acc = maximumNumber(acc, m), seeded
//         with the canonical NaN (maximumNumber's identity) or C0
//   MIN : same with minimumNumber
//   maximumNumber/minimumNumber are IEEE 754-2019 5.3.1 as the B200's FMNMX
//   implements them (measured, tools/mnmx_probe.cu): a NaN operand is ignored,
//   two NaNs give the canonical NaN 0x7fffffff, and -0 < +0.  That makes
//   max/min a function of the row's message multiset -- no fold order --
//   so a row folds two messages per 3-input FMNMX3 and products pair up in
//   FMUL2, and segments/partials combine in any order.  An all-NaN row gives
//   0x7fffffff; an empty row gives 0 (accumulate: C0, unchanged).
//   later long-row segments start from the identity (0 / NaN) and are
//   combined left to right: SUM/MEAN acc + part, MAX/MIN maxnum(acc, part).
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

// Blackwell packed fp32 multiply (FMUL2): two independent RN products v*b0,
// v*b1 -- bit-identical to two __fmul_rn.
__device__ __forceinline__ void mul2_rn(float& m0, float& m1, float v, float b0, float b1) {
  uint64_t r, bb, vv;
  asm("mov.b64 %0, {%1, %2};" : "=l"(bb) : "f"(b0), "f"(b1));
  asm("mov.b64 %0, {%1, %1};" : "=l"(vv) : "f"(v));
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(vv), "l"(bb));
  asm("mov.b64 {%0, %1}, %2;" : "=f"(m0), "=f"(m1) : "l"(r));
}

// maximumNumber / minimumNumber (FMNMX / FMNMX3)
__device__ __forceinline__ float maxnum(float a, float b) {
  float r;
  asm("max.f32 %0, %1, %2;" : "=f"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ float maxnum3(float a, float b, float c) {
  float r;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
  return r;
}
__device__ __forceinline__ float minnum(float a, float b) {
  float r;
  asm("min.f32 %0, %1, %2;" : "=f"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ float minnum3(float a, float b, float c) {
  float r;
  asm("min.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
  return r;
}

template <gespmm_reduce_t OP>
struct Semiring;

template <>
struct Semiring<GESPMM_REDUCE_SUM> {
  static constexpr bool kSeedC0 = true;   // accumulate: the chain starts at C0
  static constexpr bool kFma2 = true;     // update() is a plain FMA: pairs -> FFMA2
  static constexpr bool kMnmx = false;
  __device__ __forceinline__ static float zero() { return 0.0f; }
  __device__ __forceinline__ static float identity() { return 0.0f; }
  __device__ __forceinline__ static float chain_seed() { return -0.0f; }  // chain B: exact identity
  __device__ __forceinline__ static float update(float acc, float v, float b) {
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
  static constexpr bool kFma2 = true;
  static constexpr bool kMnmx = false;
  __device__ __forceinline__ static float zero() { return 0.0f; }
  __device__ __forceinline__ static float identity() { return 0.0f; }
  __device__ __forceinline__ static float chain_seed() { return -0.0f; }  // chain B: exact identity
  __device__ __forceinline__ static float update(float acc, float v, float b) {
    return __fmaf_rn(v, b, acc);
  }
  __device__ __forceinline__ static float combine(float acc, float part) {
    return __fadd_rn(acc, part);
  }
  __device__ __forceinline__ static float finalize(float acc, int deg, bool accumulate, float c0) {
#ifdef GESPMM_ABL_MEANMUL  // ablation builds only: the division's cost
#ifndef GESPMM_EXPERIMENT_BUILD
#error "GESPMM_ABL_MEANMUL gives wrong results: tagged experiment builds only (GESPMM_BUILD_TAG)"
#endif
    float r = deg ? acc * static_cast<float>(deg) : 0.0f;
#else
    float r = deg ? __fdiv_rn(acc, static_cast<float>(deg)) : 0.0f;
#endif
    return accumulate ? __fadd_rn(c0, r) : r;
  }
};

template <bool MAX>
struct SemiringMnmx {
  static constexpr bool kSeedC0 = true;
  static constexpr bool kFma2 = false;
  static constexpr bool kMnmx = true;  // two messages per FMNMX3, products in FMUL2
  __device__ __forceinline__ static float identity() { return __int_as_float(0x7fffffff); }
  __device__ __forceinline__ static float zero() { return identity(); }
  __device__ __forceinline__ static float chain_seed() { return identity(); }
  __device__ __forceinline__ static float pick(float a, float b) { return MAX ? maxnum(a, b) : minnum(a, b); }
  __device__ __forceinline__ static float pick3(float a, float b, float c) {
    return MAX ? maxnum3(a, b, c) : minnum3(a, b, c);
  }
  __device__ __forceinline__ static float update(float acc, float v, float b) {
    return pick(acc, __fmul_rn(v, b));
  }
  __device__ __forceinline__ static float combine(float acc, float part) { return pick(acc, part); }
  __device__ __forceinline__ static float finalize(float acc, int deg, bool accumulate, float) {
    return (deg == 0 && !accumulate) ? 0.0f : acc;
  }
};

template <>
struct Semiring<GESPMM_REDUCE_MAX> : SemiringMnmx<true> {};
template <>
struct Semiring<GESPMM_REDUCE_MIN> : SemiringMnmx<false> {};

}  // namespace gespmm
