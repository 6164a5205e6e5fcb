// gespmm_kernel.cuh -- the B200 GE-SpMM kernel family (sm_100a), instantiated
// per reduce op in gespmm_spmm_<op>.cu.
//
// What it computes: C[i, j] = reduce_{p in row i} val[p] * B[col[p], j]
// (reference kernel /root/reference/proj/fixtures/gespmm_alg2.mir:21-69;
// reduce functors in gespmm_semiring.cuh: sum/mean as two ascending FMA
// chains, max/min as the order-free maximumNumber/minimumNumber).
//
// How:
//  * One warp per work item.  An item is either a TILE of consecutive short
//    rows (deg <= kSeg, ~kTileWork work units: nnz-balanced) or one kSeg-long
//    SEGMENT of a long row.  Items come from the plan (gespmm_plan.cu).
//  * Coalesced Row Caching: the warp copies the item's whole colind/vals span
//    (<= kStageCap nonzeros) into its slice of shared memory with 16-byte
//    cp.async per lane (fully coalesced, no register cost, one commit/wait),
//    plus the tile's rowptr window; each lane then pre-scales (col -> col*ldb)
//    and pad-zeroes the entries its own copy delivered.  One __syncwarp()
//    publishes the stage -- the warp-scoped form of the reference's staging
//    barrier (gespmm_alg2.mir:36); another at the top of the next item orders
//    the stage reads before the refill (the reference's second barrier,
//    mir:65).  Certified by the reference's race checker
//    (oracle/models/gespmm_b200_stage.model).
//  * Persistent warps walk the work list (an atomic counter per column block
//    for large plans, a warp stride for small ones); a segment runs
//    through the same pipeline as a one-row tile (one code path: the kernel
//    must stay inside the instruction cache).
//  * Coarse-grained Warp Merging: each lane owns VEC consecutive columns in each
//    of CWM column tiles, so one staged (col, val) pair feeds VEC*CWM FMAs and
//    every B-row gather is one fully coalesced 32*VEC*4-byte warp access.
//  * Gather pipeline: B-row gathers are issued in batches of U = 8 nonzeros
//    (12 for sum at N=64) into one register buffer (16-24 registers at N=64;
//    32 warps/SM at 64 registers), then folded; at one column per lane (N <= 32 tiles) runs of
//    16 in-row positions are gathered at once.  The memory-level parallelism
//    this buffer allows is the kernel's bound (tools/gather_probe.cu: the
//    gather-only replay of the same stream at the same MLP takes ~90 % of
//    the kernel's time).  TMA gather4 reaches only 3-7 TB/s for 256-byte rows,
//    so the gathers stay in LDG.  At 512-byte rows (N=128 tiles) the B rows
//    instead go through a per-warp shared-memory ring with cp.async (Ring<>),
//    which wins where the gathers miss L2.
//  * Rows inside a tile are reduced sequentially in ascending p.  A batch that
//    lies inside the current row is folded check-free; a batch that crosses a
//    row end stores finished rows (streaming stores) and steps empty rows.
//  * Long-row segments publish a partial; the last segment to finish (atomic
//    ticket) combines all partials strictly in segment order and writes C, so
//    the result is deterministic and needs no second launch.
#pragma once

#include <type_traits>

#include "gespmm_internal.h"
#include "gespmm_semiring.cuh"

namespace gespmm {
namespace kern {

template <int VEC>
struct Vec;

template <>
struct Vec<1> {
  __device__ __forceinline__ static void ldg(float* d, const float* p) { d[0] = __ldg(p); }
  __device__ __forceinline__ static void ldcg(float* d, const float* p) { d[0] = __ldcg(p); }
  __device__ __forceinline__ static void ld(float* d, const float* p) { d[0] = *p; }
  __device__ __forceinline__ static void stcs(float* p, const float* s) { __stcs(p, s[0]); }
  __device__ __forceinline__ static void st(float* p, const float* s) { *p = s[0]; }
};

template <>
struct Vec<2> {
  __device__ __forceinline__ static void ldg(float* d, const float* p) {
    float2 v = __ldg(reinterpret_cast<const float2*>(p));
    d[0] = v.x, d[1] = v.y;
  }
  __device__ __forceinline__ static void ldcg(float* d, const float* p) {
    float2 v = __ldcg(reinterpret_cast<const float2*>(p));
    d[0] = v.x, d[1] = v.y;
  }
  __device__ __forceinline__ static void ld(float* d, const float* p) {
    float2 v = *reinterpret_cast<const float2*>(p);
    d[0] = v.x, d[1] = v.y;
  }
  __device__ __forceinline__ static void stcs(float* p, const float* s) {
    __stcs(reinterpret_cast<float2*>(p), make_float2(s[0], s[1]));
  }
  __device__ __forceinline__ static void st(float* p, const float* s) {
    *reinterpret_cast<float2*>(p) = make_float2(s[0], s[1]);
  }
};

template <>
struct Vec<4> {
  __device__ __forceinline__ static void ldg(float* d, const float* p) {
    float4 v = __ldg(reinterpret_cast<const float4*>(p));
    d[0] = v.x, d[1] = v.y, d[2] = v.z, d[3] = v.w;
  }
  __device__ __forceinline__ static void ldcg(float* d, const float* p) {
    float4 v = __ldcg(reinterpret_cast<const float4*>(p));
    d[0] = v.x, d[1] = v.y, d[2] = v.z, d[3] = v.w;
  }
  __device__ __forceinline__ static void ld(float* d, const float* p) {
    float4 v = *reinterpret_cast<const float4*>(p);
    d[0] = v.x, d[1] = v.y, d[2] = v.z, d[3] = v.w;
  }
  __device__ __forceinline__ static void stcs(float* p, const float* s) {
    __stcs(reinterpret_cast<float4*>(p), make_float4(s[0], s[1], s[2], s[3]));
  }
  __device__ __forceinline__ static void st(float* p, const float* s) {
    *reinterpret_cast<float4*>(p) = make_float4(s[0], s[1], s[2], s[3]);
  }
};

// A finished C row segment: the local store plus, for the fused all-gather,
// the same bytes into every peer's full C (P2P stores over NVLink, streaming).
// A compile-time switch (PEERS): the peer loop perturbs register allocation
// enough to cost 5-12 % when merely present, so only the fused-gather
// instantiations carry it.
template <int VEC, bool PEERS>
__device__ __forceinline__ void store_c(const KParams& P, float* dst, const float* o) {
  Vec<VEC>::stcs(dst, o);
  if constexpr (PEERS) {
    const int64_t off = (dst - P.C) + P.peer_shift;
    for (int q = 0; q < P.n_peers; ++q) Vec<VEC>::stcs(P.peers[q] + off, o);
  }
}

// One B-row gather: address = base + 4*off (one IMAD.WIDE.U32) and one
// non-coherent vector load.  `base` already includes the lane's column offset.
template <int VEC>
__device__ __forceinline__ void gather_off(float* d, const float* base, uint32_t off, uint64_t pol);
// GESPMM_BHINT=1: B gathers carry an L2 evict_last policy (keep B resident
// against the once-read colind/vals/C streams, which carry evict_first).
#ifndef GESPMM_BHINT
#define GESPMM_BHINT 1  // measured: +1.7% on config 2
#endif
// GESPMM_L1EV: L1 eviction priority of the B gathers (0 default allocate,
// 1 L1::no_allocate, 2 L1::evict_last, 3 L1::evict_first)
#ifndef GESPMM_L1EV
#define GESPMM_L1EV 0
#endif
#if GESPMM_L1EV == 1
#define GESPMM_L1Q ".L1::no_allocate"
#elif GESPMM_L1EV == 2
#define GESPMM_L1Q ".L1::evict_last"
#elif GESPMM_L1EV == 3
#define GESPMM_L1Q ".L1::evict_first"
#else
#define GESPMM_L1Q ""
#endif
// GESPMM_PF: L2 prefetch size qualifier of the B gathers (0 none, 1 .L2::128B,
// 2 .L2::256B)
#ifndef GESPMM_PF
#define GESPMM_PF 0
#endif
#if GESPMM_PF == 1
#define GESPMM_PFQ ".L2::128B"
#elif GESPMM_PF == 2
#define GESPMM_PFQ ".L2::256B"
#else
#define GESPMM_PFQ ""
#endif
#if GESPMM_BHINT
#define GESPMM_LDNC "ld.global.nc" GESPMM_L1Q ".L2::cache_hint" GESPMM_PFQ
#define GESPMM_POL(n) ", %" #n
#else
#define GESPMM_LDNC "ld.global.nc" GESPMM_L1Q GESPMM_PFQ
#define GESPMM_POL(n) ""
#endif
// address = base + 4 * off in one mad.wide.u32 (ptxas: LEA + LEA.HI.X; the
// single-IMAD.WIDE spelling measured no faster -- DESIGN.md 8.1)
#define GESPMM_ADDR(o, b) " .reg .u64 a;\n mad.wide.u32 a, %" #o ", 4, %" #b ";\n "
template <>
__device__ __forceinline__ void gather_off<1>(float* d, const float* base, uint32_t off, uint64_t pol) {
  asm("{\n" GESPMM_ADDR(1, 2) GESPMM_LDNC ".f32 %0, [a]" GESPMM_POL(3) ";\n}"
      : "=f"(d[0])
      : "r"(off), "l"(base), "l"(pol));
}
template <>
__device__ __forceinline__ void gather_off<2>(float* d, const float* base, uint32_t off, uint64_t pol) {
  asm("{\n" GESPMM_ADDR(2, 3) GESPMM_LDNC ".v2.f32 {%0, %1}, [a]" GESPMM_POL(4) ";\n}"
      : "=f"(d[0]), "=f"(d[1])
      : "r"(off), "l"(base), "l"(pol));
}
template <>
__device__ __forceinline__ void gather_off<4>(float* d, const float* base, uint32_t off, uint64_t pol) {
  asm("{\n" GESPMM_ADDR(4, 5) GESPMM_LDNC ".v4.f32 {%0, %1, %2, %3}, [a]" GESPMM_POL(6) ";\n}"
      : "=f"(d[0]), "=f"(d[1]), "=f"(d[2]), "=f"(d[3])
      : "r"(off), "l"(base), "l"(pol));
}
// GESPMM_SADDR=1: the batch loop reads the stage through one 32-bit shared
// address (stage entries and vals at immediate offsets) -- A/B knob
#ifndef GESPMM_SADDR
#define GESPMM_SADDR 1  // config 3 N=32: 1.271 -> 1.166 ms; configs 2/3-64 neutral
#endif
#ifndef GESPMM_MERGED_PAD
#define GESPMM_MERGED_PAD 1  // pad zeroing folded into the offset pre-scale pass
#endif
#ifndef GESPMM_FAST_VEC2
#define GESPMM_FAST_VEC2 0  // in-row fast batch at two columns per lane (0 = off)
#endif
#ifndef GESPMM_FAST_VEC1
#define GESPMM_FAST_VEC1 16  // in-row fast batch at one column per lane (0 = off)
#endif
__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t p;
  asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}

// 16-byte / 4-byte global->shared async copies (LDGSTS); the 16-byte form
// bypasses L1 for the once-read colind/vals stream.
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
#if GESPMM_BHINT
  asm volatile(
      "{\n .reg .b64 p;\n createpolicy.fractional.L2::evict_first.b64 p, 1.0;\n"
      " cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, p;\n}" ::"r"(
          static_cast<uint32_t>(__cvta_generic_to_shared(smem))),
      "l"(gmem)
      : "memory");
#else
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(
                   static_cast<uint32_t>(__cvta_generic_to_shared(smem))),
               "l"(gmem)
               : "memory");
#endif
}
// 16-byte cp.async of B-row bytes at element offset `off` from `base` (L2
// evict_last like the register gathers), bypassing L1.
#ifndef GESPMM_RING_HINT
#define GESPMM_RING_HINT 0  // no L2 hint: with one (1: policy operand, 2: createpolicy in the asm) some instantiations fault with cudaErrorIllegalInstruction at the LDGSTS (its desc operand came out as desc[UR1]); without it, configs 4/5 also run 2 % faster
#endif
__device__ __forceinline__ void cp_async16_b(void* smem, const float* base, uint32_t off, uint64_t pol) {
#if GESPMM_RING_HINT == 1
  asm volatile(
      "{\n .reg .u64 a;\n mad.wide.u32 a, %1, 4, %2;\n"
      " cp.async.cg.shared.global.L2::cache_hint [%0], [a], 16, %3;\n}" ::"r"(
          static_cast<uint32_t>(__cvta_generic_to_shared(smem))),
      "r"(off), "l"(base), "l"(pol)
      : "memory");
#elif GESPMM_RING_HINT == 2
  (void)pol;  // policy created next to its use
  asm volatile(
      "{\n .reg .u64 a;\n .reg .b64 p;\n mad.wide.u32 a, %1, 4, %2;\n"
      " createpolicy.fractional.L2::evict_last.b64 p, 1.0;\n"
      " cp.async.cg.shared.global.L2::cache_hint [%0], [a], 16, p;\n}" ::"r"(
          static_cast<uint32_t>(__cvta_generic_to_shared(smem))),
      "r"(off), "l"(base)
      : "memory");
#else
  (void)pol;
  asm volatile(
      "{\n .reg .u64 a;\n mad.wide.u32 a, %1, 4, %2;\n"
      " cp.async.cg.shared.global [%0], [a], 16;\n}" ::"r"(
          static_cast<uint32_t>(__cvta_generic_to_shared(smem))),
      "r"(off), "l"(base)
      : "memory");
#endif
}
// GESPMM_PIN=1: per-warp constants (the stage and ring shared addresses, the
// lane's B base) are pinned in registers; ptxas otherwise recomputes them
// from special registers and constants in every batch (config 5 ring: 85 ->
// 68 SASS instructions per batch of 4 nonzeros; config 2: ~19 of ~60 per
// batch of 8).
#ifndef GESPMM_PIN
#define GESPMM_PIN 1
#endif
#ifndef GESPMM_SPOS_SHFL
#define GESPMM_SPOS_SHFL 1
#endif
#ifndef GESPMM_RP_SHFL
#define GESPMM_RP_SHFL 1
#endif
#ifndef GESPMM_SEED_BRANCH
#define GESPMM_SEED_BRANCH 1
#endif
#ifndef GESPMM_SLOW_MASK
#define GESPMM_SLOW_MASK 1
#endif
#ifndef GESPMM_ITEM32
#define GESPMM_ITEM32 1
#endif
#ifndef GESPMM_RING_NOSYNC
#define GESPMM_RING_NOSYNC 1
#endif
#ifndef GESPMM_SLOW_MASK_U12
#define GESPMM_SLOW_MASK_U12 0
#endif
#ifndef GESPMM_SLOW_MASK_U4
#define GESPMM_SLOW_MASK_U4 0  // the ring's 4-row batches (512-byte rows) under the mask form (A/B)
#endif
// A value the compiler must keep in a register (an opaque move: it cannot be
// rematerialized from the special registers / constants it came from).
__device__ __forceinline__ uint32_t pin_reg(uint32_t x) {
  uint32_t y;
  asm volatile("mov.b32 %0, %1;" : "=r"(y) : "r"(x));
  return y;
}
template <typename T>
__device__ __forceinline__ T* pin_reg64(T* p) {
  uint64_t y;
  asm volatile("mov.b64 %0, %1;" : "=l"(y) : "l"(reinterpret_cast<uint64_t>(p)));
  return reinterpret_cast<T*>(y);
}
// The same copy to a 32-bit shared-window address (the ring).
__device__ __forceinline__ void cp_async16_s(uint32_t dst, const float* base, uint32_t off, uint64_t pol) {
  (void)pol;
  asm volatile(
      "{\n .reg .u64 a;\n mad.wide.u32 a, %1, 4, %2;\n"
      " cp.async.cg.shared.global [%0], [a], 16;\n}" ::"r"(dst),
      "r"(off), "l"(base)
      : "memory");
}
// VEC fp32 from a 32-bit shared-window address
template <int VEC>
__device__ __forceinline__ void lds_vec(float* d, uint32_t a);
template <>
__device__ __forceinline__ void lds_vec<1>(float* d, uint32_t a) {
  asm volatile("ld.shared.f32 %0, [%1];" : "=f"(d[0]) : "r"(a));
}
template <>
__device__ __forceinline__ void lds_vec<2>(float* d, uint32_t a) {
  asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(d[0]), "=f"(d[1]) : "r"(a));
}
template <>
__device__ __forceinline__ void lds_vec<4>(float* d, uint32_t a) {
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(d[0]), "=f"(d[1]), "=f"(d[2]), "=f"(d[3]) : "r"(a));
}
__device__ __forceinline__ void cp_async4(void* smem, const void* gmem) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(
                   static_cast<uint32_t>(__cvta_generic_to_shared(smem))),
               "l"(gmem)
               : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;" ::: "memory");
}

// Batch size U (a multiple of 4: the staged (col, val) pairs of a batch are
// read with 128-bit shared loads): 8 at <= 2 columns per lane, 4 at 4 or 8.
// One register buffer of U*VEC*CWM floats (two measured slower: they spill at
// the 64-register cap).
#ifndef GESPMM_U_NARROW
#define GESPMM_U_NARROW 8  // batch for <= 2 columns per lane
#endif
#ifndef GESPMM_ABL_NOSTORE
#define GESPMM_ABL_NOSTORE 0
#endif
#ifndef GESPMM_ABL_NOGATHER
#define GESPMM_ABL_NOGATHER 0
#endif
// the ablations skip the gathers / the C stores (wrong results by design): only
// tagged experiment builds (_build.py: GESPMM_BUILD_TAG -> libgespmm_<tag>.so,
// -DGESPMM_EXPERIMENT_BUILD) may set them, never the product library
#if (GESPMM_ABL_NOSTORE || GESPMM_ABL_NOGATHER) && !defined(GESPMM_EXPERIMENT_BUILD)
#error "GESPMM_ABL_NOSTORE/NOGATHER give wrong results: tagged experiment builds only (GESPMM_BUILD_TAG)"
#endif
// sum at two columns per lane (the 64-column tile) runs 12-row batches: 50 %
// more rows in flight for a 24-byte spill outside the batch loop -- config 4 /
// 5 at N=64 1.467 -> 1.416 / 26.3 -> 25.7 ms, config 2 0.335 -> 0.332 ms;
// max lost (0.338 -> 0.343 ms), so the other ops keep 8 (profiles/r2_pin/r2_c30_*)
#ifndef GESPMM_U_VEC4
#define GESPMM_U_VEC4 4  // register batch at four columns per lane (the ring runs that tile by default)
#endif
#ifndef GESPMM_U_SUM2
#define GESPMM_U_SUM2 12
#endif
template <int CPL, gespmm_reduce_t OP>
struct Pipe {
  static constexpr int U = CPL >= 8 ? 4 : CPL == 4 ? GESPMM_U_VEC4 : (CPL == 2 && OP == GESPMM_REDUCE_SUM) ? GESPMM_U_SUM2 : GESPMM_U_NARROW;
};

#ifndef GESPMM_MINBLOCKS
#define GESPMM_MINBLOCKS 4
#endif
// Min CTAs per SM for __launch_bounds__: caps registers so 32 warps/SM are
// resident; with two buffers in flight per warp that is ~128 KB of gathers
// per SM at N=64 (the L2 gather ceiling needs about that much).
// 8 columns per lane (N >= 256 tiles): 2 CTAs/SM, 106 registers, no spills
// (at 3 CTAs/SM the 80-register cap spilled 56-72 bytes: R-MAT 2^22 x N=256
// 7.29 -> 6.60 ms, 2^20 x 256 1.46 -> 1.32 ms)
#ifndef GESPMM_MINBLOCKS_WIDE
#define GESPMM_MINBLOCKS_WIDE 2
#endif
#ifndef GESPMM_MINBLOCKS_ONE
#define GESPMM_MINBLOCKS_ONE GESPMM_MINBLOCKS  // 1 column per lane (N <= 32 tiles)
#endif
#ifndef GESPMM_MINBLOCKS_VEC4
#define GESPMM_MINBLOCKS_VEC4 GESPMM_MINBLOCKS
#endif
template <int CPL>
struct MinBlocks {
  static constexpr int value =
      CPL >= 8 ? GESPMM_MINBLOCKS_WIDE : (CPL == 1 ? GESPMM_MINBLOCKS_ONE : CPL == 4 ? GESPMM_MINBLOCKS_VEC4 : GESPMM_MINBLOCKS);
};

// Ring mode (RING = true; DESIGN.md 5.2 "Gather ring"): B rows are copied
// into a per-warp shared-memory ring with 16-byte cp.async (no registers hold
// in-flight data) and read back with one LDS per lane per row.  kDepth
// batches of U rows are in flight per warp (~4 KB: U = 8 rows of 256 B at
// VEC = 2, U = 4 rows of 512 B at VEC = 4).  Measured ceiling on config 2's
// column stream (tools/gather_probe.cu): 0.248 ms at 24 warps/SM vs 0.311 ms
// for register gathers with 8 rows in flight at 32 warps/SM.
#ifndef GESPMM_RING_U512
#define GESPMM_RING_U512 4  // rows per ring batch at 512-byte rows
#endif
#ifndef GESPMM_RING_MINBLOCKS
#define GESPMM_RING_MINBLOCKS 3
#endif
#ifndef GESPMM_RING_DEPTH
#define GESPMM_RING_DEPTH 2  // ring batches (D - 1 in flight while one is folded); 3 measured slower (2 CTAs/SM)
#endif
template <int VEC, int CWM>
struct Ring {
  static constexpr int kRowBytes = 128 * VEC * CWM;     // one B row, the warp's columns
  static constexpr int kLanesPerRow = kRowBytes / 16;   // 16-byte chunks per row
  static constexpr int kRowsPerIssue = kLanesPerRow >= 32 ? 1 : 32 / kLanesPerRow;
  static constexpr int U = kRowBytes >= 512 ? GESPMM_RING_U512 : 8;
  static constexpr int kDepth = GESPMM_RING_DEPTH;
  static constexpr int kWarpBytes = kDepth * U * kRowBytes;
  static constexpr bool kSupported = CWM == 1 && VEC >= 2;  // N = 64 / 128 column tiles
};

template <gespmm_reduce_t OP, int VEC, int CWM, bool OFF32, bool RING, bool PEERS>
__global__ void __launch_bounds__(kWarpsPerBlock * 32, RING ? GESPMM_RING_MINBLOCKS : MinBlocks<VEC * CWM>::value)
    spmm_kernel(const KParams P) {
  using SR = Semiring<OP>;
  // sum/mean: two FMA chains per row (even/odd offsets from the row start),
  // held in accumulator slots by absolute position parity (batches are
  // 4-aligned, so the slot of batch element u is u & 1); value = slot0 + slot1
  // (fp32 addition is commutative, so it does not matter which slot holds the
  // even chain).  max/min: one chain in slot 0.
  constexpr bool TWO = SR::kFma2;
  constexpr int CPL = VEC * CWM;       // fp32 columns per lane
  constexpr int U = RING ? Ring<VEC, CWM>::U : Pipe<CPL, OP>::U;  // gathers per batch
  constexpr int FB = RING ? 0 : CPL == 1 ? GESPMM_FAST_VEC1 : CPL == 2 ? GESPMM_FAST_VEC2 : 0;  // in-row fast batch
  using RG = Ring<VEC, CWM>;
  static_assert(!RING || RG::kSupported, "ring mode: CWM == 1, VEC >= 2");
  constexpr int TW = 32 * VEC;         // columns per CWM tile
#if GESPMM_SADDR
  // one block per warp: colind slice, then vals slice (a fixed 4*kStageCap-byte
  // offset the batch loads take as an immediate)
  __shared__ __align__(16) int stg[kWarpsPerBlock][2 * kStageCap];
#else
  __shared__ __align__(16) int scol[kWarpsPerBlock][kStageCap];
  __shared__ __align__(16) float sval[kWarpsPerBlock][kStageCap];
#endif
  __shared__ int rpw[kWarpsPerBlock][kTileMaxRows + 4];

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int cb = blockIdx.y;
  const int64_t colbase = static_cast<int64_t>(cb) * (TW * CWM) + lane * VEC;
  // Lanes whose columns fall past N gather column 0 instead (always valid,
  // never stored): the gather loop carries no per-load predicate.
  bool cok[CWM];
  const float* bw[CWM];  // B + this lane's column offset, per CWM tile
  int woff[CWM];
#pragma unroll
  for (int w = 0; w < CWM; ++w) {
    // mean: woff pinned too (pin_reg) and cok derived from it -- config 2
    // mean 0.3745 -> 0.369 ms; for the other ops the extra live register
    // costs more than the rematerialization (sum 0.338 -> 0.343 ms)
    const bool ok = colbase + w * TW < P.N;
    woff[w] = ok ? static_cast<int>(colbase + w * TW) : -1;
    if (GESPMM_PIN && OP == GESPMM_REDUCE_MEAN) woff[w] = static_cast<int>(pin_reg(static_cast<uint32_t>(woff[w])));
    cok[w] = woff[w] >= 0;
    woff[w] = cok[w] ? woff[w] : 0;
    bw[w] = GESPMM_PIN ? pin_reg64(P.B + woff[w]) : P.B + woff[w];
  }
  // every lane of this column block has real columns (warp-uniform): the
  // per-lane guard (rematerialized by ptxas at every row end) is then skipped
  // -- config 2 sum / max 0.338 / 0.343 -> 0.334 / 0.338 ms; not at one column
  // per lane, where it cost config 3 N=32 1.151 -> 1.171 ms (profiles/r2_pin/)
  const bool all_ok = static_cast<int64_t>(cb + 1) * (TW * CWM) <= P.N;
  const int64_t ldb = P.ldb;
  // ring: this lane copies 16-byte chunk (lane % kLanesPerRow) of row
  // (lane / kLanesPerRow) of every kRowsPerIssue-row group; a chunk past N
  // copies column 0 (valid memory, never read back)
  extern __shared__ float4 ring_smem[];
  float4* const ring = ring_smem + warp * (RING ? RG::kWarpBytes / 16 : 0);
  const int rchunk = lane % RG::kLanesPerRow;
  const int rsub = RG::kLanesPerRow >= 32 ? 0 : lane / RG::kLanesPerRow;
  // the ring's 32-bit shared-window address, and B + this lane's column
  // inside a B row: each copy is then rsrc + 4*offset (one LEA pair)
  // (pinned in registers: ptxas otherwise recomputes them from special
  // registers and constants in every batch -- 6-12 instructions per batch)
  const uint32_t ring_s = RING ? pin_reg(static_cast<uint32_t>(__cvta_generic_to_shared(ring))) : 0u;
  const float* const rsrc = pin_reg64(P.B + [&] {
    const int64_t c = static_cast<int64_t>(cb) * TW + 4 * rchunk;
    return c < P.N ? c : 0;
  }());
#if GESPMM_SADDR
  int* const sc = stg[warp];
  float* const sv = reinterpret_cast<float*>(stg[warp] + kStageCap);
  // the stage's 32-bit shared-window address (pinned: see pin_reg)
  const uint32_t sc_s = GESPMM_PIN ? pin_reg(static_cast<uint32_t>(__cvta_generic_to_shared(sc)))
                                   : static_cast<uint32_t>(__cvta_generic_to_shared(sc));
#else
  int* const sc = scol[warp];
  float* const sv = sval[warp];
#endif
  int* const rp = rpw[warp];
  const bool accumulate = P.accumulate != 0;
  const bool seed_c0 = accumulate && SR::kSeedC0;

  float acc[2][CWM][VEC];
  // Row (segment) start: chain A -- the even offsets from `start` -- gets x
  // (or C0 when `src`), chain B gets -0.0, the exact additive identity.
  auto seed = [&](int start, float x, const float* src) {
    float c[CWM][VEC];
#pragma unroll
    for (int w = 0; w < CWM; ++w) {
      if (src) Vec<VEC>::ld(c[w], src + (woff[w] - woff[0]));
#pragma unroll
      for (int k = 0; k < VEC; ++k) {
        const float a = src ? c[w][k] : x;
        if (TWO) {
          const bool odd = start & 1;
          acc[0][w][k] = odd ? -0.0f : a;
          acc[1][w][k] = odd ? a : -0.0f;
        } else {
          acc[0][w][k] = a;
        }
      }
    }
  };
  // C rows are addressed through a running pointer (crow = C + row*ldc + the
  // lane's column), advanced by ldc per row: no 64-bit multiply per row.
  // a warp-uniform branch on the launch-wide accumulate flag, so the common
  // (no C0) path is the chain seeds alone (GESPMM_SEED_BRANCH); the select
  // form kept the C0 pointer test, the flag load and the predicated load at
  // every row end (sum only -- the other ops fold C0 in at the store: config
  // 2 sum 0.3211 -> 0.3158 ms, config 4 2.68 -> 2.64, config 3 N=64 -0.5 %;
  // profiles/r2_spos/summary_sb.txt)
  auto row_seed = [&](int start, const float* crow_) {
    if (GESPMM_SEED_BRANCH) {
      if (seed_c0) seed(start, SR::zero(), crow_);
      else seed(start, SR::zero(), nullptr);
    } else {
      seed(start, SR::zero(), seed_c0 ? crow_ : nullptr);
    }
  };
  auto value = [&](int w, int k) { return TWO ? acc[0][w][k] + acc[1][w][k] : acc[0][w][k]; };
  auto store_row = [&](float* dst, int deg) {
    if (GESPMM_ABL_NOSTORE) return;  // ablation builds only
#pragma unroll
    for (int w = 0; w < CWM; ++w) {
      if (!((CPL >= 2 && all_ok) || cok[w])) continue;
      float o[VEC];
      float c0[VEC];
      if (!SR::kSeedC0 && accumulate) Vec<VEC>::ld(c0, dst + (woff[w] - woff[0]));
#pragma unroll
      for (int k = 0; k < VEC; ++k)
        o[k] = SR::finalize(value(w, k), deg, accumulate, (!SR::kSeedC0 && accumulate) ? c0[k] : 0.f);
      store_c<VEC, PEERS>(P, dst + (woff[w] - woff[0]), o);
    }
  };
  const uint64_t bpol = GESPMM_BHINT ? policy_evict_last() : 0;
  auto gather = [&](float (&d)[CWM][VEC], int x) {
    if (GESPMM_ABL_NOGATHER) {  // ablation builds only
#pragma unroll
      for (int w = 0; w < CWM; ++w)
#pragma unroll
        for (int k = 0; k < VEC; ++k) d[w][k] = __int_as_float(x + k);
      return;
    }
#pragma unroll
    for (int w = 0; w < CWM; ++w) {
      if (OFF32) gather_off<VEC>(d[w], bw[w], static_cast<uint32_t>(x), bpol);
      else Vec<VEC>::ldg(d[w], bw[w] + static_cast<int64_t>(x) * ldb);
    }
  };

  // acc[slot] += v * b per the semiring; sum/mean column pairs go through
  // FFMA2 (Blackwell's packed fp32 FMA: two independent RN FMAs, bit-identical)
  auto fold = [&](int slot, float v, const float (&bb)[CWM][VEC]) {
    float (&a)[CWM][VEC] = acc[TWO ? slot : 0];
#pragma unroll
    for (int w = 0; w < CWM; ++w) {
      if (SR::kFma2 && VEC >= 2) {
#pragma unroll
        for (int k = 0; k < VEC; k += 2) fma2_rn(a[w][k], a[w][k + 1], v, bb[w][k], bb[w][k + 1]);
      } else {
#pragma unroll
        for (int k = 0; k < VEC; ++k) a[w][k] = SR::update(a[w][k], v, bb[w][k]);
      }
    }
  };
  // Two consecutive messages at once (sum/mean: the two chains; max/min: the
  // products in FMUL2 and one FMNMX3 per column -- the order-free fold).
  auto fold_pair = [&](float v0, const float (&b0)[CWM][VEC], float v1, const float (&b1)[CWM][VEC]) {
    if constexpr (SR::kMnmx) {
      float(&a)[CWM][VEC] = acc[0];
#pragma unroll
      for (int w = 0; w < CWM; ++w) {
        if constexpr (VEC >= 2) {
#pragma unroll
          for (int k = 0; k < VEC; k += 2) {
            float m0, m1, n0, n1;
            mul2_rn(m0, m1, v0, b0[w][k], b0[w][k + 1]);
            mul2_rn(n0, n1, v1, b1[w][k], b1[w][k + 1]);
            a[w][k] = SR::pick3(a[w][k], m0, n0);
            a[w][k + 1] = SR::pick3(a[w][k + 1], m1, n1);
          }
        } else {
          a[w][0] = SR::pick3(a[w][0], __fmul_rn(v0, b0[w][0]), __fmul_rn(v1, b1[w][0]));
        }
      }
    } else {
      fold(0, v0, b0);
      fold(1, v1, b1);
    }
  };

  // Persistent warps: warp-strided walk over the work list (no warp idles while
  // a sibling in its CTA finishes a longer item).  Control flow is warp-uniform
  // and the kernel uses no CTA-wide barrier.
  // Item indices fit 32 bits (a plan has < 2^29 items: nnz < 2^31 and a tile
  // holds >= 16 work units), so the item cursor, its bounds and the grabbed
  // index are 32-bit (GESPMM_ITEM32): fewer registers live across the item
  // (config 2 sum / max -0.9 / -0.6 %, config 3 N=16/32/64 -0.3/-1.2/-1.0 %;
  // mean lost 1.2 % and keeps 64-bit; profiles/r2_spos/summary_i32.txt)
  constexpr bool kItem32 = GESPMM_ITEM32 != 0 && OP != GESPMM_REDUCE_MEAN;
  using item_t = std::conditional_t<kItem32, int, int64_t>;
  using grab_t = std::conditional_t<kItem32, unsigned, unsigned long long>;
  const item_t wstride = static_cast<item_t>(gridDim.x) * kWarpsPerBlock;
  // the item count: on the device for plans built without a host sync
  const int64_t n_items = P.n_items_dev ? *P.n_items_dev : P.n_items;
  item_t t_begin = 0, t_end = static_cast<item_t>(n_items);
  // a failed on-device colind check earlier on the stream (host entry point,
  // single- or multi-chunk): no item is gathered through an invalid colind
  if (P.abort_flag && *reinterpret_cast<const volatile int*>(P.abort_flag)) return;
  if (P.range) {  // one chunk of the pipelined host path
    t_begin = static_cast<item_t>(P.range[0]);
    t_end = static_cast<item_t>(P.range[1]);
  }
  // Item distribution: dynamic when the launch carries a counter (P.work_ctr,
  // zeroed before the launch; one per column block): warps grab items with an
  // atomic, the next grab issued at the top of an item and consumed at its
  // end so its latency hides behind the item.  Static warp striding
  // otherwise (small launches, where the counter reset costs more than it
  // balances).  Measured dynamic vs static: config 2 0.371 -> 0.352 ms,
  // config 3 (N=64) 2.15 -> 1.81 ms, config 4 2.84 -> 2.65 ms, config 5
  // 57.5 -> 49.6 ms.
#define GESPMM_NEXT_ITEM                                                         \
  {                                                                              \
    t = dyn ? t_begin + static_cast<item_t>(__shfl_sync(0xffffffffu, next, 0)) : t + wstride; \
    continue;                                                                    \
  }
  const bool dyn = P.work_ctr != nullptr;
  unsigned long long* const wctr = dyn ? P.work_ctr + blockIdx.y : nullptr;
  auto grab = [&]() {
    grab_t v = 0;
    if (lane == 0) v = static_cast<grab_t>(atomicAdd(wctr, 1ULL));
    return v;
  };
  item_t t = dyn ? t_begin + static_cast<item_t>(__shfl_sync(0xffffffffu, grab(), 0))
                 : t_begin + static_cast<item_t>(blockIdx.x) * kWarpsPerBlock + warp;
  for (; t < t_end;) {
    const grab_t next = dyn ? grab() : grab_t(0);
    __syncwarp();  // the previous item's stage reads are done (the role of mir:65)
    const int4 it = P.items[t];
    const bool is_tile = it.y < 0;
    // ---- item decode: nonzero span [lo, hi) and its rows --------------------
    // A segment is run as a one-row tile whose row ends at the segment end.
    int lo, hi, nr, re_long = 0;
    if (is_tile) {
      int r1, pend;
      // the next item (the plan's sentinel {M, -1, nnz} after the last one)
      const int4 nx = P.items[t + 1];
      r1 = nx.x;
      pend = nx.z;
      nr = r1 - it.x;  // 1 <= nr <= kTileMaxRows (plan invariant)
      lo = it.z;
      hi = pend;
      for (int k = lane; k <= nr; k += 32) cp_async4(rp + k, P.rowptr + it.x + k);
    } else {
      nr = 1;
      lo = it.z + it.y * kSeg;
      re_long = __ldg(P.rowptr + it.x + 1);  // in flight while the stage copy is issued
      hi = min(lo + kSeg, P.nnz);  // copy bound; the segment end is applied below
    }
    // ---- CRC staging: colind/vals [sbase, hi) -> shared memory -------------
    // Batches start at 4-aligned positions sbase + k*U; entries in [sbase, lo)
    // are real neighbours (valid offsets, never folded) and the pad up to the
    // last batch end is zeroed below (offset 0: a valid row, never folded).
    const int sbase = lo & ~3;
    if (P.idx_aligned) {
      for (int e = sbase + 4 * lane; e < hi; e += 128) {
        if (e + 4 <= P.nnz) {
          cp_async16(sc + (e - sbase), P.colind + e);
          cp_async16(sv + (e - sbase), P.vals + e);
        } else {
          for (int q = e; q < P.nnz; ++q) {
            cp_async4(sc + (q - sbase), P.colind + q);
            cp_async4(sv + (q - sbase), P.vals + q);
          }
        }
      }
    } else {
      for (int e = sbase + lane; e < hi; e += 32) {
        cp_async4(sc + (e - sbase), P.colind + e);
        cp_async4(sv + (e - sbase), P.vals + e);
      }
    }
    // a segment's true end (its row's end) arrives while the copy is in flight
    // (entries copied past it are never folded: the pad and the batch bound
    // below stop at `hi`)
    if (!is_tile) hi = min(lo + kSeg, re_long);
    const int send = sbase + ((hi - sbase + U - 1) / U) * U;
    cp_async_wait_all();
    if (!P.idx_aligned) __syncwarp();  // 4-byte copies: other lanes own the entries
    if (OFF32 && GESPMM_MERGED_PAD) {
      // one pass: col -> B-row element offset col*ldb, and the pad [hi, send)
      // -> 0 (offset 0: a valid row, never folded; it overwrites whatever
      // neighbours cp.async brought in).  Each lane rewrites exactly the 4
      // entries its own 16-byte copy delivered (cp.async.wait_group orders
      // them for it), so with 16-byte staging no warp barrier is needed before this pass
      // (oracle/models/gespmm_b200_stage.model: copy and pre-scale share a
      // warp phase); the barrier after it publishes the stage.
      // The head [sbase, lo) -- up to 3 entries of the previous item, which a
      // chunked launch may not have transferred or validated yet -- is zeroed
      // the same way: a launch never gathers through an entry outside its
      // item.
      const uint32_t ldb32 = static_cast<uint32_t>(ldb);
      const int pad = hi - sbase, head = lo - sbase;
      auto keep = [&](int j) { return j >= head && j < pad; };
      for (int i = 4 * lane; i < send - sbase; i += 128) {
        int4 c = *reinterpret_cast<int4*>(sc + i);
        c.x = keep(i + 0) ? static_cast<int>(static_cast<uint32_t>(c.x) * ldb32) : 0;
        c.y = keep(i + 1) ? static_cast<int>(static_cast<uint32_t>(c.y) * ldb32) : 0;
        c.z = keep(i + 2) ? static_cast<int>(static_cast<uint32_t>(c.z) * ldb32) : 0;
        c.w = keep(i + 3) ? static_cast<int>(static_cast<uint32_t>(c.w) * ldb32) : 0;
        *reinterpret_cast<int4*>(sc + i) = c;
      }
      __syncwarp();
    } else {
      __syncwarp();
      // zero the pad [hi, send) (overwrites any neighbours cp.async brought in)
      // and the head [sbase, lo) (never gather through another item's entry)
      for (int i = hi - sbase + lane; i < send - sbase; i += 32) sc[i] = 0;
      if (lane < lo - sbase) sc[lane] = 0;
      __syncwarp();
      if (OFF32) {  // col -> B-row element offset col*ldb, once per staged entry
        const uint32_t ldb32 = static_cast<uint32_t>(ldb);
        for (int i = 4 * lane; i < send - sbase; i += 128) {
          int4 c = *reinterpret_cast<int4*>(sc + i);
          c.x = static_cast<int>(static_cast<uint32_t>(c.x) * ldb32);
          c.y = static_cast<int>(static_cast<uint32_t>(c.y) * ldb32);
          c.z = static_cast<int>(static_cast<uint32_t>(c.z) * ldb32);
          c.w = static_cast<int>(static_cast<uint32_t>(c.w) * ldb32);
          *reinterpret_cast<int4*>(sc + i) = c;
        }
        __syncwarp();
      }
    }

    // ---- row state ----------------------------------------------------------
    const int64_t grow0 = it.x;  // global row of local row 0
    const int64_t ldc = P.ldc;
    float* crow = P.C + grow0 * ldc + woff[0];
    // the rowptr window read through a 32-bit shared address that a shuffle
    // produced (GESPMM_RP_SHFL, >= 2 columns per lane): otherwise ptxas
    // rematerializes the window's address from SR_TID / SR_CgaCtaId at every
    // row end.  Config 2 sum / mean 0.3267 / 0.3670 -> 0.3221 / 0.3630 ms,
    // config 3 N=64 1.714 -> 1.710; at one column per lane (config 3 N=32)
    // and in the paired-lane kernel it lost 0.3-0.5 % (profiles/r2_spos/)
    const uint32_t rp_s = (GESPMM_RP_SHFL && CPL >= 2)
                              ? __shfl_sync(0xffffffffu, static_cast<uint32_t>(__cvta_generic_to_shared(rp)), 0)
                              : static_cast<uint32_t>(__cvta_generic_to_shared(rp));
    auto rp_at = [&](int k) {
      int x;
      asm volatile("ld.shared.s32 %0, [%1];" : "=r"(x) : "r"(rp_s + 4u * static_cast<uint32_t>(k)));
      return x;
    };
    int row = 0, rs = lo, re = is_tile ? rp_at(1) : hi;
    if (!is_tile && it.y > 0) seed(lo, SR::identity(), nullptr);
    else row_seed(lo, crow);

    // ---- gather pipeline over 4-aligned batches [qb, qb+U) ------------------
#if GESPMM_SADDR
    // 32-bit shared address of stage entry 0 relative to position 0
    // produced by a shuffle (GESPMM_SPOS_SHFL, >= 2 columns per lane), so
    // ptxas keeps it in a register instead of rematerializing it from SR_TID /
    // SR_CgaCtaId in every batch -- 10 instructions per batch of 12 at the
    // 64-column tile (the opaque mov on sc_s does not survive ptxas's copy
    // propagation).  Config 2 sum / max / mean 0.3316 / 0.3373 / 0.3697 ->
    // 0.3261 / 0.3347 / 0.3673 ms, config 3 N=64 1.740 -> 1.727, config 5
    // 52.23 -> 51.99; at one column per lane it lost (config 3 N=32 1.153 ->
    // 1.170 ms; profiles/r2_spos/)
    const uint32_t s_pos0 = (GESPMM_SPOS_SHFL && CPL >= 2)
                                ? __shfl_sync(0xffffffffu, sc_s - 4u * static_cast<uint32_t>(sbase), 0)
                                : sc_s - 4u * static_cast<uint32_t>(sbase);
#endif
    // the 4 staged offsets / values at positions qb + 4g .. qb + 4g + 3
    auto stage_off4 = [&](int qb, int g) {
      int4 o;
#if GESPMM_SADDR
      asm volatile("ld.shared.v4.s32 {%0, %1, %2, %3}, [%4];"
                   : "=r"(o.x), "=r"(o.y), "=r"(o.z), "=r"(o.w)
                   : "r"(s_pos0 + 4u * static_cast<uint32_t>(qb) + 16u * g));
#else
      o = reinterpret_cast<const int4*>(sc + (qb - sbase))[g];
#endif
      return o;
    };
    auto stage_val4 = [&](int qb, int g) {
      float4 x;
#if GESPMM_SADDR
      asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                   : "=f"(x.x), "=f"(x.y), "=f"(x.z), "=f"(x.w)
                   : "r"(s_pos0 + 4u * static_cast<uint32_t>(qb) + (4u * kStageCap + 16u * g)));
#else
      x = reinterpret_cast<const float4*>(sv + (qb - sbase))[g];
#endif
      return x;
    };
    // ring: copy batch qb into slot, one commit group per batch
    auto issue_ring = [&](int qb, int slot) {
      const uint32_t dst = ring_s + static_cast<uint32_t>((slot * U + rsub) * RG::kRowBytes + rchunk * 16);
      // the batch's offsets with 128-bit broadcast loads (no per-row LDS
      // latency chain); each lane then picks the row it copies
      int offs[U];
#pragma unroll
      for (int g = 0; g < U / 4; ++g) {
        const int4 o = stage_off4(qb, g);
        offs[4 * g] = o.x, offs[4 * g + 1] = o.y, offs[4 * g + 2] = o.z, offs[4 * g + 3] = o.w;
      }
      const uint64_t pol = policy_evict_last();
#pragma unroll
      for (int g = 0; g < U; g += RG::kRowsPerIssue) {
        int off = offs[g];
#pragma unroll
        for (int r = 1; r < RG::kRowsPerIssue; ++r) off = rsub == r ? offs[g + r] : off;
        cp_async16_s(dst + g * RG::kRowBytes, rsrc, static_cast<uint32_t>(off), pol);
      }
      asm volatile("cp.async.commit_group;" ::: "memory");
    };
    auto issue = [&](int qb, float (&b)[U][CWM][VEC]) {
#pragma unroll
      for (int g = 0; g < U / 4; ++g) {
        const int4 o = stage_off4(qb, g);
        gather(b[4 * g + 0], o.x);
        gather(b[4 * g + 1], o.y);
        gather(b[4 * g + 2], o.z);
        gather(b[4 * g + 3], o.w);
      }
    };
    auto ring_row = [&](int slot, int u, float (&d)[CWM][VEC]) {
      lds_vec<VEC>(d[0], ring_s + static_cast<uint32_t>((slot * U + u) * RG::kRowBytes + lane * VEC * 4));
    };
    auto consume = [&](int qb, const float (&b)[U][CWM][VEC]) {
      float v[U];
#pragma unroll
      for (int g = 0; g < U / 4; ++g) {
        const float4 x = stage_val4(qb, g);
        v[4 * g] = x.x, v[4 * g + 1] = x.y, v[4 * g + 2] = x.z, v[4 * g + 3] = x.w;
      }
      if (qb >= lo && qb + U <= min(hi, re)) {  // fast path: U nonzeros of the current row
#pragma unroll
        for (int u = 0; u < U; u += 2) fold_pair(v[u], b[u], v[u + 1], b[u + 1]);
        return;
      }
      if constexpr (GESPMM_SLOW_MASK && (U == 8 || (GESPMM_SLOW_MASK_U12 && U == 12) ||
                                        (GESPMM_SLOW_MASK_U4 && U == 4))) {
        // slow path by row runs: the batch's valid positions [u0, u1) split at
        // the row ends inside it; each run is folded under a bit mask of its
        // positions (predicated FFMA2s in position order), rows ending at or
        // before the run start are stored first.  One pass per row the batch
        // touches instead of a compare-and-branch chain per position: config
        // 2 max / mean 0.335 / 0.364 -> 0.328 / 0.348 ms, config 3 N=32 -0.4 %.
        // Not for sum's 12-row batches at the 64-column tile, where it adds
        // per-item spills (config 2 0.317 -> 0.311 ms, but config 3 N=64 /
        // 256 +3 / +3.5 %, config 5 at N=64 +3 %; profiles/r2_slowmask/).
        int u = max(lo - qb, 0);
        const int u1 = min(hi - qb, U);
        for (;;) {
          while (qb + u >= re) {  // rows ending at or before position qb + u are complete (tiles only)
            store_row(crow, re - rs);
            ++row;
            crow += ldc;
            rs = re;
            re = rp_at(row + 1);
            row_seed(rs, crow);
          }
          const int e = min(re - qb, u1);  // [u, e): the current row's run
          const unsigned m = ((1u << e) - 1u) & ~((1u << u) - 1u);
#pragma unroll
          for (int k = 0; k < U; ++k)
            if ((m >> k) & 1u) fold(k & 1, v[k], b[k]);
          if (e >= u1) break;
          u = e;
        }
      } else {
#pragma unroll
        for (int u = 0; u < U; ++u) {  // slow path: element by element
          const int p = qb + u;
          if (p < lo || p >= hi) continue;
          while (p >= re) {  // rows ending at or before p are complete (tiles only)
            store_row(crow, re - rs);
            ++row;
            crow += ldc;
            rs = re;
            re = rp_at(row + 1);
            row_seed(rs, crow);
          }
          fold(u & 1, v[u], b[u]);
        }
      }
    };
    if (RING && lo < hi) {
      constexpr int D = RG::kDepth;
      const int nb = (send - sbase) / U;
#pragma unroll
      for (int k = 0; k < D - 1; ++k) {  // prologue: D-1 batches in flight
        if (k < nb) issue_ring(sbase + k * U, k);
        else asm volatile("cp.async.commit_group;" ::: "memory");
      }
      for (int k = 0; k < nb; ++k) {
        if (k + D - 1 < nb) issue_ring(sbase + (k + D - 1) * U, (k + D - 1) % D);
        else asm volatile("cp.async.commit_group;" ::: "memory");
        asm volatile("cp.async.wait_group %0;" ::"n"(D - 1) : "memory");
        // At 512-byte rows (kLanesPerRow = 32) lane l copies and later reads
        // exactly bytes [16l, 16l + 16) of every row: its own wait_group
        // orders them and no other lane touches them, so the ring needs no
        // warp barrier (GESPMM_RING_NOSYNC); narrower rows map a lane's copy
        // and its read to different bytes and keep both barriers.  (Measured
        // neutral on the DRAM-bound configs 4/5, -0.3 to -0.6 % on config 4
        // sum/mean; racecheck clean: profiles/r2_ring_nosync/.)
        constexpr bool kOwn = GESPMM_RING_NOSYNC && RG::kLanesPerRow == 32 && RG::kRowsPerIssue == 1;
        if (!kOwn) __syncwarp();  // every lane's chunks of batch k are in the ring
        float ba[U][CWM][VEC];
#pragma unroll
        for (int u = 0; u < U; ++u) ring_row(k % D, u, ba[u]);
        consume(sbase + k * U, ba);
        if (!kOwn) __syncwarp();  // slot k % D is refilled at iteration k + 1
      }
    } else if (lo < hi) {
      {
        float ba[U][CWM][VEC];
        for (int qb = sbase; qb < hi; qb += U) {
          if constexpr (FB > 0) {
            // FB gathers in flight while the next FB positions lie inside the
            // current row (the bulk of long rows): FB/U times the MLP of the
            // U-batch without changing any row's fold order.  One column per
            // lane only: at 2 columns the extra buffer spills (measured
            // 0.386 vs 0.366 ms on config 2); at 1 column (N = 32) it wins
            // (config 3, N=32: 1.539 -> 1.306 ms).
            while (qb >= lo && qb + FB <= min(hi, re)) {
              float bf[FB > 0 ? FB : 4][CWM][VEC];
#pragma unroll
              for (int g = 0; g < FB / 4; ++g) {
                const int4 o = stage_off4(qb, g);
                gather(bf[4 * g + 0], o.x);
                gather(bf[4 * g + 1], o.y);
                gather(bf[4 * g + 2], o.z);
                gather(bf[4 * g + 3], o.w);
              }
#pragma unroll
              for (int g = 0; g < FB / 4; ++g) {
                const float4 x = stage_val4(qb, g);
                fold_pair(x.x, bf[4 * g + 0], x.y, bf[4 * g + 1]);
                fold_pair(x.z, bf[4 * g + 2], x.w, bf[4 * g + 3]);
              }
              qb += FB;
            }
            if (qb >= hi) break;
          }
          issue(qb, ba);
          consume(qb, ba);
        }
      }
    }

    if (is_tile) {
      // ---- the row in progress and any trailing empty rows -------------------
      for (;;) {
        store_row(crow, re - rs);
        if (++row >= nr) break;
        crow += ldc;
        rs = re;
        re = rp_at(row + 1);
        row_seed(rs, crow);
      }
      GESPMM_NEXT_ITEM;
    }
    // ---- long-row segment: publish the partial, then take a ticket -----------
    const int seg = it.y;
    const int slot = it.w;
    const int deg = re_long - it.z;
    const int nseg = (deg + kSeg - 1) / kSeg;
    float* part = P.partials + static_cast<int64_t>(slot + seg) * P.ldp;
#pragma unroll
    for (int w = 0; w < CWM; ++w)
      if (cok[w]) {
        float o[VEC];
#pragma unroll
        for (int k = 0; k < VEC; ++k) o[k] = value(w, k);
        Vec<VEC>::st(part + woff[w], o);
      }
#if GESPMM_TICKET_ACQREL
    // the warp's partial stores are ordered before lane 0's release by the
    // warp barrier; lane 0's acq_rel ticket releases them at gpu scope (and,
    // for the last segment, acquires the others') -- one lane, no full fence
    __syncwarp();
    int ticket = 0;
    int* counter = P.counters + static_cast<int64_t>(slot) * P.ncb + cb;
    if (lane == 0)
      asm volatile("atom.acq_rel.gpu.global.add.s32 %0, [%1], 1;" : "=r"(ticket) : "l"(counter) : "memory");
    ticket = __shfl_sync(0xffffffffu, ticket, 0);
    if (ticket != nseg - 1) GESPMM_NEXT_ITEM;
    __syncwarp();  // lane 0's acquire orders the whole warp's partial loads below
#else
    __threadfence();
    __syncwarp();
    int ticket = 0;
    int* counter = P.counters + static_cast<int64_t>(slot) * P.ncb + cb;
    if (lane == 0) ticket = atomicAdd(counter, 1);
    ticket = __shfl_sync(0xffffffffu, ticket, 0);
    if (ticket != nseg - 1) GESPMM_NEXT_ITEM;
#endif
    // last segment: combine all partials strictly left to right
    if (!GESPMM_TICKET_ACQREL) __threadfence();
    const float* base = P.partials + static_cast<int64_t>(slot) * P.ldp;
#pragma unroll
    for (int w = 0; w < CWM; ++w) {
      Vec<VEC>::ldcg(acc[0][w], base + woff[w]);
#pragma unroll
      for (int k = 0; k < VEC; ++k) acc[1][w][k] = -0.0f;  // value() = acc0 + -0 = acc0
    }
    constexpr int CU = 4;
    for (int s = 1; s < nseg; s += CU) {
      float pv[CU][CWM][VEC];
#pragma unroll
      for (int u = 0; u < CU; ++u) {
        const int ss = min(s + u, nseg - 1);
#pragma unroll
        for (int w = 0; w < CWM; ++w)
          Vec<VEC>::ldcg(pv[u][w], base + static_cast<int64_t>(ss) * P.ldp + woff[w]);
      }
#pragma unroll
      for (int u = 0; u < CU; ++u)
        if (s + u < nseg)
#pragma unroll
          for (int w = 0; w < CWM; ++w)
#pragma unroll
            for (int k = 0; k < VEC; ++k) acc[0][w][k] = SR::combine(acc[0][w][k], pv[u][w][k]);
    }
    store_row(crow, deg);
    if (lane == 0) *counter = 0;  // re-arm for the next launch (stream-ordered)
    t = dyn ? t_begin + static_cast<item_t>(__shfl_sync(0xffffffffu, next, 0)) : t + wstride;
  }  // item loop
#undef GESPMM_NEXT_ITEM
}

template <gespmm_reduce_t OP, int VEC, int CWM, bool OFF32, bool RING, bool PEERS = false>
cudaError_t launch_t(const KParams& p, cudaStream_t s) {
  int64_t blocks = (p.n_items + kWarpsPerBlock - 1) / kWarpsPerBlock;
  if (blocks == 0) return cudaSuccess;
  const int smem = RING ? kWarpsPerBlock * Ring<VEC, CWM>::kWarpBytes : 0;
  // persistent grid: every resident CTA slot once (per column block)
  static thread_local int cached_dev = -1, cached_slots = 0;
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev != cached_dev) {
    int sms = 0, per_sm = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (RING)
      cudaFuncSetAttribute(spmm_kernel<OP, VEC, CWM, OFF32, RING, PEERS>,
                           cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, spmm_kernel<OP, VEC, CWM, OFF32, RING, PEERS>,
                                                  kWarpsPerBlock * 32, smem);
    cached_slots = sms * (per_sm > 0 ? per_sm : 1);
    cached_dev = dev;
  }
  const int64_t slots = (cached_slots + p.ncb - 1) / p.ncb;
  if (blocks > slots) blocks = slots;
  dim3 grid(static_cast<unsigned>(blocks), static_cast<unsigned>(p.ncb), 1);
  spmm_kernel<OP, VEC, CWM, OFF32, RING, PEERS><<<grid, kWarpsPerBlock * 32, smem, s>>>(p);
  return cudaGetLastError();
}

template <gespmm_reduce_t OP, bool OFF32>
cudaError_t launch_off(const Variant& v, const KParams& p, cudaStream_t s) {
  // ring mode: 32-bit offsets, 16-byte aligned B rows, whole 16-byte chunks
  if (p.n_peers > 0) {  // fused all-gather: register-gather variants only
    if (v.vec == 4 && v.cwm == 2) return launch_t<OP, 4, 2, OFF32, false, true>(p, s);
    if (v.vec == 4 && v.cwm == 1) return launch_t<OP, 4, 1, OFF32, false, true>(p, s);
    if (v.vec == 2 && v.cwm == 2) return launch_t<OP, 2, 2, OFF32, false, true>(p, s);
    if (v.vec == 2 && v.cwm == 1) return launch_t<OP, 2, 1, OFF32, false, true>(p, s);
    if (v.vec == 1 && v.cwm == 2) return launch_t<OP, 1, 2, OFF32, false, true>(p, s);
    return launch_t<OP, 1, 1, OFF32, false, true>(p, s);
  }
  const bool ring = v.ring && OFF32 && p.ldb % 4 == 0 && p.N % 4 == 0 &&
                    reinterpret_cast<uintptr_t>(p.B) % 16 == 0;
  if (ring && v.vec == 4 && v.cwm == 1) return launch_t<OP, 4, 1, OFF32, true>(p, s);
  if (ring && v.vec == 2 && v.cwm == 1) return launch_t<OP, 2, 1, OFF32, true>(p, s);
  if (v.vec == 4 && v.cwm == 2) return launch_t<OP, 4, 2, OFF32, false>(p, s);
  if (v.vec == 4 && v.cwm == 1) return launch_t<OP, 4, 1, OFF32, false>(p, s);
  if (v.vec == 2 && v.cwm == 2) return launch_t<OP, 2, 2, OFF32, false>(p, s);
  if (v.vec == 2 && v.cwm == 1) return launch_t<OP, 2, 1, OFF32, false>(p, s);
  if (v.vec == 1 && v.cwm == 2) return launch_t<OP, 1, 2, OFF32, false>(p, s);
  return launch_t<OP, 1, 1, OFF32, false>(p, s);
}

template <gespmm_reduce_t OP>
cudaError_t launch_op(const Variant& v, const KParams& p, cudaStream_t s) {
  if (p.off32) return launch_off<OP, true>(v, p, s);
  return launch_off<OP, false>(v, p, s);
}

}  // namespace kern
}  // namespace gespmm
