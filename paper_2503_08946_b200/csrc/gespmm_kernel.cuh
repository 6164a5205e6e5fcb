// gespmm_kernel.cuh -- the B200 GE-SpMM kernel family (sm_100a), instantiated
// per reduce op in gespmm_spmm_<op>.cu.
//
// What it computes: C[i, j] = reduce_{p in row i, ascending} val[p] * B[col[p], j]
// (reference kernel /root/reference/proj/fixtures/gespmm_alg2.mir:21-69;
// reduce functors in gespmm_semiring.cuh).
//
// How:
//  * One warp per work item.  An item is either a TILE of consecutive short
//    rows (deg <= kSeg, ~kTileWork work units: nnz-balanced) or one kSeg-long
//    SEGMENT of a long row.  Items come from the plan (gespmm_plan.cu).
//  * Coalesced Row Caching: the warp streams the item's nonzeros in chunks of
//    128: every lane issues ONE 128-bit load of colind and ONE of vals and
//    writes the pairs into the warp's slice of shared memory, with col already
//    scaled to the B-row element offset col*ldb; each pair is then read back
//    as a broadcast (one LDS.64 per nonzero).  __syncwarp() orders the stage
//    writes before the reads and the reads before the next refill -- the
//    warp-scoped form of the reference's two barriers (gespmm_alg2.mir:36, :65).
//    The next chunk is prefetched into registers while the current one is used.
//  * Coarse-grained Warp Merging: each lane owns VEC consecutive columns in each
//    of CWM column tiles, so one staged pair feeds VEC*CWM FMAs and every B-row
//    gather is one fully coalesced 32*VEC*4-byte warp access.  U gathers are
//    issued before the first is consumed (memory-level parallelism).
//  * Rows inside a tile are reduced sequentially in ascending p.  A batch of U
//    nonzeros that lies inside the current row takes the check-free fast path;
//    a batch that crosses a row end takes the slow path, which stores finished
//    rows (streaming stores) and steps through empty rows.
//  * Long-row segments publish a partial; the last segment to finish (atomic
//    ticket) combines all partials strictly in segment order and writes C, so
//    the result is deterministic and needs no second launch.
#pragma once

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

// Registers per lane: U gathers of VEC*CWM floats each in flight.
template <int CPL>
struct Unroll {
  static constexpr int U = CPL >= 8 ? 2 : (CPL >= 4 ? 4 : 8);
};

// Min CTAs per SM for __launch_bounds__: caps registers so >= 32 warps/SM are
// resident (latency hiding for the dependent index->gather chain).
#ifndef GESPMM_MINBLOCKS
#define GESPMM_MINBLOCKS 4
#endif
template <int CPL>
struct MinBlocks {
  static constexpr int value = CPL >= 8 ? 3 : GESPMM_MINBLOCKS;
};

template <gespmm_reduce_t OP, int VEC, int CWM, bool OFF32>
__global__ void __launch_bounds__(kWarpsPerBlock * 32, MinBlocks<VEC * CWM>::value)
    spmm_kernel(const KParams P) {
  using SR = Semiring<OP>;
  constexpr int CPL = VEC * CWM;       // fp32 columns per lane
  constexpr int U = Unroll<CPL>::U;    // gathers in flight per lane
  constexpr int TW = 32 * VEC;         // columns per CWM tile
  constexpr int RPV = (kTileMaxRows + 32) / 32;
  __shared__ __align__(16) int2 stage[kWarpsPerBlock][kChunk];
  __shared__ int rpw[kWarpsPerBlock][kTileMaxRows + 4];

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int64_t t = static_cast<int64_t>(blockIdx.x) * kWarpsPerBlock + warp;
  if (t >= P.n_items) return;  // warp-uniform; the kernel uses no CTA-wide barrier
  const int4 it = P.items[t];
  const int cb = blockIdx.y;
  const int64_t colbase = static_cast<int64_t>(cb) * (TW * CWM) + lane * VEC;
  // Lanes whose columns fall past N gather column 0 instead (always valid,
  // never stored): the gather loop carries no per-load predicate.
  bool cok[CWM];
  int woff[CWM];
#pragma unroll
  for (int w = 0; w < CWM; ++w) {
    cok[w] = colbase + w * TW < P.N;
    woff[w] = cok[w] ? static_cast<int>(colbase + w * TW) : 0;
  }
  const float* __restrict__ B = P.B;
  const int64_t ldb = P.ldb;
  int2* st = stage[warp];
  const bool accumulate = P.accumulate != 0;

  float acc[CWM][VEC];

  auto bptr = [&](int x) -> const float* {
    if (OFF32) return B + static_cast<uint32_t>(x);
    return B + static_cast<int64_t>(x) * ldb;
  };

  // -- CRC staging: lane l covers the 4 nonzeros at cbase + 4l (128-bit loads) --
  auto fetch = [&](int cbase, int lo, int hi, int4& c, float4& v) {
    const int e = cbase + 4 * lane;
    c = make_int4(0, 0, 0, 0);
    v = make_float4(0.f, 0.f, 0.f, 0.f);
    if (e < hi && e + 4 > lo) {
      if (P.idx_aligned && e + 4 <= P.nnz) {
        c = __ldcs(reinterpret_cast<const int4*>(P.colind + e));
        v = __ldcs(reinterpret_cast<const float4*>(P.vals + e));
      } else {
        int* cc = &c.x;
        float* vv = &v.x;
#pragma unroll
        for (int q = 0; q < 4; ++q)
          if (e + q < P.nnz && e + q >= lo && e + q < hi) {
            cc[q] = __ldcs(P.colind + e + q);
            vv[q] = __ldcs(P.vals + e + q);
          }
      }
    }
  };
  auto put = [&](const int4& c, const float4& v) {
    int4 o;
    if (OFF32) {  // pre-scale to the B-row element offset (fits 32 bits: K*ldb < 2^32)
      o = make_int4(static_cast<int>(static_cast<uint32_t>(c.x) * static_cast<uint32_t>(ldb)),
                    static_cast<int>(static_cast<uint32_t>(c.y) * static_cast<uint32_t>(ldb)),
                    static_cast<int>(static_cast<uint32_t>(c.z) * static_cast<uint32_t>(ldb)),
                    static_cast<int>(static_cast<uint32_t>(c.w) * static_cast<uint32_t>(ldb)));
    } else {
      o = c;
    }
    int4* s = reinterpret_cast<int4*>(st + 4 * lane);
    s[0] = make_int4(o.x, __float_as_int(v.x), o.y, __float_as_int(v.y));
    s[1] = make_int4(o.z, __float_as_int(v.z), o.w, __float_as_int(v.w));
  };

  // Gathers for staged positions [i0, i0+U) (stage-relative), unclamped.
  auto gather = [&](int i0, float (&vv)[U], float (&b)[U][CWM][VEC]) {
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int2 e = st[i0 + u];
      vv[u] = __int_as_float(e.y);
      const float* src = bptr(e.x);
#pragma unroll
      for (int w = 0; w < CWM; ++w) Vec<VEC>::ldg(b[u][w], src + woff[w]);
    }
  };
  // Same, with positions clamped to ilast (no predicate on the loads).
  auto gather_clamped = [&](int i0, int ilast, float (&vv)[U], float (&b)[U][CWM][VEC]) {
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int2 e = st[min(i0 + u, ilast)];
      vv[u] = __int_as_float(e.y);
      const float* src = bptr(e.x);
#pragma unroll
      for (int w = 0; w < CWM; ++w) Vec<VEC>::ldg(b[u][w], src + woff[w]);
    }
  };
  auto fold = [&](float v, const float (&b)[CWM][VEC], bool first) {
#pragma unroll
    for (int w = 0; w < CWM; ++w)
#pragma unroll
      for (int k = 0; k < VEC; ++k) acc[w][k] = SR::update(acc[w][k], v, b[w][k], first);
  };

  auto seed_row = [&](int64_t grow, bool seeded) {
    if (seeded) {
      const float* src = P.C + grow * P.ldc;
#pragma unroll
      for (int w = 0; w < CWM; ++w) Vec<VEC>::ld(acc[w], src + woff[w]);
    } else {
#pragma unroll
      for (int w = 0; w < CWM; ++w)
#pragma unroll
        for (int k = 0; k < VEC; ++k) acc[w][k] = SR::zero();
    }
  };
  auto store_row = [&](int64_t grow, int deg, const float (&r)[CWM][VEC]) {
    float* dst = P.C + grow * P.ldc;
#pragma unroll
    for (int w = 0; w < CWM; ++w) {
      if (!cok[w]) continue;
      float o[VEC];
      float c0[VEC];
      if (!SR::kSeedC0 && accumulate) Vec<VEC>::ld(c0, dst + woff[w]);
#pragma unroll
      for (int k = 0; k < VEC; ++k)
        o[k] = SR::finalize(r[w][k], deg, accumulate, (!SR::kSeedC0 && accumulate) ? c0[k] : 0.f);
      Vec<VEC>::stcs(dst + woff[w], o);
    }
  };

  if (it.y < 0) {
    // ---------------- tile of consecutive short rows [r0, r1) ----------------
    const int r0 = it.x;
    int r1, pend;
    if (t + 1 < P.n_items) {
      const int4 nx = P.items[t + 1];
      r1 = nx.x;
      pend = nx.z;
    } else {
      r1 = P.M;
      pend = P.nnz;
    }
    const int nr = r1 - r0;  // 1 <= nr <= kTileMaxRows (plan invariant)
    const int pbeg = it.z;
    int rpv[RPV];
#pragma unroll
    for (int i = 0; i < RPV; ++i) {
      const int k = lane + 32 * i;
      rpv[i] = (k <= nr) ? __ldg(P.rowptr + r0 + k) : 0;
    }
    int4 c;
    float4 v;
    fetch(pbeg & ~3, pbeg, pend, c, v);
    int* rp = rpw[warp];
#pragma unroll
    for (int i = 0; i < RPV; ++i) {
      const int k = lane + 32 * i;
      if (k <= nr) rp[k] = rpv[i];
    }
    __syncwarp();
    const bool seed = accumulate && SR::kSeedC0;
    int row = 0;
    int rs = pbeg;
    int re = rp[1];
    seed_row(r0, seed);
    // advance past every row that ends at or before position q
    auto advance_to = [&](int q) {
      while (q >= re) {
        store_row(r0 + row, re - rs, acc);
        ++row;
        rs = re;
        re = rp[row + 1];
        seed_row(r0 + row, seed);
      }
    };
    if (pbeg < pend) {
      int cbase = pbeg & ~3;
      while (true) {
        put(c, v);
        __syncwarp();
        const int nbase = cbase + kChunk;
        const bool more = nbase < pend;
        if (more) fetch(nbase, pbeg, pend, c, v);  // next chunk in flight during this one
        const int q1 = min(pend, nbase);
        for (int q = max(pbeg, cbase); q < q1; q += U) {
          float vv[U];
          float b[U][CWM][VEC];
          if (q + U <= q1 && q + U <= re) {
            // fast path: U nonzeros of the current row
            gather(q - cbase, vv, b);
            const bool first = SR::kFirstMsg && !accumulate && q == rs;
#pragma unroll
            for (int u = 0; u < U; ++u) fold(vv[u], b[u], first && u == 0);
          } else {
            // slow path: the batch crosses a row end or the chunk end
            gather_clamped(q - cbase, q1 - 1 - cbase, vv, b);
#pragma unroll
            for (int u = 0; u < U; ++u) {
              if (q + u < q1) {
                advance_to(q + u);
                fold(vv[u], b[u], SR::kFirstMsg && !accumulate && q + u == rs);
              }
            }
          }
        }
        __syncwarp();  // stage reads complete before the refill
        if (!more) break;
        cbase = nbase;
      }
    }
    for (;;) {  // the row in progress and any trailing empty rows
      store_row(r0 + row, re - rs, acc);
      if (++row >= nr) break;
      rs = re;
      re = rp[row + 1];
      seed_row(r0 + row, seed);
    }
  } else {
    // ---------------- one segment of a long row ------------------------------
    const int row = it.x;
    const int seg = it.y;
    const int rs = it.z;
    const int slot = it.w;
    const int ps = rs + seg * kSeg;
    int4 c;
    float4 v;
    fetch(ps & ~3, ps, ps + kSeg, c, v);  // issued before rowptr[row+1] returns
    const int re = __ldg(P.rowptr + row + 1);
    const int pe = min(ps + kSeg, re);
    const int deg = re - rs;
    const int nseg = (deg + kSeg - 1) / kSeg;
    if (seg == 0) {
      seed_row(row, accumulate && SR::kSeedC0);
    } else {
#pragma unroll
      for (int w = 0; w < CWM; ++w)
#pragma unroll
        for (int k = 0; k < VEC; ++k) acc[w][k] = SR::identity();
    }
    const bool first0 = SR::kFirstMsg && !accumulate && seg == 0;
    int cbase = ps & ~3;
    while (true) {
      put(c, v);
      __syncwarp();
      const int nbase = cbase + kChunk;
      const bool more = nbase < pe;
      if (more) fetch(nbase, ps, pe, c, v);
      const int q1 = min(pe, nbase);
      int q = max(ps, cbase);
      for (; q + U <= q1; q += U) {
        float vv[U];
        float b[U][CWM][VEC];
        gather(q - cbase, vv, b);
#pragma unroll
        for (int u = 0; u < U; ++u) fold(vv[u], b[u], first0 && u == 0 && q == ps);
      }
      if (q < q1) {
        float vv[U];
        float b[U][CWM][VEC];
        gather_clamped(q - cbase, q1 - 1 - cbase, vv, b);
#pragma unroll
        for (int u = 0; u < U; ++u)
          if (q + u < q1) fold(vv[u], b[u], first0 && q + u == ps);
      }
      __syncwarp();
      if (!more) break;
      cbase = nbase;
    }
    // publish this segment's partial, then take a ticket
    float* part = P.partials + static_cast<int64_t>(slot + seg) * P.ldp;
#pragma unroll
    for (int w = 0; w < CWM; ++w)
      if (cok[w]) Vec<VEC>::st(part + woff[w], acc[w]);
    __threadfence();
    __syncwarp();
    int ticket = 0;
    int* counter = P.counters + static_cast<int64_t>(slot) * P.ncb + cb;
    if (lane == 0) ticket = atomicAdd(counter, 1);
    ticket = __shfl_sync(0xffffffffu, ticket, 0);
    if (ticket == nseg - 1) {
      // last segment: combine all partials strictly left to right
      __threadfence();
      const float* base = P.partials + static_cast<int64_t>(slot) * P.ldp;
      float r[CWM][VEC];
#pragma unroll
      for (int w = 0; w < CWM; ++w) Vec<VEC>::ldcg(r[w], base + woff[w]);
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
              for (int k = 0; k < VEC; ++k) r[w][k] = SR::combine(r[w][k], pv[u][w][k]);
      }
      store_row(row, deg, r);
      if (lane == 0) *counter = 0;  // re-arm for the next launch (stream-ordered)
    }
  }
}

template <gespmm_reduce_t OP, int VEC, int CWM, bool OFF32>
cudaError_t launch_t(const KParams& p, cudaStream_t s) {
  const int64_t blocks = (p.n_items + kWarpsPerBlock - 1) / kWarpsPerBlock;
  if (blocks == 0) return cudaSuccess;
  dim3 grid(static_cast<unsigned>(blocks), static_cast<unsigned>(p.ncb), 1);
  spmm_kernel<OP, VEC, CWM, OFF32><<<grid, kWarpsPerBlock * 32, 0, s>>>(p);
  return cudaGetLastError();
}

template <gespmm_reduce_t OP, bool OFF32>
cudaError_t launch_off(const Variant& v, const KParams& p, cudaStream_t s) {
  if (v.vec == 4 && v.cwm == 2) return launch_t<OP, 4, 2, OFF32>(p, s);
  if (v.vec == 4 && v.cwm == 1) return launch_t<OP, 4, 1, OFF32>(p, s);
  if (v.vec == 2 && v.cwm == 2) return launch_t<OP, 2, 2, OFF32>(p, s);
  if (v.vec == 2 && v.cwm == 1) return launch_t<OP, 2, 1, OFF32>(p, s);
  if (v.vec == 1 && v.cwm == 2) return launch_t<OP, 1, 2, OFF32>(p, s);
  return launch_t<OP, 1, 1, OFF32>(p, s);
}

template <gespmm_reduce_t OP>
cudaError_t launch_op(const Variant& v, const KParams& p, cudaStream_t s) {
  if (p.off32) return launch_off<OP, true>(v, p, s);
  return launch_off<OP, false>(v, p, s);
}

}  // namespace kern
}  // namespace gespmm
