// gespmm_spmm.cu -- the B200 GE-SpMM kernel family (sm_100a).
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
//    128: every lane issues ONE 128-bit load of colind and ONE of vals, and the
//    (col, val) pairs are staged in the warp's slice of shared memory; each pair
//    is then read back as a broadcast (one LDS.64 per nonzero).  __syncwarp()
//    orders stage writes before reads and reads before the next refill -- the
//    warp-scoped form of the reference's two barriers (gespmm_alg2.mir:36, :65).
//    The next chunk is prefetched into registers while the current one is used.
//  * Coarse-grained Warp Merging: each lane owns VEC consecutive columns in each
//    of CWM column tiles, so one staged pair feeds VEC*CWM FMAs and every B-row
//    gather is a fully coalesced 32*VEC*4-byte warp access.  U gathers are in
//    flight per lane before the first is consumed (memory-level parallelism).
//  * Rows inside a tile are reduced sequentially in ascending p; the warp
//    switches rows as the stream crosses rowptr boundaries (rowptr window held
//    in shared memory) and stores each C row once (streaming store).
//  * Long-row segments publish a partial; the last segment to finish (atomic
//    ticket) combines all partials strictly in segment order and writes C, so
//    the result is deterministic and needs no second launch.
#include "gespmm_internal.h"
#include "gespmm_semiring.cuh"

namespace gespmm {
namespace {

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

// Streaming (evict-first) 128-bit loads for the once-read colind/vals stream.
__device__ __forceinline__ int4 ld_stream_i4(const int* p) {
  return __ldcs(reinterpret_cast<const int4*>(p));
}
__device__ __forceinline__ float4 ld_stream_f4(const float* p) {
  return __ldcs(reinterpret_cast<const float4*>(p));
}

template <gespmm_reduce_t OP, int VEC, int CWM>
__global__ void __launch_bounds__(kWarpsPerBlock * 32)
    spmm_kernel(const KParams P) {
  using SR = Semiring<OP>;
  constexpr int CPL = VEC * CWM;                      // fp32 columns per lane
  constexpr int U = CPL >= 8 ? 2 : 16 / CPL;          // gathers in flight per lane
  constexpr int TW = 32 * VEC;                        // columns per CWM tile
  __shared__ __align__(16) int2 stage[kWarpsPerBlock][kChunk];
  __shared__ int rpw[kWarpsPerBlock][kTileMaxRows + 4];

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int64_t t = static_cast<int64_t>(blockIdx.x) * kWarpsPerBlock + warp;
  if (t >= P.n_items) return;  // warp-uniform; the kernel uses no CTA-wide barrier
  const int cb = blockIdx.y;
  const int4 it = P.items[t];
  const int64_t colbase = static_cast<int64_t>(cb) * (TW * CWM) + lane * VEC;
  bool cok[CWM];
#pragma unroll
  for (int w = 0; w < CWM; ++w) cok[w] = colbase + w * TW < P.N;
  const float* Bl = P.B + colbase;
  int2* st = stage[warp];
  const bool accumulate = P.accumulate != 0;

  float acc[CWM][VEC];

  // -- CRC staging: lane l covers the 4 nonzeros at cbase + 4l (128-bit loads) --
  auto fetch = [&](int cbase, int lo, int hi, int4& c, float4& v) {
    const int e = cbase + 4 * lane;
    c = make_int4(0, 0, 0, 0);
    v = make_float4(0.f, 0.f, 0.f, 0.f);
    if (e < hi && e + 4 > lo) {
      if (P.idx_aligned && e + 4 <= P.nnz) {
        c = ld_stream_i4(P.colind + e);
        v = ld_stream_f4(P.vals + e);
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
    int4* s = reinterpret_cast<int4*>(st + 4 * lane);
    s[0] = make_int4(c.x, __float_as_int(v.x), c.y, __float_as_int(v.y));
    s[1] = make_int4(c.z, __float_as_int(v.z), c.w, __float_as_int(v.w));
  };

  // Streams nonzeros [lo, hi) (first chunk already fetched into c/v) and calls
  // step(q, val, b) for q ascending.
  auto stream_span = [&](int lo, int hi, int4 c, float4 v, auto&& step) {
    if (lo >= hi) return;
    int cbase = lo & ~3;
    while (true) {
      put(c, v);
      __syncwarp();
      const int nbase = cbase + kChunk;
      const bool more = nbase < hi;
      if (more) fetch(nbase, lo, hi, c, v);  // next chunk in flight during this one
      const int q0 = max(lo, cbase);
      const int q1 = min(hi, nbase);
      for (int q = q0; q < q1; q += U) {
        int2 e[U];
        float b[U][CWM][VEC];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          if (q + u < q1) {
            e[u] = st[q + u - cbase];
            const float* src = Bl + static_cast<int64_t>(e[u].x) * P.ldb;
#pragma unroll
            for (int w = 0; w < CWM; ++w)
              if (cok[w]) Vec<VEC>::ldg(b[u][w], src + w * TW);
          }
        }
#pragma unroll
        for (int u = 0; u < U; ++u)
          if (q + u < q1) step(q + u, __int_as_float(e[u].y), b[u]);
      }
      __syncwarp();  // stage reads complete before the refill
      if (!more) break;
      cbase = nbase;
    }
  };

  auto seed_row = [&](int64_t grow, bool seeded) {
    if (seeded) {
      const float* src = P.C + grow * P.ldc + colbase;
#pragma unroll
      for (int w = 0; w < CWM; ++w)
        if (cok[w]) Vec<VEC>::ld(acc[w], src + w * TW);
    } else {
#pragma unroll
      for (int w = 0; w < CWM; ++w)
#pragma unroll
        for (int k = 0; k < VEC; ++k) acc[w][k] = SR::zero();
    }
  };
  auto store_row = [&](int64_t grow, int deg, const float (&r)[CWM][VEC]) {
    float* dst = P.C + grow * P.ldc + colbase;
#pragma unroll
    for (int w = 0; w < CWM; ++w) {
      if (!cok[w]) continue;
      float o[VEC];
      float c0[VEC];
      if (!SR::kSeedC0 && accumulate) Vec<VEC>::ld(c0, dst + w * TW);
#pragma unroll
      for (int k = 0; k < VEC; ++k)
        o[k] = SR::finalize(r[w][k], deg, accumulate, (!SR::kSeedC0 && accumulate) ? c0[k] : 0.f);
      Vec<VEC>::stcs(dst + w * TW, o);
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
    int rpv[(kTileMaxRows + 32) / 32];
#pragma unroll
    for (int i = 0; i < (kTileMaxRows + 32) / 32; ++i) {
      const int k = lane + 32 * i;
      rpv[i] = (k <= nr) ? __ldg(P.rowptr + r0 + k) : 0;
    }
    int4 c;
    float4 v;
    fetch(pbeg & ~3, pbeg, pend, c, v);
    int* rp = rpw[warp];
#pragma unroll
    for (int i = 0; i < (kTileMaxRows + 32) / 32; ++i) {
      const int k = lane + 32 * i;
      if (k <= nr) rp[k] = rpv[i];
    }
    __syncwarp();
    const bool seed = accumulate && SR::kSeedC0;
    int row = 0;
    int rs = pbeg;
    int re = rp[1];
    seed_row(r0, seed);
    stream_span(pbeg, pend, c, v, [&](int q, float val, const float (&b)[CWM][VEC]) {
      while (q >= re) {  // rows [.., q) are complete: store and advance (warp-uniform)
        store_row(r0 + row, re - rs, acc);
        ++row;
        rs = re;
        re = rp[row + 1];
        seed_row(r0 + row, seed);
      }
      const bool first = SR::kFirstMsg && !accumulate && q == rs;
#pragma unroll
      for (int w = 0; w < CWM; ++w)
#pragma unroll
        for (int k = 0; k < VEC; ++k) acc[w][k] = SR::update(acc[w][k], val, b[w][k], first);
    });
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
    stream_span(ps, pe, c, v, [&](int q, float val, const float (&b)[CWM][VEC]) {
      const bool first = SR::kFirstMsg && !accumulate && seg == 0 && q == ps;
#pragma unroll
      for (int w = 0; w < CWM; ++w)
#pragma unroll
        for (int k = 0; k < VEC; ++k) acc[w][k] = SR::update(acc[w][k], val, b[w][k], first);
    });
    // publish this segment's partial, then take a ticket
    float* part = P.partials + static_cast<int64_t>(slot + seg) * P.ldp + colbase;
#pragma unroll
    for (int w = 0; w < CWM; ++w)
      if (cok[w]) Vec<VEC>::st(part + w * TW, acc[w]);
    __threadfence();
    __syncwarp();
    int ticket = 0;
    int* counter = P.counters + static_cast<int64_t>(slot) * P.ncb + cb;
    if (lane == 0) ticket = atomicAdd(counter, 1);
    ticket = __shfl_sync(0xffffffffu, ticket, 0);
    if (ticket == nseg - 1) {
      // last segment: combine all partials strictly left to right
      __threadfence();
      const float* base = P.partials + static_cast<int64_t>(slot) * P.ldp + colbase;
      float r[CWM][VEC];
#pragma unroll
      for (int w = 0; w < CWM; ++w)
        if (cok[w]) Vec<VEC>::ldcg(r[w], base + w * TW);
      constexpr int CU = 4;
      for (int s = 1; s < nseg; s += CU) {
        float pv[CU][CWM][VEC];
#pragma unroll
        for (int u = 0; u < CU; ++u)
          if (s + u < nseg)
#pragma unroll
            for (int w = 0; w < CWM; ++w)
              if (cok[w]) Vec<VEC>::ldcg(pv[u][w], base + static_cast<int64_t>(s + u) * P.ldp + w * TW);
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

template <gespmm_reduce_t OP, int VEC, int CWM>
cudaError_t launch_t(const KParams& p, cudaStream_t s) {
  const int64_t blocks = (p.n_items + kWarpsPerBlock - 1) / kWarpsPerBlock;
  if (blocks == 0) return cudaSuccess;
  dim3 grid(static_cast<unsigned>(blocks), static_cast<unsigned>(p.ncb), 1);
  spmm_kernel<OP, VEC, CWM><<<grid, kWarpsPerBlock * 32, 0, s>>>(p);
  return cudaGetLastError();
}

template <gespmm_reduce_t OP>
cudaError_t launch_op(const Variant& v, const KParams& p, cudaStream_t s) {
  if (v.vec == 4 && v.cwm == 2) return launch_t<OP, 4, 2>(p, s);
  if (v.vec == 4 && v.cwm == 1) return launch_t<OP, 4, 1>(p, s);
  if (v.vec == 2 && v.cwm == 2) return launch_t<OP, 2, 2>(p, s);
  if (v.vec == 2 && v.cwm == 1) return launch_t<OP, 2, 1>(p, s);
  if (v.vec == 1 && v.cwm == 2) return launch_t<OP, 1, 2>(p, s);
  return launch_t<OP, 1, 1>(p, s);
}

}  // namespace

cudaError_t launch_spmm(gespmm_reduce_t op, const Variant& v, const KParams& p,
                        cudaStream_t stream) {
  switch (op) {
    case GESPMM_REDUCE_SUM: return launch_op<GESPMM_REDUCE_SUM>(v, p, stream);
    case GESPMM_REDUCE_MAX: return launch_op<GESPMM_REDUCE_MAX>(v, p, stream);
    case GESPMM_REDUCE_MIN: return launch_op<GESPMM_REDUCE_MIN>(v, p, stream);
    case GESPMM_REDUCE_MEAN: return launch_op<GESPMM_REDUCE_MEAN>(v, p, stream);
  }
  return cudaErrorInvalidValue;
}

int variant_cols(const Variant& v) { return 32 * v.vec * v.cwm; }

std::string variant_name(const Variant& v) {
  return "vec" + std::to_string(v.vec) + "_lpr32_cwm" + std::to_string(v.cwm);
}

bool parse_variant(const char* name, Variant* v) {
  for (int vec : {1, 2, 4})
    for (int cwm : {1, 2}) {
      Variant c{vec, cwm};
      if (variant_name(c) == name) {
        *v = c;
        return true;
      }
    }
  return false;
}

// Tile shape selected by N (north star item (1)): fewest idle lanes, then fewest
// column blocks, then the widest loads the alignment of B/C allows.
Variant choose_variant(int64_t N, const float* B, int64_t ldb, const float* C, int64_t ldc) {
  auto aligned = [&](int vec) {
    const uintptr_t a = static_cast<uintptr_t>(vec) * 4;
    return reinterpret_cast<uintptr_t>(B) % a == 0 && reinterpret_cast<uintptr_t>(C) % a == 0 &&
           ldb % vec == 0 && ldc % vec == 0 && N % vec == 0;
  };
  Variant best{1, 1};
  int64_t best_idle = -1, best_ncb = 0;
  for (int vec : {4, 2, 1}) {
    if (!aligned(vec)) continue;
    for (int cwm : {1, 2}) {
      Variant c{vec, cwm};
      const int64_t cols = variant_cols(c);
      const int64_t ncb = (N + cols - 1) / cols;
      const int64_t idle = ncb * cols - N;
      if (best_idle < 0 || idle < best_idle || (idle == best_idle && ncb < best_ncb)) {
        best = c;
        best_idle = idle;
        best_ncb = ncb;
      }
    }
  }
  return best;
}

}  // namespace gespmm
