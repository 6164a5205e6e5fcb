// gespmm_kernel_pair.cuh -- paired-lane GE-SpMM kernel for N < 32 (all ops).
//
// Same work items, staging and row walk as gespmm_kernel.cuh (read that file
// first); what differs is the lane mapping.  The sum/mean contract reduces each
// row (segment) as two FMA chains -- the nonzeros at even and at odd offsets
// from its start -- added at the end; max/min have no
// fold order at all (maximumNumber), so any split of the positions works.
// Here the two chains live in the two 16-lane halves of the warp: half g folds
// the staged positions of absolute parity g, each lane owning VEC (<= 4)
// consecutive columns, so every warp instruction gathers two B rows (two
// 128-bit loads per lane pair at N=64) and the address math / load count per
// nonzero halve compared with the 32-lane kernel.  Row control stays
// warp-uniform (both halves walk the same rows); at a row end the halves'
// chains are combined with one shfl_xor(16) -- fp32 addition and
// maximumNumber are commutative, so both halves hold the same bits -- and the
// lower half stores.
//
// The stage is permuted per 8-entry block to [0,2,4,6,1,3,5,7] so a half reads
// its four (col, val) pairs of a batch with one 128-bit shared load each.
#pragma once

#include "gespmm_kernel.cuh"

namespace gespmm {
namespace kern {

#ifndef GESPMM_PAIR_MINBLOCKS
#define GESPMM_PAIR_MINBLOCKS GESPMM_MINBLOCKS
#endif
#ifndef GESPMM_PAIR_U
#define GESPMM_PAIR_U 16  // measured: config 3 N=16 1.356 -> 1.255 ms vs 8
#endif
#ifndef GESPMM_SPOS_SHFL_PAIR
#define GESPMM_SPOS_SHFL_PAIR 1
#endif
#ifndef GESPMM_PAIR_U1
#define GESPMM_PAIR_U1 GESPMM_PAIR_U  // one column per lane (N <= 16)
#endif
template <gespmm_reduce_t OP, int VEC, bool OFF32>
__global__ void __launch_bounds__(kWarpsPerBlock * 32, GESPMM_PAIR_MINBLOCKS)
    spmm_pair_kernel(const KParams P) {
  using SR = Semiring<OP>;
  static_assert(SR::kFma2 || SR::kMnmx, "paired lanes: two-chain sum/mean or order-free max/min");
  constexpr int U = VEC == 1 ? GESPMM_PAIR_U1 : GESPMM_PAIR_U;  // positions per batch (U/2 per half; 8, 16 or 32)
  constexpr int H = U / 2;
  static_assert(U % 8 == 0 && kTileWork + kSeg + kRowCost + 2 + 3 + U <= kStageCap,
                "the stage holds the largest item rounded up to a batch");
  constexpr int TW = 16 * VEC;   // columns per column block
  constexpr unsigned FULL = 0xffffffffu;
  // per warp: colind slice then vals slice (vals at an immediate offset)
  __shared__ __align__(16) int stg[kWarpsPerBlock][2 * kStageCap];
  __shared__ int rpw[kWarpsPerBlock][kTileMaxRows + 4];

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int g = lane >> 4;       // my half = the parity of the positions I fold
  const int gl = lane & 15;
  const int cb = blockIdx.y;
  const int64_t colbase = static_cast<int64_t>(cb) * TW + gl * VEC;
  const bool cok = colbase < P.N;
  const int woff = cok ? static_cast<int>(colbase) : 0;
  const float* bw = GESPMM_PIN ? pin_reg64(P.B + woff) : P.B + woff;  // pinned: see pin_reg
  const int64_t ldb = P.ldb;
  const int64_t ldc = P.ldc;
  int* const sc = stg[warp];
  const uint32_t sc_s = GESPMM_PIN ? pin_reg(static_cast<uint32_t>(__cvta_generic_to_shared(sc)))
                                   : static_cast<uint32_t>(__cvta_generic_to_shared(sc));
  float* const sv = reinterpret_cast<float*>(stg[warp] + kStageCap);
  int* const rp = rpw[warp];
  const bool accumulate = P.accumulate != 0;
  const bool seed_c0 = accumulate && SR::kSeedC0;
  const bool storer = g == 0 && cok;
  const uint64_t bpol = GESPMM_BHINT ? policy_evict_last() : 0;

  float acc[VEC];
  // chain A (even offsets from `start`) is held by the half whose parity is
  // start's; it gets x (or C0), the other half the chain identity (sum: -0.0,
  // max/min: NaN).
  auto seed = [&](int start, float x, const float* src) {
    float c[VEC];
    if (src) Vec<VEC>::ld(c, src);
    const bool mine = g == (start & 1);
#pragma unroll
    for (int k = 0; k < VEC; ++k) acc[k] = mine ? (src ? c[k] : x) : SR::chain_seed();
  };
  auto row_seed = [&](int start, const float* crow_) {
    seed(start, SR::zero(), seed_c0 ? crow_ : nullptr);
  };
  // A (+) B across the halves (both halves end with the same bits)
  auto combined = [&](float (&o)[VEC]) {
#pragma unroll
    for (int k = 0; k < VEC; ++k) o[k] = SR::combine(acc[k], __shfl_xor_sync(FULL, acc[k], 16));
  };
  auto store_row = [&](float* dst, int deg) {
    float o[VEC];
    combined(o);
    // max/min over an empty row with accumulate: C0 untouched (the halves'
    // combine would canonicalize a NaN C0)
    if (!storer || (SR::kMnmx && accumulate && deg == 0)) return;
    float c0[VEC];
    if (!SR::kSeedC0 && accumulate) Vec<VEC>::ld(c0, dst);
#pragma unroll
    for (int k = 0; k < VEC; ++k)
      o[k] = SR::finalize(o[k], deg, accumulate, (!SR::kSeedC0 && accumulate) ? c0[k] : 0.f);
    Vec<VEC>::stcs(dst, o);
  };
  auto gather = [&](float (&d)[VEC], int x) {
    if (OFF32) gather_off<VEC>(d, bw, static_cast<uint32_t>(x), bpol);
    else Vec<VEC>::ldg(d, bw + static_cast<int64_t>(x) * ldb);
  };
  auto fold = [&](float v, const float (&b)[VEC]) {
    if (SR::kFma2 && VEC >= 2) {
#pragma unroll
      for (int k = 0; k < VEC; k += 2) fma2_rn(acc[k], acc[k + 1], v, b[k], b[k + 1]);
    } else {
#pragma unroll
      for (int k = 0; k < VEC; ++k) acc[k] = SR::update(acc[k], v, b[k]);
    }
  };
  // two of my half's entries (max/min: products in FMUL2, one FMNMX3 per column)
  auto fold_pair = [&](float v0, const float (&b0)[VEC], float v1, const float (&b1)[VEC]) {
    if constexpr (SR::kMnmx) {
      if constexpr (VEC >= 2) {
#pragma unroll
        for (int k = 0; k < VEC; k += 2) {
          float m0, m1, n0, n1;
          mul2_rn(m0, m1, v0, b0[k], b0[k + 1]);
          mul2_rn(n0, n1, v1, b1[k], b1[k + 1]);
          acc[k] = SR::pick3(acc[k], m0, n0);
          acc[k + 1] = SR::pick3(acc[k + 1], m1, n1);
        }
      } else {
        acc[0] = SR::pick3(acc[0], __fmul_rn(v0, b0[0]), __fmul_rn(v1, b1[0]));
      }
    } else {
      fold(v0, b0);
      fold(v1, b1);
    }
  };

  // 32-bit item cursor (GESPMM_ITEM32; gespmm_kernel.cuh)
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
    t = dyn ? t_begin + static_cast<item_t>(__shfl_sync(FULL, next, 0)) : t + wstride; \
    continue;                                                                    \
  }
  const bool dyn = P.work_ctr != nullptr;
  unsigned long long* const wctr = dyn ? P.work_ctr + blockIdx.y : nullptr;
  auto grab = [&]() {
    grab_t v = 0;
    if (lane == 0) v = static_cast<grab_t>(atomicAdd(wctr, 1ULL));
    return v;
  };
  item_t t = dyn ? t_begin + static_cast<item_t>(__shfl_sync(FULL, grab(), 0))
                 : t_begin + static_cast<item_t>(blockIdx.x) * kWarpsPerBlock + warp;
  for (; t < t_end;) {
    const grab_t next = dyn ? grab() : grab_t(0);
    __syncwarp();  // the previous item's stage reads are done (the role of mir:65)
    const int4 it = P.items[t];
    const bool is_tile = it.y < 0;
    int lo, hi, nr, re_long = 0;
    if (is_tile) {
      int r1, pend;
      // the next item (the plan's sentinel {M, -1, nnz} after the last one)
      const int4 nx = P.items[t + 1];
      r1 = nx.x;
      pend = nx.z;
      nr = r1 - it.x;
      lo = it.z;
      hi = pend;
      for (int k = lane; k <= nr; k += 32) cp_async4(rp + k, P.rowptr + it.x + k);
    } else {
      nr = 1;
      lo = it.z + it.y * kSeg;
      re_long = __ldg(P.rowptr + it.x + 1);  // in flight while the stage copy is issued
      hi = min(lo + kSeg, P.nnz);  // copy bound; the segment end is applied below
    }
    // ---- CRC staging (as in gespmm_kernel.cuh), then the parity permutation --
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
    __syncwarp();
    for (int i = hi - sbase + lane; i < send - sbase; i += 32) sc[i] = 0;  // pad: row 0, never folded
    if (lane < lo - sbase) sc[lane] = 0;  // head: another item's entries, never gathered through
    __syncwarp();
    {
      // per 8-entry block: the 4 even positions, then the 4 odd ones (a half's
      // 4 entries of the block contiguous).  Lane l holds entries 4l..4l+3
      // (coalesced 128-bit loads and stores, no bank conflicts); lane pairs
      // (2m, 2m+1) own block m and swap one entry pair with shfl_xor(1): the
      // even lane keeps its evens and takes its partner's, the odd lane the
      // odds.  (A lane-per-block permutation reads and writes at a 64-byte
      // lane stride: 16-way bank conflicts, ~25 % of the L1 data-pipe
      // wavefronts at config 3 N=16.)  The trip count is warp-uniform for the
      // shuffles; the span is a multiple of U >= 8, so a pair is in or out
      // together.
      const uint32_t ldb32 = static_cast<uint32_t>(ldb);
      const bool odd = lane & 1;
      const int len = send - sbase;
      for (int i0 = 0; i0 < len; i0 += 128) {
        const int i = i0 + 4 * lane;
        const bool in = i < len;
        int4 a = make_int4(0, 0, 0, 0);
        float4 f = make_float4(0.f, 0.f, 0.f, 0.f);
        if (in) {
          a = *reinterpret_cast<int4*>(sc + i);
          f = *reinterpret_cast<float4*>(sv + i);
        }
        const int ra = __shfl_xor_sync(FULL, odd ? a.x : a.y, 1);
        const int rb = __shfl_xor_sync(FULL, odd ? a.z : a.w, 1);
        const float ga = __shfl_xor_sync(FULL, odd ? f.x : f.y, 1);
        const float gb = __shfl_xor_sync(FULL, odd ? f.z : f.w, 1);
        int d[4] = {odd ? ra : a.x, odd ? rb : a.z, odd ? a.y : ra, odd ? a.w : rb};
        const float x[4] = {odd ? ga : f.x, odd ? gb : f.z, odd ? f.y : ga, odd ? f.w : gb};
        if (OFF32) {
#pragma unroll
          for (int r = 0; r < 4; ++r) d[r] = static_cast<int>(static_cast<uint32_t>(d[r]) * ldb32);
        }
        if (in) {
          *reinterpret_cast<int4*>(sc + i) = make_int4(d[0], d[1], d[2], d[3]);
          *reinterpret_cast<float4*>(sv + i) = make_float4(x[0], x[1], x[2], x[3]);
        }
      }
      __syncwarp();
    }

    // ---- row state (warp-uniform) --------------------------------------------
    float* crow = P.C + static_cast<int64_t>(it.x) * ldc + woff;
    int row = 0, rs = lo, re = is_tile ? rp[1] : hi;
    if (!is_tile && it.y > 0) seed(lo, SR::identity(), nullptr);
    else row_seed(lo, crow);

    // 32-bit shared address of my half's entries of 8-entry block 0
    // through a shuffle (GESPMM_SPOS_SHFL_PAIR, one column per lane): ptxas
    // otherwise recomputes the half's offset from SR_TID in every batch
    // (DESIGN.md 5.2 item 11): config 3 N=16 sum / max / mean 1.071 / 1.090 /
    // 1.083 -> 1.040 / 1.057 / 1.051 ms; pair_vec2 (N=32 max) +0.3 %, so not there
    const uint32_t s_pos0 = (GESPMM_SPOS_SHFL_PAIR && VEC == 1)
                                ? __shfl_sync(FULL, sc_s + 4u * static_cast<uint32_t>(4 * g - sbase), lane)
                                : sc_s + 4u * static_cast<uint32_t>(4 * g - sbase);
    for (int qb = sbase; qb < hi; qb += U) {
      // my half's staged entries of this batch, four per 8-entry block:
      // entry i is position qb + 2i + g
      float b[H][VEC];
      float v[H];
#pragma unroll
      for (int q4 = 0; q4 < H / 4; ++q4) {
        int4 o;
        asm volatile("ld.shared.v4.s32 {%0, %1, %2, %3}, [%4];"
                     : "=r"(o.x), "=r"(o.y), "=r"(o.z), "=r"(o.w)
                     : "r"(s_pos0 + 4u * static_cast<uint32_t>(qb) + 32u * q4));
        gather(b[4 * q4 + 0], o.x);
        gather(b[4 * q4 + 1], o.y);
        gather(b[4 * q4 + 2], o.z);
        gather(b[4 * q4 + 3], o.w);
      }
#pragma unroll
      for (int q4 = 0; q4 < H / 4; ++q4) {
        float4 vv;
        asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                     : "=f"(vv.x), "=f"(vv.y), "=f"(vv.z), "=f"(vv.w)
                     : "r"(s_pos0 + 4u * static_cast<uint32_t>(qb) + (4u * kStageCap + 32u * q4)));
        v[4 * q4] = vv.x, v[4 * q4 + 1] = vv.y, v[4 * q4 + 2] = vv.z, v[4 * q4 + 3] = vv.w;
      }
      if (qb >= lo && qb + U <= min(hi, re)) {  // fast path: the batch is in the current row
#pragma unroll
        for (int i = 0; i < H; i += 2) fold_pair(v[i], b[i], v[i + 1], b[i + 1]);
        continue;
      }
#pragma unroll
      for (int j = 0; j < U; ++j) {  // slow path: positions in order
        const int p = qb + j;
        if (p < lo || p >= hi) continue;
        while (p >= re) {  // rows ending at or before p are complete (tiles only)
          store_row(crow, re - rs);
          ++row;
          crow += ldc;
          rs = re;
          re = rp[row + 1];
          row_seed(rs, crow);
        }
        if (g == (j & 1)) fold(v[j >> 1], b[j >> 1]);  // my entry j/2 is position qb + j
      }
    }

    if (is_tile) {
      for (;;) {  // the row in progress and any trailing empty rows
        store_row(crow, re - rs);
        if (++row >= nr) break;
        crow += ldc;
        rs = re;
        re = rp[row + 1];
        row_seed(rs, crow);
      }
      GESPMM_NEXT_ITEM;
    }
    // ---- long-row segment: publish A + B, then take a ticket ------------------
    const int seg = it.y;
    const int slot = it.w;
    const int deg = re_long - it.z;
    const int nseg = (deg + kSeg - 1) / kSeg;
    {
      float o[VEC];
      combined(o);
      if (storer) Vec<VEC>::st(P.partials + static_cast<int64_t>(slot + seg) * P.ldp + woff, o);
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
    ticket = __shfl_sync(FULL, ticket, 0);
    if (ticket != nseg - 1) GESPMM_NEXT_ITEM;
    __syncwarp();  // lane 0's acquire orders the whole warp's partial loads below
#else
    __threadfence();
    __syncwarp();
    int ticket = 0;
    int* counter = P.counters + static_cast<int64_t>(slot) * P.ncb + cb;
    if (lane == 0) ticket = atomicAdd(counter, 1);
    ticket = __shfl_sync(FULL, ticket, 0);
    if (ticket != nseg - 1) GESPMM_NEXT_ITEM;
#endif
    // last segment: combine the partials left to right (both halves compute
    // it; the lower half stores)
    if (!GESPMM_TICKET_ACQREL) __threadfence();
    const float* base = P.partials + static_cast<int64_t>(slot) * P.ldp + woff;
    float r[VEC];
    Vec<VEC>::ldcg(r, base);
    for (int s = 1; s < nseg; ++s) {
      float pv[VEC];
      Vec<VEC>::ldcg(pv, base + static_cast<int64_t>(s) * P.ldp);
#pragma unroll
      for (int k = 0; k < VEC; ++k) r[k] = SR::combine(r[k], pv[k]);
    }
    if (storer) {
      float c0[VEC];
      if (!SR::kSeedC0 && accumulate) Vec<VEC>::ld(c0, crow);
#pragma unroll
      for (int k = 0; k < VEC; ++k)
        r[k] = SR::finalize(r[k], deg, accumulate, (!SR::kSeedC0 && accumulate) ? c0[k] : 0.f);
      Vec<VEC>::stcs(crow, r);
    }
    if (lane == 0) *counter = 0;  // re-arm for the next launch (stream-ordered)
    t = dyn ? t_begin + static_cast<item_t>(__shfl_sync(FULL, next, 0)) : t + wstride;
  }  // item loop
#undef GESPMM_NEXT_ITEM
}

template <gespmm_reduce_t OP, int VEC, bool OFF32>
cudaError_t launch_pair_t(const KParams& p, cudaStream_t s) {
  int64_t blocks = (p.n_items + kWarpsPerBlock - 1) / kWarpsPerBlock;
  if (blocks == 0) return cudaSuccess;
  static thread_local int cached_dev = -1, cached_slots = 0;
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev != cached_dev) {
    int sms = 0, per_sm = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, spmm_pair_kernel<OP, VEC, OFF32>,
                                                  kWarpsPerBlock * 32, 0);
    cached_slots = sms * (per_sm > 0 ? per_sm : 1);
    cached_dev = dev;
  }
  const int64_t slots = (cached_slots + p.ncb - 1) / p.ncb;
  if (blocks > slots) blocks = slots;
  dim3 grid(static_cast<unsigned>(blocks), static_cast<unsigned>(p.ncb), 1);
  spmm_pair_kernel<OP, VEC, OFF32><<<grid, kWarpsPerBlock * 32, 0, s>>>(p);
  return cudaGetLastError();
}

template <gespmm_reduce_t OP>
cudaError_t launch_pair(const Variant& v, const KParams& p, cudaStream_t s) {
  if (p.off32) {
    if (v.vec == 4) return launch_pair_t<OP, 4, true>(p, s);
    if (v.vec == 2) return launch_pair_t<OP, 2, true>(p, s);
    return launch_pair_t<OP, 1, true>(p, s);
  }
  if (v.vec == 4) return launch_pair_t<OP, 4, false>(p, s);
  if (v.vec == 2) return launch_pair_t<OP, 2, false>(p, s);
  return launch_pair_t<OP, 1, false>(p, s);
}

}  // namespace kern
}  // namespace gespmm
