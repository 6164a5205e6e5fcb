// gespmm_plan.cu -- nnz-balanced work decomposition, built on the GPU
// (BASELINE.json north star item (2): "nnz-balanced row-partitioner with a
// power-law/long-row split path").
//
// Input: rowptr of one CSR (plus colind for optional validation).
// Output: a list of work items, one warp each, in row order:
//   TILE    {r0, -1, rowptr[r0], 0}: consecutive short rows (deg <= kSeg); the
//           tile ends where the next item starts.  A short row costs
//           w = deg + kRowCost work units; row i joins tile floor(E_i / tw)
//           where E is the exclusive prefix of w and tw the plan's tile_work,
//           so a tile holds ~tw units (<= tw + kSeg + kRowCost) and <= tw /
//           kRowCost rows.
//   SEGMENT {row, s, rowptr[row], slot}: nonzeros [rs + s*kSeg, rs + (s+1)*kSeg)
//           of a long row; `slot` is the row's first partial-buffer slot.
// A long row always ends the tile before it.  The decomposition depends only
// on rowptr -- never on the device or grid -- which is what makes results
// reproducible across GPUs and across row-sharding.
//
// Steps: k_rows (per-row work, packed 40|24-bit, + CSR validation)
//        -> exclusive scan (CUB) -> k_count (items per row) -> exclusive scan
//        -> one D2H of the totals (the only host sync) -> k_emit.
// The reference validates the same CSR rules on the host (src/oracle.cpp:291-316).
#include <cub/device/device_scan.cuh>

#include <cstdio>
#include <cstdlib>

#include "gespmm_internal.h"

namespace gespmm {
namespace {

constexpr uint64_t kLowMask = (uint64_t(1) << kPackShift) - 1;

enum : int { kErrRowptr0 = 1, kErrMonotone = 2, kErrEnd = 4, kErrColRange = 8 };

__global__ void k_rows(const int* __restrict__ rowptr, int M, int nnz,
                       uint64_t* __restrict__ packed, int* __restrict__ err) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= M) return;
  const int a = rowptr[i];
  const int b = rowptr[i + 1];
  int e = 0;
  if (i == 0 && a != 0) e |= kErrRowptr0;
  if (b < a) e |= kErrMonotone;
  if (i == M - 1 && b != nnz) e |= kErrEnd;
  if (e) atomicOr(err, e);
  const int deg = b >= a ? b - a : 0;
  const bool lng = deg > kSeg;
  if (lng) atomicAdd(err + 1, 1);  // long-row count (plan info)
  const uint64_t w = lng ? 0 : static_cast<uint64_t>(deg + kRowCost);
  const uint64_t ns = lng ? static_cast<uint64_t>((deg + kSeg - 1) / kSeg) : 0;
  packed[i] = (ns << kPackShift) | w;
}

__global__ void k_colind(const int* __restrict__ colind, int64_t nnz, int K, int* __restrict__ err) {
  int bad = 0;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t p = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; p < nnz; p += stride) {
    const int c = __ldcs(colind + p);
    bad |= (c < 0) | (c >= K);
  }
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(err, kErrColRange);
}

__device__ __forceinline__ bool tile_start(int i, const uint64_t* packed, const uint64_t* E, int tw) {
  const uint64_t pi = packed[i];
  if ((pi & kLowMask) == 0) return false;  // long row: no tile starts here
  if (i == 0) return true;
  const uint64_t pp = packed[i - 1];
  if ((pp & kLowMask) == 0) return true;   // previous row is long
  return ((E[i] & kLowMask) / tw) != ((E[i - 1] & kLowMask) / tw);
}

__global__ void k_count(const uint64_t* __restrict__ packed, const uint64_t* __restrict__ E, int M, int tw,
                        int* __restrict__ cnt) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= M) return;
  cnt[i] = (tile_start(i, packed, E, tw) ? 1 : 0) + static_cast<int>(packed[i] >> kPackShift);
}

__global__ void k_emit(const int* __restrict__ rowptr, const uint64_t* __restrict__ packed,
                       const uint64_t* __restrict__ E, const int* __restrict__ pos, int M, int tw,
                       int4* __restrict__ items, int64_t cap) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= M) return;
  int64_t p = pos[i];
  const int rs = rowptr[i];
  // cap: the async build's upper bound (a valid CSR never reaches it; an
  // invalid rowptr may -- its launches abort on the error bit)
  if (tile_start(i, packed, E, tw) && p < cap) items[p] = make_int4(i, -1, rs, 0);
  if (tile_start(i, packed, E, tw)) ++p;
  const int ns = static_cast<int>(packed[i] >> kPackShift);
  const int slot = static_cast<int>(E[i] >> kPackShift);
  for (int s = 0; s < ns && p < cap; ++s) items[p++] = make_int4(i, s, rs, slot);
}

struct Totals {
  uint64_t last_packed;
  uint64_t last_E;
  int last_cnt;
  int last_pos;
  int err;
  int n_long;
};

__global__ void k_totals(const uint64_t* packed, const uint64_t* E, const int* cnt, const int* pos,
                         int M, const int* err, Totals* out) {
  out->last_packed = packed[M - 1];
  out->last_E = E[M - 1];
  out->last_cnt = cnt[M - 1];
  out->last_pos = pos[M - 1];
  out->err = err[0];
  out->n_long = err[1];
}

// items[n_items] = {M, -1, nnz, 0}: a tile "starting" at row M, position
// nnz -- so every item's end is items[t + 1] with no bound check in the
// kernel (the last real tile ends at row M / position nnz).
__global__ void k_sentinel(int4* items, int64_t n, int M, int nnz) { items[n] = make_int4(M, -1, nnz, 0); }

// The async build's counts (one thread): n_items, n_segs, error bits.
constexpr int kErrItemCap = 16;  // more items than the bound (invalid rowptr only)
__global__ void k_meta(const uint64_t* packed, const uint64_t* E, const int* cnt, const int* pos, int M,
                       int nnz, const int* err, int64_t cap, int4* items, gespmm_plan_s::Meta* out) {
  const int64_t n = static_cast<int64_t>(pos[M - 1]) + cnt[M - 1];
  out->n_items = n < cap ? n : cap;
  items[out->n_items] = make_int4(M, -1, nnz, 0);  // the sentinel (k_sentinel)
  out->n_segs = static_cast<int64_t>(E[M - 1] >> kPackShift) + static_cast<int64_t>(packed[M - 1] >> kPackShift);
  out->err = err[0] | (n > cap ? kErrItemCap : 0);
  out->n_long = err[1];
}

std::string csr_error_text(int err, int64_t K) {
  // wording follows raceset::validate_instance (src/oracle.cpp:302-315)
  if (err & kErrRowptr0) return "invalid csr: rowPtr[0] must be 0";
  if (err & kErrMonotone) return "invalid csr: rowPtr must be nondecreasing";
  if (err & kErrEnd) return "invalid csr: rowPtr end differs from nnz of colInd";
  if (err & kErrColRange) return "invalid csr: colInd entry out of [0," + std::to_string(K) + ")";
  return "invalid csr";
}

struct ChunkRows {
  int64_t r[kMaxChunks + 1];
};

// ranges[c] = first item whose row is >= rows[c] (items are in row order; a
// long row's segment 0 precedes its other segments), ranges[nc] = n_items.
// pin = 1 (chunk partitions): ranges[0] = 0 and ranges[nc] = n_items;
// pin = 0: every entry is the lower bound of rows[c], c < nc.
__global__ void k_chunk_ranges(const int4* __restrict__ items, int64_t n_items, ChunkRows rows, int nc,
                               int64_t* __restrict__ ranges, int pin) {
  const int c = threadIdx.x;
  if (pin ? c > nc : c >= nc) return;
  if (pin && c == nc) {
    ranges[c] = n_items;
    return;
  }
  int64_t lo = 0, hi = n_items;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (items[mid].x < rows.r[c]) lo = mid + 1;
    else hi = mid;
  }
  ranges[c] = (pin && c == 0) ? 0 : lo;
}

// Item-aligned chunk rows: out_rows[c] = the first row of the first item whose
// row is >= rows.r[c] (so no tile spans two chunks), out_rows[nc] = M, and
// ranges[c] = that item (ranges[nc] = n_items).
__global__ void k_chunk_rows_aligned(const int4* __restrict__ items, int64_t n_items, int64_t M,
                                     ChunkRows rows, int nc, int64_t* __restrict__ ranges,
                                     int64_t* __restrict__ out_rows) {
  const int c = threadIdx.x;
  if (c > nc) return;
  if (c == nc) {
    ranges[c] = n_items;
    out_rows[c] = M;
    return;
  }
  int64_t lo = 0, hi = n_items;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (items[mid].x < rows.r[c]) lo = mid + 1;
    else hi = mid;
  }
  if (c == 0) lo = 0;
  ranges[c] = lo;
  out_rows[c] = c == 0 ? 0 : (lo < n_items ? static_cast<int64_t>(items[lo].x) : M);
}

}  // namespace

cudaError_t chunk_rows_aligned(const gespmm_plan_s* plan, const int64_t* rows, int nc, int64_t* d_ranges,
                               int64_t* d_rows, cudaStream_t s) {
  if (nc < 1 || nc > kMaxChunks) return cudaErrorInvalidValue;
  ChunkRows cr{};
  for (int c = 0; c <= nc; ++c) cr.r[c] = rows[c];
  k_chunk_rows_aligned<<<1, kMaxChunks + 1, 0, s>>>(plan->items, plan->n_items, plan->M, cr, nc, d_ranges, d_rows);
  return cudaGetLastError();
}

cudaError_t chunk_ranges(const gespmm_plan_s* plan, const int64_t* rows, int nc, int64_t* d_ranges,
                         cudaStream_t s) {
  if (nc < 1 || nc > kMaxChunks) return cudaErrorInvalidValue;
  ChunkRows cr{};
  for (int c = 0; c <= nc; ++c) cr.r[c] = rows[c];
  k_chunk_ranges<<<1, kMaxChunks + 1, 0, s>>>(plan->items, plan->n_items, cr, nc, d_ranges, 1);
  return cudaGetLastError();
}

// d_range[k] = first item whose row is >= rows[k], k = 0, 1 (any row range).
cudaError_t row_item_range(const gespmm_plan_s* plan, const int64_t* rows, int64_t* d_range,
                           cudaStream_t s) {
  ChunkRows cr{};
  cr.r[0] = rows[0];
  cr.r[1] = rows[1];
  k_chunk_ranges<<<1, 32, 0, s>>>(plan->items, plan->n_items, cr, 2, d_range, 0);
  return cudaGetLastError();
}

// Validates colind[p0, p1) on the device, OR-ing an error bit into *err (no sync).
cudaError_t validate_colind_async(const int* colind, int64_t p0, int64_t p1, int64_t K, int* err,
                                  cudaStream_t s) {
  if (p1 <= p0) return cudaSuccess;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  int64_t blocks = (p1 - p0 + 255) / 256;
  if (blocks > 4 * sms) blocks = 4 * sms;
  k_colind<<<static_cast<unsigned>(blocks), 256, 0, s>>>(colind + p0, p1 - p0, static_cast<int>(K), err);
  return cudaGetLastError();
}

std::string csr_error_message(int err, int64_t K) { return csr_error_text(err, K); }

int g_tile_work_override = 0;  // > 0: forced tile_work (tests/tuning)

// The plan's tile_work: the largest power of two in [kMinTileWork, kTileWork]
// with at least 2 x 148 x 32 tiles' worth of work (148 SMs x 32 resident
// warps), from (nnz, M) only so the decomposition stays device-independent.
// Results never depend on it (short rows stay whole).  Measured on config 1
// (4096^2, 168 K nnz, picks 16): 256 / 64 / 32 / 16 / 8 units -> 20.3 / 12.5 /
// 12.3 / 11.6 / 11.5 us; config 3 (picks 256) within 1 % for 16..256.
int tile_work_for(int64_t M, int64_t nnz) {
  if (g_tile_work_override > 0) return g_tile_work_override;
  const int64_t work = nnz + kRowCost * M;
  int tw = kTileWork;
  while (tw > kMinTileWork && work < static_cast<int64_t>(tw) * 2 * 148 * 32) tw >>= 1;
  return tw;
}

// Validates colind on the device; returns the error bits via *err_host (sync).
gespmm_status_t device_validate_colind(const int* colind, int64_t nnz, int64_t K,
                                       cudaStream_t s) {
  int* err = nullptr;
  cudaError_t ce = cudaMallocAsync(&err, sizeof(int), s);
  if (ce != cudaSuccess) return cuda_fail(ce, "cudaMallocAsync");
  cudaMemsetAsync(err, 0, sizeof(int), s);
  if (nnz > 0) {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    int64_t blocks = (nnz + 255) / 256;
    if (blocks > 4 * sms) blocks = 4 * sms;
    k_colind<<<static_cast<unsigned>(blocks), 256, 0, s>>>(colind, nnz, static_cast<int>(K), err);
  }
  int h = 0;
  cudaMemcpyAsync(&h, err, sizeof(int), cudaMemcpyDeviceToHost, s);
  cudaFreeAsync(err, s);
  ce = cudaStreamSynchronize(s);
  if (ce != cudaSuccess) return cuda_fail(ce, "validate colind");
  if (h) return fail(GESPMM_CSR_INVALID, csr_error_text(h, K));
  return GESPMM_OK;
}

// Plan temporaries are stream-ordered allocations from the device's default
// memory pool; keep that pool's memory mapped across synchronizations
// (release threshold 0 would unmap and remap ~25 MB per plan build).
static void keep_pool_resident() {
  static bool done[64] = {};
  if (std::getenv("GESPMM_NO_POOL_RESIDENT")) return;  // debug switch
  int dev = 0;
  cudaGetDevice(&dev);
  if (done[dev & 63]) return;
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
    uint64_t threshold = UINT64_MAX;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &threshold);
  }
  done[dev & 63] = true;
}

gespmm_status_t build_plan(gespmm_plan_s* plan, const int* rowptr, const int* colind,
                           bool check_colind, cudaStream_t s) {
  NvtxRange nvtx("gespmm:plan_build");
  keep_pool_resident();
  plan->async_counts = false;
  const int64_t M = plan->M;
  const int M32 = static_cast<int>(M);
  const int nnz32 = static_cast<int>(plan->nnz);
  cudaError_t ce;
  if (M == 0) {
    plan->n_items = plan->n_tiles = plan->n_long = plan->n_segs = 0;
    if (plan->nnz != 0) return fail(GESPMM_CSR_INVALID, "invalid csr: rowPtr end differs from nnz of colInd");
    return GESPMM_OK;
  }
  // temporaries (stream-ordered)
  uint64_t *packed = nullptr, *E = nullptr;
  int *cnt = nullptr, *pos = nullptr, *err = nullptr;
  Totals* tot = nullptr;
  void* tmp = nullptr;
  size_t tmp1 = 0, tmp2 = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, tmp1, packed, E, M32, s);
  cub::DeviceScan::ExclusiveSum(nullptr, tmp2, cnt, pos, M32, s);
  const size_t tmp_bytes = tmp1 > tmp2 ? tmp1 : tmp2;
  const size_t bytes = M * (8 + 8 + 4 + 4) + 64 + sizeof(Totals) + tmp_bytes + 8 * 256;
  char* arena = nullptr;
  ce = cudaMallocAsync(&arena, bytes, s);
  if (ce != cudaSuccess) return cuda_fail(ce, "plan temporaries");
  {
    char* p = arena;
    auto take = [&](size_t n) {
      char* r = p;
      p += (n + 255) & ~size_t(255);
      return r;
    };
    packed = reinterpret_cast<uint64_t*>(take(M * 8));
    E = reinterpret_cast<uint64_t*>(take(M * 8));
    cnt = reinterpret_cast<int*>(take(M * 4));
    pos = reinterpret_cast<int*>(take(M * 4));
    err = reinterpret_cast<int*>(take(64));
    tot = reinterpret_cast<Totals*>(take(sizeof(Totals)));
    tmp = take(tmp_bytes);
    (void)bytes;
  }
  Trace tr("plan");
  tr.mark("alloc temporaries", s);
  const unsigned blocks = static_cast<unsigned>((M + 255) / 256);
  cudaMemsetAsync(err, 0, 2 * sizeof(int), s);
  k_rows<<<blocks, 256, 0, s>>>(rowptr, M32, nnz32, packed, err);
  if (check_colind && plan->nnz > 0) {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    int64_t cblocks = (plan->nnz + 255) / 256;
    if (cblocks > 4 * sms) cblocks = 4 * sms;
    k_colind<<<static_cast<unsigned>(cblocks), 256, 0, s>>>(colind, plan->nnz,
                                                            static_cast<int>(plan->K), err);
  }
  size_t tb = tmp_bytes;
  cub::DeviceScan::ExclusiveSum(tmp, tb, packed, E, M32, s);
  const int tw = tile_work_for(M, plan->nnz);
  plan->tile_work = tw;
  k_count<<<blocks, 256, 0, s>>>(packed, E, M32, tw, cnt);
  tb = tmp_bytes;
  cub::DeviceScan::ExclusiveSum(tmp, tb, cnt, pos, M32, s);
  k_totals<<<1, 1, 0, s>>>(packed, E, cnt, pos, M32, err, tot);
  tr.mark("rows/validate/scan/count", s);
  Totals h{};
  cudaMemcpyAsync(&h, tot, sizeof(Totals), cudaMemcpyDeviceToHost, s);
  ce = cudaStreamSynchronize(s);
  if (ce != cudaSuccess) {
    cudaFreeAsync(arena, s);
    return cuda_fail(ce, "plan build");
  }
  if (h.err) {
    cudaFreeAsync(arena, s);
    return fail(GESPMM_CSR_INVALID, csr_error_text(h.err, plan->K));
  }
  plan->n_items = static_cast<int64_t>(h.last_pos) + h.last_cnt;
  plan->n_segs = static_cast<int64_t>(h.last_E >> kPackShift) + static_cast<int64_t>(h.last_packed >> kPackShift);
  plan->n_long = h.n_long;
  plan->n_tiles = plan->n_items - plan->n_segs;
  if (!plan->items || plan->items_cap < plan->n_items) {  // grow-only (re-planned plans reuse it)
    if (plan->items) cudaFree(plan->items);
    plan->items = nullptr;
    plan->items_cap = 0;
    const int64_t cap = plan->n_items + 1;  // + the sentinel
    ce = cudaMallocAsync(&plan->items, static_cast<size_t>(cap) * sizeof(int4), s);
    if (ce != cudaSuccess) {
      cudaFreeAsync(arena, s);
      return cuda_fail(ce, "plan items");
    }
    plan->items_cap = cap;
  }
  tr.mark("totals D2H + items alloc", s);
  k_emit<<<blocks, 256, 0, s>>>(rowptr, packed, E, pos, M32, tw, plan->items, plan->n_items);
  k_sentinel<<<1, 1, 0, s>>>(plan->items, plan->n_items, M32, nnz32);
  ce = cudaGetLastError();
  cudaFreeAsync(arena, s);
  tr.mark("emit", s);
  if (ce != cudaSuccess) return cuda_fail(ce, "plan emit");
  return GESPMM_OK;
}

// Upper bounds of the decomposition from (M, nnz, tile_work) alone: tiles <=
// (nnz + kRowCost M) / tw + n_long + 2 (a tile closes after ~tw units or at a
// long row), n_long <= nnz / (kSeg + 1), segments <= nnz / kSeg + n_long.
static void plan_bounds(int64_t M, int64_t nnz, int tw, int64_t* items, int64_t* segs) {
  const int64_t n_long = nnz / (kSeg + 1) + 1;
  const int64_t sg = nnz / kSeg + n_long + 1;
  const int64_t tiles = (nnz + kRowCost * M) / tw + n_long + 2;
  *segs = sg;
  *items = tiles + sg;
}

// The one-shot plan build (gespmm_csr_spmm): the same kernels as build_plan,
// but nothing comes back to the host -- items are emitted into a buffer sized
// by plan_bounds, and the true counts and the CSR error bits land in
// plan->meta on the device.  Every launch of this plan reads the count from
// there and returns at once on an error bit; the caller copies meta to the
// host after its one trailing synchronization (VERDICT r1 Next 7: one sync
// per one-shot call instead of two).
gespmm_status_t build_plan_async(gespmm_plan_s* plan, const int* rowptr, const int* colind,
                                 bool check_colind, cudaStream_t s) {
  NvtxRange nvtx("gespmm:plan_build_async");
  keep_pool_resident();
  const int64_t M = plan->M;
  const int M32 = static_cast<int>(M);
  const int nnz32 = static_cast<int>(plan->nnz);
  cudaError_t ce;
  plan->async_counts = true;
  if (!plan->meta) {
    ce = cudaMallocAsync(&plan->meta, sizeof(gespmm_plan_s::Meta), s);
    if (ce == cudaSuccess) ce = cudaMallocHost(&plan->meta_host, sizeof(gespmm_plan_s::Meta));
    if (ce != cudaSuccess) return cuda_fail(ce, "plan meta");
  }
  const int tw = tile_work_for(M, plan->nnz);
  plan->tile_work = tw;
  int64_t ub_items = 0, ub_segs = 0;
  plan_bounds(M, plan->nnz, tw, &ub_items, &ub_segs);
  plan->n_items = M > 0 ? ub_items : 0;
  plan->n_segs = ub_segs;
  plan->n_tiles = plan->n_long = -1;  // known on the device only
  if (M == 0) {
    plan->n_items = 0;
    if (plan->nnz != 0) return fail(GESPMM_CSR_INVALID, "invalid csr: rowPtr end differs from nnz of colInd");
    return GESPMM_OK;
  }
  if (!plan->items || plan->items_cap < ub_items + 1) {
    if (plan->items) cudaFree(plan->items);
    plan->items = nullptr;
    plan->items_cap = 0;
    ce = cudaMallocAsync(&plan->items, static_cast<size_t>(ub_items + 1) * sizeof(int4), s);
    if (ce != cudaSuccess) return cuda_fail(ce, "plan items");
    plan->items_cap = ub_items + 1;
  }
  uint64_t *packed = nullptr, *E = nullptr;
  int *cnt = nullptr, *pos = nullptr, *err = nullptr;
  void* tmp = nullptr;
  size_t tmp1 = 0, tmp2 = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, tmp1, packed, E, M32, s);
  cub::DeviceScan::ExclusiveSum(nullptr, tmp2, cnt, pos, M32, s);
  const size_t tmp_bytes = tmp1 > tmp2 ? tmp1 : tmp2;
  const size_t bytes = M * (8 + 8 + 4 + 4) + 64 + tmp_bytes + 8 * 256;
  char* arena = nullptr;
  ce = cudaMallocAsync(&arena, bytes, s);
  if (ce != cudaSuccess) return cuda_fail(ce, "plan temporaries");
  {
    char* p = arena;
    auto take = [&](size_t n) {
      char* r = p;
      p += (n + 255) & ~size_t(255);
      return r;
    };
    packed = reinterpret_cast<uint64_t*>(take(M * 8));
    E = reinterpret_cast<uint64_t*>(take(M * 8));
    cnt = reinterpret_cast<int*>(take(M * 4));
    pos = reinterpret_cast<int*>(take(M * 4));
    err = reinterpret_cast<int*>(take(64));
    tmp = take(tmp_bytes);
  }
  const unsigned blocks = static_cast<unsigned>((M + 255) / 256);
  cudaMemsetAsync(err, 0, 2 * sizeof(int), s);
  k_rows<<<blocks, 256, 0, s>>>(rowptr, M32, nnz32, packed, err);
  if (check_colind && plan->nnz > 0) {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    int64_t cblocks = (plan->nnz + 255) / 256;
    if (cblocks > 4 * sms) cblocks = 4 * sms;
    k_colind<<<static_cast<unsigned>(cblocks), 256, 0, s>>>(colind, plan->nnz, static_cast<int>(plan->K), err);
  }
  size_t tb = tmp_bytes;
  cub::DeviceScan::ExclusiveSum(tmp, tb, packed, E, M32, s);
  k_count<<<blocks, 256, 0, s>>>(packed, E, M32, tw, cnt);
  tb = tmp_bytes;
  cub::DeviceScan::ExclusiveSum(tmp, tb, cnt, pos, M32, s);
  k_emit<<<blocks, 256, 0, s>>>(rowptr, packed, E, pos, M32, tw, plan->items, ub_items);
  k_meta<<<1, 1, 0, s>>>(packed, E, cnt, pos, M32, nnz32, err, ub_items, plan->items, plan->meta);
  ce = cudaGetLastError();
  cudaFreeAsync(arena, s);
  if (ce != cudaSuccess) return cuda_fail(ce, "plan build");
  return GESPMM_OK;
}

}  // namespace gespmm
