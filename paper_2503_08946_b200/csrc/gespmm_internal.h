// gespmm_internal.h -- shared between the plan builder, the SpMM kernels and
// the C-ABI layer.  Not part of the public boundary (include/gespmm.h is).
#pragma once

#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>

#include <cstdint>
#include <string>

#include "gespmm.h"

namespace gespmm {

// ---- work decomposition constants ------------------------
// Long rows (deg > kSeg) are cut into kSeg-long segments from the row start.
constexpr int kSeg = GESPMM_SEGMENT_LEN;
// A tile is a run of consecutive short rows worth ~tile_work work units, where a
// row costs deg + kRowCost (the row cost accounts for its C-row store).
// tile_work is a power of two in [kMinTileWork, kTileWork], chosen per plan
// from (nnz, M) alone (never the device): the largest one that still gives
// every warp slot of a 148-SM B200 (x2) an item, so small matrices are not
// latency-bound on a few long warps (tile_work_for).
#ifndef GESPMM_TILE_MAX
#define GESPMM_TILE_MAX 256
#endif
constexpr int kTileWork = GESPMM_TILE_MAX;
constexpr int kMinTileWork = 16;
constexpr int kRowCost = 2;
// Rows per tile are bounded: every short row advances the work prefix by >= kRowCost.
constexpr int kTileMaxRows = kTileWork / kRowCost;
// Kernel geometry: one warp per work item, 8 warps per CTA.
constexpr int kWarpsPerBlock = 8;
// Per-warp shared-memory stage for one item's (col, val) stream.  An item holds
// at most kTileWork + kSeg + kRowCost - 1 nonzeros (a tile) or kSeg (a segment);
// staging starts at the 16-byte-aligned position below the item start.
// 576: 8 warps x 576 x 8 B = 36.9 KB per CTA, so three CTAs fit per SM next
// to the gather ring (8 x 4 KB); the bound below covers the 4-alignment of the
// stage start and the rounding of its end up to a batch of (at most) 12.
#ifndef GESPMM_STAGE_CAP
#define GESPMM_STAGE_CAP 576
#endif
constexpr int kStageCap = GESPMM_STAGE_CAP;
static_assert(kTileWork + kSeg + kRowCost + 2 + 3 + 12 <= kStageCap, "stage too small for the largest item");
// Low 40 bits of the packed plan scan carry tile work, high 24 bits segment counts.
constexpr int kPackShift = 40;
// Column panels: B slabs larger than this are processed in column panels
// (gespmm_capi.cu panel_width); panels are at least GESPMM_PANEL_MIN columns.
#ifndef GESPMM_PANEL_L2_MB
#define GESPMM_PANEL_L2_MB 80
#endif
#ifndef GESPMM_PANEL_MIN
#define GESPMM_PANEL_MIN 64
#endif

// Pipelined host path: at most this many row chunks per call.
constexpr int kMaxChunks = 64;
// Items are distributed to warps dynamically (an atomic counter per column
// block) rather than by static warp striding.
#ifndef GESPMM_DYN
#define GESPMM_DYN 1
#endif
constexpr int64_t kDynMinItems = 16384;  // below: static warp striding
// Long-row segment tickets: acq_rel atomic by one lane (1) or full fences (0).
#ifndef GESPMM_TICKET_ACQREL
#define GESPMM_TICKET_ACQREL 1
#endif
// Fused all-gather: at most this many destination buffers (one node's GPUs).
constexpr int kMaxPeers = 8;

// Kernel variant: VEC fp32 columns per lane per load (1, 2 or 4) and CWM column
// tiles per warp (Coarse-grained Warp Merging); one warp covers 32*VEC*CWM
// columns of one column block.  `pair`: the paired-lane sum/mean kernel
// (gespmm_kernel_pair.cuh), 16 lanes x VEC columns, two nonzeros per warp step.
struct Variant {
  int vec = 1;
  int cwm = 1;
  bool pair = false;
  bool ring = false;  // B rows through the shared-memory cp.async ring (gespmm_kernel.cuh Ring)
};

// Everything the SpMM kernel reads.  Passed by value (kernel parameter space).
struct KParams {
  const int* rowptr;
  const int* colind;
  const float* vals;
  const float* B;
  float* C;
  int64_t ldb, ldc, N;
  int64_t ldp;             // leading dimension of the long-row partials
  const int4* items;       // {row, seg (-1 = tile), rowptr[row], slot base}
  int64_t n_items;
  int M;
  int nnz;
  float* partials;         // [n_segments][ldp]
  int* counters;           // [n_segments][ncb], zero between launches
  int accumulate;
  int ncb;                 // column blocks (gridDim.y)
  int idx_aligned;         // colind and vals 16-byte aligned -> 128-bit staging loads
  int off32;               // K*ldb <= 2^32: stage 32-bit B-row element offsets
  // Pipelined host path (gespmm_csr_spmm_host): the launch runs items
  // [range[0], range[1]) only (nullptr: all); it returns at once when
  // abort_flag is non-null and *abort_flag is set (a failed on-device colind
  // check of this or an earlier chunk, with or without a range).
  const int64_t* range;
  const int* abort_flag;
  // one-shot plans built without a host sync (build_plan_async): the true
  // item count lives on the device (n_items above is its upper bound)
  const int64_t* n_items_dev;
  // Fused C all-gather (gespmm_plan_execute_peers): every C row is also stored
  // at peers[q] + peer_shift + (its offset from C), q < n_peers -- peer GPUs'
  // full-C buffers (CUDA IPC over NVLink) or this GPU's own.
  float* peers[kMaxPeers];
  int n_peers;
  int64_t peer_shift;
  // dynamic item distribution: one counter per column block, zero at launch
  unsigned long long* work_ctr;
};

// GESPMM_TRACE=1: phase timings of the host entry point and the plan build on
// stderr (each phase is synchronized; diagnostics only).
struct Trace {
  bool on = false, sync = false;
  double t0 = 0, last = 0;
  const char* scope = "";
  explicit Trace(const char* s);
  void mark(const char* phase, cudaStream_t stream);
};

// NVTX range for the host-side phases (plan build, execute, the pipelined
// host entry point, the sharded path): visible in nsys / ncu --nvtx timelines.
// Header-only NVTX v3: a no-op unless a profiler injects its library.
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};

void set_error(const std::string& msg);
gespmm_status_t fail(gespmm_status_t s, const std::string& msg);
gespmm_status_t cuda_fail(cudaError_t e, const char* what);

Variant choose_variant(int64_t N, const float* B, int64_t ldb, const float* C, int64_t ldc,
                       gespmm_reduce_t op);
int variant_cols(const Variant& v);
std::string variant_name(const Variant& v);
bool parse_variant(const char* name, Variant* v);

cudaError_t launch_spmm(gespmm_reduce_t op, const Variant& v, const KParams& p,
                        cudaStream_t stream);

}  // namespace gespmm

// Plan object behind the opaque gespmm_plan_t.
struct gespmm_plan_s {
  int64_t M = 0, K = 0, nnz = 0;
  int4* items = nullptr;
  int64_t items_cap = 0;
  int64_t n_items = 0, n_tiles = 0, n_long = 0, n_segs = 0;
  float* partials = nullptr;
  int64_t partial_floats = 0;
  int* counters = nullptr;
  int64_t* row_range = nullptr;
  unsigned long long* work_ctr = nullptr;  // per column block item counters (GESPMM_DYN)
  int64_t work_ctr_n = 0;  // [2] items of the current execute_rows chunk (+ a zero abort flag)
  int64_t counter_ints = 0;
  int tile_work = gespmm::kTileWork;
  int device = 0;
  // build_plan_async (the one-shot entry point): counts and the CSR error
  // bits stay on the device (meta); n_items / n_segs hold upper bounds and
  // every launch reads the true count and aborts on an error bit
  struct Meta {
    int64_t n_items, n_segs;
    int err, n_long;
  };
  Meta* meta = nullptr;       // device (pool)
  Meta* meta_host = nullptr;  // pinned mirror, read after the caller's sync
  bool async_counts = false;
  std::string last_variant;  // the kernel variant of the last execute (diagnostics)
};

namespace gespmm {
// The one-shot plan build with no host synchronization (gespmm_plan.cu).
gespmm_status_t build_plan_async(gespmm_plan_s* plan, const int* rowptr, const int* colind,
                                 bool check_colind, cudaStream_t s);
std::string csr_error_message(int err, int64_t K);
}  // namespace gespmm
