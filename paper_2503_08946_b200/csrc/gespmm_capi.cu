// gespmm_capi.cu -- the extern "C" boundary (include/gespmm.h).
//
// Replaces the reference's hot-path surface:
//   raceset::validate_instance  (src/oracle.cpp:291-316)  -> gespmm_validate_csr[_device]
//   raceset::run on gespmm_alg2 (src/oracle.cpp:699-736)  -> gespmm_csr_spmm[_host]
// Reference errors are C++ exceptions raceset::Error{ErrorKind}
// (include/raceset/error.hpp:36-56); here they are status codes plus a
// thread-local detail string with the same wording.
#include <dlfcn.h>

#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <algorithm>
#include <mutex>
#include <string>

#include "gespmm_internal.h"

namespace gespmm {

gespmm_status_t build_plan(gespmm_plan_s* plan, const int* rowptr, const int* colind,
                           bool check_colind, cudaStream_t s);
gespmm_status_t device_validate_colind(const int* colind, int64_t nnz, int64_t K, cudaStream_t s);
cudaError_t chunk_ranges(const gespmm_plan_s* plan, const int64_t* rows, int nc, int64_t* d_ranges,
                         cudaStream_t s);
cudaError_t row_item_range(const gespmm_plan_s* plan, const int64_t* rows, int64_t* d_range,
                           cudaStream_t s);
cudaError_t chunk_rows_aligned(const gespmm_plan_s* plan, const int64_t* rows, int nc, int64_t* d_ranges,
                               int64_t* d_rows, cudaStream_t s);
cudaError_t validate_colind_async(const int* colind, int64_t p0, int64_t p1, int64_t K, int* err,
                                  cudaStream_t s);
std::string csr_error_message(int err, int64_t K);
extern int g_tile_work_override;

namespace {
thread_local std::string g_last_error;
std::string g_variant_override;  // test hook; "" = heuristic
}  // namespace

void set_error(const std::string& msg) { g_last_error = msg; }

static double now_ms() {
  return std::chrono::duration<double, std::milli>(
             std::chrono::steady_clock::now().time_since_epoch())
      .count();
}

// GESPMM_TRACE=1: synchronize at each mark (device phase times);
// GESPMM_TRACE=2: host timestamps only (where the host thread blocks);
// GESPMM_TRACE=3: no marks; the pipelined host entry prints its device
// timeline (per-chunk copy / launch completion events, no added syncs).
Trace::Trace(const char* s) : scope(s) {
  const char* e = std::getenv("GESPMM_TRACE");
  on = e && *e && *e != '0' && *e != '3';
  sync = on && *e != '2';
  if (on) t0 = last = now_ms();
}

void Trace::mark(const char* phase, cudaStream_t stream) {
  if (!on) return;
  if (sync) cudaStreamSynchronize(stream);
  const double t = now_ms();
  std::fprintf(stderr, "[gespmm trace] %s %-24s %8.3f ms (total %8.3f)\n", scope, phase, t - last,
               t - t0);
  last = t;
}

gespmm_status_t fail(gespmm_status_t s, const std::string& msg) {
  g_last_error = msg;
  return s;
}

gespmm_status_t cuda_fail(cudaError_t e, const char* what) {
  g_last_error = std::string(what) + ": " + cudaGetErrorString(e);
  return GESPMM_CUDA_ERROR;
}

namespace {

cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

// A plan lives on the device it was built on: its calls switch to that device
// for their duration (workspace allocations, counters and launches) and
// restore the caller's current device afterwards.
struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    if (cudaGetDevice(&prev) == cudaSuccess && prev != dev) cudaSetDevice(dev);
    else prev = -1;
  }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

// Shape/argument checks shared by the device and host entry points.
gespmm_status_t check_shape(int64_t M, int64_t K, int64_t N, int64_t nnz, int64_t ldb,
                            int64_t ldc) {
  if (M < 0 || K < 0 || N < 1 || nnz < 0)
    return fail(GESPMM_INVALID_ARG, "invalid argument: need M, K, nnz >= 0 and N >= 1");
  if (ldb < N || ldc < N) return fail(GESPMM_INVALID_ARG, "invalid argument: ldb and ldc must be >= N");
  // int32 indices: nonzero positions and rows are int32 (gespmm_alg2.mir:5 i32
  // params); leave headroom for the 128-wide staging arithmetic.
  if (nnz > (int64_t(1) << 31) - 1024 || M > (int64_t(1) << 31) - 2 || K > (int64_t(1) << 31) - 1)
    return fail(GESPMM_INVALID_ARG, "invalid argument: M, K and nnz must fit int32 indexing");
  return GESPMM_OK;
}

Variant pick_variant(int64_t N, const float* B, int64_t ldb, const float* C, int64_t ldc,
                     gespmm_reduce_t op) {
  Variant v = choose_variant(N, B, ldb, C, ldc, op);
  if (!g_variant_override.empty()) {
    Variant o;
    if (parse_variant(g_variant_override.c_str(), &o)) {
      auto ok = [&](int vec) {
        const uintptr_t a = static_cast<uintptr_t>(vec) * 4;
        return reinterpret_cast<uintptr_t>(B) % a == 0 && reinterpret_cast<uintptr_t>(C) % a == 0 &&
               ldb % vec == 0 && ldc % vec == 0 && N % vec == 0;
      };
      if (ok(o.vec)) v = o;
    }
  }
  return v;
}

// Plan-owned device buffers (items, partials, counters, work counters, the
// one-shot plan's meta) come from the device's stream-ordered pool (cudaMallocAsync on the
// plan's stream; the pool keeps its memory mapped, gespmm_plan.cu
// keep_pool_resident), so a fresh plan costs no cudaMalloc round trip
// (config 2: 1.46 ms per fresh Plan with cudaMalloc); grow-only, released with
// cudaFree (synchronizing) in gespmm_plan_destroy.
gespmm_status_t ensure_workspace(gespmm_plan_s* plan, int64_t ldp, int ncb, cudaStream_t s) {
  if (plan->n_segs == 0) return GESPMM_OK;
  const int64_t need_p = plan->n_segs * ldp;
  if (need_p > plan->partial_floats) {
    if (plan->partials) cudaFree(plan->partials);
    plan->partials = nullptr;
    plan->partial_floats = 0;
    cudaError_t e = cudaMallocAsync(&plan->partials, static_cast<size_t>(need_p) * sizeof(float), s);
    if (e != cudaSuccess) return cuda_fail(e, "plan partials");
    plan->partial_floats = need_p;
  }
  const int64_t need_c = plan->n_segs * ncb;
  if (need_c > plan->counter_ints) {
    if (plan->counters) cudaFree(plan->counters);
    plan->counters = nullptr;
    plan->counter_ints = 0;
    cudaError_t e = cudaMallocAsync(&plan->counters, static_cast<size_t>(need_c) * sizeof(int), s);
    if (e != cudaSuccess) return cuda_fail(e, "plan counters");
    e = cudaMemsetAsync(plan->counters, 0, static_cast<size_t>(need_c) * sizeof(int), s);
    if (e != cudaSuccess) return cuda_fail(e, "plan counters memset");
    plan->counter_ints = need_c;
  }
  return GESPMM_OK;
}

std::mutex& host_ws_mutex() {
  static std::mutex m;
  return m;
}

// The host entry point's plan, one per device, re-planned in place per call.
gespmm_plan_s* host_plan() {
  static gespmm_plan_s* plans[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  gespmm_plan_s*& p = plans[dev & 63];
  if (!p) {
    p = new gespmm_plan_s();
    p->device = dev;
  }
  return p;
}

// Copy streams + events of the pipelined host entry point, one set per device.
struct Pipe {
  cudaStream_t in = nullptr, out = nullptr;
  cudaEvent_t ev[2 + 2 * kMaxChunks] = {};
};
gespmm_status_t pipe_streams(Pipe** out) {
  static Pipe pipes[64];
  int dev = 0;
  cudaGetDevice(&dev);
  Pipe& x = pipes[dev & 63];
  if (!x.in) {
    cudaError_t e = cudaStreamCreateWithFlags(&x.in, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&x.out, cudaStreamNonBlocking);
    for (auto& ev : x.ev)
      if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
    if (e != cudaSuccess) return cuda_fail(e, "host pipeline streams");
  }
  *out = &x;
  return GESPMM_OK;
}

// Grow-only device workspace for the host entry point, one per device.
gespmm_status_t host_workspace(int64_t bytes, char** out) {
  struct Ws {
    char* p = nullptr;
    int64_t cap = 0;
  };
  static Ws ws[64];
  int dev = 0;
  cudaGetDevice(&dev);
  Ws& w = ws[dev & 63];
  if (bytes > w.cap) {
    if (w.p) cudaFree(w.p);
    w.p = nullptr;
    w.cap = 0;
    cudaError_t e = cudaMalloc(&w.p, static_cast<size_t>(bytes > 0 ? bytes : 256));
    if (e != cudaSuccess) return cuda_fail(e, "host-path workspace");
    w.cap = bytes;
  }
  *out = w.p;
  return GESPMM_OK;
}

// Panel width for an N-column product over K B-rows.  GESPMM_PANEL=<cols>
// overrides (0 = one panel); otherwise a single panel unless K x N x 4 bytes
// exceeds the L2 budget, then the widest power-of-two panel (>= kMinPanel
// columns) whose slab fits; no panels when even the narrowest slab does not fit.
int g_schedule_override = -1;  // -1 auto, 0 static striding, 1 dynamic counter

int64_t g_panel_override = [] {
  const char* e = std::getenv("GESPMM_PANEL");
  return e ? static_cast<int64_t>(std::atoll(e)) : int64_t(-1);
}();

int64_t panel_width(int64_t K, int64_t N) {
  const int64_t forced = g_panel_override;
  if (forced == 0) return N;
  if (forced > 0) return forced < N ? forced : N;
  constexpr int64_t kL2Budget = int64_t(GESPMM_PANEL_L2_MB) << 20;
  constexpr int64_t kMinPanel = GESPMM_PANEL_MIN;
  // measured (profiles/r1_panels.txt): Reddit-like K=233K, N=256 -> 64-column
  // panels (60 MB slabs) 12.47 -> 9.05 ms; R-MAT K=4M, N=128, where even a
  // 64-column slab (1 GB) exceeds L2, panels only re-stream the CSR (3.04 ->
  // 3.29 ms): so panel only when the narrowest panel's slab fits.
  if (K * N * 4 <= kL2Budget || K * kMinPanel * 4 > kL2Budget) return N;
  int64_t w = 256;
  while (w > kMinPanel && K * w * 4 > kL2Budget) w /= 2;
  return w < N ? w : N;
}

// The launches of one execute (one per column panel), optionally restricted
// to the item range *range (device memory) with an on-device abort flag.
gespmm_status_t execute_range(gespmm_plan_s* plan, int64_t N, const int32_t* rowptr,
                              const int32_t* colind, const float* vals, const float* B, int64_t ldb,
                              float* C, int64_t ldc, gespmm_reduce_t op, int accumulate,
                              const int64_t* range, const int* abort_flag, cudaStream_t s,
                              float* const* peers = nullptr, int n_peers = 0, int64_t peer_shift = 0) {
  NvtxRange nvtx(n_peers > 0 ? "gespmm:execute_peers" : range ? "gespmm:execute_range" : "gespmm:execute");
  gespmm_status_t st = GESPMM_OK;
  // Column panels (DESIGN.md 5.2 "Panels"): when B's row slab K x N does not
  // fit in L2, the columns are processed in panels of `pw` columns, one launch
  // per panel on the same stream, so the gathered B working set of each launch
  // is K x pw and stays L2-resident; colind/vals are re-streamed per panel.
  // Per-column arithmetic is unchanged (columns are independent).
  const int64_t pw = panel_width(plan->K, N);
  const int64_t ldp = (N + 3) & ~int64_t(3);
  for (int64_t c0 = 0; c0 < N; c0 += pw) {
    const int64_t n = N - c0 < pw ? N - c0 : pw;
    Variant v = pick_variant(n, B + c0, ldb, C + c0, ldc, op);
    if (n_peers > 0) {  // the fused-gather stores live in the 32-lane register kernel
      v.pair = false;
      v.ring = false;
    }
    const int ncb = static_cast<int>((n + variant_cols(v) - 1) / variant_cols(v));
    if (ncb > 65535) return fail(GESPMM_INVALID_ARG, "invalid argument: N too large");
    st = ensure_workspace(plan, ldp, ncb, s);
    if (st != GESPMM_OK) return st;
    KParams p{};
    p.rowptr = rowptr;
    p.colind = colind;
    p.vals = vals;
    p.B = B + c0;
    p.C = C + c0;
    p.ldb = ldb;
    p.ldc = ldc;
    p.N = n;
    p.ldp = ldp;
    p.items = plan->items;
    p.n_items = plan->n_items;
    p.M = static_cast<int>(plan->M);
    p.nnz = static_cast<int>(plan->nnz);
    p.partials = plan->partials;
    p.counters = plan->counters;
    p.accumulate = accumulate ? 1 : 0;
    p.ncb = ncb;
    p.idx_aligned = (reinterpret_cast<uintptr_t>(colind) % 16 == 0) &&
                    (reinterpret_cast<uintptr_t>(vals) % 16 == 0);
    p.off32 = plan->K * ldb <= (int64_t(1) << 32);
    p.range = range;
    p.abort_flag = abort_flag;
    p.n_items_dev = nullptr;
    if (plan->async_counts) {  // build_plan_async: true count + error bits on the device
      p.n_items_dev = &plan->meta->n_items;
      if (!p.abort_flag) p.abort_flag = &plan->meta->err;
    }
    // Dynamic item distribution for launches with enough items to balance
    // (config 1's 1.3 K items ran 0.018 -> 0.029 ms dynamic: the counter reset
    // dominates); the counters (one per column block) are zeroed on the
    // stream ahead of the launch.
    p.work_ctr = nullptr;
    // (item-range launches -- row chunks of the pipelined host path and of
    // execute_rows -- are a few thousand items each: static)
    const bool dyn = g_schedule_override >= 0 ? g_schedule_override == 1
                                              : (GESPMM_DYN && !range && plan->n_items >= kDynMinItems);
    if (dyn) {
      if (plan->work_ctr_n < ncb) {
        if (plan->work_ctr) cudaFree(plan->work_ctr);
        plan->work_ctr = nullptr;
        plan->work_ctr_n = 0;
        cudaError_t e = cudaMallocAsync(&plan->work_ctr, static_cast<size_t>(ncb) * 8, s);
        if (e != cudaSuccess) return cuda_fail(e, "plan work counters");
        plan->work_ctr_n = ncb;
      }
      cudaError_t e = cudaMemsetAsync(plan->work_ctr, 0, static_cast<size_t>(ncb) * 8, s);
      if (e != cudaSuccess) return cuda_fail(e, "work counter reset");
      p.work_ctr = plan->work_ctr;
    }
    p.n_peers = n_peers;
    p.peer_shift = peer_shift;
    for (int q = 0; q < n_peers; ++q) p.peers[q] = peers[q] + c0;  // this panel's columns
    plan->last_variant = variant_name(v);
    cudaError_t e = launch_spmm(op, v, p, s);
    if (e != cudaSuccess) return cuda_fail(e, "spmm launch");
  }
  return GESPMM_OK;
}

}  // namespace
}  // namespace gespmm

using namespace gespmm;

extern "C" {

int gespmm_version(void) { return GESPMM_VERSION_MAJOR * 100 + GESPMM_VERSION_MINOR; }

const char* gespmm_status_string(gespmm_status_t s) {
  switch (s) {
    case GESPMM_OK: return "ok";
    case GESPMM_CSR_INVALID: return "invalid csr";          // ErrorKind::CsrInvalid
    case GESPMM_OUT_OF_BOUNDS: return "out of bounds";      // ErrorKind::OutOfBounds
    case GESPMM_INVALID_ARG: return "invalid argument";
    case GESPMM_CUDA_ERROR: return "cuda error";
    case GESPMM_NCCL_ERROR: return "nccl error";
    case GESPMM_NOT_SUPPORTED: return "not supported";
  }
  return "unknown status";
}

const char* gespmm_last_error(void) { return g_last_error.c_str(); }

gespmm_status_t gespmm_validate_csr(int64_t M, int64_t K, int64_t rowptr_len,
                                    const int32_t* rowptr, int64_t colind_len,
                                    const int32_t* colind, int64_t vals_len) {
  g_last_error.clear();
  if (M < 0 || K < 0 || rowptr_len < 0 || colind_len < 0 || vals_len < 0)
    return fail(GESPMM_INVALID_ARG, "invalid argument: negative size");
  if ((rowptr_len > 0 && !rowptr) || (colind_len > 0 && !colind))
    return fail(GESPMM_INVALID_ARG, "invalid argument: null pointer");
  // reference src/oracle.cpp:302-315, in the same order
  if (rowptr_len == 0 || rowptr[0] != 0) return fail(GESPMM_CSR_INVALID, "invalid csr: rowPtr[0] must be 0");
  for (int64_t i = 1; i < rowptr_len; ++i)
    if (rowptr[i] < rowptr[i - 1])
      return fail(GESPMM_CSR_INVALID, "invalid csr: rowPtr must be nondecreasing");
  if (static_cast<int64_t>(rowptr[rowptr_len - 1]) != colind_len)
    return fail(GESPMM_CSR_INVALID, "invalid csr: rowPtr end differs from nnz of colInd");
  if (colind_len != vals_len)
    return fail(GESPMM_CSR_INVALID, "invalid csr: colInd and val lengths differ");
  for (int64_t p = 0; p < colind_len; ++p)
    if (colind[p] < 0 || colind[p] >= K)
      return fail(GESPMM_CSR_INVALID,
                  "invalid csr: colInd entry out of [0," + std::to_string(K) + ")");
  // added: the kernel reads rowPtr[i+1] for every row i < M (gespmm_alg2.mir:16-18)
  if (rowptr_len != M + 1) return fail(GESPMM_CSR_INVALID, "invalid csr: rowPtr length must be M + 1");
  return GESPMM_OK;
}

gespmm_status_t gespmm_validate_csr_device(int64_t M, int64_t K, int64_t nnz,
                                           const int32_t* rowptr, const int32_t* colind,
                                           void* stream) {
  g_last_error.clear();
  if (M < 0 || K < 0 || nnz < 0) return fail(GESPMM_INVALID_ARG, "invalid argument: negative size");
  gespmm_status_t st0 = check_shape(M, K, 1, nnz, 1, 1);
  if (st0 != GESPMM_OK) return st0;
  if ((M > 0 && !rowptr) || (nnz > 0 && !colind))
    return fail(GESPMM_INVALID_ARG, "invalid argument: null pointer");
  gespmm_plan_s tmp;
  tmp.M = M;
  tmp.K = K;
  tmp.nnz = nnz;
  gespmm_status_t st = build_plan(&tmp, rowptr, colind, true, as_stream(stream));
  if (tmp.items) cudaFree(tmp.items);
  return st;
}

gespmm_status_t gespmm_plan_create(gespmm_plan_t* plan, int64_t M, int64_t K, int64_t nnz,
                                   const int32_t* rowptr, const int32_t* colind, int flags,
                                   void* stream) {
  g_last_error.clear();
  if (!plan) return fail(GESPMM_INVALID_ARG, "invalid argument: plan is null");
  *plan = nullptr;
  gespmm_status_t st = check_shape(M, K, 1, nnz, 1, 1);
  if (st != GESPMM_OK) return st;
  if (M > 0 && !rowptr) return fail(GESPMM_INVALID_ARG, "invalid argument: rowptr is null");
  auto* p = new gespmm_plan_s();
  p->M = M;
  p->K = K;
  p->nnz = nnz;
  cudaGetDevice(&p->device);
  st = build_plan(p, rowptr, colind, (flags & 1) != 0, as_stream(stream));
  if (st != GESPMM_OK) {
    gespmm_plan_destroy(p);
    return st;
  }
  *plan = p;
  return GESPMM_OK;
}

gespmm_status_t gespmm_plan_execute(gespmm_plan_t plan, int64_t N, const int32_t* rowptr,
                                    const int32_t* colind, const float* vals, const float* B,
                                    int64_t ldb, float* C, int64_t ldc, gespmm_reduce_t op,
                                    int accumulate, void* stream) {
  if (!plan) return fail(GESPMM_INVALID_ARG, "invalid argument: plan is null");
  gespmm_status_t st = check_shape(plan->M, plan->K, N, plan->nnz, ldb, ldc);
  if (st != GESPMM_OK) return st;
  if (op < GESPMM_REDUCE_SUM || op > GESPMM_REDUCE_MEAN)
    return fail(GESPMM_INVALID_ARG, "invalid argument: unknown reduce op");
  if (plan->n_items == 0) return GESPMM_OK;  // M == 0
  if (!rowptr || (plan->nnz > 0 && (!colind || !vals || !B)) || !C)
    return fail(GESPMM_INVALID_ARG, "invalid argument: null pointer");
  DeviceGuard dg(plan->device);
  return execute_range(plan, N, rowptr, colind, vals, B, ldb, C, ldc, op, accumulate, nullptr,
                       nullptr, as_stream(stream));
}

gespmm_status_t gespmm_plan_execute_rows(gespmm_plan_t plan, int64_t row_begin, int64_t row_end,
                                         int64_t N, const int32_t* rowptr, const int32_t* colind,
                                         const float* vals, const float* B, int64_t ldb, float* C,
                                         int64_t ldc, gespmm_reduce_t op, int accumulate,
                                         void* stream) {
  if (!plan) return fail(GESPMM_INVALID_ARG, "invalid argument: plan is null");
  gespmm_status_t st = check_shape(plan->M, plan->K, N, plan->nnz, ldb, ldc);
  if (st != GESPMM_OK) return st;
  if (op < GESPMM_REDUCE_SUM || op > GESPMM_REDUCE_MEAN)
    return fail(GESPMM_INVALID_ARG, "invalid argument: unknown reduce op");
  if (row_begin < 0 || row_end < row_begin || row_end > plan->M)
    return fail(GESPMM_INVALID_ARG, "invalid argument: need 0 <= row_begin <= row_end <= M");
  if (plan->n_items == 0 || row_end == row_begin) return GESPMM_OK;
  if (!rowptr || (plan->nnz > 0 && (!colind || !vals || !B)) || !C)
    return fail(GESPMM_INVALID_ARG, "invalid argument: null pointer");
  DeviceGuard dg(plan->device);
  cudaStream_t s = as_stream(stream);
  if (!plan->row_range) {
    cudaError_t e = cudaMallocAsync(&plan->row_range, 4 * sizeof(int64_t), s);
    if (e == cudaSuccess) e = cudaMemsetAsync(plan->row_range, 0, 4 * sizeof(int64_t), s);
    if (e != cudaSuccess) return cuda_fail(e, "plan row range");
  }
  const int64_t rows[2] = {row_begin, row_end};
  cudaError_t e = row_item_range(plan, rows, plan->row_range, s);
  if (e != cudaSuccess) return cuda_fail(e, "row chunk range");
  return execute_range(plan, N, rowptr, colind, vals, B, ldb, C, ldc, op, accumulate,
                       plan->row_range, reinterpret_cast<const int*>(plan->row_range + 2), s);
}

gespmm_status_t gespmm_plan_execute_peers(gespmm_plan_t plan, int64_t N, const int32_t* rowptr,
                                          const int32_t* colind, const float* vals, const float* B,
                                          int64_t ldb, float* C, int64_t ldc, gespmm_reduce_t op,
                                          int accumulate, float* const* peers, int n_peers,
                                          int64_t peer_row0, void* stream) {
  if (!plan) return fail(GESPMM_INVALID_ARG, "invalid argument: plan is null");
  gespmm_status_t st = check_shape(plan->M, plan->K, N, plan->nnz, ldb, ldc);
  if (st != GESPMM_OK) return st;
  if (op < GESPMM_REDUCE_SUM || op > GESPMM_REDUCE_MEAN)
    return fail(GESPMM_INVALID_ARG, "invalid argument: unknown reduce op");
  if (n_peers < 0 || n_peers > kMaxPeers || (n_peers > 0 && !peers) || peer_row0 < 0)
    return fail(GESPMM_INVALID_ARG, "invalid argument: need 0 <= n_peers <= 8 and peer_row0 >= 0");
  for (int q = 0; q < n_peers; ++q)
    if (!peers[q]) return fail(GESPMM_INVALID_ARG, "invalid argument: null peer buffer");
  if (plan->n_items == 0) return GESPMM_OK;
  if (!rowptr || (plan->nnz > 0 && (!colind || !vals || !B)) || !C)
    return fail(GESPMM_INVALID_ARG, "invalid argument: null pointer");
  DeviceGuard dg(plan->device);
  return execute_range(plan, N, rowptr, colind, vals, B, ldb, C, ldc, op, accumulate, nullptr, nullptr,
                       as_stream(stream), peers, n_peers, peer_row0 * ldc);
}

gespmm_status_t gespmm_ipc_get_handle(void* dev_ptr, char handle[64], int64_t* offset) {
  if (!dev_ptr || !handle || !offset) return fail(GESPMM_INVALID_ARG, "invalid argument: ipc handle");
  // the handle names the whole allocation (e.g. a torch caching-allocator
  // segment); the peer adds the offset of dev_ptr inside it
  using GetRange = int (*)(unsigned long long*, size_t*, unsigned long long);
  static GetRange get_range = [] {
    void* h = dlopen("libcuda.so.1", RTLD_NOW | RTLD_GLOBAL);
    return h ? reinterpret_cast<GetRange>(dlsym(h, "cuMemGetAddressRange_v2")) : nullptr;
  }();
  if (!get_range) return fail(GESPMM_NOT_SUPPORTED, "cuMemGetAddressRange_v2 unavailable");
  unsigned long long base = 0;
  size_t size = 0;
  if (get_range(&base, &size, reinterpret_cast<unsigned long long>(dev_ptr)) != 0)
    return fail(GESPMM_INVALID_ARG, "invalid argument: not a device allocation");
  cudaIpcMemHandle_t h;
  cudaError_t e = cudaIpcGetMemHandle(&h, reinterpret_cast<void*>(base));
  if (e != cudaSuccess) return cuda_fail(e, "cudaIpcGetMemHandle");
  static_assert(sizeof(h) == 64, "cudaIpcMemHandle_t is 64 bytes");
  std::memcpy(handle, &h, 64);
  *offset = static_cast<int64_t>(reinterpret_cast<unsigned long long>(dev_ptr) - base);
  return GESPMM_OK;
}

gespmm_status_t gespmm_ipc_open_handle(const char handle[64], void** dev_ptr) {
  if (!dev_ptr || !handle) return fail(GESPMM_INVALID_ARG, "invalid argument: ipc handle");
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle, 64);
  cudaError_t e = cudaIpcOpenMemHandle(dev_ptr, h, cudaIpcMemLazyEnablePeerAccess);
  if (e != cudaSuccess) return cuda_fail(e, "cudaIpcOpenMemHandle");
  return GESPMM_OK;
}

gespmm_status_t gespmm_ipc_close_handle(void* dev_ptr) {
  if (!dev_ptr) return GESPMM_OK;
  cudaError_t e = cudaIpcCloseMemHandle(dev_ptr);
  if (e != cudaSuccess) return cuda_fail(e, "cudaIpcCloseMemHandle");
  return GESPMM_OK;
}

gespmm_status_t gespmm_plan_destroy(gespmm_plan_t plan) {
  if (!plan) return GESPMM_OK;
  DeviceGuard dg(plan->device);
  if (plan->work_ctr) cudaFree(plan->work_ctr);
  if (plan->row_range) cudaFree(plan->row_range);
  if (plan->items) cudaFree(plan->items);
  if (plan->partials) cudaFree(plan->partials);
  if (plan->counters) cudaFree(plan->counters);
  if (plan->meta) cudaFree(plan->meta);
  if (plan->meta_host) cudaFreeHost(plan->meta_host);
  delete plan;
  return GESPMM_OK;
}

gespmm_status_t gespmm_plan_get_info(gespmm_plan_t plan, gespmm_plan_info_t* info) {
  if (!plan || !info) return fail(GESPMM_INVALID_ARG, "invalid argument: null");
  info->M = plan->M;
  info->nnz = plan->nnz;
  info->n_items = plan->n_items;
  info->n_tiles = plan->n_tiles;
  info->n_long_rows = plan->n_long;
  info->n_segments = plan->n_segs;
  info->segment_len = kSeg;
  info->tile_work = plan->tile_work;
  info->kernel_launches_per_execute = plan->n_items > 0 ? 1 : 0;
  return GESPMM_OK;
}

gespmm_status_t gespmm_csr_spmm(int64_t M, int64_t K, int64_t N, int64_t nnz,
                                const int32_t* rowptr, const int32_t* colind,
                                const float* vals, const float* B, int64_t ldb, float* C,
                                int64_t ldc, gespmm_reduce_t op, int accumulate, void* stream) {
  NvtxRange nvtx("gespmm:csr_spmm");
  g_last_error.clear();
  gespmm_status_t st = check_shape(M, K, N, nnz, ldb, ldc);
  if (st != GESPMM_OK) return st;
  if ((M > 0 && !rowptr) || (nnz > 0 && (!colind || !vals)) || (K * N > 0 && !B) || (M * N > 0 && !C))
    return fail(GESPMM_INVALID_ARG, "invalid argument: null pointer");
  if (op < GESPMM_REDUCE_SUM || op > GESPMM_REDUCE_MEAN)
    return fail(GESPMM_INVALID_ARG, "invalid argument: unknown reduce op");
  // A per-device plan object re-planned in place (no cudaMalloc/cudaFree per
  // call: cudaFree synchronizes the device); the call returns after its
  // launches drain, so the next call may reuse the plan's buffers.
  static std::mutex mu;
  std::lock_guard<std::mutex> lock(mu);
  static gespmm_plan_s* plans[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  gespmm_plan_s*& plan = plans[dev & 63];
  if (!plan) {
    plan = new gespmm_plan_s();
    plan->device = dev;
  }
  plan->M = M;
  plan->K = K;
  plan->nnz = nnz;
  // one synchronization per call: the plan is built on the device without a
  // host round trip (build_plan_async), the kernel reads its item count and
  // error bits there, and the bits come back with the trailing sync
  cudaStream_t cs = as_stream(stream);
  st = build_plan_async(plan, rowptr, colind, /*validate colind*/ true, cs);
  if (st != GESPMM_OK) return st;
  st = gespmm_plan_execute(plan, N, rowptr, colind, vals, B, ldb, C, ldc, op, accumulate, stream);
  if (st != GESPMM_OK) {
    cudaStreamSynchronize(cs);
    return st;
  }
  cudaError_t e = plan->n_items > 0 ? cudaMemcpyAsync(plan->meta_host, plan->meta, sizeof(*plan->meta),
                                                     cudaMemcpyDeviceToHost, cs)
                                   : cudaSuccess;
  const cudaError_t e2 = cudaStreamSynchronize(cs);
  if (e == cudaSuccess) e = e2;
  if (e != cudaSuccess) return cuda_fail(e, "spmm");
  if (plan->n_items > 0 && plan->meta_host->err)
    return fail(GESPMM_CSR_INVALID, csr_error_message(plan->meta_host->err, K));
  return GESPMM_OK;
}

gespmm_status_t gespmm_csr_spmm_host(int64_t M, int64_t K, int64_t N, int64_t nnz,
                                     const int32_t* rowptr, const int32_t* colind,
                                     const float* vals, const float* B, int64_t ldb, float* C,
                                     int64_t ldc, gespmm_reduce_t op, int accumulate,
                                     void* stream) {
  NvtxRange nvtx("gespmm:csr_spmm_host");
  g_last_error.clear();
  gespmm_status_t st = check_shape(M, K, N, nnz, ldb, ldc);
  if (st != GESPMM_OK) return st;
  if (op < GESPMM_REDUCE_SUM || op > GESPMM_REDUCE_MEAN)
    return fail(GESPMM_INVALID_ARG, "invalid argument: unknown reduce op");
  if ((M > 0 && !rowptr) || (nnz > 0 && (!colind || !vals)) || (K * N > 0 && !B) || (M * N > 0 && !C))
    return fail(GESPMM_INVALID_ARG, "invalid argument: null pointer");
  // The rowptr contract (reference src/oracle.cpp:302-307): its ends here,
  // monotonicity by the plan build on the device (before any launch); colind
  // range on the device per chunk, before that chunk's launch.
  if (M > 0 && rowptr[0] != 0) return fail(GESPMM_CSR_INVALID, "invalid csr: rowPtr[0] must be 0");
  if ((M > 0 ? static_cast<int64_t>(rowptr[M]) : 0) != nnz)
    return fail(GESPMM_CSR_INVALID, "invalid csr: rowPtr end differs from nnz of colInd");
  if (M == 0 || N == 0) return GESPMM_OK;
  cudaStream_t s = as_stream(stream);
  // One grow-only device workspace per device, reused across calls (a fresh
  // 0.7 GB allocation per call costs more than the kernel).
  std::lock_guard<std::mutex> lock(host_ws_mutex());
  Trace tr("host");
  auto al = [](int64_t bytes) { return (bytes + 255) & ~int64_t(255); };
  const int64_t b_rp = al((M + 1) * 4), b_ci = al(nnz * 4), b_v = al(nnz * 4),
                b_B = al(K * N * 4), b_C = al(M * N * 4), b_x = al(16 * (kMaxChunks + 1) + 64);
  char* ws = nullptr;
  st = host_workspace(b_rp + b_ci + b_v + b_B + b_C + b_x, &ws);
  if (st != GESPMM_OK) return st;
  auto* d_rp = reinterpret_cast<int32_t*>(ws);
  auto* d_ci = reinterpret_cast<int32_t*>(ws + b_rp);
  auto* d_v = reinterpret_cast<float*>(ws + b_rp + b_ci);
  auto* d_B = reinterpret_cast<float*>(ws + b_rp + b_ci + b_v);
  auto* d_C = reinterpret_cast<float*>(ws + b_rp + b_ci + b_v + b_B);
  auto* d_ranges = reinterpret_cast<int64_t*>(ws + b_rp + b_ci + b_v + b_B + b_C);
  auto* d_rows = d_ranges + kMaxChunks + 1;
  auto* d_err = reinterpret_cast<int*>(d_rows + kMaxChunks + 1);
  Pipe* pp = nullptr;
  st = pipe_streams(&pp);
  if (st != GESPMM_OK) return st;
  cudaStream_t s_in = pp->in, s_out = pp->out;
  tr.mark("workspace", s);

  // Row chunks of ~equal rows (= equal C bytes, equal D2H time), their
  // boundaries moved to item starts so every chunk's launch writes exactly
  // its own C rows (no tile spans two chunks); processed in order of
  // increasing nonzeros: C rows that need the least colind/vals go back to
  // the host first, so the D2H stream starts right after B arrives and the
  // heavy chunks' H2D overlaps the C drain (PCIe is full duplex).  R-MAT puts
  // a third of the nonzeros in the first 1/16 of the rows; in row order the
  // D2H stream idled behind them (11.3 ms).  Chunks of equal
  // PCIe bytes (8 rowptr[i] + 4 N i; GESPMM_HOST_EQUAL_BYTES=1) shrink the
  // last chunk's tail but measured no better: after B the call is bound by
  // duplex PCIe (config 5: 8.2 GB in + 8.6 GB out at ~45 GB/s each way),
  // 354.8 vs 358.6 ms on config 5, 83.0 vs 80.7 on config 4, 11.0 vs 10.8 on
  // config 2 (profiles/r2_chunks/).
  const int64_t c_bytes = M * N * 4;
  int nc = static_cast<int>(std::min<int64_t>(c_bytes / (8 << 20), 16));
  if (const char* x = std::getenv("GESPMM_HOST_CHUNKS")) nc = std::atoi(x);  // tests / A/B, <= kMaxChunks
  if (nc > kMaxChunks) nc = kMaxChunks;
  if (nc < 1 || std::getenv("GESPMM_HOST_NO_PIPELINE")) nc = 1;
  const bool in_row_order = std::getenv("GESPMM_HOST_ROW_ORDER") != nullptr;  // A/B switch
  const bool equal_rows = std::getenv("GESPMM_HOST_EQUAL_BYTES") == nullptr;
  // A launch reads its item's colind/vals up to the 16-byte staging granule
  // past the item end (never folded); chunk transfers cover that overhang.
  const int64_t overhang = 16;

  cudaError_t e = cudaSuccess;
  auto chk = [&](cudaError_t x) {
    if (e == cudaSuccess) e = x;
  };
  // GESPMM_TRACE=3: device timeline of this call (timing events, no syncs)
  const char* trace_env = std::getenv("GESPMM_TRACE");
  const bool tl = trace_env && *trace_env == '3';
  cudaEvent_t tev[3 + 3 * kMaxChunks] = {};
  auto tmark = [&](int i, cudaStream_t st) {
    if (!tl) return;
    if (!tev[i]) cudaEventCreate(&tev[i]);
    cudaEventRecord(tev[i], st);
  };
  // ---- host -> device on s_in: rowptr, B (and C0) ----------------------------
  chk(cudaEventRecord(pp->ev[0], s));  // s_in must not overtake prior work on s
  chk(cudaStreamWaitEvent(s_in, pp->ev[0], 0));
  tmark(0, s_in);
  chk(cudaMemcpyAsync(d_rp, rowptr, static_cast<size_t>(M + 1) * 4, cudaMemcpyHostToDevice, s_in));
  chk(cudaEventRecord(pp->ev[1], s_in));  // rowptr resident
  if (K > 0) {
    if (ldb == N) chk(cudaMemcpyAsync(d_B, B, static_cast<size_t>(K * N) * 4, cudaMemcpyHostToDevice, s_in));
    else chk(cudaMemcpy2DAsync(d_B, N * 4, B, ldb * 4, N * 4, K, cudaMemcpyHostToDevice, s_in));
  }
  tmark(1, s_in);  // rowptr + B resident
  if (e != cudaSuccess) {
    cudaStreamSynchronize(s_in);
    return cuda_fail(e, "host to device copy");
  }
  tr.mark("H2D issued", s);
  // ---- plan from rowptr (overlaps the B transfer), item-aligned chunks -------
  chk(cudaStreamWaitEvent(s, pp->ev[1], 0));
  chk(cudaMemsetAsync(d_err, 0, sizeof(int), s));
  // The plan object is cached per device with the workspace and re-planned in
  // place: no cudaMalloc/cudaFree per call (cudaFree synchronizes the device
  // and costs milliseconds at these sizes).
  gespmm_plan_s* plan = host_plan();
  plan->M = M;
  plan->K = K;
  plan->nnz = nnz;
  if (e == cudaSuccess) st = build_plan(plan, d_rp, nullptr, false, s);
  if (e != cudaSuccess || st != GESPMM_OK) {
    cudaStreamSynchronize(s_in);
    return e != cudaSuccess ? cuda_fail(e, "plan") : st;
  }
  int64_t rows[kMaxChunks + 1];
  if (equal_rows) {
    for (int c = 0; c <= nc; ++c) rows[c] = M * c / nc;
  } else {  // first row i with cost(i) >= c / nc of the total (host rowptr)
    const int64_t wr = 4 * N;
    auto cost = [&](int64_t i) { return 8 * static_cast<int64_t>(rowptr[i]) + wr * i; };
    const int64_t total = cost(M);
    rows[0] = 0;
    for (int c = 1; c <= nc; ++c) {
      const int64_t target = static_cast<int64_t>(static_cast<double>(total) * c / nc);
      int64_t lo = rows[c - 1], hi = M;
      while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (cost(mid) < target) lo = mid + 1;
        else hi = mid;
      }
      rows[c] = c == nc ? M : lo;
    }
  }
  chk(chunk_rows_aligned(plan, rows, nc, d_ranges, d_rows, s));
  chk(cudaMemcpyAsync(rows, d_rows, static_cast<size_t>(nc + 1) * sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  chk(cudaStreamSynchronize(s));  // ~20 us; B is still in flight
  int order[kMaxChunks];
  for (int c = 0; c < nc; ++c) order[c] = c;
  auto nnz_of = [&](int c) { return static_cast<int64_t>(rowptr[rows[c + 1]]) - rowptr[rows[c]]; };
  if (!in_row_order)
    std::stable_sort(order, order + nc, [&](int a, int b) { return nnz_of(a) < nnz_of(b); });
  // ---- colind/vals per chunk, in processing order, behind B on s_in ----------
  for (int k = 0; k < nc && e == cudaSuccess; ++k) {
    const int c = order[k];
    const int64_t p0 = rowptr[rows[c]];
    int64_t p1 = static_cast<int64_t>(rowptr[rows[c + 1]]) + overhang;
    if (p1 > nnz) p1 = nnz;
    if (p1 > p0) {
      chk(cudaMemcpyAsync(d_ci + p0, colind + p0, static_cast<size_t>(p1 - p0) * 4, cudaMemcpyHostToDevice, s_in));
      chk(cudaMemcpyAsync(d_v + p0, vals + p0, static_cast<size_t>(p1 - p0) * 4, cudaMemcpyHostToDevice, s_in));
    }
    const int64_t r0 = rows[c], nr = rows[c + 1] - rows[c];
    if (accumulate && nr > 0) {  // C0 rows of this chunk (its launch touches only these)
      if (ldc == N)
        chk(cudaMemcpyAsync(d_C + r0 * N, C + r0 * N, static_cast<size_t>(nr * N) * 4, cudaMemcpyHostToDevice, s_in));
      else
        chk(cudaMemcpy2DAsync(d_C + r0 * N, N * 4, C + r0 * ldc, ldc * 4, N * 4, nr, cudaMemcpyHostToDevice, s_in));
    }
    chk(cudaEventRecord(pp->ev[2 + k], s_in));  // chunk c's nonzeros resident
    tmark(3 + k, s_in);
  }
  tr.mark("rowptr H2D + plan", s);
  // ---- per chunk: colind check, the launch(es), C rows back on s_out --------
  for (int k = 0; k < nc && e == cudaSuccess; ++k) {
    const int c = order[k];
    chk(cudaStreamWaitEvent(s, pp->ev[2 + k], 0));
    chk(validate_colind_async(d_ci, rowptr[rows[c]], rowptr[rows[c + 1]], K, d_err, s));
    if (e != cudaSuccess) break;
    st = execute_range(plan, N, d_rp, d_ci, d_v, d_B, N, d_C, N, op, accumulate,
                       nc > 1 ? d_ranges + c : nullptr, d_err, s);
    if (st != GESPMM_OK) break;
    chk(cudaEventRecord(pp->ev[2 + kMaxChunks + k], s));
    tmark(3 + kMaxChunks + k, s);
    chk(cudaStreamWaitEvent(s_out, pp->ev[2 + kMaxChunks + k], 0));
    const int64_t r0 = rows[c], nr = rows[c + 1] - rows[c];
    if (nr > 0) {
      if (ldc == N)
        chk(cudaMemcpyAsync(C + r0 * N, d_C + r0 * N, static_cast<size_t>(nr * N) * 4,
                            cudaMemcpyDeviceToHost, s_out));
      else
        chk(cudaMemcpy2DAsync(C + r0 * ldc, ldc * 4, d_C + r0 * N, N * 4, N * 4, nr,
                              cudaMemcpyDeviceToHost, s_out));
    }
    tmark(3 + 2 * kMaxChunks + k, s_out);
  }
  tmark(2, s);  // plan + all launches done (s)
  tr.mark("chunks issued", s);
  int h_err = 0;
  chk(cudaMemcpyAsync(&h_err, d_err, sizeof(int), cudaMemcpyDeviceToHost, s));
  const cudaError_t e1 = cudaStreamSynchronize(s_out);
  tr.mark("sync out", s);
  const cudaError_t e2 = cudaStreamSynchronize(s_in);
  const cudaError_t e3 = cudaStreamSynchronize(s);
  chk(e1);
  chk(e2);
  chk(e3);
  tr.mark("chunks + C D2H", s);
  if (tl) {  // ms from the first copy: inputs resident / chunk c H2D, launch, D2H done
    auto at = [&](int i) {
      float ms = -1.f;
      if (tev[i] && tev[0]) cudaEventElapsedTime(&ms, tev[0], tev[i]);
      return ms;
    };
    std::fprintf(stderr, "[gespmm timeline] rowptr+B resident %.3f ms, %d chunks\n", at(1), nc);
    for (int k = 0; k < nc; ++k) {
      const int c = order[k];
      std::fprintf(stderr, "[gespmm timeline] chunk %2d rows %9lld nnz %10lld: H2D %.3f  kernel %.3f  D2H %.3f\n",
                   c, static_cast<long long>(rows[c + 1] - rows[c]), static_cast<long long>(nnz_of(c)),
                   at(3 + k), at(3 + kMaxChunks + k), at(3 + 2 * kMaxChunks + k));
    }
    for (cudaEvent_t x : tev)
      if (x) cudaEventDestroy(x);
  }
  if (st != GESPMM_OK) return st;
  if (e != cudaSuccess) return cuda_fail(e, "pipelined host spmm");
  // C's contents are unspecified after CSR_INVALID (earlier chunks may have
  // been written back); no launch ever read an out-of-range colind: every
  // launch follows its chunk's colind check on `s` and returns at once when
  // the flag is set (single chunk included).
  if (h_err) return fail(GESPMM_CSR_INVALID, csr_error_message(h_err, K));
  return GESPMM_OK;
}

const char* gespmm_variant_name(int64_t N, const float* B, int64_t ldb, const float* C,
                                int64_t ldc, gespmm_reduce_t op) {
  static thread_local std::string name;
  name = variant_name(pick_variant(N, B, ldb, C, ldc, op));
  return name.c_str();
}

int64_t gespmm_panel_width(int64_t K, int64_t N) { return N < 1 ? 0 : panel_width(K, N); }

gespmm_status_t gespmm_set_schedule_override(int mode) {
  if (mode < -1 || mode > 1) return fail(GESPMM_INVALID_ARG, "invalid argument: schedule mode -1/0/1");
  g_schedule_override = mode;
  return GESPMM_OK;
}

gespmm_status_t gespmm_set_tile_work_override(int32_t units) {
  if (units != 0 && (units < kRowCost || units > kTileWork))
    return fail(GESPMM_INVALID_ARG, "invalid argument: tile work must be 0 (auto) or in [2, 256]");
  g_tile_work_override = units;
  return GESPMM_OK;
}

const char* gespmm_plan_last_variant(gespmm_plan_t plan) {
  return plan ? plan->last_variant.c_str() : "";
}

gespmm_status_t gespmm_set_panel_override(int64_t cols) {
  g_panel_override = cols < 0 ? -1 : cols;
  return GESPMM_OK;
}

gespmm_status_t gespmm_set_variant_override(const char* name) {
  if (!name || !*name) {
    g_variant_override.clear();
    return GESPMM_OK;
  }
  Variant v;
  if (!parse_variant(name, &v)) return fail(GESPMM_INVALID_ARG, std::string("unknown variant ") + name);
  g_variant_override = name;
  return GESPMM_OK;
}

gespmm_status_t gespmm_partition_rows(int64_t M, const int32_t* rowptr, int parts,
                                      int64_t* bounds) {
  if (M < 0 || parts < 1 || !rowptr || !bounds)
    return fail(GESPMM_INVALID_ARG, "invalid argument: partition_rows");
  // balance nnz + rows (a row's C store costs about one nonzero's gather)
  const int64_t total = static_cast<int64_t>(rowptr[M]) + M;
  bounds[0] = 0;
  for (int r = 1; r < parts; ++r) {
    const int64_t target = total * r / parts;
    int64_t lo = bounds[r - 1], hi = M;
    while (lo < hi) {  // first row i with rowptr[i] + i >= target
      const int64_t mid = (lo + hi) / 2;
      if (static_cast<int64_t>(rowptr[mid]) + mid < target) lo = mid + 1;
      else hi = mid;
    }
    bounds[r] = lo;
  }
  bounds[parts] = M;
  return GESPMM_OK;
}

}  // extern "C"
