// gespmm_comm.cu -- row-block sharding over NVLink/NVSwitch.
//
// The path's only exchange step is the broadcast of B: every C row depends
// only on its own CSR row and B, so each rank computes its C slab from its row
// block with no collective inside the compute.  B goes out once with
// ncclBroadcast (NVLink 5 / NVSwitch; NVLS when NCCL enables it); the optional
// C all-gather is one grouped ncclBroadcast per slab owner (slabs are uneven).
// Per-row reduction order is untouched by sharding and the plan depends only on
// rowptr, so results are bit-identical at 1/2/4/8 GPUs.
//
// NCCL is resolved at run time: if the process already loaded a libnccl.so.2
// (e.g. torch's), dlopen returns that copy, so two NCCLs never coexist.
#include <dlfcn.h>

#include <chrono>
#include <cstdlib>
#include <algorithm>
#include <cstring>
#include <mutex>
#include <set>
#include <thread>

#include "gespmm_internal.h"

namespace {

typedef int nccl_result_t;
typedef struct {
  char internal[128];
} nccl_unique_id_t;
typedef void* nccl_comm_t;

struct Nccl {
  nccl_result_t (*GetUniqueId)(nccl_unique_id_t*) = nullptr;
  nccl_result_t (*CommInitRank)(nccl_comm_t*, int, nccl_unique_id_t, int) = nullptr;
  nccl_result_t (*CommDestroy)(nccl_comm_t) = nullptr;
  nccl_result_t (*Broadcast)(const void*, void*, size_t, int, int, nccl_comm_t, cudaStream_t) = nullptr;
  nccl_result_t (*GroupStart)() = nullptr;
  nccl_result_t (*GroupEnd)() = nullptr;
  nccl_result_t (*AllReduce)(const void*, void*, size_t, int, int, nccl_comm_t, cudaStream_t) = nullptr;
  nccl_result_t (*CommGetAsyncError)(nccl_comm_t, nccl_result_t*) = nullptr;
  nccl_result_t (*CommAbort)(nccl_comm_t) = nullptr;
  const char* (*GetErrorString)(nccl_result_t) = nullptr;
  bool ok = false;
  std::string why;
};

constexpr int kNcclChar = 0;   // ncclChar / ncclInt8: byte-wise broadcast
constexpr int kNcclInt32 = 2;  // ncclInt32
constexpr int kNcclMax = 2;    // ncclMax
constexpr nccl_result_t kNcclInProgress = 7;  // ncclInProgress (non-blocking comms)

Nccl& nccl() {
  static Nccl n;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      n.why = std::string("cannot load libnccl.so.2: ") + dlerror();
      return;
    }
    auto sym = [&](const char* name) { return dlsym(h, name); };
    n.GetUniqueId = reinterpret_cast<decltype(n.GetUniqueId)>(sym("ncclGetUniqueId"));
    n.CommInitRank = reinterpret_cast<decltype(n.CommInitRank)>(sym("ncclCommInitRank"));
    n.CommDestroy = reinterpret_cast<decltype(n.CommDestroy)>(sym("ncclCommDestroy"));
    n.Broadcast = reinterpret_cast<decltype(n.Broadcast)>(sym("ncclBroadcast"));
    n.GroupStart = reinterpret_cast<decltype(n.GroupStart)>(sym("ncclGroupStart"));
    n.GroupEnd = reinterpret_cast<decltype(n.GroupEnd)>(sym("ncclGroupEnd"));
    n.GetErrorString = reinterpret_cast<decltype(n.GetErrorString)>(sym("ncclGetErrorString"));
    n.AllReduce = reinterpret_cast<decltype(n.AllReduce)>(sym("ncclAllReduce"));
    n.CommGetAsyncError = reinterpret_cast<decltype(n.CommGetAsyncError)>(sym("ncclCommGetAsyncError"));
    n.CommAbort = reinterpret_cast<decltype(n.CommAbort)>(sym("ncclCommAbort"));
    n.ok = n.GetUniqueId && n.CommInitRank && n.CommDestroy && n.Broadcast && n.GroupStart &&
           n.GroupEnd && n.GetErrorString && n.AllReduce && n.CommGetAsyncError && n.CommAbort;
    if (!n.ok) n.why = "libnccl.so.2 lacks required symbols";
  });
  return n;
}

gespmm_status_t nccl_fail(nccl_result_t r, const char* what) {
  Nccl& n = nccl();
  return gespmm::fail(GESPMM_NCCL_ERROR,
                      std::string(what) + ": " + (n.GetErrorString ? n.GetErrorString(r) : "?"));
}

// Communicators torn down by gespmm_comm_wait (ncclCommAbort frees them): any
// later use returns GESPMM_NCCL_ERROR instead of touching freed state.
std::mutex g_aborted_mu;
std::set<void*> g_aborted;
bool aborted(void* comm) {
  std::lock_guard<std::mutex> l(g_aborted_mu);
  return g_aborted.count(comm) != 0;
}
gespmm_status_t abort_comm(void* comm, const std::string& why) {
  Nccl& n = nccl();
  {
    std::lock_guard<std::mutex> l(g_aborted_mu);
    if (!g_aborted.insert(comm).second) return gespmm::fail(GESPMM_NCCL_ERROR, why);
  }
  n.CommAbort(comm);
  return gespmm::fail(GESPMM_NCCL_ERROR, why + " (communicator aborted)");
}

// Default wait bound of the sharded entry points (GESPMM_NCCL_TIMEOUT_MS,
// default 10 min): a dead peer turns into GESPMM_NCCL_ERROR, not a hang.
int64_t default_timeout_ms() {
  const char* e = std::getenv("GESPMM_NCCL_TIMEOUT_MS");
  const long long v = e ? std::atoll(e) : 0;
  return v > 0 ? v : 600000;
}

}  // namespace

extern "C" {

gespmm_status_t gespmm_comm_get_unique_id(char id[128]) {
  Nccl& n = nccl();
  if (!n.ok) return gespmm::fail(GESPMM_NOT_SUPPORTED, n.why);
  nccl_unique_id_t u;
  nccl_result_t r = n.GetUniqueId(&u);
  if (r != 0) return nccl_fail(r, "ncclGetUniqueId");
  std::memcpy(id, u.internal, 128);
  return GESPMM_OK;
}

gespmm_status_t gespmm_comm_init(void** comm, int world, const char id[128], int rank) {
  Nccl& n = nccl();
  if (!n.ok) return gespmm::fail(GESPMM_NOT_SUPPORTED, n.why);
  if (!comm || world < 1 || rank < 0 || rank >= world)
    return gespmm::fail(GESPMM_INVALID_ARG, "invalid argument: comm_init");
  nccl_unique_id_t u;
  std::memcpy(u.internal, id, 128);
  nccl_comm_t c = nullptr;
  nccl_result_t r = n.CommInitRank(&c, world, u, rank);
  if (r != 0) return nccl_fail(r, "ncclCommInitRank");
  {  // a new communicator may reuse the address of an aborted (freed) one
    std::lock_guard<std::mutex> l(g_aborted_mu);
    g_aborted.erase(c);
  }
  *comm = c;
  return GESPMM_OK;
}

gespmm_status_t gespmm_comm_destroy(void* comm) {
  Nccl& n = nccl();
  if (!comm) return GESPMM_OK;
  if (!n.ok) return gespmm::fail(GESPMM_NOT_SUPPORTED, n.why);
  if (aborted(comm)) return GESPMM_OK;  // already freed by ncclCommAbort
  nccl_result_t r = n.CommDestroy(comm);
  if (r != 0) return nccl_fail(r, "ncclCommDestroy");
  return GESPMM_OK;
}

gespmm_status_t gespmm_comm_wait(void* comm, void* stream, int64_t timeout_ms) {
  gespmm::NvtxRange nvtx("gespmm:comm_wait");
  Nccl& n = nccl();
  if (!n.ok) return gespmm::fail(GESPMM_NOT_SUPPORTED, n.why);
  if (!comm) return gespmm::fail(GESPMM_INVALID_ARG, "invalid argument: comm is null");
  if (aborted(comm)) return gespmm::fail(GESPMM_NCCL_ERROR, "communicator was aborted");
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const auto t0 = std::chrono::steady_clock::now();
  for (int spin = 0;; ++spin) {
    const cudaError_t q = cudaStreamQuery(s);
    if (q == cudaSuccess) return GESPMM_OK;
    if (q != cudaErrorNotReady) return gespmm::cuda_fail(q, "comm wait");
    nccl_result_t ae = 0;
    const nccl_result_t r = n.CommGetAsyncError(comm, &ae);
    if (r != 0) return abort_comm(comm, std::string("ncclCommGetAsyncError: ") + n.GetErrorString(r));
    if (ae != 0 && ae != kNcclInProgress)
      return abort_comm(comm, std::string("NCCL asynchronous error: ") + n.GetErrorString(ae));
    if (timeout_ms > 0 && std::chrono::steady_clock::now() - t0 > std::chrono::milliseconds(timeout_ms))
      return abort_comm(comm, "NCCL wait timed out after " + std::to_string(timeout_ms) +
                                  " ms (a peer stalled or died)");
    if (spin > 64) std::this_thread::sleep_for(std::chrono::microseconds(200));
  }
}

gespmm_status_t gespmm_sharded_spmm_ex(void* comm, int world, int rank, int root, gespmm_plan_t plan,
                                       int64_t M_local, int64_t K, int64_t N, int64_t nnz_local,
                                       const int32_t* rowptr, const int32_t* colind, const float* vals,
                                       float* B, int64_t ldb, float* C, int64_t ldc, gespmm_reduce_t op,
                                       int accumulate, float* C_full, int64_t ldc_full,
                                       const int64_t* row_bounds, const gespmm_shard_opts_t* opts,
                                       void* stream) {
  gespmm::NvtxRange nvtx("gespmm:sharded_spmm");
  Nccl& n = nccl();
  if (!n.ok) return gespmm::fail(GESPMM_NOT_SUPPORTED, n.why);
  gespmm_shard_opts_t o = {1, nullptr, 1, 0};
  if (opts) o = *opts;
  if (!comm || world < 1 || rank < 0 || rank >= world || root < 0 || root >= world)
    return gespmm::fail(GESPMM_INVALID_ARG, "invalid argument: comm/world/rank/root");
  if (aborted(comm)) return gespmm::fail(GESPMM_NCCL_ERROR, "communicator was aborted");
  if (ldb != N) return gespmm::fail(GESPMM_INVALID_ARG, "invalid argument: sharded B needs ldb == N");
  if (o.c_chunks < 1 || o.b_panels < 1)
    return gespmm::fail(GESPMM_INVALID_ARG, "invalid argument: chunks and panels must be >= 1");
  if (o.b_panels > 1 && o.c_chunks > 1)
    return gespmm::fail(GESPMM_INVALID_ARG, "invalid argument: b_panels > 1 needs c_chunks == 1");
  if (C_full && (!row_bounds || ldc != N || ldc_full != N))
    return gespmm::fail(GESPMM_INVALID_ARG,
                        "invalid argument: C all-gather needs row_bounds and ldc == ldc_full == N");
  if (C_full && row_bounds[rank + 1] - row_bounds[rank] != M_local)
    return gespmm::fail(GESPMM_INVALID_ARG, "invalid argument: row_bounds disagree with M_local");
  if (K * N > 0 && !B) return gespmm::fail(GESPMM_INVALID_ARG, "invalid argument: B is null");
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  nccl_result_t r = 0;

  // 0. a temporary plan validates this rank's CSR (colind range included)
  //    BEFORE any collective, and the ranks agree on the outcome (one int32
  //    max all-reduce): every rank returns the error, none is left waiting in
  //    a broadcast its failed peer never posts.
  gespmm_plan_t p = plan;
  gespmm_status_t st = GESPMM_OK;
  std::string local_err;
  if (!p) {
    st = gespmm_plan_create(&p, M_local, K, nnz_local, rowptr, colind, /*validate colind*/ 1, stream);
    if (st != GESPMM_OK) {
      local_err = gespmm_last_error();
      p = nullptr;
    }
  }
  auto done = [&](gespmm_status_t x) {
    if (!plan && p) {
      cudaStreamSynchronize(s);
      gespmm_plan_destroy(p);
    }
    return x;
  };
  if (!plan && world > 1) {
    // host words in pinned memory: a copy to or from pageable memory can block
    // inside cudaMemcpyAsync -- forever, if a peer never joins the all-reduce --
    // before the bounded wait below could see it.  [0] = this rank's status,
    // [1] = the agreed (max) status.
    static thread_local int* words = [] {
      int* p = nullptr;
      return cudaMallocHost(reinterpret_cast<void**>(&p), 2 * sizeof(int)) == cudaSuccess ? p : nullptr;
    }();
    if (!words) return done(gespmm::fail(GESPMM_CUDA_ERROR, "status agreement: pinned host words"));
    words[0] = st == GESPMM_OK ? 0 : static_cast<int>(st);
    words[1] = 0;
    int* flag = nullptr;
    cudaError_t ce = cudaMallocAsync(reinterpret_cast<void**>(&flag), sizeof(int), s);
    if (ce == cudaSuccess) ce = cudaMemcpyAsync(flag, words, sizeof(int), cudaMemcpyHostToDevice, s);
    if (ce != cudaSuccess) return done(gespmm::cuda_fail(ce, "status agreement"));
    r = n.AllReduce(flag, flag, 1, kNcclInt32, kNcclMax, comm, s);
    if (r == 0) ce = cudaMemcpyAsync(words + 1, flag, sizeof(int), cudaMemcpyDeviceToHost, s);
    cudaFreeAsync(flag, s);
    if (r != 0) return done(nccl_fail(r, "ncclAllReduce(status)"));
    const gespmm_status_t w = gespmm_comm_wait(comm, stream, o.timeout_ms > 0 ? o.timeout_ms : default_timeout_ms());
    if (w != GESPMM_OK) {
      if (!plan) p = nullptr;  // the stream may never drain: do not synchronize on it
      return w;
    }
    if (ce != cudaSuccess) return done(gespmm::cuda_fail(ce, "status agreement"));
    const int agreed = words[1];
    if (st != GESPMM_OK) return done(gespmm::fail(st, local_err));
    if (agreed != 0)
      return done(gespmm::fail(static_cast<gespmm_status_t>(agreed),
                               "sharded spmm: another rank's row block failed validation"));
  } else if (st != GESPMM_OK) {
    return done(gespmm::fail(st, local_err));
  }

  cudaStream_t cs = nullptr;
  cudaEvent_t ev = nullptr;
  auto streams = [&]() {
    if (cs) return cudaSuccess;
    cudaError_t ce = cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking);
    if (ce == cudaSuccess) ce = cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
    return ce;
  };
  auto release = [&]() {
    if (cs) {
      cudaStreamSynchronize(cs);
      cudaEventDestroy(ev);
      cudaStreamDestroy(cs);
      cs = nullptr;
    }
  };

  if (o.b_panels <= 1) {
    // 1. the exchange: B from root, in place
    r = n.Broadcast(B, B, static_cast<size_t>(K * N) * sizeof(float), kNcclChar, root, comm, s);
    if (r != 0) return done(nccl_fail(r, "ncclBroadcast(B)"));
  } else {
    // 1+2. SURVEY 8 f4: B in column panels [c0, c1) packed into contiguous
    // K x w buffers (the root packs with one 2-D copy each), panel p broadcast
    // on a comm stream while panel p-1 computes on `stream`; each panel is a
    // plain execute with ldb = w into C[:, c0:c1].  A column's result does not
    // depend on which columns share its launch, so this is bit-identical to
    // the unpanelled path.
    cudaError_t ce = streams();
    if (ce != cudaSuccess) return done(gespmm::cuda_fail(ce, "sharded comm stream"));
    const int P = static_cast<int>(std::min<int64_t>(o.b_panels, std::max<int64_t>(1, (N + 31) / 32)));
    int64_t step = (N + P - 1) / P;
    if (N >= 32) step = (step + 31) / 32 * 32;
    float* ws = o.b_panel_ws;
    if (!ws) {
      ce = cudaMallocAsync(reinterpret_cast<void**>(&ws), static_cast<size_t>(K * N) * sizeof(float), s);
      if (ce != cudaSuccess) return done(gespmm::cuda_fail(ce, "B panel workspace"));
    }
    cudaEventRecord(ev, s);
    cudaStreamWaitEvent(cs, ev, 0);  // B, the workspace and the plan are ready
    for (int64_t c0 = 0; c0 < N && st == GESPMM_OK; c0 += step) {
      const int64_t w = std::min(step, N - c0);
      float* pan = ws + K * c0;  // panel p: K x w, contiguous
      if (rank == root && K > 0) {
        ce = cudaMemcpy2DAsync(pan, w * sizeof(float), B + c0, ldb * sizeof(float), w * sizeof(float), K,
                               cudaMemcpyDeviceToDevice, cs);
        if (ce != cudaSuccess) {
          st = gespmm::cuda_fail(ce, "B panel pack");
          break;
        }
      }
      r = n.Broadcast(pan, pan, static_cast<size_t>(K * w) * sizeof(float), kNcclChar, root, comm, cs);
      if (r != 0) {
        st = nccl_fail(r, "ncclBroadcast(B panel)");
        break;
      }
      cudaEventRecord(ev, cs);
      cudaStreamWaitEvent(s, ev, 0);
      st = gespmm_plan_execute(p, w, rowptr, colind, vals, pan, w, C + c0, ldc, op, accumulate, stream);
    }
    if (!o.b_panel_ws) cudaFreeAsync(ws, s);
    if (st != GESPMM_OK) {
      release();
      return done(st);
    }
  }

  if (o.b_panels <= 1 && (!C_full || o.c_chunks == 1)) {
    // 2. the local slab
    st = gespmm_plan_execute(p, N, rowptr, colind, vals, B, ldb, C, ldc, op, accumulate, stream);
    if (st != GESPMM_OK) return done(st);
  }
  if (C_full && (o.c_chunks == 1 || o.b_panels > 1)) {
    // 3. the optional all-gather of the uneven slabs
    r = n.GroupStart();
    if (r != 0) return done(nccl_fail(r, "ncclGroupStart"));
    for (int w = 0; w < world; ++w) {
      const int64_t rows = row_bounds[w + 1] - row_bounds[w];
      if (rows <= 0) continue;
      float* recv = C_full + row_bounds[w] * N;
      const float* send = (w == rank) ? C : recv;
      r = n.Broadcast(send, recv, static_cast<size_t>(rows * N) * sizeof(float), kNcclChar, w, comm, s);
      if (r != 0) {
        n.GroupEnd();
        release();
        return done(nccl_fail(r, "ncclBroadcast(C slab)"));
      }
    }
    r = n.GroupEnd();
    if (r != 0) {
      release();
      return done(nccl_fail(r, "ncclGroupEnd"));
    }
  } else if (C_full) {
    // compute-overlapped all-gather.  Chunk j of every slab is
    // rows [a + (b-a)j/chunks, a + (b-a)(j+1)/chunks) of that slab (computable
    // by all ranks from row_bounds).  Chunk j runs on `stream`
    // (gespmm_plan_execute_rows: rows < its end are final afterwards); the
    // broadcasts of every owner's chunk j run on a comm stream that waits for
    // it, while chunk j+1 computes.
    const int chunks = o.c_chunks;
    cudaError_t ce = streams();
    if (ce != cudaSuccess) return done(gespmm::cuda_fail(ce, "sharded comm stream"));
    const int64_t a_me = row_bounds[rank];
    for (int j = 0; j < chunks && st == GESPMM_OK; ++j) {
      const int64_t lo = M_local * j / chunks, hi = M_local * (j + 1) / chunks;
      st = gespmm_plan_execute_rows(p, lo, hi, N, rowptr, colind, vals, B, ldb, C, ldc, op, accumulate,
                                    stream);
      if (st != GESPMM_OK) break;
      cudaEventRecord(ev, s);
      cudaStreamWaitEvent(cs, ev, 0);
      r = n.GroupStart();
      for (int w = 0; w < world && r == 0; ++w) {
        const int64_t a = row_bounds[w], m = row_bounds[w + 1] - row_bounds[w];
        const int64_t r0 = a + m * j / chunks, r1 = a + m * (j + 1) / chunks;
        if (r1 <= r0) continue;
        float* recv = C_full + r0 * N;
        const float* send = (w == rank) ? C + (r0 - a_me) * N : recv;
        r = n.Broadcast(send, recv, static_cast<size_t>((r1 - r0) * N) * sizeof(float), kNcclChar, w, comm, cs);
      }
      const nccl_result_t r2 = n.GroupEnd();
      if (r == 0) r = r2;
      if (r != 0) st = nccl_fail(r, "ncclBroadcast(C chunk)");
    }
    cudaEventRecord(ev, cs);
    cudaStreamWaitEvent(s, ev, 0);  // the caller's stream sees the gathered C
  }
  if (cs) {
    // the comm stream's work is ordered before `stream` (event above / the
    // panel loop); bounded, error-polled wait when asked or when the C
    // all-gather ran on it
    if (o.timeout_ms > 0 || (C_full && o.c_chunks > 1)) {
      const gespmm_status_t w = gespmm_comm_wait(comm, stream, o.timeout_ms > 0 ? o.timeout_ms : default_timeout_ms());
      if (w != GESPMM_OK) {
        // the comm stream may never drain (aborted collective): leak it
        // rather than block in its destruction
        if (plan == nullptr) p = nullptr;
        return w;
      }
    }
    release();
  } else if (o.timeout_ms > 0 && st == GESPMM_OK) {
    const gespmm_status_t w = gespmm_comm_wait(comm, stream, o.timeout_ms);
    if (w != GESPMM_OK) {
      if (plan == nullptr) p = nullptr;
      return w;
    }
  }
  return done(st);
}

gespmm_status_t gespmm_sharded_spmm_chunked(void* comm, int world, int rank, int root,
                                            gespmm_plan_t plan, int64_t M_local, int64_t K, int64_t N,
                                            int64_t nnz_local, const int32_t* rowptr,
                                            const int32_t* colind, const float* vals, float* B,
                                            int64_t ldb, float* C, int64_t ldc, gespmm_reduce_t op,
                                            int accumulate, float* C_full, int64_t ldc_full,
                                            const int64_t* row_bounds, int chunks, void* stream) {
  const gespmm_shard_opts_t o = {1, nullptr, chunks, 0};
  return gespmm_sharded_spmm_ex(comm, world, rank, root, plan, M_local, K, N, nnz_local, rowptr, colind, vals,
                                B, ldb, C, ldc, op, accumulate, C_full, ldc_full, row_bounds, &o, stream);
}

gespmm_status_t gespmm_sharded_spmm(void* comm, int world, int rank, int root,
                                    gespmm_plan_t plan, int64_t M_local, int64_t K, int64_t N,
                                    int64_t nnz_local, const int32_t* rowptr,
                                    const int32_t* colind, const float* vals, float* B,
                                    int64_t ldb, float* C, int64_t ldc, gespmm_reduce_t op,
                                    int accumulate, float* C_full, int64_t ldc_full,
                                    const int64_t* row_bounds, void* stream) {
  return gespmm_sharded_spmm_chunked(comm, world, rank, root, plan, M_local, K, N, nnz_local, rowptr,
                                     colind, vals, B, ldb, C, ldc, op, accumulate, C_full, ldc_full,
                                     row_bounds, 1, stream);
}
}  // extern "C"
