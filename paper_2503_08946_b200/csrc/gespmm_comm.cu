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

#include <cstring>
#include <mutex>

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
  const char* (*GetErrorString)(nccl_result_t) = nullptr;
  bool ok = false;
  std::string why;
};

constexpr int kNcclChar = 0;  // ncclChar / ncclInt8: byte-wise broadcast

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
    n.ok = n.GetUniqueId && n.CommInitRank && n.CommDestroy && n.Broadcast && n.GroupStart &&
           n.GroupEnd && n.GetErrorString;
    if (!n.ok) n.why = "libnccl.so.2 lacks required symbols";
  });
  return n;
}

gespmm_status_t nccl_fail(nccl_result_t r, const char* what) {
  Nccl& n = nccl();
  return gespmm::fail(GESPMM_NCCL_ERROR,
                      std::string(what) + ": " + (n.GetErrorString ? n.GetErrorString(r) : "?"));
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
  *comm = c;
  return GESPMM_OK;
}

gespmm_status_t gespmm_comm_destroy(void* comm) {
  Nccl& n = nccl();
  if (!comm) return GESPMM_OK;
  if (!n.ok) return gespmm::fail(GESPMM_NOT_SUPPORTED, n.why);
  nccl_result_t r = n.CommDestroy(comm);
  if (r != 0) return nccl_fail(r, "ncclCommDestroy");
  return GESPMM_OK;
}

gespmm_status_t gespmm_sharded_spmm_chunked(void* comm, int world, int rank, int root,
                                            gespmm_plan_t plan, int64_t M_local, int64_t K, int64_t N,
                                            int64_t nnz_local, const int32_t* rowptr,
                                            const int32_t* colind, const float* vals, float* B,
                                            int64_t ldb, float* C, int64_t ldc, gespmm_reduce_t op,
                                            int accumulate, float* C_full, int64_t ldc_full,
                                            const int64_t* row_bounds, int chunks, void* stream) {
  Nccl& n = nccl();
  if (!n.ok) return gespmm::fail(GESPMM_NOT_SUPPORTED, n.why);
  if (!comm || world < 1 || rank < 0 || rank >= world || root < 0 || root >= world)
    return gespmm::fail(GESPMM_INVALID_ARG, "invalid argument: comm/world/rank/root");
  if (ldb != N) return gespmm::fail(GESPMM_INVALID_ARG, "invalid argument: sharded B needs ldb == N");
  if (chunks < 1) return gespmm::fail(GESPMM_INVALID_ARG, "invalid argument: chunks must be >= 1");
  if (C_full && (!row_bounds || ldc != N || ldc_full != N))
    return gespmm::fail(GESPMM_INVALID_ARG,
                        "invalid argument: C all-gather needs row_bounds and ldc == ldc_full == N");
  if (C_full && row_bounds[rank + 1] - row_bounds[rank] != M_local)
    return gespmm::fail(GESPMM_INVALID_ARG, "invalid argument: row_bounds disagree with M_local");
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  // 1. the exchange: B from root, in place
  nccl_result_t r = n.Broadcast(B, B, static_cast<size_t>(K * N) * sizeof(float), kNcclChar, root,
                                comm, s);
  if (r != 0) return nccl_fail(r, "ncclBroadcast(B)");
  gespmm_plan_t p = plan;
  gespmm_status_t st = GESPMM_OK;
  if (!p) st = gespmm_plan_create(&p, M_local, K, nnz_local, rowptr, colind, 0, stream);
  auto done = [&](gespmm_status_t x) {
    if (!plan && p) {
      cudaStreamSynchronize(s);
      gespmm_plan_destroy(p);
    }
    return x;
  };
  if (st != GESPMM_OK) return done(st);
  if (!C_full || chunks == 1 || world == 0) {
    // 2. the local slab, then 3. the optional all-gather of the uneven slabs
    st = gespmm_plan_execute(p, N, rowptr, colind, vals, B, ldb, C, ldc, op, accumulate, stream);
    if (st != GESPMM_OK || !C_full) return done(st);
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
        return done(nccl_fail(r, "ncclBroadcast(C slab)"));
      }
    }
    r = n.GroupEnd();
    if (r != 0) return done(nccl_fail(r, "ncclGroupEnd"));
    return done(GESPMM_OK);
  }
  // compute-overlapped all-gather.  Chunk j of every slab is rows
  // [a + (b-a)j/chunks, a + (b-a)(j+1)/chunks) of that slab (computable by all
  // ranks from row_bounds).  Chunk j runs on `stream` (gespmm_plan_execute_rows:
  // rows < its end are final afterwards); the broadcasts of every owner's
  // chunk j run on a comm stream that waits for it, while chunk j+1 computes.
  cudaStream_t cs = nullptr;
  cudaEvent_t ev = nullptr;
  cudaError_t ce = cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking);
  if (ce == cudaSuccess) ce = cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
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
  cudaStreamSynchronize(cs);
  cudaEventDestroy(ev);
  cudaStreamDestroy(cs);
  return done(st);
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
