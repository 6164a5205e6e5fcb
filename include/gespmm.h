/*
 * gespmm.h -- C-ABI of the B200-native GE-SpMM hot path (libgespmm.so).
 *
 * Drop-in boundary for the reference's CSR x dense SpMM path.  The reference
 * (arXiv 2503.08946's `raceset` artifact) exposes that path as
 *
 *   kernel @gespmm_alg2(%rowPtr: i32*, %colInd: i32*, %val: f32*, %B: f32*,
 *                       %C: f32*, %M, %N, %K)
 *        -- /root/reference/proj/fixtures/gespmm_alg2.mir:5
 *   raceset::run(const ConcreteInstance&, const Function&, const RunOptions&)
 *        -- /root/reference/proj/include/raceset/oracle.hpp:71-74
 *   raceset::validate_instance(const ConcreteInstance&)   (CSR contract)
 *        -- /root/reference/proj/include/raceset/oracle.hpp:38-39,
 *           src/oracle.cpp:291-316
 *
 * Conventions:
 *   - CSR: rowptr int32[M+1], colind int32[nnz], vals fp32[nnz]; colind need
 *     not be sorted or unique (the reference does not require it).
 *   - B fp32 [K x N] row-major with leading dimension ldb >= N; C fp32 [M x N]
 *     row-major with ldc >= N (gespmm_alg2.mir:51-56 uses ld = N).
 *   - 64-bit sizes and 64-bit B/C address arithmetic (K*N may exceed 2^31).
 *   - Device pointers are caller-owned; nothing is copied behind the caller's
 *     back; work is enqueued on `stream` (a cudaStream_t, 0 = legacy default).
 *   - No exceptions cross the ABI: every entry point returns a status; the
 *     thread-local detail string is gespmm_last_error().
 *   - Thread safety: distinct plans may be used concurrently from distinct
 *     threads; one plan must not be executed concurrently with itself.
 *
 * Semantics (normative, oracle/gespmm_oracle.c), fp32:
 *   SUM : two ascending FMA chains per row, over the nonzeros at even (A) and
 *         odd (B) offsets from the row start: A = fmaf(val[p], B[col[p]][j], A)
 *         from A = 0 (accumulate: C0), B likewise from -0.0; value = A + B
 *   MEAN: the SUM value from A = 0, then / deg(i) (correctly rounded);
 *         accumulate adds C0
 *   MAX/MIN: m = val[p]*B[col[p]][j] (rounded, unfused); the value is IEEE
 *         754-2019 maximumNumber (MIN: minimumNumber) over the row's messages
 *         and, with accumulate, C0: NaN operands ignored, all-NaN -> the
 *         canonical NaN 0x7fffffff, -0 < +0 (the B200's FMNMX); order-free
 *   empty rows give 0 (accumulate: C0 for sum/max/min, C0 + 0 for mean).
 *   Rows with more than GESPMM_SEGMENT_LEN nonzeros are reduced in fixed
 *   GESPMM_SEGMENT_LEN-long segments from the row start (each segment as above,
 *   later segments seeded with 0 / NaN), combined left to right (sum/mean: +,
 *   max/min: maximumNumber/minimumNumber).  Results are deterministic and
 *   independent of device, grid and sharding.
 */
#ifndef GESPMM_H_
#define GESPMM_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GESPMM_VERSION_MAJOR 0
#define GESPMM_VERSION_MINOR 1
/* Long-row segment length (nonzeros).  Part of the numerical contract. */
#ifndef GESPMM_SEGMENT_LEN
#define GESPMM_SEGMENT_LEN 256
#endif

/* Status codes.  Mirrors the reference's ErrorKind values that can arise on
 * this path (reference include/raceset/error.hpp:10-32):
 *   CsrInvalid -> GESPMM_CSR_INVALID (src/oracle.cpp:291-316),
 *   OutOfBounds -> GESPMM_OUT_OF_BOUNDS (src/oracle.cpp:673-677),
 * plus the host-API failures a C-ABI needs. */
typedef enum gespmm_status {
  GESPMM_OK = 0,
  GESPMM_CSR_INVALID = 1,
  GESPMM_OUT_OF_BOUNDS = 2,
  GESPMM_INVALID_ARG = 3,
  GESPMM_CUDA_ERROR = 4,
  GESPMM_NCCL_ERROR = 5,
  GESPMM_NOT_SUPPORTED = 6
} gespmm_status_t;

/* Reduce operator (compile-time functor inside the kernels).  The reference
 * has SUM only (gespmm_alg2.mir:57-59); MAX/MIN/MEAN are the generalized
 * semiring of BASELINE.json's north star. */
typedef enum gespmm_reduce {
  GESPMM_REDUCE_SUM = 0,
  GESPMM_REDUCE_MAX = 1,
  GESPMM_REDUCE_MIN = 2,
  GESPMM_REDUCE_MEAN = 3
} gespmm_reduce_t;

typedef struct gespmm_plan_s* gespmm_plan_t;

/* Library version as MAJOR*100 + MINOR. */
int gespmm_version(void);
/* Static description of a status code. */
const char* gespmm_status_string(gespmm_status_t s);
/* Detail of the last failure on the calling thread ("" if none), in the style
 * of raceset::Error::what() ("invalid csr: rowPtr must be nondecreasing"). */
const char* gespmm_last_error(void);

/* Host-side CSR validation with the reference's rules
 * (validate_instance, src/oracle.cpp:291-316): rowptr non-empty, rowptr[0] == 0,
 * nondecreasing, rowptr[rowptr_len-1] == colind_len, colind_len == vals_len,
 * 0 <= colind < K.  Added: rowptr_len == M + 1.  Pointers are HOST memory. */
gespmm_status_t gespmm_validate_csr(int64_t M, int64_t K, int64_t rowptr_len,
                                    const int32_t* rowptr, int64_t colind_len,
                                    const int32_t* colind, int64_t vals_len);

/* The same rules checked on the GPU for DEVICE pointers (one pass over rowptr
 * and colind; synchronizes `stream` to return the verdict). */
gespmm_status_t gespmm_validate_csr_device(int64_t M, int64_t K, int64_t nnz,
                                           const int32_t* rowptr, const int32_t* colind,
                                           void* stream);

/* One-shot SpMM on device buffers: C = A (op) B, or C = C0 (op-combine) A (op) B
 * when accumulate != 0 (the reference kernel's C read-modify-write,
 * gespmm_alg2.mir:55-59).  Validates the CSR on the device (the reference
 * validates inside run(), src/oracle.cpp:700), re-plans a cached per-device
 * plan in place (no allocation per call: cudaFree would synchronize the
 * device), launches, and returns after the launches complete -- it
 * synchronizes `stream` twice (the plan's totals, the end of the call; calls
 * are serialized by a process-wide lock).  For asynchronous repeated
 * execution build a plan once (gespmm_plan_create) and use
 * gespmm_plan_execute, which never synchronizes. */
gespmm_status_t gespmm_csr_spmm(int64_t M, int64_t K, int64_t N, int64_t nnz,
                                const int32_t* rowptr, const int32_t* colind,
                                const float* vals, const float* B, int64_t ldb, float* C,
                                int64_t ldc, gespmm_reduce_t op, int accumulate, void* stream);

/* One-shot SpMM on HOST buffers (the C++-host drop-in for raceset::run, which
 * takes its instance by value, src/oracle.cpp:381-399): copies the CSR and B
 * to the device, validates, plans, computes and copies C back (C is read first
 * when accumulate != 0).  Blocking; `stream` may be 0.  Host buffers may be
 * pageable; pinned buffers copy at full link speed. */
gespmm_status_t gespmm_csr_spmm_host(int64_t M, int64_t K, int64_t N, int64_t nnz,
                                     const int32_t* rowptr, const int32_t* colind,
                                     const float* vals, const float* B, int64_t ldb, float* C,
                                     int64_t ldc, gespmm_reduce_t op, int accumulate,
                                     void* stream);

/* Plan = the nnz-balanced work decomposition of one sparsity structure
 * (tiles of consecutive short rows + fixed segments of long rows), built on
 * the GPU.  Depends only on (M, nnz, rowptr); reusable for any vals/B/N/op.
 * flags: bit 0 = also validate colind against K on the device.
 * Synchronizes `stream` once to size the work list. */
gespmm_status_t gespmm_plan_create(gespmm_plan_t* plan, int64_t M, int64_t K, int64_t nnz,
                                   const int32_t* rowptr, const int32_t* colind, int flags,
                                   void* stream);
/* Launch with a plan (asynchronous on `stream`, no host synchronization once
 * the plan's workspace -- long-row partials and counters, sized by N -- has
 * been allocated; growing it, on the first call or a wider N, uses
 * cudaMalloc/cudaFree, which may synchronize the device). */
gespmm_status_t gespmm_plan_execute(gespmm_plan_t plan, int64_t N, const int32_t* rowptr,
                                    const int32_t* colind, const float* vals, const float* B,
                                    int64_t ldb, float* C, int64_t ldc, gespmm_reduce_t op,
                                    int accumulate, void* stream);

/* One row chunk of an execute (compute overlapped with the
 * C all-gather / the D2H of finished rows).  Runs the plan's work items whose
 * first row lies in [row_begin, row_end).  Executing consecutive chunks
 * [r0=0, r1), [r1, r2), ..., [r_j, r_j+1) in order on ONE stream makes every C
 * row < r_j+1 final once chunk j has run (a tile that starts before r_j+1 and
 * runs past it is finished by chunk j); all chunks together equal one
 * gespmm_plan_execute bit for bit.  Not concurrent with another execute of
 * the same plan. */
gespmm_status_t gespmm_plan_execute_rows(gespmm_plan_t plan, int64_t row_begin, int64_t row_end,
                                         int64_t N, const int32_t* rowptr, const int32_t* colind,
                                         const float* vals, const float* B, int64_t ldb, float* C,
                                         int64_t ldc, gespmm_reduce_t op, int accumulate,
                                         void* stream);
gespmm_status_t gespmm_plan_destroy(gespmm_plan_t plan);

/* Plan introspection (tests, benches). */
typedef struct gespmm_plan_info {
  int64_t M, nnz;
  int64_t n_items;        /* work items (short-row tiles + long-row segments) */
  int64_t n_tiles;        /* short-row tiles */
  int64_t n_long_rows;    /* rows with deg > GESPMM_SEGMENT_LEN */
  int64_t n_segments;     /* segments of long rows */
  int64_t segment_len;    /* GESPMM_SEGMENT_LEN */
  int64_t tile_work;      /* target work units per tile */
  int64_t kernel_launches_per_execute;
} gespmm_plan_info_t;
gespmm_status_t gespmm_plan_get_info(gespmm_plan_t plan, gespmm_plan_info_t* info);

/* Which kernel variant a given N / alignment / op selects ("pair_vec4",
 * "vec4_lpr32_cwm2", ...), and a test-only override ("" = heuristic).
 * Not thread-safe. */
const char* gespmm_variant_name(int64_t N, const float* B, int64_t ldb, const float* C,
                                int64_t ldc, gespmm_reduce_t op);
gespmm_status_t gespmm_set_variant_override(const char* name);

/* gespmm_plan_execute with a FUSED C all-gather (SURVEY.md 8 e "fusion
 * option", f4): the kernel stores every finished C row both into C (this
 * rank's slab, ld = ldc) and into each of peers[0..n_peers) -- full-C buffers
 * of the node's GPUs (opened with gespmm_ipc_open_handle; P2P stores over
 * NVLink) or this GPU's own -- at row peer_row0 + (local row), same ld.  The
 * transfer overlaps the computation row by row; no collective call.  The
 * caller synchronizes the ranks afterwards (stream sync + a barrier) before
 * reading the full C.  n_peers <= 8. */
gespmm_status_t gespmm_plan_execute_peers(gespmm_plan_t plan, int64_t N, const int32_t* rowptr,
                                          const int32_t* colind, const float* vals, const float* B,
                                          int64_t ldb, float* C, int64_t ldc, gespmm_reduce_t op,
                                          int accumulate, float* const* peers, int n_peers,
                                          int64_t peer_row0, void* stream);
/* CUDA IPC of a device buffer for the fused all-gather (64-byte handles).
 * get: the handle of the allocation containing dev_ptr and dev_ptr's byte
 * offset in it; open (in another process): the allocation's base -- add the
 * offset.  close takes the base open returned. */
gespmm_status_t gespmm_ipc_get_handle(void* dev_ptr, char handle[64], int64_t* offset);
gespmm_status_t gespmm_ipc_open_handle(const char handle[64], void** dev_ptr);
gespmm_status_t gespmm_ipc_close_handle(void* dev_ptr);

/* Column-panel width for gespmm_plan_execute (DESIGN.md 5.2 "Panels"): -1 =
 * heuristic (panels of the widest power-of-two width whose K x width B slab
 * fits the L2 budget, only when B itself does not), 0 = never split, > 0 =
 * force panels of `cols` columns.  Results are identical for every width
 * (columns are independent).  Test/tuning knob; not thread-safe. */
gespmm_status_t gespmm_set_panel_override(int64_t cols);
/* Item distribution across warps: -1 = automatic (a dynamic atomic counter
 * when the plan has >= 16384 work items, static warp striding below), 0 =
 * static, 1 = dynamic.  Results are identical either way.  Test/tuning
 * knob; not thread-safe. */
gespmm_status_t gespmm_set_schedule_override(int mode);
/* Tile size of plans built after the call, in work units (a row costs deg +
 * 2): 0 = automatic (the largest power of two in [16, 256] that still gives
 * every warp slot of the GPU work; 256 for large matrices), or a forced value
 * in [2, 256].  Results are identical for every value (rows stay whole).
 * Test/tuning knob; not thread-safe. */
gespmm_status_t gespmm_set_tile_work_override(int32_t units);
/* The kernel variant the plan's last execute launched (diagnostics; "" before
 * the first execute), e.g. "vec4_lpr32_cwm1_ring". */
const char* gespmm_plan_last_variant(gespmm_plan_t plan);
/* The panel width gespmm_plan_execute uses for a K-row B with N columns: one
 * kernel launch per panel, ceil(N / width) launches per execute. */
int64_t gespmm_panel_width(int64_t K, int64_t N);

/* nnz-balanced row partition for row-block sharding over `parts` ranks
 * (HOST rowptr): bounds[0..parts] with bounds[0] = 0, bounds[parts] = M,
 * cut so that (nnz + rows) per part is balanced.  Rows never span parts. */
gespmm_status_t gespmm_partition_rows(int64_t M, const int32_t* rowptr, int parts,
                                      int64_t* bounds);

/* ---- synthetic inputs on the GPU ------------
 * R-MAT (Graph500 quadrant recursion with probabilities a, b, c, d = 1-a-b-c;
 * no vertex permutation) with 2^scale rows/cols and `edges` sampled edges,
 * deduplicated and sorted by (row, col), as CSR into caller DEVICE buffers:
 * rowptr int32[2^scale + 1], colind int32[edges], vals fp32[edges] (U[-1,1)).
 * *nnz_out = unique edges (<= edges).  Uniforms are Philox4x32-10 keyed by
 * `seed` and counted by (edge, level): the graph depends on the arguments only.
 * Synchronizes `stream` once (the unique count). */
gespmm_status_t gespmm_rmat_csr(int32_t scale, int64_t edges, double a, double b, double c,
                                uint64_t seed, int32_t* rowptr, int32_t* colind, float* vals,
                                int64_t* nnz_out, void* stream);
/* out[i] = lo + (hi - lo) * u_i, u_i = Philox(seed, i) in [0, 1) (24-bit), on `stream`. */
gespmm_status_t gespmm_uniform_fill(float* out, int64_t n, float lo, float hi, uint64_t seed,
                                    void* stream);

/* ---- format conversions on the GPU (the data formats around the path) ----
 * COO -> CSR: rows/cols/vals[nnz] (DEVICE) -> rowptr[M+1], colind/vals_out[nnz];
 * entries keep their input order within a row (stable), duplicates are kept
 * (the CSR contract allows both; the within-row order is the fold order).
 * GESPMM_OUT_OF_BOUNDS when a row index lies outside [0, M).  Synchronizes
 * `stream` once (the range check). */
gespmm_status_t gespmm_coo_to_csr(int64_t M, int64_t nnz, const int32_t* rows, const int32_t* cols,
                                  const float* vals, int32_t* rowptr, int32_t* colind, float* vals_out,
                                  void* stream);
/* CSR of A (M x K, DEVICE) -> CSR of A^T (K x M): t_rowptr[K+1],
 * t_colind/t_vals[nnz]; row j of A^T lists column j's nonzeros in ascending
 * row order (the CSC of A).  GESPMM_OUT_OF_BOUNDS for a column outside
 * [0, K).  Synchronizes `stream` once. */
gespmm_status_t gespmm_csr_transpose(int64_t M, int64_t K, int64_t nnz, const int32_t* rowptr,
                                     const int32_t* colind, const float* vals, int32_t* t_rowptr,
                                     int32_t* t_colind, float* t_vals, void* stream);

/* ---- multi-GPU (row-block sharding) -------------
 * NCCL is resolved at run time (dlopen "libnccl.so.2"; the copy already loaded
 * in the process wins), so the library never drags in a second NCCL. */

/* NCCL unique id (128 bytes) for gespmm_comm_init; call on one rank and ship
 * the bytes to the others out of band. */
gespmm_status_t gespmm_comm_get_unique_id(char id[128]);
/* Creates an ncclComm_t on the current device; *comm receives it. */
gespmm_status_t gespmm_comm_init(void** comm, int world, const char id[128], int rank);
gespmm_status_t gespmm_comm_destroy(void* comm);

/* Row-sharded SpMM on `comm`.  Each rank passes its row block of the CSR
 * (rowptr rebased to 0, M_local rows) and a B buffer of K x N (ldb); B is
 * broadcast from `root` over NVLink (ncclBroadcast, in place) -- the only
 * exchange -- then each rank computes its C slab (M_local x N, ldc).  If
 * C_full != NULL, the slabs are additionally all-gathered into C_full
 * (M_global x N, ld = ldc_full) with one ncclBroadcast per slab owner, using
 * row_bounds[0..world] (global row offsets of every rank's slab).  `plan`
 * may be NULL (a temporary plan is built).  Asynchronous on `stream` except
 * for temporary-plan creation. */
gespmm_status_t gespmm_sharded_spmm(void* comm, int world, int rank, int root,
                                    gespmm_plan_t plan, int64_t M_local, int64_t K, int64_t N,
                                    int64_t nnz_local, const int32_t* rowptr,
                                    const int32_t* colind, const float* vals, float* B,
                                    int64_t ldb, float* C, int64_t ldc, gespmm_reduce_t op,
                                    int accumulate, float* C_full, int64_t ldc_full,
                                    const int64_t* row_bounds, void* stream);

/* As gespmm_sharded_spmm, with the C all-gather overlapped with the
 * computation: each slab is computed in `chunks` row
 * chunks (gespmm_plan_execute_rows) and chunk j of every slab is broadcast by
 * its owner on an internal comm stream while chunk j+1 is computed.
 * chunks = 1 is gespmm_sharded_spmm.  Returns after the gather has drained. */
gespmm_status_t gespmm_sharded_spmm_chunked(void* comm, int world, int rank, int root,
                                            gespmm_plan_t plan, int64_t M_local, int64_t K, int64_t N,
                                            int64_t nnz_local, const int32_t* rowptr,
                                            const int32_t* colind, const float* vals, float* B,
                                            int64_t ldb, float* C, int64_t ldc, gespmm_reduce_t op,
                                            int accumulate, float* C_full, int64_t ldc_full,
                                            const int64_t* row_bounds, int chunks, void* stream);

/* Options of gespmm_sharded_spmm_ex. */
typedef struct {
  /* > 1: B is broadcast in this many column panels (widths multiples of 32
   * where N allows), panel p on an internal comm stream while panel p-1
   * computes; non-root ranks' B is then NOT written --
   * the panels live in b_panel_ws.  1: one in-place broadcast of B. */
  int b_panels;
  /* K*N floats of device workspace for the panels; NULL: allocated and freed
   * stream-ordered per call. */
  float* b_panel_ws;
  /* > 1: C all-gather overlapped with the compute in this many row chunks
   * (needs b_panels == 1). */
  int c_chunks;
  /* > 0: return only after the work drained, polling ncclCommGetAsyncError;
   * an asynchronous NCCL error or a wait longer than timeout_ms ABORTS the
   * communicator (ncclCommAbort) and returns GESPMM_NCCL_ERROR -- a dead peer
   * is an error, not a hang.  0: asynchronous on `stream` (the internal
   * waits use GESPMM_NCCL_TIMEOUT_MS, default 600000). */
  int64_t timeout_ms;
} gespmm_shard_opts_t;

/* Row-sharded SpMM with options (the two entry points above are this with
 * {1, NULL, 1, 0} and {1, NULL, chunks, 0}).  With plan == NULL a temporary
 * plan VALIDATES this rank's CSR (colind range included) before any
 * collective, and the ranks agree on the outcome with one all-reduce: a rank
 * whose block is invalid returns GESPMM_CSR_INVALID and every other rank
 * returns it too (no rank is left waiting in a broadcast). */
gespmm_status_t gespmm_sharded_spmm_ex(void* comm, int world, int rank, int root, gespmm_plan_t plan,
                                       int64_t M_local, int64_t K, int64_t N, int64_t nnz_local,
                                       const int32_t* rowptr, const int32_t* colind, const float* vals,
                                       float* B, int64_t ldb, float* C, int64_t ldc, gespmm_reduce_t op,
                                       int accumulate, float* C_full, int64_t ldc_full,
                                       const int64_t* row_bounds, const gespmm_shard_opts_t* opts,
                                       void* stream);

/* Waits for `stream` while polling ncclCommGetAsyncError(comm): GESPMM_OK when
 * the stream drained; on an asynchronous NCCL error or after timeout_ms (> 0)
 * the communicator is aborted (ncclCommAbort; a later gespmm_comm_destroy is a
 * no-op) and GESPMM_NCCL_ERROR is returned. */
gespmm_status_t gespmm_comm_wait(void* comm, void* stream, int64_t timeout_ms);

#ifdef __cplusplus
}
#endif

#endif /* GESPMM_H_ */
