/*
 * gespmm_oracle.c -- CPU ORACLE for the GE-SpMM hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library, and
 * only as the checker or the timed CPU baseline -- never as the product path.
 * The product path (paper_2503_08946_b200/) never links or calls it.
 *
 * Two restatements of the reference algorithm live here:
 *
 *  1. oracle_spmm_ref_f64 -- what the reference interpreter computes when it
 *     executes /root/reference/proj/fixtures/gespmm_alg2.mir:
 *       - per output cell (i, j), nonzeros in ascending p
 *         (gespmm_alg2.mir:21-24 tile loop, :38-41 inner loop, :61-69 latches);
 *       - C[i*N+j] is read-modified-written: c1 = c0 + (val * B)
 *         (gespmm_alg2.mir:51-59);
 *       - arithmetic in fp64, product and sum rounded separately, no FMA
 *         (oracle.cpp:593-613), arrays held as double (oracle.cpp:337-352).
 *     Parity pinned against the goldens derived from the reference interpreter
 *     by log replay (tests/golden/, made by oracle/ref_replay.cpp).
 *
 *  2. oracle_spmm_f32 -- the fp32 "twin": the normative fp32 semantics of the
 *     B200 path: fp32 with explicit fused multiply-adds
 *     (fmaf); sum/mean reduce each row (segment) as two ascending FMA chains
 *     over the even- and odd-offset positions, added at the end; max/min are
 *     maximumNumber/minimumNumber over the row's messages; long rows (more than seg_len nonzeros) are reduced in
 *     seg_len-long segments combined left to right.  The GPU result is
 *     bit-identical to this twin.
 *
 * Build: oracle/Makefile (-O2 -fopenmp -ffp-contract=off, never -ffast-math).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

enum { OR_SUM = 0, OR_MAX = 1, OR_MIN = 2, OR_MEAN = 3 };

enum {
  OR_OK = 0,
  OR_CSR_INVALID = 1,
  OR_INVALID_ARG = 3,
};

/* Same rules as validate_instance (reference oracle.cpp:291-316): rowPtr
 * non-empty with rowPtr[0] == 0, nondecreasing, rowPtr.back() == |colInd|,
 * |colInd| == |val|, 0 <= colInd < cols.  Plus |rowPtr| == M + 1 (the kernel
 * reads rowPtr[i+1] for every i < M, gespmm_alg2.mir:17-18). */
int oracle_validate_csr(int64_t M, int64_t K, int64_t rowptr_len, const int32_t* rowptr,
                        int64_t colind_len, const int32_t* colind, int64_t vals_len) {
  if (M < 0 || K < 0) return OR_INVALID_ARG;
  if (rowptr_len < 1 || rowptr[0] != 0) return OR_CSR_INVALID;
  for (int64_t i = 1; i < rowptr_len; ++i)
    if (rowptr[i] < rowptr[i - 1]) return OR_CSR_INVALID;
  if ((int64_t)rowptr[rowptr_len - 1] != colind_len) return OR_CSR_INVALID;
  if (colind_len != vals_len) return OR_CSR_INVALID;
  for (int64_t p = 0; p < colind_len; ++p)
    if (colind[p] < 0 || (int64_t)colind[p] >= K) return OR_CSR_INVALID;
  if (rowptr_len != M + 1) return OR_CSR_INVALID;
  return OR_OK;
}

/* (1) fp64 restatement of the interpreter run.  C is in/out (the reference
 * kernel accumulates into C, gespmm_alg2.mir:55-59). */
void oracle_spmm_ref_f64(int64_t M, int64_t N, const int32_t* rowptr, const int32_t* colind,
                         const double* vals, const double* B, int64_t ldb, double* C,
                         int64_t ldc, int nthreads) {
#ifdef _OPENMP
  if (nthreads > 0) omp_set_num_threads(nthreads);
#pragma omp parallel for schedule(dynamic, 64)
#endif
  for (int64_t i = 0; i < M; ++i) {
    for (int64_t j = 0; j < N; ++j) {
      double c = C[i * ldc + j];
      for (int64_t p = rowptr[i]; p < rowptr[i + 1]; ++p) {
        double prod = vals[p] * B[(int64_t)colind[p] * ldb + j]; /* %prod = mul %vv, %b */
        c = c + prod;                                             /* %c1 = add %c0, %prod */
      }
      C[i * ldc + j] = c;
    }
  }
}

/* Companion bound used by the 1e-5 norm-wise tolerance: sum_p |val*B|. */
void oracle_spmm_absbound_f64(int64_t M, int64_t N, const int32_t* rowptr, const int32_t* colind,
                              const float* vals, const float* B, int64_t ldb, double* out,
                              int64_t ldo, int nthreads) {
#ifdef _OPENMP
  if (nthreads > 0) omp_set_num_threads(nthreads);
#pragma omp parallel for schedule(dynamic, 64)
#endif
  for (int64_t i = 0; i < M; ++i)
    for (int64_t j = 0; j < N; ++j) {
      double s = 0.0;
      for (int64_t p = rowptr[i]; p < rowptr[i + 1]; ++p)
        s += fabs((double)vals[p] * (double)B[(int64_t)colind[p] * ldb + j]);
      out[i * ldo + j] = s;
    }
}

/* (1b) The reference restatement for every reduce op, on fp32 inputs, in
 * fp64 (the interpreter's number type, oracle.cpp:337-352): products
 * val*B are exact in fp64 (24 + 24 significand bits); SUM is the reference's
 * ascending, unfused c = c + prod from c = 0 (gespmm_alg2.mir:51-59,
 * oracle.cpp:593-613); MEAN = SUM / deg; MAX/MIN = the largest/smallest exact
 * product (the semiring extension).  Empty rows give 0.
 * bound[i,j] = sum_p |val*B| (MEAN: / deg), the scale of the north star's
 * norm-wise 1e-5 tolerance.  Because fp32 rounding is monotone, a correct fp32
 * MAX/MIN equals (float) of this value exactly. */
void oracle_spmm_ref64_op(int64_t M, int64_t N, const int32_t* rowptr, const int32_t* colind,
                          const float* vals, const float* B, int64_t ldb, double* out,
                          double* bound, int op, int nthreads) {
#ifdef _OPENMP
  if (nthreads > 0) omp_set_num_threads(nthreads);
#pragma omp parallel for schedule(dynamic, 16)
#endif
  for (int64_t i = 0; i < M; ++i) {
    const int64_t rs = rowptr[i], re = rowptr[i + 1], deg = re - rs;
    for (int64_t j = 0; j < N; ++j) {
      double c = 0.0, s = 0.0;
      for (int64_t p = rs; p < re; ++p) {
        const double prod = (double)vals[p] * (double)B[(int64_t)colind[p] * ldb + j];
        s += fabs(prod);
        if (op == OR_SUM || op == OR_MEAN) c = c + prod;
        else if (p == rs) c = prod;
        else if (op == OR_MAX) c = prod > c ? prod : c;
        else c = prod < c ? prod : c;
      }
      if (op == OR_MEAN && deg) {
        c /= (double)deg;
        s /= (double)deg;
      }
      out[i * N + j] = c;
      bound[i * N + j] = s;
    }
  }
}

/* ---- (2) the fp32 twin ---------------------------------------------------- */

/* pick(op, a, b): the max/min fold step, IEEE 754-2019 maximumNumber /
 * minimumNumber (5.3.1) exactly as the B200's FMNMX computes them (measured,
 * tools/mnmx_probe.cu): a NaN operand is ignored, two NaNs give the canonical
 * NaN 0x7fffffff, and -0 < +0.  Commutative and associative, so a row's
 * max/min depends on its message multiset only (the GPU folds two messages
 * per FMNMX3).  Products are plain fp32 multiplies; the Makefile builds with
 * -ffp-contract=off so they are never contracted into an FMA. */
static inline float canonical_nan(void) {
  union { uint32_t u; float f; } x = {0x7fffffffu};
  return x.f;
}
static inline float pick(int op, float a, float b) {
  if (isnan(a)) return isnan(b) ? canonical_nan() : b;
  if (isnan(b)) return a;
  if (a == b) return (signbit(a) != 0) == (op == OR_MAX) ? b : a; /* +-0 tie; else identical */
  if (op == OR_MAX) return a > b ? a : b;
  return a < b ? a : b;
}

/* Reduce nonzeros [ps, pe) of one row into acc[0..N).  Per column j the order
 * is p ascending, exactly as in the reference (gespmm_alg2.mir:38-59).
 * mode: 0 = first segment without an initial value (sum: +0; max/min: the
 *           canonical NaN, maximumNumber's identity),
 *       1 = first segment seeded with init[] (accumulate=1: C0),
 *       2 = later segment (sum: +0; max/min: the canonical NaN). */
static void fold_span(int op, int64_t ps, int64_t pe, int64_t N, const int32_t* colind,
                      const float* vals, const float* B, int64_t ldb, int mode,
                      const float* init, float* acc) {
  int64_t p = ps;
  if (op == OR_SUM || op == OR_MEAN) {
    /* Two FMA chains: positions at even offsets from the span start (chain A,
     * seeded with init or +0) and at odd offsets (chain B, seeded with -0.0,
     * the exact additive identity); the span's value is A + B. */
    float* accb = acc + N;
    for (int64_t j = 0; j < N; ++j) {
      acc[j] = (mode == 1) ? init[j] : 0.0f;
      accb[j] = -0.0f;
    }
    for (; p < pe; ++p) {
      const float v = vals[p];
      const float* b = B + (int64_t)colind[p] * ldb;
      float* a = ((p - ps) & 1) ? accb : acc;
      for (int64_t j = 0; j < N; ++j) a[j] = fmaf(v, b[j], a[j]);
    }
    for (int64_t j = 0; j < N; ++j) acc[j] = acc[j] + accb[j];
    return;
  }
  for (int64_t j = 0; j < N; ++j) acc[j] = (mode == 1) ? init[j] : canonical_nan();
  for (; p < pe; ++p) {
    const float v = vals[p];
    const float* b = B + (int64_t)colind[p] * ldb;
    for (int64_t j = 0; j < N; ++j) {
      const float m = v * b[j];
      acc[j] = pick(op, acc[j], m);
    }
  }
}

/* C = A (op) B, or C = C0 (+) A (op) B with accumulate=1.  seg_len <= 0 means
 * "never split"; otherwise rows with deg > seg_len are reduced per segment
 * [rs + k*seg_len, rs + (k+1)*seg_len) and combined left to right:
 *   sum/mean: acc = acc + part;  max/min: acc = pick(acc, part).
 * Empty rows: sum/mean/max/min give 0 (accumulate=1: C0). */
int oracle_spmm_f32(int64_t M, int64_t N, const int32_t* rowptr, const int32_t* colind,
                    const float* vals, const float* B, int64_t ldb, float* C, int64_t ldc, int op,
                    int accumulate, int64_t seg_len, int nthreads) {
  if (op < OR_SUM || op > OR_MEAN || N < 0 || M < 0) return OR_INVALID_ARG;
  if (N == 0 || M == 0) return OR_OK;
#ifdef _OPENMP
  if (nthreads > 0) omp_set_num_threads(nthreads);
#pragma omp parallel
#endif
  {
    float* acc = (float*)malloc(sizeof(float) * (size_t)N * 5);
    float* part = acc + 2 * N;  /* fold_span uses [x, x + 2N) as its two chains */
    float* c0 = acc + 4 * N;
#ifdef _OPENMP
#pragma omp for schedule(dynamic, 256)
#endif
    for (int64_t i = 0; i < M; ++i) {
      const int64_t rs = rowptr[i], re = rowptr[i + 1], deg = re - rs;
      const int split = seg_len > 0 && deg > seg_len;
      const int64_t e0 = split ? rs + seg_len : re;
      float* out = C + i * ldc;
      for (int64_t j = 0; j < N; ++j) c0[j] = accumulate ? out[j] : 0.0f;
      if (op == OR_MAX || op == OR_MIN) {
        if (deg == 0) {
          for (int64_t j = 0; j < N; ++j) out[j] = c0[j];
          continue;
        }
        fold_span(op, rs, e0, N, colind, vals, B, ldb, accumulate ? 1 : 0, c0, acc);
        for (int64_t s = e0; s < re; s += seg_len) {
          int64_t e = s + seg_len < re ? s + seg_len : re;
          fold_span(op, s, e, N, colind, vals, B, ldb, 2, c0, part);
          for (int64_t j = 0; j < N; ++j) acc[j] = pick(op, acc[j], part[j]);
        }
        for (int64_t j = 0; j < N; ++j) out[j] = acc[j];
      } else {
        /* SUM seeds the chain with C0 (the reference's c0 + prod order);
         * MEAN reduces from +0 and adds C0 after the division. */
        const int seed = accumulate && op == OR_SUM;
        fold_span(op, rs, e0, N, colind, vals, B, ldb, seed ? 1 : 0, c0, acc);
        for (int64_t s = e0; s < re; s += seg_len) {
          int64_t e = s + seg_len < re ? s + seg_len : re;
          fold_span(op, s, e, N, colind, vals, B, ldb, 2, c0, part);
          for (int64_t j = 0; j < N; ++j) acc[j] = acc[j] + part[j];
        }
        if (op == OR_MEAN) {
          for (int64_t j = 0; j < N; ++j) {
            float r = deg ? acc[j] / (float)deg : 0.0f;
            out[j] = accumulate ? c0[j] + r : r;
          }
        } else {
          for (int64_t j = 0; j < N; ++j) out[j] = acc[j];
        }
      }
    }
    free(acc);
  }
  return OR_OK;
}

int oracle_num_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}
