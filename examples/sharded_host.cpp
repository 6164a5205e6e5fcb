// sharded_host.cpp -- a C++ host driving the multi-GPU path through the C-ABI
// alone (no Python, no torch): one thread per visible GPU, one NCCL rank per
// thread, row-block sharding with the column-panelled B broadcast overlapped
// with the compute, the C all-gather, and a bounded error-polled wait
// (gespmm_sharded_spmm_ex).
//
//   examples/sharded_host [M K N nnz_per_row panels]      (defaults 200000 50000 128 24 4)
//
// Every rank ends with the full C; rank 0 checks sampled rows against a
// host-side fp64 sum (north-star bound |c - ref| <= 1e-5 max(|ref|, sum|v b|))
// and prints one line: "sharded_host ok ..." or the first failure.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <string>
#include <thread>
#include <vector>

#include "gespmm.h"

namespace {

struct Problem {
  int64_t M, K, N;
  std::vector<int32_t> rowptr, colind;
  std::vector<float> vals, B;
};

Problem make_problem(int64_t M, int64_t K, int64_t N, int per_row) {
  Problem p{M, K, N, {}, {}, {}, {}};
  std::mt19937_64 rng(7);
  std::uniform_real_distribution<float> u(-1.f, 1.f);
  p.rowptr.assign(M + 1, 0);
  for (int64_t i = 0; i < M; ++i) {
    // skewed degrees (some empty rows, some long rows that are split in segments)
    const int64_t r = static_cast<int64_t>(rng() % 1000);
    const int64_t d = r < 300 ? 0 : r > 995 ? 40 * per_row : static_cast<int64_t>(rng() % (2 * per_row + 1));
    p.rowptr[i + 1] = static_cast<int32_t>(p.rowptr[i] + d);
  }
  const int64_t nnz = p.rowptr[M];
  p.colind.resize(nnz);
  p.vals.resize(nnz);
  for (int64_t e = 0; e < nnz; ++e) {
    p.colind[e] = static_cast<int32_t>(rng() % static_cast<uint64_t>(K));
    p.vals[e] = u(rng);
  }
  p.B.resize(K * N);
  for (auto& x : p.B) x = u(rng);
  return p;
}

#define CK(x)                                                                                   \
  do {                                                                                          \
    cudaError_t e_ = (x);                                                                       \
    if (e_ != cudaSuccess) {                                                                    \
      std::fprintf(stderr, "rank %d: %s:%d %s\n", rank, __FILE__, __LINE__, cudaGetErrorString(e_)); \
      return 1;                                                                                 \
    }                                                                                           \
  } while (0)
#define GK(x)                                                                                      \
  do {                                                                                             \
    gespmm_status_t s_ = (x);                                                                      \
    if (s_ != GESPMM_OK) {                                                                         \
      std::fprintf(stderr, "rank %d: %s -> %s: %s\n", rank, #x, gespmm_status_string(s_), gespmm_last_error()); \
      return 1;                                                                                    \
    }                                                                                              \
  } while (0)

int rank_main(int rank, int world, const char* id, const Problem& P, const std::vector<int64_t>& bounds,
              int panels, std::vector<float>* C_out) {
  CK(cudaSetDevice(rank));
  void* comm = nullptr;
  GK(gespmm_comm_init(&comm, world, id, rank));
  const int64_t a = bounds[rank], b = bounds[rank + 1];
  const int64_t p0 = P.rowptr[a], p1 = P.rowptr[b];
  const int64_t M_loc = b - a, nnz_loc = p1 - p0, K = P.K, N = P.N, M = P.M;
  std::vector<int32_t> rp(M_loc + 1);
  for (int64_t i = 0; i <= M_loc; ++i) rp[i] = P.rowptr[a + i] - static_cast<int32_t>(p0);
  cudaStream_t s;
  CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  int32_t *d_rp, *d_ci;
  float *d_v, *d_B, *d_C, *d_Cf;
  CK(cudaMalloc(&d_rp, (M_loc + 1) * 4));
  CK(cudaMalloc(&d_ci, (nnz_loc > 0 ? nnz_loc : 1) * 4));
  CK(cudaMalloc(&d_v, (nnz_loc > 0 ? nnz_loc : 1) * 4));
  CK(cudaMalloc(&d_B, K * N * 4));
  CK(cudaMalloc(&d_C, (M_loc > 0 ? M_loc : 1) * N * 4));
  CK(cudaMalloc(&d_Cf, M * N * 4));
  CK(cudaMemcpyAsync(d_rp, rp.data(), (M_loc + 1) * 4, cudaMemcpyHostToDevice, s));
  CK(cudaMemcpyAsync(d_ci, P.colind.data() + p0, nnz_loc * 4, cudaMemcpyHostToDevice, s));
  CK(cudaMemcpyAsync(d_v, P.vals.data() + p0, nnz_loc * 4, cudaMemcpyHostToDevice, s));
  if (rank == 0) CK(cudaMemcpyAsync(d_B, P.B.data(), K * N * 4, cudaMemcpyHostToDevice, s));
  // plan = NULL: this rank's block is validated before any collective and the
  // ranks agree on the outcome; B goes out in `panels` column panels
  // overlapped with the compute; every rank receives the full C; the call
  // returns after the work drained (or GESPMM_NCCL_ERROR after 2 minutes)
  const gespmm_shard_opts_t opts = {panels, nullptr, 1, 120000};
  GK(gespmm_sharded_spmm_ex(comm, world, rank, /*root*/ 0, nullptr, M_loc, K, N, nnz_loc, d_rp, d_ci, d_v, d_B, N,
                            d_C, N, GESPMM_REDUCE_SUM, 0, d_Cf, N, bounds.data(), &opts, s));
  if (rank == 0) {
    C_out->resize(M * N);
    CK(cudaMemcpyAsync(C_out->data(), d_Cf, M * N * 4, cudaMemcpyDeviceToHost, s));
  }
  CK(cudaStreamSynchronize(s));
  cudaFree(d_rp);
  cudaFree(d_ci);
  cudaFree(d_v);
  cudaFree(d_B);
  cudaFree(d_C);
  cudaFree(d_Cf);
  cudaStreamDestroy(s);
  GK(gespmm_comm_destroy(comm));
  return 0;
}

}  // namespace

int main(int argc, char** argv) {
  const int64_t M = argc > 1 ? std::atoll(argv[1]) : 200000;
  const int64_t K = argc > 2 ? std::atoll(argv[2]) : 50000;
  const int64_t N = argc > 3 ? std::atoll(argv[3]) : 128;
  const int per_row = argc > 4 ? std::atoi(argv[4]) : 24;
  const int panels = argc > 5 ? std::atoi(argv[5]) : 4;
  int world = 0;
  if (cudaGetDeviceCount(&world) != cudaSuccess || world < 1) {
    std::printf("sharded_host: no GPU\n");
    return 2;
  }
  const Problem P = make_problem(M, K, N, per_row);
  std::vector<int64_t> bounds(world + 1);
  int rank = -1;
  GK(gespmm_partition_rows(M, P.rowptr.data(), world, bounds.data()));
  char id[128];
  GK(gespmm_comm_get_unique_id(id));
  std::vector<int> rc(world, 0);
  std::vector<float> C;
  std::vector<std::thread> th;
  for (int r = 0; r < world; ++r)
    th.emplace_back([&, r] { rc[r] = rank_main(r, world, id, P, bounds, panels, &C); });
  for (auto& t : th) t.join();
  for (int r = 0; r < world; ++r)
    if (rc[r]) return 1;
  // rank 0's full C against a host fp64 sum on every 97th row
  double worst = 0;
  for (int64_t i = 0; i < M; i += 97)
    for (int64_t j = 0; j < N; ++j) {
      double ref = 0, mag = 0;
      for (int32_t e = P.rowptr[i]; e < P.rowptr[i + 1]; ++e) {
        const double t = static_cast<double>(P.vals[e]) * P.B[static_cast<int64_t>(P.colind[e]) * N + j];
        ref += t;
        mag += std::fabs(t);
      }
      const double bound = 1e-5 * std::fmax(std::fabs(ref), mag);
      const double err = std::fabs(C[i * N + j] - ref);
      if (bound > 0) worst = std::fmax(worst, err / bound);
      else if (err != 0) worst = 1e30;
    }
  std::printf("sharded_host %s: world=%d M=%lld K=%lld N=%lld nnz=%d panels=%d worst=%.4f of the 1e-5 bound\n",
              worst <= 1.0 ? "ok" : "FAILED", world, static_cast<long long>(M), static_cast<long long>(K),
              static_cast<long long>(N), P.rowptr[M], panels, worst);
  return worst <= 1.0 ? 0 : 1;
}
