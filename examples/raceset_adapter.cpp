// raceset_adapter.cpp -- the binding a raceset maintainer adds to compute the
// GE-SpMM values of a ConcreteInstance on a B200 through libgespmm.so.
//
// Reference types: raceset::ConcreteInstance (proj/include/raceset/oracle.hpp:17-35),
// raceset::validate_instance (oracle.hpp:38-39), raceset::Error (error.hpp:36-56).
// The reference's run(inst, gespmm_alg2) (oracle.cpp:699-736) returns only the
// access log; this returns the C it would have computed (fp32).
//
// Build (examples/Makefile):  g++ -std=c++20 -I<ref>/proj/include -I<repo>/include
//   raceset_adapter.cpp <ref objects> -L<repo>/paper_2503_08946_b200 -lgespmm
#include <cstdint>
#include <stdexcept>
#include <vector>

#include "gespmm.h"
#include "raceset/error.hpp"
#include "raceset/oracle.hpp"

namespace raceset_b200 {

// C = C0 + A*B for the instance's gespmm_alg2 arrays (rowPtr, colInd, val, B,
// C; params M, N, K).  Throws raceset::Error with the reference's kinds.
std::vector<float> gespmm_values(const raceset::ConcreteInstance& inst,
                                 gespmm_reduce_t op = GESPMM_REDUCE_SUM) {
  raceset::validate_instance(inst);  // the reference's own CSR rules first
  const int64_t M = inst.params.at("M"), N = inst.params.at("N"), K = inst.params.at("K");
  const auto& a = inst.arrays;
  std::vector<int32_t> rowptr(a.at("rowPtr").ints.begin(), a.at("rowPtr").ints.end());
  std::vector<int32_t> colind(a.at("colInd").ints.begin(), a.at("colInd").ints.end());
  std::vector<float> vals(a.at("val").floats.begin(), a.at("val").floats.end());
  std::vector<float> B(a.at("B").floats.begin(), a.at("B").floats.end());
  std::vector<float> C(a.at("C").floats.begin(), a.at("C").floats.end());
  if (static_cast<int64_t>(rowptr.size()) < M + 1 || static_cast<int64_t>(B.size()) < K * N ||
      static_cast<int64_t>(C.size()) < M * N)
    throw raceset::Error(raceset::ErrorKind::OutOfBounds, "instance arrays smaller than M/N/K");
  rowptr.resize(M + 1);
  gespmm_status_t st = gespmm_csr_spmm_host(M, K, N, rowptr[M], rowptr.data(), colind.data(),
                                            vals.data(), B.data(), N, C.data(), N, op,
                                            /*accumulate (mir:55-59)*/ 1, nullptr);
  if (st == GESPMM_CSR_INVALID) throw raceset::Error(raceset::ErrorKind::CsrInvalid, gespmm_last_error());
  if (st == GESPMM_OUT_OF_BOUNDS) throw raceset::Error(raceset::ErrorKind::OutOfBounds, gespmm_last_error());
  if (st != GESPMM_OK) throw std::runtime_error(gespmm_last_error());
  C.resize(M * N);
  return C;
}

}  // namespace raceset_b200

#ifdef RACESET_ADAPTER_MAIN
#include <cstdio>
int main(int argc, char** argv) {
  if (argc < 2) {
    std::fprintf(stderr, "usage: %s <instance.inst>\n", argv[0]);
    return 2;
  }
  try {
    raceset::ConcreteInstance inst = raceset::load_instance_file(argv[1]);
    std::vector<float> C = raceset_b200::gespmm_values(inst);
    for (float c : C) std::printf("%g ", c);
    std::printf("\n");
  } catch (const std::exception& e) {
    std::fprintf(stderr, "%s\n", e.what());
    return 1;
  }
  return 0;
}
#endif
