// ref_replay.cpp -- drives the UNMODIFIED reference interpreter (raceset::run,
// /root/reference/proj/src/oracle.cpp:699-736) on the reference's own GE-SpMM
// kernel (/root/reference/proj/fixtures/gespmm_alg2.mir, embedded at build
// time) and recovers the C values it computed by replaying its access log.
//
// TEST INFRASTRUCTURE ONLY: linked into oracle/_ref/libgespmm_ref.so by
// oracle/Makefile from the reference sources where they lie (never copied into
// this repo).  Used (a) to generate / re-check the golden fixtures under
// tests/golden/, (b) to pin oracle/gespmm_oracle.c, and (c) as the timed CPU
// implementation of `bench.py --impl reference`.
//
// Why replay: run() returns only the AccessLog (oracle.cpp:735); the fp64 C it
// computed is discarded.  The log is in execution order (phase-synchronous
// rounds, oracle.cpp:718-734), so re-executing the kernel's dataflow over it
// reproduces every value the interpreter held:
//     %k = load colInd[pt]; %v = load val[pt]; store %k, sm_k[tx]; store %v, sm_v[tx]
//     %ki = load sm_k[kk]; %vv = load sm_v[kk]; %b = load B[..]; %c0 = load C[..]
//     store (%c0 + %vv * %b), C[..]          (gespmm_alg2.mir:29-34, :50-59)
// with the interpreter's arithmetic: fp64, product and sum rounded separately
// (oracle.cpp:599-604).
#include <atomic>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>
#include <map>
#include <string>
#include <thread>
#include <vector>

#include "raceset/error.hpp"
#include "raceset/miniir.hpp"
#include "raceset/oracle.hpp"

namespace {

const char* kGespmmMir =
#include "gespmm_alg2_mir.inc"
    ;

thread_local std::string g_err;

struct ThreadRegs {
  int64_t k = 0;     // last colInd load
  double v = 0;      // last val load
  double vv = 0;     // last sm_v load
  double b = 0;      // last B load
  double c0 = 0;     // last C load
};

int64_t linear_thread(const raceset::AccessLogEntry& e, const int64_t grid[3],
                      const int64_t block[3]) {
  int64_t b = (e.block[2] * grid[1] + e.block[1]) * grid[0] + e.block[0];
  int64_t t = (e.thread[2] * block[1] + e.thread[1]) * block[0] + e.thread[0];
  return b * block[0] * block[1] * block[2] + t;
}

// Replays the gespmm_alg2 dataflow over `log`; C (in/out) receives the values.
void replay(const raceset::AccessLog& log, const raceset::ConcreteInstance& inst,
            std::vector<double>& C) {
  const auto& colInd = inst.arrays.at("colInd").ints;
  const auto& val = inst.arrays.at("val").floats;
  const auto& Bv = inst.arrays.at("B").floats;
  int64_t nblocks = inst.grid[0] * inst.grid[1] * inst.grid[2];
  int64_t bsz = inst.block[0] * inst.block[1] * inst.block[2];
  std::vector<ThreadRegs> regs(static_cast<size_t>(nblocks * bsz));
  // shared arrays, per linear block (extent 4 in gespmm_alg2.mir:5)
  std::vector<std::vector<int64_t>> sm_k(static_cast<size_t>(nblocks), std::vector<int64_t>(4, 0));
  std::vector<std::vector<double>> sm_v(static_cast<size_t>(nblocks), std::vector<double>(4, 0.0));
  for (const auto& e : log) {
    ThreadRegs& r = regs[static_cast<size_t>(linear_thread(e, inst.grid, inst.block))];
    int64_t blk = (e.block[2] * inst.grid[1] + e.block[1]) * inst.grid[0] + e.block[0];
    int64_t cell = e.cell.at(0);
    bool rd = e.kind == raceset::AccessKind::Read;
    const std::string& a = e.array;
    if (a == "colInd") {
      r.k = colInd[static_cast<size_t>(cell)];
    } else if (a == "val") {
      r.v = val[static_cast<size_t>(cell)];
    } else if (a == "sm_k") {
      if (!rd) sm_k[static_cast<size_t>(blk)][static_cast<size_t>(cell)] = r.k;
    } else if (a == "sm_v") {
      if (rd) r.vv = sm_v[static_cast<size_t>(blk)][static_cast<size_t>(cell)];
      else sm_v[static_cast<size_t>(blk)][static_cast<size_t>(cell)] = r.v;
    } else if (a == "B") {
      r.b = Bv[static_cast<size_t>(cell)];
    } else if (a == "C") {
      if (rd) {
        r.c0 = C[static_cast<size_t>(cell)];
      } else {
        double prod = r.vv * r.b;  // %prod = mul %vv, %b
        C[static_cast<size_t>(cell)] = r.c0 + prod;  // %c1 = add %c0, %prod
      }
    }
    // rowPtr reads carry no value into C
  }
}

const raceset::Function& gespmm_function() {
  static const raceset::Function f = raceset::parse_miniir(kGespmmMir);
  return f;
}

// One instance covering rows [r0, r1) of the CSR, with B compacted to the
// referenced rows (values unchanged, so every C value is unchanged).
struct Piece {
  raceset::ConcreteInstance inst;
  int64_t r0 = 0, r1 = 0;
};

Piece make_piece(int64_t r0, int64_t r1, int64_t N, const int32_t* rowptr,
                 const int32_t* colind, const float* vals, const float* B, int64_t ldb,
                 const double* C0) {
  Piece pc;
  pc.r0 = r0;
  pc.r1 = r1;
  auto& inst = pc.inst;
  inst.name = "sample";
  int64_t M = r1 - r0;
  int64_t p0 = rowptr[r0], p1 = rowptr[r1];
  std::map<int32_t, int64_t> remap;
  for (int64_t p = p0; p < p1; ++p) remap.emplace(colind[p], 0);
  int64_t Kc = 0;
  for (auto& kv : remap) kv.second = Kc++;
  auto& rp = inst.arrays["rowPtr"];
  rp.elem = raceset::ElemKind::I32;
  for (int64_t i = r0; i <= r1; ++i) rp.ints.push_back(rowptr[i] - p0);
  auto& ci = inst.arrays["colInd"];
  ci.elem = raceset::ElemKind::I32;
  auto& vl = inst.arrays["val"];
  vl.elem = raceset::ElemKind::F32;
  for (int64_t p = p0; p < p1; ++p) {
    ci.ints.push_back(remap[colind[p]]);
    vl.floats.push_back(static_cast<double>(vals[p]));
  }
  auto& bb = inst.arrays["B"];
  bb.elem = raceset::ElemKind::F32;
  bb.floats.resize(static_cast<size_t>(Kc * N));
  for (auto& kv : remap)
    for (int64_t j = 0; j < N; ++j)
      bb.floats[static_cast<size_t>(kv.second * N + j)] =
          static_cast<double>(B[static_cast<int64_t>(kv.first) * ldb + j]);
  auto& cc = inst.arrays["C"];
  cc.elem = raceset::ElemKind::F32;
  cc.floats.assign(static_cast<size_t>(M * N), 0.0);
  if (C0)
    for (int64_t i = 0; i < M; ++i)
      for (int64_t j = 0; j < N; ++j)
        cc.floats[static_cast<size_t>(i * N + j)] = C0[(r0 + i) * N + j];
  inst.params["M"] = M;
  inst.params["N"] = N;
  inst.params["K"] = Kc > 0 ? Kc : 1;
  inst.params["A_S"] = p1 - p0;
  // one block per row, blockDim 4 (the kernel's shared extent, mir:5), and
  // enough column blocks to cover N.
  inst.grid[0] = M > 0 ? M : 1;
  inst.grid[1] = (N + 3) / 4;
  inst.grid[2] = 1;
  inst.block[0] = 4;
  inst.block[1] = 1;
  inst.block[2] = 1;
  raceset::ConcreteInstance::CsrSpec cs;
  cs.row_ptr = "rowPtr";
  cs.col_ind = "colInd";
  cs.val = "val";
  cs.cols = Kc > 0 ? Kc : 1;
  inst.csr = cs;
  return pc;
}

}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

// Runs the reference interpreter on a .inst text exactly as `raceset oracle`
// does (cli.cpp:192-199) and replays C.  c_out receives M*N doubles (the C
// array after the run); *log_len the number of logged accesses.
// Returns 0 on success, 1 + ErrorKind on a reference Error, -1 otherwise.
int ref_run_instance_text(const char* inst_text, double* c_out, int64_t c_cap,
                          int64_t* c_len, int64_t* log_len) {
  try {
    raceset::ConcreteInstance inst = raceset::parse_instance(inst_text);
    raceset::AccessLog log = raceset::run(inst, gespmm_function());
    std::vector<double> C = inst.arrays.at("C").floats;
    replay(log, inst, C);
    *c_len = static_cast<int64_t>(C.size());
    *log_len = static_cast<int64_t>(log.size());
    if (static_cast<int64_t>(C.size()) > c_cap) return -2;
    std::memcpy(c_out, C.data(), C.size() * sizeof(double));
    return 0;
  } catch (const raceset::Error& e) {
    g_err = e.what();
    return 1 + static_cast<int>(e.kind());
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

// Reference SpMM over a CSR: the rows are cut into `nthreads` contiguous
// pieces, each an independent ConcreteInstance run by raceset::run on its own
// std::thread ("instances may run in parallel", reference SPEC.md:478-479).
// seconds_out = wall time of the parallel run() calls only.  If C != nullptr
// the replayed fp64 result (C = C0 + A*B, C0 taken from C) is written back.
// Returns 0 on success, 1 + ErrorKind / -1 on failure.
int ref_spmm_csr(int64_t M, int64_t N, const int32_t* rowptr, const int32_t* colind,
                 const float* vals, const float* B, int64_t ldb, double* C, int nthreads,
                 int64_t step_limit, double* seconds_out, int64_t* log_entries_out) {
  try {
    if (nthreads < 1) nthreads = 1;
    if (nthreads > M) nthreads = M > 0 ? static_cast<int>(M) : 1;
    // nnz-balanced contiguous pieces
    int64_t nnz = rowptr[M];
    std::vector<int64_t> cut(static_cast<size_t>(nthreads) + 1, M);
    cut[0] = 0;
    for (int t = 1; t < nthreads; ++t) {
      int64_t target = nnz * t / nthreads;
      int64_t lo = cut[static_cast<size_t>(t) - 1], hi = M;
      while (lo < hi) {
        int64_t mid = (lo + hi) / 2;
        if (rowptr[mid] < target) lo = mid + 1;
        else hi = mid;
      }
      cut[static_cast<size_t>(t)] = lo;
    }
    std::vector<Piece> pieces;
    for (int t = 0; t < nthreads; ++t)
      pieces.push_back(make_piece(cut[static_cast<size_t>(t)], cut[static_cast<size_t>(t) + 1], N,
                                  rowptr, colind, vals, B, ldb, C));
    const raceset::Function& f = gespmm_function();
    std::vector<raceset::AccessLog> logs(pieces.size());
    std::vector<std::string> errs(pieces.size());
    std::vector<int> codes(pieces.size(), 0);
    raceset::RunOptions ro;
    ro.step_limit = step_limit > 0 ? step_limit : ro.step_limit;
    auto t0 = std::chrono::steady_clock::now();
    std::vector<std::thread> th;
    for (size_t t = 0; t < pieces.size(); ++t)
      th.emplace_back([&, t] {
        try {
          logs[t] = raceset::run(pieces[t].inst, f, ro);
        } catch (const raceset::Error& e) {
          errs[t] = e.what();
          codes[t] = 1 + static_cast<int>(e.kind());
        } catch (const std::exception& e) {
          errs[t] = e.what();
          codes[t] = -1;
        }
      });
    for (auto& x : th) x.join();
    auto t1 = std::chrono::steady_clock::now();
    if (seconds_out) *seconds_out = std::chrono::duration<double>(t1 - t0).count();
    int64_t total = 0;
    for (size_t t = 0; t < pieces.size(); ++t) {
      if (codes[t] != 0) {
        g_err = errs[t];
        return codes[t];
      }
      total += static_cast<int64_t>(logs[t].size());
    }
    if (log_entries_out) *log_entries_out = total;
    if (C) {
      for (size_t t = 0; t < pieces.size(); ++t) {
        std::vector<double> Cp = pieces[t].inst.arrays.at("C").floats;
        replay(logs[t], pieces[t].inst, Cp);
        int64_t rows = pieces[t].r1 - pieces[t].r0;
        std::memcpy(C + pieces[t].r0 * N, Cp.data(), static_cast<size_t>(rows * N) * sizeof(double));
      }
    }
    return 0;
  } catch (const raceset::Error& e) {
    g_err = e.what();
    return 1 + static_cast<int>(e.kind());
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

}  // extern "C"
