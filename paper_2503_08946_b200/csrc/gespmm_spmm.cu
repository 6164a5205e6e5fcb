// gespmm_spmm.cu -- kernel dispatch and tile-shape selection.  The kernel
// family itself is gespmm_kernel.cuh, instantiated per reduce op in
// gespmm_spmm_{sum,max,min,mean}.cu.
#include <cstdlib>

#include "gespmm_internal.h"

namespace gespmm {

cudaError_t launch_spmm_sum(const Variant& v, const KParams& p, cudaStream_t s);
cudaError_t launch_spmm_max(const Variant& v, const KParams& p, cudaStream_t s);
cudaError_t launch_spmm_min(const Variant& v, const KParams& p, cudaStream_t s);
cudaError_t launch_spmm_mean(const Variant& v, const KParams& p, cudaStream_t s);

cudaError_t launch_spmm(gespmm_reduce_t op, const Variant& v, const KParams& p,
                        cudaStream_t stream) {
  switch (op) {
    case GESPMM_REDUCE_SUM: return launch_spmm_sum(v, p, stream);
    case GESPMM_REDUCE_MAX: return launch_spmm_max(v, p, stream);
    case GESPMM_REDUCE_MIN: return launch_spmm_min(v, p, stream);
    case GESPMM_REDUCE_MEAN: return launch_spmm_mean(v, p, stream);
  }
  return cudaErrorInvalidValue;
}

int variant_cols(const Variant& v) { return v.pair ? 16 * v.vec : 32 * v.vec * v.cwm; }

std::string variant_name(const Variant& v) {
  if (v.pair) return "pair_vec" + std::to_string(v.vec);
  return "vec" + std::to_string(v.vec) + "_lpr32_cwm" + std::to_string(v.cwm) + (v.ring ? "_ring" : "");
}

namespace {
// in preference order for equal idle lanes / column blocks.  The paired-lane
// kernel comes last: at N=64 the 32-lane kernel measured faster (0.362 vs
// 0.382 ms on config 2); it wins only where 32 lanes would idle (N < 32).
const Variant kVariants[] = {{4, 1, false, false}, {4, 2, false, false}, {2, 1, false, false},
                             {2, 2, false, false}, {1, 1, false, false}, {1, 2, false, false},
                             {4, 1, true, false},  {2, 1, true, false},  {1, 1, true, false},
                             {4, 1, false, true},  {2, 1, false, true}};
}  // namespace

bool parse_variant(const char* name, Variant* v) {
  for (const Variant& c : kVariants)
    if (variant_name(c) == name) {
      *v = c;
      return true;
    }
  return false;
}

// Tile shape selected by N and op (north star item (1)): fewest idle lanes,
// then fewest column blocks, then the table order above.
Variant choose_variant(int64_t N, const float* B, int64_t ldb, const float* C, int64_t ldc,
                       gespmm_reduce_t op /* every variant implements every op */) {
  auto aligned = [&](int vec) {
    const uintptr_t a = static_cast<uintptr_t>(vec) * 4;
    return reinterpret_cast<uintptr_t>(B) % a == 0 && reinterpret_cast<uintptr_t>(C) % a == 0 &&
           ldb % vec == 0 && ldc % vec == 0 && N % vec == 0;
  };
  Variant best{1, 1, false};
  int64_t best_idle = -1, best_ncb = 0;
  // max/min at the 32-column tile: the paired-lane kernel first (FMUL2 +
  // FMNMX3 over two positions per warp instruction; config 3 N=32 max 1.286
  // -> 1.218 ms); sum/mean keep the 32-lane kernel there (1.159 vs 1.186 ms,
  // profiles/r2_pairperm/)
  const bool pair_first = (op == GESPMM_REDUCE_MAX || op == GESPMM_REDUCE_MIN) && N > 16 && N <= 32;
  if (pair_first && aligned(2)) {
    best = Variant{2, 1, true, false};
    best_idle = 32 - N;
    best_ncb = 1;
  }
  for (const Variant& c : kVariants) {
    if (!aligned(c.vec) || c.ring) continue;
    const int64_t cols = variant_cols(c);
    const int64_t ncb = (N + cols - 1) / cols;
    const int64_t idle = ncb * cols - N;
    if (best_idle < 0 || idle < best_idle || (idle == best_idle && ncb < best_ncb)) {
      best = c;
      best_idle = idle;
      best_ncb = ncb;
    }
  }
  // The shared-memory gather ring (gespmm_kernel.cuh Ring): on for the
  // 128-column tile (VEC = 4: 512-byte rows, DRAM-bound R-MAT configs 4/5,
  // config 4: 3.09 -> 2.82 ms), off for the 64-column tile where the register
  // pipeline wins (config 2: 0.367 vs 0.485 ms).  GESPMM_RING=0 / 1 / 2 forces
  // off / on for VEC = 4 (default) / on for VEC >= 2.
  static const int ring_mode = [] {
    const char* e = std::getenv("GESPMM_RING");
    return e ? std::atoi(e) : 1;
  }();
  if (!best.pair && best.cwm == 1 && ((ring_mode >= 1 && best.vec == 4) || (ring_mode == 2 && best.vec >= 2)))
    best.ring = true;
  return best;
}

}  // namespace gespmm
