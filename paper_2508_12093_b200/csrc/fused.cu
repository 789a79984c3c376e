// fused.cu — E6/E7: the standalone per-slot program kernel (k_prog).
//
// Every inverse-root / Chebyshev / Newton entry point is slot-wise: no rotation
// occurs between its input and its output, and its op DAG (chebyshev.hpp:
// 113-163, primitives.hpp:105-217) is data-independent.  The host replays the
// DAG's control flow symbolically (flow.h, SymB) for levels and meter, then
// launches one kernel that evaluates the whole DAG per slot in registers:
// ~1,050 quantised ops per slot for a degree-511 seed plus 6 Newton steps, with
// no HBM traffic between ops (16 B/slot algorithmic).  The program is a short
// list of macro instructions (kernels.h MOp) read from the constant bank; the
// evaluator itself is prog.cuh (shared with the statistics kernel, stat.cu).
// Geometry: one block per SM, each owning an equal contiguous slot range, P
// lanes per slot (prog.cuh prog_geometry).
#include <cstdio>

#include "core.h"
#include "kernels.h"
#include "quant.cuh"
#include "prog.cuh"

namespace hsg {
namespace k {
namespace {

// ---- the interpreter kernel --------------------------------------------------------------
template <class Q, int P>
__global__ void __launch_bounds__(prog_max_threads<P>(), 1) k_prog(Q q, const __grid_constant__ Prog pg) {
  extern __shared__ double stab[];
  for (int i = threadIdx.x; i < pg.ntab; i += blockDim.x) stab[i] = __ldg(pg.tabs + i);
  __syncthreads();
  const Range R = block_range(pg.S);
  if (R.lo >= R.hi) return;
  const unsigned iters = (R.spb * P + blockDim.x - 1) / blockDim.x;
  for (unsigned it = 0; it < iters; ++it) {
    const unsigned g = threadIdx.x + it * blockDim.x;
    const unsigned slot = R.lo + g / P;
    const bool live = slot < R.hi;
    // dead lanes shadow a live slot so lane-group shuffles stay converged
    exec<Q, P>(q, pg, stab, live ? slot : R.hi - 1, static_cast<int>(g % P), live, nullptr);
  }
}

// Fused kernels only run on-grid inputs (QGrid) or unquantised ones (QNone).
template <class F>
void with_q(QSpec qs, F&& f) {
  const double s = ldexp(1.0, qs.bits), inv = ldexp(1.0, -qs.bits);
  switch (qs.mode) {
    case QMode::None: f(QNone{}); break;
    case QMode::Grid: f(QGrid{s, inv}); break;
    default: fail(HS_E_ERROR, "fused kernels take QNone or QGrid only");
  }
}

}  // namespace

void run_prog(QSpec qs, const Prog& p, int lanes, cudaStream_t s) {
  if (p.S == 0) return;
  with_q(qs, [&](auto Q) {
    using QT = decltype(Q);
    const size_t smem = static_cast<size_t>(p.ntab) * sizeof(double);
    auto go = [&](auto kern, int P, int maxt) {
      if (smem > 48 * 1024)
        cuda_ok(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)),
                "prog smem attr");
      const Geo g = prog_geometry(p.S, P, Runtime::get().sm_count(), maxt);
      kern<<<g.blocks, g.threads, smem, s>>>(Q, p);
    };
    if (lanes == 8) go(k_prog<QT, 8>, 8, prog_max_threads<8>());
    else if (lanes == 4) go(k_prog<QT, 4>, 4, prog_max_threads<4>());
    else if (lanes == 2) go(k_prog<QT, 2>, 2, prog_max_threads<2>());
    else go(k_prog<QT, 1>, 1, prog_max_threads<1>());
  });
  cuda_ok(cudaGetLastError(), "prog launch");
  Runtime::get().note_launch();
}

}  // namespace k
}  // namespace hsg
