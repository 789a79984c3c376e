// fused.cu — E6-E8: per-slot fused programs and the statistics reduction kernels.
//
// Per-slot program (k_prog).  Every inverse-root / Chebyshev / Newton entry
// point is slot-wise: no rotation occurs between its input and its output, and
// its op DAG (chebyshev.hpp:113-163, primitives.hpp:105-217) is data-independent.
// The host replays the DAG's control flow symbolically (flow.h, SymB) for
// levels and meter, then launches one kernel that evaluates the whole DAG per
// slot in registers: ~1,050 quantised ops per slot for a degree-511 seed plus
// 6 Newton steps, with no HBM traffic between ops (16 B/slot algorithmic).
// The program is a short list of macro instructions (kernels.h MOp) read from
// the constant bank; the Chebyshev BSGS tree itself is straight-line code
// (cheb_full<K>) keeping T_1..T_{2^(K-1)} and the recursion partials in
// registers.  With `lanes` > 1 the top log2(lanes) levels of a full-degree
// (2^K - 1) tree are split across adjacent threads and recombined with warp
// shuffles, so 32768 slots fill the 148 SMs.
//
// Reduction kernels (moments / central).  The statistics pipelines'
// rotate-and-sum reductions (stats.hpp:41-87) run through slotsum.cuh with the
// producing slot-wise ops fused into the prologue and the consuming ones into
// the epilogue.
#include <cstdio>

#include "core.h"
#include "kernels.h"
#include "quant.cuh"
#include "prog.cuh"
#include "slotsum.cuh"

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

// ---- statistics reduction functors -----------------------------------------------------
constexpr int kMaxCols = 2;

template <class Q>
struct MomPro {
  Q q;
  MomArgs a[kMaxCols];
  template <int NA>
  __device__ void operator()(unsigned b, unsigned i, double (&v)[NA]) const {
    const MomArgs& A = a[b];
    for (int c = 0; c < A.nchunks; ++c) {
      const double X = q.in(__ldg(A.x[c] + i));
      double t[3];
      int k = 0;
      if (A.mode & MOM_MEAN) t[k++] = q.mulc(X, A.cm);  // mul_pt(chunk, 1/(B n))
      if (A.mode & MOM_VAR) {
        const double s = q.mulc(X, A.ca);               // mul_pt(chunk, 1/sqrt(S n))
        t[k++] = q.mul(s, s);                           // mul_ct(a, a)
        t[k++] = q.mulc(X, A.cmp);                      // mul_pt(chunk, 1/(n sqrt(S)))
      }
#pragma unroll
      for (int j = 0; j < NA; ++j) v[j] = c == 0 ? t[j] : q.add(v[j], t[j]);
    }
  }
};

template <class Q>
struct MomEpi {
  Q q;
  int mode[kMaxCols];
  double* mu[kMaxCols];
  double* var[kMaxCols];
  template <int NA>
  __device__ void operator()(unsigned b, unsigned i, const double (&v)[NA]) const {
    int k = 0;
    if (mode[b] & MOM_MEAN) mu[b][i] = q.out(v[k++]);
    if (mode[b] & MOM_VAR) {
      const double sq_sum = v[k], mp = v[k + 1];
      var[b][i] = q.out(q.sub(sq_sum, q.mul(mp, mp)));  // sub_ct(sq_sum, mul_ct(mp, mp))
    }
  }
};

template <class Q>
struct CentPro {
  Q q;
  CentArgs a;
  unsigned S;
  template <int NA>
  __device__ void operator()(unsigned, unsigned i, double (&v)[NA]) const {
    const double mux = q.in(__ldg(a.mux + i));
    const double muy = a.power == 2 ? q.in(__ldg(a.muy + i)) : 0.0;
    for (int c = 0; c < a.nchunks; ++c) {
      const double mm = a.valid[c] < S ? q.mulc(mux, i < a.valid[c] ? 1.0 : 0.0) : mux;  // mul_pt(mu, mask)
      const double cx = q.sub(q.in(__ldg(a.x[c] + i)), mm);
      double p;
      if (a.power == 4) {
        const double sq = q.mul(cx, cx);
        p = q.mul(sq, sq);
      } else if (a.power == 3) {
        const double sq = q.mul(cx, cx);
        p = q.mul(sq, cx);
      } else {
        p = q.mul(cx, q.sub(q.in(__ldg(a.y[c] + i)), muy));
      }
      const double term = q.mulc(p, a.inv_n);  // mean_of_chunks: mul_pt(chunk, 1/n)
      v[0] = c == 0 ? term : q.add(v[0], term);
    }
  }
};

template <class Q>
struct CentEpi {
  Q q;
  double* out;
  template <int NA>
  __device__ void operator()(unsigned, unsigned i, const double (&v)[NA]) const {
    out[i] = q.out(v[0]);
  }
};

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

void moments(QSpec qs, const MomArgs* cols, int ncols, size_t S, cudaStream_t s) {
  if (ncols < 1 || ncols > kMaxCols) fail(HS_E_ERROR, "moments: bad column batch");
  const int mode = cols[0].mode;
  for (int c = 1; c < ncols; ++c)
    if (cols[c].mode != mode) fail(HS_E_ERROR, "moments: mixed modes in one batch");
  const int NA = (mode & MOM_MEAN ? 1 : 0) + (mode & MOM_VAR ? 2 : 0);
  with_q(qs, [&](auto Q) {
    using QT = decltype(Q);
    MomPro<QT> pro{};
    MomEpi<QT> epi{};
    pro.q = Q;
    epi.q = Q;
    for (int c = 0; c < ncols; ++c) {
      pro.a[c] = cols[c];
      epi.mode[c] = cols[c].mode;
      epi.mu[c] = cols[c].mu;
      epi.var[c] = cols[c].var;
    }
    if (NA == 1) launch_slotsum<QT, 1>(Q, pro, epi, S, ncols, s);
    else if (NA == 2) launch_slotsum<QT, 2>(Q, pro, epi, S, ncols, s);
    else launch_slotsum<QT, 3>(Q, pro, epi, S, ncols, s);
  });
}

void central(QSpec qs, const CentArgs& a, size_t S, cudaStream_t s) {
  with_q(qs, [&](auto Q) {
    using QT = decltype(Q);
    CentPro<QT> pro{Q, a, static_cast<unsigned>(S)};
    CentEpi<QT> epi{Q, a.out};
    launch_slotsum<QT, 1>(Q, pro, epi, S, 1, s);
  });
}

}  // namespace k
}  // namespace hsg
