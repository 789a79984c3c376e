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
#include "slotsum.cuh"

namespace hsg {
namespace k {
namespace {

constexpr int kProgThreads = 256;
constexpr int kMaxK = 10;  // T_{2^0} .. T_{2^9}; degree <= 1023

// ---- Chebyshev evaluation ------------------------------------------------------
// Series tables live in shared memory (staged once per block).  A table of a
// lane-split series is interleaved by part (element e of part l at e*P + l) so
// the P lanes of a slot read consecutive words (conflict-free) and all slots of
// a warp read the same words (broadcast).
//
// F_K: full tree of degree 2^K - 1 (K >= 1) or a degree-0 leaf (K == 0).
// Table layout [F_{K-1}(q) | F_{K-1}(r)], leaves (c1, c0).  chebyshev.hpp:140-158.
template <int K, int ST, class F>
__device__ __forceinline__ double ffull(const F& f, const double* t, const double (&T)[kMaxK]) {
  if constexpr (K <= 1) {
    return f.addc(f.mulc(T[0], t[0]), t[ST]);  // add_pt(mul_pt(x, c1), c0)
  } else {
    constexpr int H = (1 << (K - 1)) * ST;
    const double head = f.mul(ffull<K - 1, ST>(f, t, T), T[K - 1]);  // mul_ct(eval(q), T_g)
    const double rest = ffull<K - 1, ST>(f, t + H, T);
    return f.add(head, rest);                                       // add_ct(head, eval(r))
  }
}

template <int ST, class F>
__device__ __forceinline__ double ffull_dyn(int K, const F& f, const double* t, const double (&T)[kMaxK]) {
  switch (K) {
    case 0: return ffull<0, ST>(f, t, T);
    case 1: return ffull<1, ST>(f, t, T);
    case 2: return ffull<2, ST>(f, t, T);
    case 3: return ffull<3, ST>(f, t, T);
    case 4: return ffull<4, ST>(f, t, T);
    case 5: return ffull<5, ST>(f, t, T);
    case 6: return ffull<6, ST>(f, t, T);
    case 7: return ffull<7, ST>(f, t, T);
    case 8: return ffull<8, ST>(f, t, T);
    default: return ffull<9, ST>(f, t, T);
  }
}

__device__ __forceinline__ double tpow(int k, const double (&T)[kMaxK]) {
  switch (k) {
    case 0: return T[0];
    case 1: return T[1];
    case 2: return T[2];
    case 3: return T[3];
    case 4: return T[4];
    case 5: return T[5];
    case 6: return T[6];
    case 7: return T[7];
    case 8: return T[8];
    default: return T[9];
  }
}

// Exact iterative evaluation of F_k (post-order with an explicit stack):
// compact code for slots outside the fast path's range.
template <class Q>
__device__ double fslow(const Q& q, const double* t, int st, int k, const double* T) {
  if (k <= 1) return q.addc(q.mulc(T[0], t[0]), t[st]);
  double stack[kMaxK + 1];
  const int n = 1 << (k - 1);
  for (int j = 0; j < n; ++j) {
    double v = q.addc(q.mulc(T[0], t[(2 * j) * st]), t[(2 * j + 1) * st]);
    int m = 1;
    while (j & (1 << (m - 1))) {
      v = q.add(q.mul(stack[m], T[m]), v);
      ++m;
    }
    stack[m] = v;
  }
  return stack[k];
}

template <class Q>
__device__ __noinline__ double cheb_exact(Q q, const double* t, int d, double x, int P, int split) {
  const int K = 32 - __clz(d);
  double T[kMaxK];
  T[0] = x;
  for (int j = 1; j < K; ++j) {
    const double sq = q.mul(T[j - 1], T[j - 1]);
    T[j] = q.addc(q.add(sq, sq), q.in(-1.0));
  }
  if (split) {
    int p = 0;
    while ((1 << p) < P) ++p;
    const int Ks = K - p;
    double v[8];
    for (int l = 0; l < P; ++l) v[l] = fslow(q, t + l, P, Ks, T);
    for (int r = 0; r < p; ++r)
      for (int l = 0; l < P; l += 2 << r) v[l] = q.add(q.mul(v[l], T[Ks + r]), v[l + (1 << r)]);
    return v[0];
  }
  int gk[kMaxK];
  int m = 0, dd = d;
  bool pt = false;
  while (dd > 1) {
    const int k = 31 - __clz(dd);
    gk[m++] = k;
    dd -= 1 << k;
    if (dd == 0) {
      pt = true;
      break;
    }
  }
  const double* c = t;
  double v;
  if (pt) {
    v = q.mulc(T[gk[m - 1]], c[0]);
    c += 1;
  } else {
    v = q.addc(q.mulc(x, c[0]), c[1]);
    c += 2;
  }
  for (int i = m - 1; i >= 0; --i) {
    const int k = gk[i];
    const double head = (pt && i == m - 1) ? v : q.mul(v, T[k]);
    const double rest = fslow(q, c, 1, k, T);
    c += (k == 0) ? 2 : (1 << k);
    v = q.add(head, rest);
  }
  return v;
}

// ChebEncryptedEval::run (chebyshev.hpp:117-125) for degree d <= 1023; t in smem.
template <class Q, int P>
__device__ __forceinline__ double cheb_eval(const Q& q, const double* t, int d, double x, int lane, bool split,
                                            bool fast_ok) {
  if (d <= 0) return q.addc(q.sub(x, x), t[0]);        // add_pt(sub_ct(x, x), c0)
  if (d == 1) return q.addc(q.mulc(x, t[0]), t[1]);     // a single leaf
  if (!(fast_ok && FastOf<Q>::in_range(q, x))) return cheb_exact<Q>(q, t, d, x, P, split ? 1 : 0);
  using FF = typename FastOf<Q>::type;
  const FF ff = FastOf<Q>::make(q);
  const int K = 32 - __clz(d);
  double T[kMaxK];
  T[0] = x;
#pragma unroll
  for (int j = 1; j < kMaxK; ++j) {  // build_powers (chebyshev.hpp:130-138)
    if (j < K) {
      const double sq = ff.mul(T[j - 1], T[j - 1]);
      T[j] = ff.addc(ff.add(sq, sq), q.in(-1.0));
    } else {
      T[j] = 0.0;
    }
  }
  constexpr int p = P == 8 ? 3 : (P == 4 ? 2 : (P == 2 ? 1 : 0));
  if (P > 1 && split) {
    // lane-split full tree: lane l evaluates F_{K-p} on (interleaved) part l,
    // then the top p levels are recombined pairwise (partner = lane ^ (1 << r)).
    const int Ks = K - p;
    double v = ffull_dyn<P>(Ks, ff, t + lane, T);
    const unsigned gmask = ((1u << P) - 1u) << (threadIdx.x & 31u & ~static_cast<unsigned>(P - 1));
#pragma unroll
    for (int r = 0; r < p; ++r) {
      const double o = __shfl_xor_sync(gmask, v, 1 << r, P);
      const bool left = ((lane >> r) & 1) == 0;
      v = ff.add(ff.mul(left ? v : o, tpow(Ks + r, T)), left ? o : v);
    }
    return v;
  }
  // general degree: peel the top bit repeatedly (p = q*T_g + r, r full)
  int gk[kMaxK];
  int m = 0, dd = d;
  bool pt = false;
  while (dd > 1) {
    const int k = 31 - __clz(dd);
    gk[m++] = k;
    dd -= 1 << k;
    if (dd == 0) {
      pt = true;
      break;
    }
  }
  const double* c = t;
  double v;
  if (pt) {
    v = ff.mulc(tpow(gk[m - 1], T), c[0]);  // head = mul_pt(T_g, q0)
    c += 1;
  } else {
    v = ff.addc(ff.mulc(x, c[0]), c[1]);  // degree-1 leaf of the last quotient
    c += 2;
  }
  for (int i = m - 1; i >= 0; --i) {
    const int k = gk[i];
    const double head = (pt && i == m - 1) ? v : ff.mul(v, tpow(k, T));
    const double rest = ffull_dyn<1>(k, ff, c, T);
    c += (k == 0) ? 2 : (1 << k);
    v = ff.add(head, rest);
  }
  return v;
}

// ---- Newton (primitives.hpp:105-132) -----------------------------------------------
template <class Q>
__device__ double newton(const Q& q, double x, double y, int n, int iters, double lin) {
  for (int it = 0; it < iters; ++it) {
    double prod;
    if (n == 2) {
      prod = q.mul(q.mul(x, y), q.mul(y, y));  // [x,y,y,y] -> [xy, yy] -> [xy*yy]
    } else if (n == 1) {
      prod = q.mul(q.mul(x, y), y);            // [x,y,y] -> [xy, y] -> [xy*y]
    } else {
      double f[kMaxFusedNewtonN + 2];
      int nf = 0;
      f[nf++] = x;
      for (int j = 0; j < n + 1; ++j) f[nf++] = y;
      while (nf > 1) {
        int w = 0, k = 0;
        for (; k + 1 < nf; k += 2) f[w++] = q.mul(f[k], f[k + 1]);
        if (nf & 1) f[w++] = f[nf - 1];
        nf = w;
      }
      prod = f[0];
    }
    y = q.sub(q.mulc(y, lin), prod);  // sub_ct(mul_pt(y, (n+1)/n), prod)
  }
  return y;
}

// ---- the interpreter ---------------------------------------------------------------------
template <class Q, int P>
__global__ void __launch_bounds__(kProgThreads) k_prog(Q q, const __grid_constant__ Prog pg) {
  extern __shared__ double stab[];
  for (int i = threadIdx.x; i < pg.ntab; i += blockDim.x) stab[i] = __ldg(pg.tabs + i);
  __syncthreads();
  const unsigned gid = blockIdx.x * blockDim.x + threadIdx.x;
  const unsigned slot_raw = gid / P;
  const int lane = static_cast<int>(gid % P);
  const bool live = slot_raw < pg.S;
  const unsigned s = live ? slot_raw : pg.S - 1;  // dead lanes shadow the last slot (shuffles stay converged)
  double r[kRegs];
#pragma unroll 1
  for (int k = 0; k < pg.n; ++k) {
    const MInst& I = pg.ins[k];
    switch (I.op) {
      case M_LD: r[I.dst] = q.in(__ldg(pg.in[I.i0] + s)); break;
      case M_ST:
        if (live && lane == 0) pg.out[I.i0][s] = q.out(r[I.a]);
        break;
      case M_CONST: r[I.dst] = I.c; break;
      case M_ADD: r[I.dst] = q.add(r[I.a], r[I.b]); break;
      case M_SUB: r[I.dst] = q.sub(r[I.a], r[I.b]); break;
      case M_MUL: r[I.dst] = q.mul(r[I.a], r[I.b]); break;
      case M_ADDC: r[I.dst] = q.addc(r[I.a], I.c); break;
      case M_MULC: r[I.dst] = q.mulc(r[I.a], I.c); break;
      case M_CHEB: r[I.dst] = cheb_eval<Q, P>(q, stab + I.i0, I.i1, r[I.a], lane, I.b != 0, I.c != 0.0); break;
      case M_NEWTON: r[I.dst] = newton<Q>(q, r[I.a], r[I.b], I.i0, I.i1, I.c); break;
      case M_ZAPPLY:
        if (live)
          for (int c = lane; c < pg.nchunks; c += P)
            pg.zout[c][s] = q.out(q.mul(q.sub(q.in(__ldg(pg.zin[c] + s)), r[I.a]), r[I.b]));
        break;
      default: break;
    }
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
    const size_t threads = static_cast<size_t>(p.S) * lanes;
    const unsigned grid = static_cast<unsigned>((threads + kProgThreads - 1) / kProgThreads);
    const size_t smem = static_cast<size_t>(p.ntab) * sizeof(double);
    auto go = [&](auto kern) {
      if (smem > 48 * 1024)
        cuda_ok(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)),
                "prog smem attr");
      kern<<<grid, kProgThreads, smem, s>>>(Q, p);
    };
    if (lanes == 8) go(k_prog<QT, 8>);
    else if (lanes == 4) go(k_prog<QT, 4>);
    else if (lanes == 2) go(k_prog<QT, 2>);
    else go(k_prog<QT, 1>);
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
