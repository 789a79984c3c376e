// prog.cuh — device side of the per-slot fused programs (kernels.h MOp):
// the Chebyshev BSGS evaluator (chebyshev.hpp:113-163), the Newton loop
// (primitives.hpp:105-132) and the macro-instruction interpreter shared by the
// standalone program kernel (fused.cu) and the cooperative statistics kernel
// (stat.cu).
#pragma once

#include "kernels.h"
#include "quant.cuh"

namespace hsg {
namespace k {

constexpr int kMaxK = 10;  // T_{2^0} .. T_{2^9}; degree <= 1023

// ---- Chebyshev evaluation ------------------------------------------------------
// Series tables live in shared memory (staged once per block).  A table of a
// lane-split series is interleaved by part (element e of part l at e*P + l) so
// the P lanes of a slot read consecutive words (conflict-free) and all slots of
// a warp read the same words (broadcast).
//
// F_K: full tree of degree 2^K - 1 (K >= 1) or a degree-0 leaf (K == 0).
// Table layout [F_{K-1}(q) | F_{K-1}(r)], leaves (c1, c0).  chebyshev.hpp:140-158.
//
// Pipe balance (sm_100a, ncu of k_zbatch): a magic-constant rounding is two FP64-pipe
// instructions (add M, subtract M; the add folds into an FMA for products), FRND.F64 is one XU
// instruction at a quarter of the FP64 rate, and the two pipes issue side by side.  All-magic
// leaves the XU pipe idle with the FP64 pipe at 81 %; all-FRND is XU bound.  The leaves
// (mul_pt + add_pt, two roundings each, two thirds of the tree's roundings) therefore round with
// FRND on the leaf positions selected by kLeafMulX / kLeafAddX (bit j: leaves with index = j
// mod 8), everything else with the magic constant: both forms give the same bits (quant.cuh).
#ifndef HS_LEAF_MULX
#define HS_LEAF_MULX 0xFF
#endif
#ifndef HS_LEAF_ADDX
#define HS_LEAF_ADDX 0x55
#endif
constexpr unsigned kLeafMulX = HS_LEAF_MULX, kLeafAddX = HS_LEAF_ADDX;

template <int K, int ST, int J = 0, class F>
__device__ __forceinline__ double ffull(const F& f, const double* t, const double (&T)[kMaxK]) {
  if constexpr (K <= 1) {  // add_pt(mul_pt(x, c1), c0)
    constexpr bool mx = (kLeafMulX >> (J & 7)) & 1u, ax = (kLeafAddX >> (J & 7)) & 1u;
    const double m = mx ? f.mulc_x(T[0], t[0]) : f.mulc(T[0], t[0]);
    return ax ? f.addc_x(m, t[ST]) : f.addc(m, t[ST]);
  } else {
    constexpr int H = (1 << (K - 1)) * ST;
    const double head = f.mul(ffull<K - 1, ST, 2 * J>(f, t, T), T[K - 1]);  // mul_ct(eval(q), T_g)
    const double rest = ffull<K - 1, ST, 2 * J + 1>(f, t + H, T);
    return f.add(head, rest);                                              // add_ct(head, eval(r))
  }
}

// Any F_K as a loop over 2^(K-kBK) unrolled F_kBK blocks, combined by a carry
// chain over the upper levels: block j finishes every level m whose bit
// (m - kBK) of j is set (F_{m+1} = add(mul(F_m(left), T_m), F_m(right))).  The
// branches are warp-uniform and stk[]/T[] stay in registers (static indices in
// the unrolled carry loop); the code stays ~3 KB so it lives in the I-cache
// (a fully unrolled degree-511 tree is ~32 KB of SASS per lane and stalled on
// instruction fetch).  Same ops on the same operands as ffull<K>: bit-identical.
#ifndef HS_KBK
#define HS_KBK 5
#endif
constexpr int kBK = HS_KBK;

template <int ST, class F>
__device__ __forceinline__ double ffull_small(int K, const F& f, const double* t, const double (&T)[kMaxK]) {
  switch (K) {
    case 0: return ffull<0, ST>(f, t, T);
    case 1: return ffull<1, ST>(f, t, T);
    case 2: return ffull<2, ST>(f, t, T);
    case 3: return ffull<3, ST>(f, t, T);
    case 4: return ffull<4, ST>(f, t, T);
    case 5: return ffull<5, ST>(f, t, T);
    default: return ffull<(kBK > 5 ? kBK : 5), ST>(f, t, T);
  }
}

#ifndef HS_BLK_UNROLL
#define HS_BLK_UNROLL 4
#endif
constexpr int kBlkUnroll = HS_BLK_UNROLL;  // leaf blocks in flight per thread (ILP of the tree walk)
template <int ST, class F>
__device__ __forceinline__ double ffull_dyn(int K, const F& f, const double* t, const double (&T)[kMaxK]) {
  if (K <= kBK) return ffull_small<ST>(K, f, t, T);
  const int nb = 1 << (K - kBK);
  constexpr int BS = (1 << kBK) * ST;
  double stk[kMaxK];
  double v = 0.0;
#pragma unroll(kBlkUnroll)
  for (int j = 0; j < nb; ++j) {
    v = ffull<kBK, ST>(f, t + j * BS, T);
#pragma unroll
    for (int m = kBK; m < kMaxK - 1; ++m) {
      if ((j >> (m - kBK)) & 1) {
        v = f.add(f.mul(stk[m], T[m]), v);
      } else {
        stk[m] = v;
        break;
      }
    }
  }
  return v;
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

// ---- degree-511 tree with its table in the constant bank (batched Z-score, one lane per slot) ----
// The coefficients are operands of the FP64 instructions themselves (c[bank][immediate]): no
// coefficient loads, no table addressing and no block loop, at the price of a fully unrolled tree.
// Each translation unit that includes this header has its own copy of the table; only stat.cu's is
// ever filled (upload_const_table) and read (k_zbatch with CT = true).
__constant__ double c_cheb511[512];

template <int K, int OFF, int J, class F>
__device__ __forceinline__ double ffull_c(const F& f, const double (&T)[kMaxK]) {
  if constexpr (K <= 1) {
    constexpr bool mx = (kLeafMulX >> (J & 7)) & 1u, ax = (kLeafAddX >> (J & 7)) & 1u;
    const double m = mx ? f.mulc_x(T[0], c_cheb511[OFF]) : f.mulc(T[0], c_cheb511[OFF]);
    return ax ? f.addc_x(m, c_cheb511[OFF + 1]) : f.addc(m, c_cheb511[OFF + 1]);
  } else {
    constexpr int H = 1 << (K - 1);
    const double head = f.mul(ffull_c<K - 1, OFF, 2 * J>(f, T), T[K - 1]);
    const double rest = ffull_c<K - 1, OFF + H, 2 * J + 1>(f, T);
    return f.add(head, rest);
  }
}

// the d = 511 instance of cheb_eval's peel-the-top-bit loop: leaf (c[0], c[1]), then F_k at c[2^k]
template <int KK, class F>
__device__ __forceinline__ double cheb511_c(const F& f, double v, const double (&T)[kMaxK]) {
  if constexpr (KK > 8) {
    return v;
  } else {
    const double head = f.mul(v, T[KK]);
    const double rest = ffull_c<KK, (1 << KK), 0>(f, T);
    return cheb511_c<KK + 1>(f, f.add(head, rest), T);
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
template <class Q, int P, bool CT = false>
__device__ __forceinline__ double cheb_eval(const Q& q, const double* t, int d, double x, int lane, bool split,
                                            bool fast_ok, bool in_const = false) {
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
    // a zero result may carry the wrong zero sign (quant.cuh magic_round_nz): redo exactly
    return v == 0.0 ? cheb_exact<Q>(q, t, d, x, P, 1) : v;
  }
  if constexpr (CT && P == 1) {
    if (in_const && d == 511) {  // uniform: the table of this series is also in the constant bank
      const double v0 = ff.addc(ff.mulc(x, c_cheb511[0]), c_cheb511[1]);
      const double v = cheb511_c<1>(ff, v0, T);
      return v == 0.0 ? cheb_exact<Q>(q, t, d, x, P, 0) : v;
    }
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
  return v == 0.0 ? cheb_exact<Q>(q, t, d, x, P, 0) : v;  // zero sign: see quant.cuh magic_round_nz
}

// ---- Newton (primitives.hpp:105-132) -----------------------------------------------
// flag (debug_checks, this slot checked): check_divergence after every iteration
template <class Q>
__device__ double newton(const Q& q, double x, double y, int n, int iters, double lin, unsigned* flag = nullptr) {
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
    if (flag && !(fabs(q.out(y)) <= 1e6)) atomicOr(flag, 1u);  // primitives.hpp:89-96
  }
  return y;
}

// The reference's debug predicates (kernels.h ChkKind) on a slot value in real units
__device__ __forceinline__ bool chk_fails(int kind, double v, double c, double c2) {
  switch (kind) {
    case CK_OPEN: return !(v > c) || !(v <= c2);
    case CK_RANGE: return v < c || v > c2;
    case CK_LT: return v < c;
    case CK_SCALED_LT: return __dmul_rn(__dmul_rn(v, c), c) < c2;
    default: return fabs(v) < c;
  }
}

// ---- launch geometry ---------------------------------------------------------------------
// One block per SM (148 on B200), each owning a contiguous, equal range of slots,
// P threads per slot: every SM gets the same amount of FP64 work.
#ifndef HS_P1_THREADS
#define HS_P1_THREADS 256
#endif
template <int P>
constexpr int prog_max_threads() {
  return P == 1 ? HS_P1_THREADS : (P == 2 ? 512 : 1024);
}

struct Geo {
  unsigned blocks, threads;
};

inline Geo prog_geometry(size_t S, int P, int sms, int max_threads) {
  const size_t work = S * static_cast<size_t>(P);
  size_t blocks = (work + 31) / 32;
  if (blocks > static_cast<size_t>(sms)) blocks = static_cast<size_t>(sms);
  if (blocks < 1) blocks = 1;
  const size_t spb = (S + blocks - 1) / blocks;
  size_t threads = ((spb * P + 31) / 32) * 32;
  if (threads > static_cast<size_t>(max_threads)) threads = static_cast<size_t>(max_threads);
  return Geo{static_cast<unsigned>(blocks), static_cast<unsigned>(threads)};
}

// This block's slot range [lo, hi)
struct Range {
  unsigned lo, hi, spb;
};
__device__ __forceinline__ Range block_range(unsigned S) {
  const unsigned spb = (S + gridDim.x - 1) / gridDim.x;
  const unsigned lo = blockIdx.x * spb;
  return Range{lo, lo + spb < S ? lo + spb : S, spb};
}

// ---- one slot's program ------------------------------------------------------------
// r: the slot's register file; sv: per-slot statistic values (M_LDR), if any.
template <class Q, int P, bool CT = false>
__device__ __forceinline__ void exec(const Q& q, const Prog& pg, const double* stab, unsigned s, int lane,
                                     bool live, const double* sv) {
  double r[kRegs];
#pragma unroll 1
  for (int k = 0; k < pg.n; ++k) {
    const MInst& I = pg.ins[k];
    switch (I.op) {
      case M_LD: r[I.dst] = q.in(__ldg(pg.in[I.i0] + s)); break;
      case M_LDR: r[I.dst] = sv[I.i0]; break;
      case M_ST:
        if (live && lane == 0) pg.out[I.i0][s] = q.out(r[I.a]);
        break;
      case M_CONST: r[I.dst] = I.c; break;
      case M_ADD: r[I.dst] = q.add(r[I.a], r[I.b]); break;
      case M_SUB: r[I.dst] = q.sub(r[I.a], r[I.b]); break;
      case M_MUL: r[I.dst] = q.mul(r[I.a], r[I.b]); break;
      case M_ADDC: r[I.dst] = q.addc(r[I.a], I.c); break;
      case M_MULC: r[I.dst] = q.mulc(r[I.a], I.c); break;
      case M_CHEB:
        r[I.dst] = cheb_eval<Q, P, CT>(q, stab + I.i0, I.i1, r[I.a], lane, I.b != 0, I.c != 0.0, I.i2 != 0);
        break;
      case M_NEWTON:
        r[I.dst] = newton<Q>(q, r[I.a], r[I.b], I.i0, I.i1, I.c,
                             pg.flags && live && lane == 0 && s < static_cast<unsigned>(I.i2) ? pg.flags : nullptr);
        break;
      case M_CHK:
        if (pg.flags && live && lane == 0 && s < static_cast<unsigned>(I.i1) && chk_fails(I.i0, q.out(r[I.a]), I.c, I.c2))
          atomicOr(pg.flags, 1u);
        break;
      case M_ZAPPLY:
        if (live)
          for (int c = lane; c < pg.nchunks; c += P)
            pg.zout[c][s] = q.out(q.mul(q.sub(q.in(__ldg(pg.zin[c] + s)), r[I.a]), r[I.b]));
        break;
      default: break;
    }
  }
}

}  // namespace k
}  // namespace hsg
