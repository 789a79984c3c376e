// quant.cuh — slot arithmetic policies shared by every kernel.
//
// The reference applies q(v) = nearbyint(v * 2^s) * 2^-s after every op
// (ckks.hpp:247-252) when CkksParams::quantize is set.  Three policies:
//
//   QNone   quantize == false: plain IEEE fp64 ops.
//   QExact  the reference formula literally, on plain slot values; valid for
//           ANY input (used by the op-by-op kernels).
//   QGrid   values carried in grid units A = v * 2^s (exact power-of-two
//           scaling).  For on-grid inputs (every output of a quantising op) this
//           reproduces QExact bit-for-bit with fewer fp64 instructions:
//             q(a+b)  ->  A + B                 (sum of grid integers is exact or
//                                                already integral: no rint)
//             q(a*b)  ->  rint((A * B) * 2^-s)  (fl(A*B) = fl(a*b) * 2^2s)
//             q(a*c)  ->  rint(A * c)
//             q(a+c)  ->  rint(A + c*2^s)       (c*2^s pre-scaled on the host)
//           Power-of-two scalings are exact away from overflow (|v| < 2^(1023-2s)),
//           and underflowing products round to the same signed zero in both
//           forms.  Fused kernels use QGrid only when every input ciphertext is
//           known to be on the 2^-s grid (CtData::grid), otherwise the host
//           falls back to the op-by-op QExact path.
//
// All arithmetic goes through __d*_rn intrinsics (never contracted into FMA),
// and rint() lowers to FRND.F64 (round-half-even == std::nearbyint under the
// default rounding mode).  The library is also compiled with -fmad=false.
#pragma once

#include <cuda_runtime.h>

namespace hsg {

struct QNone {
  static constexpr bool kExactSum = false;  // fp64 rounding: sums are order-dependent
  __device__ __forceinline__ double in(double v) const { return v; }
  __device__ __forceinline__ double out(double v) const { return v; }
  __device__ __forceinline__ double add(double a, double b) const { return __dadd_rn(a, b); }
  __device__ __forceinline__ double sub(double a, double b) const { return __dsub_rn(a, b); }
  __device__ __forceinline__ double mul(double a, double b) const { return __dmul_rn(a, b); }
  __device__ __forceinline__ double mulc(double a, double c) const { return __dmul_rn(a, c); }
  __device__ __forceinline__ double addc(double a, double c) const { return __dadd_rn(a, c); }
  __device__ __forceinline__ double mulc_x(double a, double c) const { return __dmul_rn(a, c); }
  __device__ __forceinline__ double addc_x(double a, double c) const { return __dadd_rn(a, c); }
  __device__ __forceinline__ double req(double a) const { return a; }
};

struct QExact {
  static constexpr bool kExactSum = false;  // inputs may be off-grid
  double s, inv;  // 2^scale_bits, 2^-scale_bits
  __device__ __forceinline__ double q(double v) const { return __dmul_rn(rint(__dmul_rn(v, s)), inv); }
  __device__ __forceinline__ double in(double v) const { return v; }
  __device__ __forceinline__ double out(double v) const { return v; }
  __device__ __forceinline__ double add(double a, double b) const { return q(__dadd_rn(a, b)); }
  __device__ __forceinline__ double sub(double a, double b) const { return q(__dsub_rn(a, b)); }
  __device__ __forceinline__ double mul(double a, double b) const { return q(__dmul_rn(a, b)); }
  __device__ __forceinline__ double mulc(double a, double c) const { return q(__dmul_rn(a, c)); }
  __device__ __forceinline__ double addc(double a, double c) const { return q(__dadd_rn(a, c)); }
  __device__ __forceinline__ double req(double a) const { return q(a); }
};

struct QGrid {
  static constexpr bool kExactSum = true;  // integer grid units: see slotsum.cuh
  double s, inv;
  __device__ __forceinline__ double in(double v) const { return __dmul_rn(v, s); }
  __device__ __forceinline__ double out(double a) const { return __dmul_rn(a, inv); }
  __device__ __forceinline__ double add(double a, double b) const { return __dadd_rn(a, b); }
  __device__ __forceinline__ double sub(double a, double b) const { return __dsub_rn(a, b); }
  __device__ __forceinline__ double mul(double a, double b) const {
    return rint(__dmul_rn(__dmul_rn(a, b), inv));
  }
  __device__ __forceinline__ double mulc(double a, double c) const { return rint(__dmul_rn(a, c)); }
  // c must be pre-scaled by 2^s on the host (prep_addc)
  __device__ __forceinline__ double addc(double a, double cs) const { return rint(__dadd_rn(a, cs)); }
  __device__ __forceinline__ double req(double a) const { return a; }
};

// ---- fast rounding for the Chebyshev core -----------------------------------------
// FRND.F64 issues at a quarter of the DMUL rate on sm_100 (measured:
// hs_diag_fp64_rate), so the fused Chebyshev tree rounds with the magic
// constant M = 1.5 * 2^52 instead:
//     for |t| < 2^51:  rint(t) == copysign(fl(t + M) - M, t)
// (fl(t + M) is t + M rounded half-even to an integer; M is even, so ties go to
// the same integer as rint; the copysign restores rint's signed zero).  For
// q(a*b) the 2^-s scaling folds into one FMA: fma(p, 2^-s, M) rounds
// p * 2^-s + M once, and p * 2^-s is exact, so it equals fl(fl(p*2^-s) + M).
//
// Range: the host enables this path for a series only when the sum of its
// table's |coefficients| B satisfies 1.001 * B < 2^11 (real units), and the
// kernel takes it only for slots with |x| <= 1.  Then every T_k stays within
// 1 + 2^-20 (one 2^-41 rounding per op, amplified at most 4x per doubling over
// <= 9 doublings) and every leaf, product and partial sum of the BSGS tree is
// bounded by 1.001 * B < 2^11, i.e. |t| < 2^51 in grid units: the identity
// holds for every rounding.  Other slots take the FRND path (bit-identical).
constexpr double kMagic = 6755399441055744.0;  // 1.5 * 2^52

__device__ __forceinline__ double magic_round(double s, double sign_src) {
  return copysign(__dsub_rn(s, kMagic), sign_src);
}
// Without the copysign the result differs from rint only in the SIGN OF A ZERO (t in
// [-0.5, 0) gives +0 instead of -0).  Inside a Chebyshev tree a zero's sign only ever flows
// into other zeros (x + 0 = x for x != 0; 0 * y and rint(0 + c) keep or drop it), so every
// nonzero value of the tree, and in particular a nonzero result, is bit-identical to the
// rint() evaluation; prog.cuh re-evaluates a slot exactly when the tree's result is zero.
__device__ __forceinline__ double magic_round_nz(double s) { return __dsub_rn(s, kMagic); }

struct QGridFast {
  double inv;
  __device__ __forceinline__ double add(double a, double b) const { return __dadd_rn(a, b); }
  __device__ __forceinline__ double mul(double a, double b) const {
    return magic_round_nz(__fma_rn(__dmul_rn(a, b), inv, kMagic));
  }
  __device__ __forceinline__ double mulc(double a, double c) const {
    return magic_round_nz(__dadd_rn(__dmul_rn(a, c), kMagic));
  }
  __device__ __forceinline__ double addc(double a, double cs) const {
    return magic_round_nz(__dadd_rn(__dadd_rn(a, cs), kMagic));
  }
  // the same roundings on the XU pipe (FRND.F64): QGrid's own forms, valid for any magnitude
  __device__ __forceinline__ double mulc_x(double a, double c) const { return rint(__dmul_rn(a, c)); }
  __device__ __forceinline__ double addc_x(double a, double cs) const { return rint(__dadd_rn(a, cs)); }
};

template <class Q>
struct FastOf;
template <>
struct FastOf<QGrid> {
  using type = QGridFast;
  __device__ static QGridFast make(const QGrid& q) { return QGridFast{q.inv}; }
  __device__ static bool in_range(const QGrid& q, double x) { return fabs(x) <= q.s; }  // |x| <= 1
};
template <>
struct FastOf<QNone> {  // no rounding at all: the "fast" core is the exact one
  using type = QNone;
  __device__ static QNone make(const QNone& q) { return q; }
  __device__ static bool in_range(const QNone&, double) { return true; }
};

}  // namespace hsg
