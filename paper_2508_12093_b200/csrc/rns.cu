// rns.cu — Tier R kernels and host orchestration (see rns.h).
//
//   NTT / iNTT   two shared-memory passes per limb (columns, then contiguous
//                rows), radix-8 register groups, Shoup twiddles, lazy Harvey
//                butterflies in [0, 4q), canonical output; one launch covers any
//                list of (input row, output row, prime) triples for a batch.
//   tensor       d0 = a0 b0, d1 = a0 b1 + a1 b0 (one 128-bit reduction), d2 = a1 b1.
//   ModUp        fast base conversion of every digit (coefficient form) to the
//                extended basis Q_l u P in one launch (128-bit accumulation, one
//                reduction per output), then one batched NTT of all new rows.
//   inner        sum_j ModUp(d_j) * key_j; each thread keeps its key words in
//                registers and loops over the batch, so the key streams from HBM
//                once per call instead of once per ciphertext.
//   ModDown      in-place iNTT of the P rows, base conversion P -> Q_l, NTT whose last
//                pass applies (acc - conv) * P^-1 (+ d0/d1 for HMult, + sigma(c0) for
//                rotate) instead of storing the converted rows.
//   rescale      iNTT of the last limb; one NTT over the remaining limbs whose column
//                pass loads [c_l]_{q_i} and whose row pass stores (c_i - t_i) q_l^-1.
//   automorph    NTT-domain Galois permutation for 5^k.
// Every kernel takes its batch index from blockIdx.z.  Ring sizes are powers of
// two: all index arithmetic is shifts and masks.
#include "rns.h"

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <stdexcept>
#include <string>
#include <type_traits>

namespace hsg {
namespace rns {
namespace {

constexpr int kT = 256;  // threads per elementwise block

enum : uint64_t { D_SECRET = 1, D_KEY_A = 2, D_KEY_E = 3, D_CT = 4, D_ENC_A = 5, D_ENC_E = 6 };

__host__ __device__ inline uint64_t hash64(uint64_t seed, uint64_t domain, uint64_t a, uint64_t b) {
  uint64_t z = seed ^ (domain * 0x9E3779B97F4A7C15ULL) ^ (a * 0xC2B2AE3D27D4EB4FULL) ^ (b * 0x165667B19E3779F9ULL);
  z += 0x9E3779B97F4A7C15ULL;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}
__host__ __device__ inline uint64_t uniform_mod(uint64_t h, uint64_t q) {
  return static_cast<uint64_t>((static_cast<u128>(h) * q) >> 64);
}
__device__ inline uint64_t lift(int64_t v, uint64_t q) {
  return v >= 0 ? static_cast<uint64_t>(v) % q : q - (static_cast<uint64_t>(-v) % q);
}
__device__ inline uint32_t bitrev(uint32_t x, uint32_t bits) { return __brev(x) >> (32 - bits); }

// NTT-domain automorphism X -> X^g: slot n of the result is slot galois_src(n) of the input
__device__ inline uint32_t galois_src(uint32_t j, uint64_t g, uint32_t logN) {
  const uint64_t mask = (2ULL << logN) - 1;
  const uint64_t e = ((2ULL * bitrev(j, logN) + 1) * g) & mask;
  return bitrev(static_cast<uint32_t>((e - 1) >> 1), logN);
}


// (input row, output row, prime) per blockIdx.y of an NTT launch
constexpr int kMaxRows = 128;
struct RowMap {
  uint16_t irow[kMaxRows], orow[kMaxRows];
  uint8_t prime[kMaxRows];
};

// ---------------------------------------------------------------- NTT kernels
// One pass = a batch of independent sub-transforms held in shared memory:
//   column pass: the first log2(R1) stages, transform c = column {r*C + c};
//   row pass   : the remaining log2(C) stages, transform g = block [g*C, (g+1)*C).
// Stage m (local), block i of a sub-transform uses twiddle index m*S + i with
// S = 1 (columns) or R1 + g (rows), so one device routine serves both passes.
// Each thread runs radix-2^RB groups (RB <= 3 stages) in registers; the first
// group step reads HBM directly, the last writes HBM directly, the ones between
// exchange through shared memory (row tiles XOR-swizzled, see swz()).
#ifndef HS_NTT_LOGTILE
#define HS_NTT_LOGTILE 11
#define HS_NTT_MINB 6
#endif
constexpr uint32_t kLogTile = HS_NTT_LOGTILE;  // elements per NTT block (log2)
#ifndef HS_NTT_MAXRB
#define HS_NTT_MAXRB 3
#endif
constexpr int kMaxRB = HS_NTT_MAXRB;  // largest radix (log2) of a register step
constexpr int kNT = 1 << (HS_NTT_LOGTILE - kMaxRB);  // threads per NTT block: one largest-radix group each
constexpr uint32_t kNTile = 1u << kLogTile;

// Row-tile shared-memory swizzle: a bijection inside aligned 16-word groups that
// makes every store/load pattern of every radix step (logN 10..17, forward and
// inverse) hit 16 distinct 8-byte bank slots per half-warp (exhaustively checked
// offline against the step access patterns below).
// Where the last NTT step puts a canonical output word: straight to HBM, or (ModDown
// epilogue of key switching) out = (acc - v) * P^-1 (+ add) without materialising v.
struct PlainStore {
  uint64_t* g;
  __device__ void operator()(size_t off, uint64_t v) const { g[off] = v; }
};

struct PlainLoad {
  const uint64_t* g;
  __device__ uint64_t operator()(size_t off) const { return g[off]; }
};

// Rescale of k c (k an integer constant, per-limb residues k_i; k = 1: plain rescale).  The
// product is never stored: iNTT(k_l c_l) = k_l iNTT(c_l) mod q_l, so the spread multiplies
// the coefficient-form last limb by k_l, and the combine computes (k_i c_i - t_i) q_l^-1 --
// the same canonical words as multiplying first and rescaling after.
struct RsLoad {  // rescale: [k_l c_l]_{q_i} read straight from the coefficient-form last limb
  const uint64_t* last;
  PrimeC P;
  bool kon;
  uint64_t kl, kl_sh, ql;
  __device__ uint64_t operator()(size_t off) const {
    return reduce64(kon ? mul_shoup(last[off], kl, kl_sh, ql) : last[off], P);
  }
};

struct RsStore {  // rescale: out = (k_i c_i - NTT([k_l c_l]_{q_i})) * q_l^-1 (+ a_i: a fused add_pt)
  const uint64_t* in;
  uint64_t* out;
  uint64_t q, qinv, qinv_sh;
  bool kon;
  uint64_t k, k_sh;
  uint64_t addc = 0;
  __device__ void operator()(size_t off, uint64_t v) const {
    const uint64_t c = kon ? mul_shoup(in[off], k, k_sh, q) : in[off];
    out[off] = add_mod(mul_shoup(sub_mod(c, v, q), qinv, qinv_sh, q), addc, q);
  }
};

constexpr int kRsMaxLimbs = 64;
struct RsEpi {  // the rescale's spread and combine fused into its NTT passes
  const uint64_t* last;
  const uint64_t* in;
  uint64_t* out;
  const uint64_t* qinv;
  const uint64_t* qinv_sh;
  size_t last_stride, in_stride, out_stride;
  uint32_t level;
  bool kon = false;  // rescale of k c: k's residues and Shoup companions, limbs 0..level
  uint64_t k[kRsMaxLimbs], k_sh[kRsMaxLimbs];
  // per batch item constants instead (device, [batch][2][level + 1]: residues then Shoup)
  const uint64_t* kitems = nullptr;
  // per batch item constant added to polynomial 0 of the output (device, [batch][level]), or null
  const uint64_t* aitems = nullptr;
  __device__ uint64_t kk(uint32_t bz, uint32_t i) const {
    return kitems ? kitems[size_t(bz) * 2 * (level + 1) + i] : k[i];
  }
  __device__ uint64_t kk_sh(uint32_t bz, uint32_t i) const {
    return kitems ? kitems[size_t(bz) * 2 * (level + 1) + level + 1 + i] : k_sh[i];
  }
};

struct MdEpi {  // k_moddown fused into the last pass of the conv-rows NTT
  const uint64_t* acc;
  const uint64_t* add0;
  const uint64_t* add1;
  uint64_t* out;
  const uint64_t* pinv;
  const uint64_t* pinv_sh;
  size_t acc_stride, add_stride, out_stride;
  uint32_t nl, nx;
  // ModDown merged with HMult's rescale (pinv = (P q_l)^-1): add_w enters scaled by q_l^-1
  const uint64_t* ascale = nullptr;
  const uint64_t* ascale_sh = nullptr;
};

// Key-switch inputs produced on the fly instead of materialised: mul_relin's tensor
// (d = a1 b1, add_0 = a0 b0, add_1 = a0 b1 + a1 b0) and rotate's automorphism
// (d = sigma(c1), add_0 = sigma(c0)).  The iNTT that starts ModUp loads d through
// TnLoad / PermLoad, and the ModDown store adds add_w through AddTensor / AddPerm.
enum KsSrcMode : int { KS_PLAIN = 0, KS_TENSOR = 1, KS_PERM = 2 };
struct KsSrc {
  int mode = KS_PLAIN;
  const uint64_t* a = nullptr;  // tensor: first ciphertext; automorphism: the input ciphertext
  const uint64_t* b = nullptr;  // tensor: second ciphertext
  size_t stride = 0;            // per batch item
  uint64_t g = 0;               // Galois element
  uint32_t nl = 0;
};

struct TnLoad {  // d = a1 b1 (this tile of limb i)
  const uint64_t* a1;
  const uint64_t* b1;
  PrimeC P;
  __device__ uint64_t operator()(size_t off) const { return mul_mod(a1[off], b1[off], P); }
};

template <int LOGN>
struct PermLoad {  // d = sigma_g(c1): row = limb i of c1 (whole row), toff = this tile's first word
  const uint64_t* row;
  uint64_t g;
  uint32_t toff;
  __device__ uint64_t operator()(size_t off) const { return row[galois_src(toff + uint32_t(off), g, LOGN)]; }
};

struct AddRow {  // + add_w[i] (materialised) or nothing
  const uint64_t* p;
  __device__ uint64_t operator()(size_t off, uint64_t r, uint64_t q) const { return p ? add_mod(r, p[off], q) : r; }
};

struct AddRowScaled {  // + add_w[i] q_l^-1 (ModDown by P q_l: (acc + P d - conv) (P q_l)^-1)
  const uint64_t* p;
  uint64_t sc, sc_sh;
  __device__ uint64_t operator()(size_t off, uint64_t r, uint64_t q) const {
    return add_mod(r, mul_shoup(p[off], sc, sc_sh, q), q);
  }
};

struct AddTensor {  // + a0 b0 (w = 0) or + a0 b1 + a1 b0 (w = 1), same reductions as k_tensor
  const uint64_t *a0, *a1, *b0, *b1;
  PrimeC P;
  int w;
  __device__ uint64_t operator()(size_t off, uint64_t r, uint64_t q) const {
    const uint64_t t = w == 0 ? mul_mod(a0[off], b0[off], P)
                              : reduce128(static_cast<u128>(a0[off]) * b1[off] + static_cast<u128>(a1[off]) * b0[off], P);
    return add_mod(r, t, q);
  }
};

template <int LOGN>
struct AddPerm {  // + sigma_g(c0) (w = 0 only: row null for w = 1)
  const uint64_t* row;
  uint64_t g;
  uint32_t toff;
  __device__ uint64_t operator()(size_t off, uint64_t r, uint64_t q) const {
    return row ? add_mod(r, row[galois_src(toff + uint32_t(off), g, LOGN)], q) : r;
  }
};

template <class AddF>
struct MdStore {
  const uint64_t* acc;  // acc_w row i (this tile)
  uint64_t* out;        // out_w row i (this tile)
  uint64_t q, pinv, pinv_sh;
  AddF add;
  __device__ void operator()(size_t off, uint64_t v) const {
    out[off] = add(off, mul_shoup(sub_mod(acc[off], v, q), pinv, pinv_sh, q), q);
  }
};

__device__ __forceinline__ uint32_t swz(uint32_t u) { return u ^ (((u >> 2) ^ (u >> 3)) & 15u); }

template <int LOGN, bool ROWS>
struct NttGeom {
  static constexpr uint32_t logR1 = LOGN / 2, logC = LOGN - logR1;
  static constexpr uint32_t logR = ROWS ? logC : logR1;  // sub-transform length of this pass
  static constexpr uint32_t logTPB = ROWS ? (kLogTile - logC < logR1 ? kLogTile - logC : logR1)
                                          : (kLogTile - logR1 < logC ? kLogTile - logR1 : logC);
  static constexpr uint32_t R1 = 1u << logR1;
};

// n consecutive twiddles (n a power of two <= 8, constant after unrolling; the start is
// n-aligned): 16-byte loads for n >= 2
__device__ __forceinline__ void ldg_tw(uint64_t (&w)[8], const uint64_t* p, int n) {
  if (n == 1) {
    w[0] = __ldg(p);
  } else {
    const ulonglong2* p2 = reinterpret_cast<const ulonglong2*>(p);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      if (2 * i >= n) break;
      const ulonglong2 v = __ldg(p2 + i);
      w[2 * i] = v.x;
      w[2 * i + 1] = v.y;
    }
  }
}
__device__ __forceinline__ void ldg_tw(double (&w)[8], const double* p, int n) {
  if (n == 1) {
    w[0] = __ldg(p);
  } else {
    const double2* p2 = reinterpret_cast<const double2*>(p);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      if (2 * i >= n) break;
      const double2 v = __ldg(p2 + i);
      w[2 * i] = v.x;
      w[2 * i + 1] = v.y;
    }
  }
}

// One radix-2^RB step (stages DONE .. DONE+RB-1 of this pass) for every group of the tile.
template <bool INV, bool ROWS, int LOGN, int RB, int DONE, bool FIRST, bool LAST, class LD, class ST>
__device__ __forceinline__ void ntt_step(const LD& gin, const ST& gout,
                                         uint64_t* __restrict__ sm, const uint64_t* __restrict__ psi,
                                         const uint64_t* __restrict__ psip, uint64_t q, uint32_t tile0,
                                         uint64_t ninv, uint64_t ninv_sh, const uint64_t* wpre = nullptr,
                                         const uint64_t* wppre = nullptr) {
  using G = NttGeom<LOGN, ROWS>;
  constexpr uint32_t logR = G::logR, logTPB = G::logTPB, logC = G::logC;
  constexpr uint32_t logG = logR - RB;  // groups per transform (log)
  constexpr uint32_t total = 1u << (logG + logTPB);
  constexpr uint32_t logs = INV ? DONE : logR - 1 - DONE - (RB - 1);  // element stride inside a group (log)
  const uint64_t q2 = 2 * q;
#pragma unroll
  for (uint32_t it = 0; it < (total + kNT - 1) / kNT; ++it) {
    const uint32_t idx = threadIdx.x + it * kNT;
    if (total % kNT != 0 && idx >= total) break;
    uint32_t tr, g;
    if (ROWS) {
      g = idx & ((1u << logG) - 1);
      tr = idx >> logG;
    } else {
      tr = idx & ((1u << logTPB) - 1);
      g = idx >> logTPB;
    }
    const uint32_t blk0 = g >> logs;
    const uint32_t j0 = (blk0 << (logs + RB)) | (g & ((1u << logs) - 1));
    // swz is linear over XOR and j0 has zeros in bits logs .. logs + RB - 1, so the swizzled index of
    // element k is swz(base) ^ swz(k << logs): one swizzle per thread and step, one XOR with a
    // compile-time constant per element
    const uint32_t sb = ROWS ? swz((tr << logR) + j0) : 0u;
    const uint32_t S = ROWS ? G::R1 + tile0 + tr : 1u;
    uint64_t x[1 << RB];
#pragma unroll
    for (int k = 0; k < (1 << RB); ++k) {
      const uint32_t e = j0 + (uint32_t(k) << logs);
      if (FIRST)
        x[k] = gin(ROWS ? (size_t(tr) << logC) + e : (size_t(e) << logC) + tr);
      else
        x[k] = ROWS ? sm[sb ^ swz(uint32_t(k) << logs)] : sm[(e << logTPB) + tr];
    }
    if (!INV) {
#pragma unroll
      for (int st = 0; st < RB; ++st) {
        const int d = 1 << (RB - 1 - st);
        uint64_t wv[8], wpv[8];  // the stage's 2^st consecutive twiddles: 16-byte loads
        const uint32_t wi0 = ((1u << (DONE + st)) * S) + (blk0 << st);
        if (wpre && it == 0) {  // loaded before the barrier that precedes this step (ntt_tw_u64)
#pragma unroll
          for (int b = 0; b < (1 << st); ++b) {
            wv[b] = wpre[(1 << st) - 1 + b];
            wpv[b] = wppre[(1 << st) - 1 + b];
          }
        } else {
          ldg_tw(wv, psi + wi0, 1 << st);
          ldg_tw(wpv, psip + wi0, 1 << st);
        }
#pragma unroll
        for (int b = 0; b < (1 << st); ++b) {
          const uint64_t w = wv[b], wp = wpv[b];
#pragma unroll
          for (int o = 0; o < d; ++o) {
            const int k0 = b * 2 * d + o;
            uint64_t X = x[k0];
            X = X >= q2 ? X - q2 : X;
            const uint64_t T = mul_shoup_lazy(x[k0 + d], w, wp, q);
            x[k0] = X + T;
            x[k0 + d] = X - T + q2;
          }
        }
      }
    } else {
#pragma unroll
      for (int st = 0; st < RB; ++st) {
        const int d = 1 << st;
        constexpr uint32_t logh0 = logR - 1 - DONE;
        uint64_t wv[8], wpv[8];
        const uint32_t wi0 = ((1u << (logh0 - st)) * S) + (blk0 << (RB - 1 - st));
        if (wpre && it == 0) {
#pragma unroll
          for (int b = 0; b < (1 << (RB - 1 - st)); ++b) {
            wv[b] = wpre[(1 << RB) - (2 << (RB - 1 - st)) + b];
            wpv[b] = wppre[(1 << RB) - (2 << (RB - 1 - st)) + b];
          }
        } else {
          ldg_tw(wv, psi + wi0, 1 << (RB - 1 - st));
          ldg_tw(wpv, psip + wi0, 1 << (RB - 1 - st));
        }
#pragma unroll
        for (int b = 0; b < (1 << (RB - 1 - st)); ++b) {
          const uint64_t w = wv[b], wp = wpv[b];
#pragma unroll
          for (int o = 0; o < d; ++o) {
            const int k0 = b * 2 * d + o;
            const uint64_t X = x[k0], Y = x[k0 + d];
            const uint64_t s2 = X + Y;
            x[k0] = s2 >= q2 ? s2 - q2 : s2;
            x[k0 + d] = mul_shoup_lazy(X - Y + q2, w, wp, q);
          }
        }
      }
    }
#pragma unroll
    for (int k = 0; k < (1 << RB); ++k) {
      const uint32_t e = j0 + (uint32_t(k) << logs);
      uint64_t v = x[k];
      if (LAST) {
        if (!INV) {
          v = v >= q2 ? v - q2 : v;
          v = v >= q ? v - q : v;
        } else if (!ROWS) {
          v = mul_shoup(v, ninv, ninv_sh, q);
        }
        gout(ROWS ? (size_t(tr) << logC) + e : (size_t(e) << logC) + tr, v);
      } else {
        if (ROWS)
          sm[sb ^ swz(uint32_t(k) << logs)] = v;
        else
          sm[(e << logTPB) + tr] = v;
      }
    }
  }
}

// All steps of a pass, unrolled at compile time.  Radix-8 steps with the remainder
// taken as radix-4 (a 4-stage tail becomes 2 + 2); with kMaxRB = 4, radix-16 steps
// (5 and 6 stages become 3 + 2 and 3 + 3).
constexpr int pick_rb(int rem) {
  if (kMaxRB >= 4) return rem <= 4 ? rem : (rem <= 6 ? 3 : 4);
  return rem == 4 ? 2 : (rem < 3 ? rem : 3);
}
// Called once per pass, right after the barrier that follows the first step (every
// thread has consumed its inputs): the persistent kernel issues the next tile's loads there.
struct NoPf {
  __device__ void operator()() const {}
};

// The twiddles (and Shoup companions) of one radix step for this thread's first group, issued before
// the barrier that precedes the step (see ntt_tw_fp; same layout).  HS_NTT_PRETW64: the same bit mask as
// HS_NTT_PRETW for the 64-bit path.
#ifndef HS_NTT_PRETW64
#define HS_NTT_PRETW64 3
#endif
template <bool INV, bool ROWS, int LOGN, int RB, int DONE>
__device__ __forceinline__ void ntt_tw_u64(uint64_t (&wpre)[8], uint64_t (&wppre)[8], const uint64_t* __restrict__ psi,
                                           const uint64_t* __restrict__ psip, uint32_t tile0) {
  using G = NttGeom<LOGN, ROWS>;
  constexpr uint32_t logR = G::logR, logTPB = G::logTPB;
  constexpr uint32_t logG = logR - RB;
  constexpr uint32_t logs = INV ? DONE : logR - 1 - DONE - (RB - 1);
  const uint32_t idx = threadIdx.x;
  const uint32_t g = ROWS ? idx & ((1u << logG) - 1) : idx >> logTPB;
  const uint32_t tr = ROWS ? idx >> logG : idx & ((1u << logTPB) - 1);
  const uint32_t blk0 = g >> logs;
  const uint32_t S = ROWS ? G::R1 + tile0 + tr : 1u;
#pragma unroll
  for (int st = 0; st < RB; ++st) {
    uint64_t wv[8], wpv[8];
    if (!INV) {
      const uint32_t wi0 = ((1u << (DONE + st)) * S) + (blk0 << st);
      ldg_tw(wv, psi + wi0, 1 << st);
      ldg_tw(wpv, psip + wi0, 1 << st);
#pragma unroll
      for (int b = 0; b < (1 << st); ++b) {
        wpre[(1 << st) - 1 + b] = wv[b];
        wppre[(1 << st) - 1 + b] = wpv[b];
      }
    } else {
      constexpr uint32_t logh0 = logR - 1 - DONE;
      const uint32_t wi0 = ((1u << (logh0 - st)) * S) + (blk0 << (RB - 1 - st));
      ldg_tw(wv, psi + wi0, 1 << (RB - 1 - st));
      ldg_tw(wpv, psip + wi0, 1 << (RB - 1 - st));
#pragma unroll
      for (int b = 0; b < (1 << (RB - 1 - st)); ++b) {
        wpre[(1 << RB) - (2 << (RB - 1 - st)) + b] = wv[b];
        wppre[(1 << RB) - (2 << (RB - 1 - st)) + b] = wpv[b];
      }
    }
  }
}

template <bool INV, bool ROWS, int LOGN, int DONE, class LD, class ST, class PF = NoPf>
__device__ __forceinline__ void ntt_steps(const LD& gin, const ST& gout, uint64_t* sm, const uint64_t* psi,
                                          const uint64_t* psip, uint64_t q, uint32_t tile0, uint64_t ninv,
                                          uint64_t ninv_sh, const PF& pf = PF{}) {
  constexpr int logR = NttGeom<LOGN, ROWS>::logR;
  if constexpr (DONE < logR) {
    constexpr int rem = logR - DONE;
    constexpr int RB = pick_rb(rem);
    constexpr bool pre = ((HS_NTT_PRETW64 >> ((INV ? 2 : 0) + (ROWS ? 0 : 1))) & 1) != 0 && DONE > 0 && RB <= 3;
    uint64_t wpre[8], wppre[8];
    if constexpr (pre) ntt_tw_u64<INV, ROWS, LOGN, RB, DONE>(wpre, wppre, psi, psip, tile0);
    if constexpr (DONE > 0) __syncthreads();
    if constexpr (DONE > 0 && DONE == pick_rb(logR)) pf();
    ntt_step<INV, ROWS, LOGN, RB, DONE, DONE == 0, DONE + RB == logR, LD, ST>(
        gin, gout, sm, psi, psip, q, tile0, ninv, ninv_sh, pre ? wpre : nullptr, pre ? wppre : nullptr);
    ntt_steps<INV, ROWS, LOGN, DONE + RB, LD, ST, PF>(gin, gout, sm, psi, psip, q, tile0, ninv, ninv_sh, pf);
  } else if constexpr (DONE == pick_rb(logR) && !std::is_same_v<PF, NoPf>) {  // single-step pass
    __syncthreads();
    pf();
  }
}

// ---- FP64 path for primes below 2^45 (40-bit q_i, <= 44-bit special primes) --------
// Residues are carried as exact integers in fp64 registers.  A twiddle product
// y*w mod q is hi = fl(y w), lo = fma(y, w, -hi) (exact), k = rint(hi / q) (magic
// constant), r = fma(-k, q, hi) + lo: every step is exact because all values are
// integers below 2^53, and |r| < 1.5 q.  Forward (Cooley-Tukey) outputs X +- T grow
// by at most 1.5 q per stage (< 26 q < 2^49.7 after 16 stages, so hi/q stays inside
// the magic constant's 2^51 range), so no reduction is needed inside a pass; inverse (Gentleman-Sande) sums double per stage and are folded
// back below 0.6 q after every radix step.  Pass outputs are canonical u64.  The
// arithmetic runs on the FP64 pipe, leaving the integer ALU (the bottleneck of the
// 64-bit Shoup path) to addressing.  Results are identical: the NTT of canonical
// input is a unique canonical vector.
constexpr double kMagic = 6755399441055744.0;  // 1.5 * 2^52: fl(x + M) - M = rint(x), |x| < 2^51
#ifndef HS_NTT_RAW
#define HS_NTT_RAW 1
#endif
// intermediate between the two passes as raw fp64 (HS_NTT_RAW=0: canonical u64 words)
constexpr int kRawOut = HS_NTT_RAW ? 1 : 0, kRawIn = HS_NTT_RAW ? 2 : 0;
constexpr double kTwo52 = 4503599627370496.0;

__device__ __forceinline__ double u2d(uint64_t v) {  // exact for v < 2^52
  return __dadd_rn(__longlong_as_double(static_cast<long long>(v | 0x4330000000000000ULL)), -kTwo52);
}
__device__ __forceinline__ uint64_t d2u(double r) {  // r integer in [0, 2^52)
  return static_cast<uint64_t>(__double_as_longlong(__dadd_rn(r, kTwo52))) & 0xFFFFFFFFFFFFFULL;
}
__device__ __forceinline__ double fp_mulmod(double y, double w, double q, double qinv) {
  const double hi = __dmul_rn(y, w);
  const double lo = __fma_rn(y, w, -hi);
  const double k = __dadd_rn(__fma_rn(hi, qinv, kMagic), -kMagic);
  return __dadd_rn(__fma_rn(-k, q, hi), lo);
}
__device__ __forceinline__ double fp_fold(double x, double q, double qinv) {  // -> |r| < 0.6 q
  const double k = __dadd_rn(__fma_rn(x, qinv, kMagic), -kMagic);
  return __fma_rn(-k, q, x);
}
__device__ __forceinline__ uint64_t fp_canon(double x, double q, double qinv) {
  double r = fp_fold(x, q, qinv);
  r = r < 0.0 ? __dadd_rn(r, q) : r;
  return d2u(r);
}

// Row-pass twiddles staged in shared memory: for local stage m the tile's rows use the
// contiguous run tw[2^m (R1 + tile0) + (0 .. TPB 2^m)), stored at tws[TPB (2^m - 1) + ...].
template <int LOGN>
struct RowTw {
  using G = NttGeom<LOGN, true>;
  static constexpr uint32_t TPB = 1u << G::logTPB;
  static constexpr uint32_t words = TPB * ((1u << G::logC) - 1);
  __device__ static constexpr uint32_t off(uint32_t m) { return TPB * ((1u << m) - 1); }
};

template <int LOGN>
__device__ __forceinline__ void stage_row_tw(double* tws, const double* tw, uint32_t tile0) {
  using T = RowTw<LOGN>;
#pragma unroll
  for (uint32_t m = 0; m < T::G::logC; ++m) {
    const double* src = tw + (size_t(1) << m) * (T::G::R1 + tile0);
    double* dst = tws + T::off(m);
    for (uint32_t k = threadIdx.x; k < (T::TPB << m); k += kNT) dst[k] = __ldg(src + k);
  }
}

// RAWM: 0 canonical u64 in and out; 1 (first pass of a two-pass NTT) the output stays as raw
// fp64 bits (unreduced forward / folded inverse values) for the second pass; 2 (second pass)
// the input is those raw fp64 bits.  Saves the canonicalisation and the integer-to-double
// conversion between the passes (the intermediate is read by nothing else).
template <bool INV, bool ROWS, int LOGN, int RB, int DONE, bool FIRST, bool LAST, class LD, class ST, int RAWM = 0>
__device__ __forceinline__ void ntt_step_fp(const LD& gin, const ST& gout,
                                            double* __restrict__ sm, const double* __restrict__ tw, double q,
                                            double qinv, uint32_t tile0, double ninv,
                                            const double* __restrict__ tws, const double* wpre = nullptr) {
  using G = NttGeom<LOGN, ROWS>;
  constexpr uint32_t logR = G::logR, logTPB = G::logTPB, logC = G::logC;
  constexpr uint32_t logG = logR - RB;
  constexpr uint32_t total = 1u << (logG + logTPB);
  constexpr uint32_t logs = INV ? DONE : logR - 1 - DONE - (RB - 1);
#pragma unroll
  for (uint32_t it = 0; it < (total + kNT - 1) / kNT; ++it) {
    const uint32_t idx = threadIdx.x + it * kNT;
    if (total % kNT != 0 && idx >= total) break;
    uint32_t tr, g;
    if (ROWS) {
      g = idx & ((1u << logG) - 1);
      tr = idx >> logG;
    } else {
      tr = idx & ((1u << logTPB) - 1);
      g = idx >> logTPB;
    }
    const uint32_t blk0 = g >> logs;
    const uint32_t j0 = (blk0 << (logs + RB)) | (g & ((1u << logs) - 1));
    // swz is linear over XOR and j0 has zeros in bits logs .. logs + RB - 1, so the swizzled index of
    // element k is swz(base) ^ swz(k << logs): one swizzle per thread and step, one XOR with a
    // compile-time constant per element
    const uint32_t sb = ROWS ? swz((tr << logR) + j0) : 0u;
    const uint32_t S = ROWS ? G::R1 + tile0 + tr : 1u;
    double x[1 << RB];
#pragma unroll
    for (int k = 0; k < (1 << RB); ++k) {
      const uint32_t e = j0 + (uint32_t(k) << logs);
      if (FIRST) {
        const uint64_t g = gin(ROWS ? (size_t(tr) << logC) + e : (size_t(e) << logC) + tr);
        x[k] = RAWM == 2 ? __longlong_as_double(static_cast<long long>(g)) : u2d(g);
      } else {
        x[k] = ROWS ? sm[sb ^ swz(uint32_t(k) << logs)] : sm[(e << logTPB) + tr];
      }
    }
    if (!INV) {
#pragma unroll
      for (int st = 0; st < RB; ++st) {
        const int d = 1 << (RB - 1 - st);
        double wv[8];  // the stage's 2^st twiddles are consecutive: 16-byte loads
        if (wpre && it == 0) {  // loaded before the barrier that precedes this step (ntt_tw_fp)
#pragma unroll
          for (int b = 0; b < (1 << st); ++b) wv[b] = wpre[(1 << st) - 1 + b];
        } else if (!(ROWS && tws)) {
          ldg_tw(wv, tw + ((1u << (DONE + st)) * S) + (blk0 << st), 1 << st);
        }
#pragma unroll
        for (int b = 0; b < (1 << st); ++b) {
          const double w = ROWS && tws ? tws[RowTw<LOGN>::off(DONE + st) + (tr << (DONE + st)) + (blk0 << st) + b]
                                       : wv[b];
#pragma unroll
          for (int o = 0; o < d; ++o) {
            const int k0 = b * 2 * d + o;
            const double T = fp_mulmod(x[k0 + d], w, q, qinv);
            const double X = x[k0];
            x[k0] = __dadd_rn(X, T);
            x[k0 + d] = __dadd_rn(X, -T);
          }
        }
      }
    } else {
      constexpr uint32_t logh0 = logR - 1 - DONE;
#pragma unroll
      for (int st = 0; st < RB; ++st) {
        const int d = 1 << st;
        double wv[8];
        if (wpre && it == 0) {
#pragma unroll
          for (int b = 0; b < (1 << (RB - 1 - st)); ++b) wv[b] = wpre[(1 << RB) - (2 << (RB - 1 - st)) + b];
        } else if (!(ROWS && tws)) {
          ldg_tw(wv, tw + ((1u << (logh0 - st)) * S) + (blk0 << (RB - 1 - st)), 1 << (RB - 1 - st));
        }
#pragma unroll
        for (int b = 0; b < (1 << (RB - 1 - st)); ++b) {
          const double w = ROWS && tws
                               ? tws[RowTw<LOGN>::off(logh0 - st) + (tr << (logh0 - st)) + (blk0 << (RB - 1 - st)) + b]
                               : wv[b];
#pragma unroll
          for (int o = 0; o < d; ++o) {
            const int k0 = b * 2 * d + o;
            const double X = x[k0], Y = x[k0 + d];
            x[k0] = __dadd_rn(X, Y);
            x[k0 + d] = fp_mulmod(__dadd_rn(X, -Y), w, q, qinv);
          }
        }
      }
      if (!LAST || RAWM == 1) {
#pragma unroll
        for (int k = 0; k < (1 << RB); ++k) x[k] = fp_fold(x[k], q, qinv);
      }
    }
#pragma unroll
    for (int k = 0; k < (1 << RB); ++k) {
      const uint32_t e = j0 + (uint32_t(k) << logs);
      if (LAST && RAWM == 1) {
        gout(ROWS ? (size_t(tr) << logC) + e : (size_t(e) << logC) + tr,
             static_cast<uint64_t>(__double_as_longlong(x[k])));
      } else if (LAST) {
        const double v = (INV && !ROWS) ? fp_mulmod(x[k], ninv, q, qinv) : x[k];
        gout(ROWS ? (size_t(tr) << logC) + e : (size_t(e) << logC) + tr, fp_canon(v, q, qinv));
      } else {
        if (ROWS)
          sm[sb ^ swz(uint32_t(k) << logs)] = x[k];
        else
          sm[(e << logTPB) + tr] = x[k];
      }
    }
  }
}

// The twiddles of one radix step for this thread's first group (it = 0), issued before the barrier
// that precedes the step: their L1/L2 latency overlaps the barrier wait and the shared-memory reads
// instead of following them (a row pass's twiddles are distinct per row: L1 misses).  Forward: stage
// st's 2^st values at wpre[2^st - 1 ..]; inverse: stage st's 2^(RB-1-st) values after the earlier stages'.
// HS_NTT_PRETW: bit 0 forward rows, bit 1 forward columns, bit 2 inverse rows, bit 3 inverse columns.
#ifndef HS_NTT_PRETW
#define HS_NTT_PRETW 3
#endif
template <bool INV, bool ROWS, int LOGN, int RB, int DONE>
__device__ __forceinline__ void ntt_tw_fp(double (&wpre)[8], const double* __restrict__ tw, uint32_t tile0) {
  using G = NttGeom<LOGN, ROWS>;
  constexpr uint32_t logR = G::logR, logTPB = G::logTPB;
  constexpr uint32_t logG = logR - RB;
  constexpr uint32_t logs = INV ? DONE : logR - 1 - DONE - (RB - 1);
  const uint32_t idx = threadIdx.x;
  const uint32_t g = ROWS ? idx & ((1u << logG) - 1) : idx >> logTPB;
  const uint32_t tr = ROWS ? idx >> logG : idx & ((1u << logTPB) - 1);
  const uint32_t blk0 = g >> logs;
  const uint32_t S = ROWS ? G::R1 + tile0 + tr : 1u;
#pragma unroll
  for (int st = 0; st < RB; ++st) {
    double wv[8];
    if (!INV) {
      ldg_tw(wv, tw + ((1u << (DONE + st)) * S) + (blk0 << st), 1 << st);
#pragma unroll
      for (int b = 0; b < (1 << st); ++b) wpre[(1 << st) - 1 + b] = wv[b];
    } else {
      constexpr uint32_t logh0 = logR - 1 - DONE;
      ldg_tw(wv, tw + ((1u << (logh0 - st)) * S) + (blk0 << (RB - 1 - st)), 1 << (RB - 1 - st));
#pragma unroll
      for (int b = 0; b < (1 << (RB - 1 - st)); ++b) wpre[(1 << RB) - (2 << (RB - 1 - st)) + b] = wv[b];
    }
  }
}

template <bool INV, bool ROWS, int LOGN, int DONE, class LD, class ST, class PF = NoPf, int RAWM = 0>
__device__ __forceinline__ void ntt_steps_fp(const LD& gin, const ST& gout, double* sm, const double* tw,
                                             double q, double qinv, uint32_t tile0, double ninv,
                                             const double* tws = nullptr, const PF& pf = PF{}) {
  constexpr int logR = NttGeom<LOGN, ROWS>::logR;
  if constexpr (DONE < logR) {
    constexpr int rem = logR - DONE;
    constexpr int RB = pick_rb(rem);
    constexpr bool pre = ((HS_NTT_PRETW >> ((INV ? 2 : 0) + (ROWS ? 0 : 1))) & 1) != 0 && DONE > 0 && RB <= 3;
    double wpre[8];
    if constexpr (pre) {
      if (!(ROWS && tws)) ntt_tw_fp<INV, ROWS, LOGN, RB, DONE>(wpre, tw, tile0);
    }
    if constexpr (DONE > 0) __syncthreads();
    if constexpr (DONE > 0 && DONE == pick_rb(logR)) pf();
    ntt_step_fp<INV, ROWS, LOGN, RB, DONE, DONE == 0, DONE + RB == logR, LD, ST, RAWM>(
        gin, gout, sm, tw, q, qinv, tile0, ninv, tws, pre && !(ROWS && tws) ? wpre : nullptr);
    ntt_steps_fp<INV, ROWS, LOGN, DONE + RB, LD, ST, PF, RAWM>(gin, gout, sm, tw, q, qinv, tile0, ninv, tws, pf);
  } else if constexpr (DONE == pick_rb(logR) && !std::is_same_v<PF, NoPf>) {
    __syncthreads();
    pf();
  }
}

// Forward: columns then rows; inverse: rows then columns.  Reads `in`, writes
// `out` (may alias: every block reads its whole tile before its last step writes).
// 3 blocks of 512 threads per SM (40 registers): measured 1.3x over 2 blocks.
// MODE 0: plain; 1: ModDown epilogue (forward row pass); 2: rescale spread as the
// load of the forward column pass; 3: rescale combine as the store of the row pass.
struct PassEpi {
  MdEpi md;
  RsEpi rs;
  KsSrc ks;
};

template <class L>
__device__ __forceinline__ L mk_ld(const uint64_t* g) {
  return L{g};
}

// One pass over tile bx of row-map entry by, batch item bz (the body of k_ntt_pass).
// sm: kNTile words for the tile, plus (row passes) RowTw<LOGN>::words doubles of staged twiddles.
template <bool INV, bool ROWS, int LOGN, int MODE, int LDK, class PF = NoPf>
__device__ __forceinline__ void ntt_pass_dev(uint32_t bx, uint32_t by, uint32_t bz, uint64_t* sm, const uint64_t* in,
                                             size_t in_stride, uint64_t* out, size_t out_stride, const RowMap& rm,
                                             const PrimeC* pcs, const uint64_t* tw, const double* twd,
                                             const PassEpi& epi, bool use_row_tw = true,
                                             const uint64_t* stage = nullptr, const PF& pf = PF{}) {
  using G = NttGeom<LOGN, ROWS>;
  using PlainLd = PlainLoad;
  constexpr uint32_t N = 1u << LOGN;
  const uint32_t pi = rm.prime[by];
  const PrimeC& P = pcs[pi];
  const uint64_t* psi = tw + size_t(pi) * 4 * N + (INV ? 2 * N : 0);
  const uint64_t* psip = psi + N;
  const uint32_t tile0 = bx << G::logTPB;  // first sub-transform of this block
  const size_t toff = ROWS ? (size_t(tile0) << G::logC) : size_t(tile0);
  const uint64_t* gi = in + bz * in_stride + (size_t(rm.irow[by]) << LOGN) + toff;
  uint64_t* go = out + bz * out_stride + (size_t(rm.orow[by]) << LOGN) + toff;
  const double* twp = twd + size_t(pi) * 2 * N + (INV ? N : 0);
  double* tws = nullptr;
  if constexpr (ROWS) {
    if (P.fp && use_row_tw) {  // uniform per block
      tws = reinterpret_cast<double*>(sm) + kNTile;
      stage_row_tw<LOGN>(tws, twp, tile0);
      __syncthreads();
    }
  }
  auto run = [&](const auto& ld, const auto& st) {
    if (P.fp)  // first pass (forward columns / inverse rows) leaves raw fp64 words for the second
      ntt_steps_fp<INV, ROWS, LOGN, 0, std::decay_t<decltype(ld)>, std::decay_t<decltype(st)>, PF,
                   (ROWS == INV) ? kRawOut : kRawIn>(ld, st, reinterpret_cast<double*>(sm), twp, P.qd, P.qinvd, tile0,
                                                    static_cast<double>(P.ninv), tws, pf);
    else
      ntt_steps<INV, ROWS, LOGN, 0>(ld, st, sm, psi, psip, P.q, tile0, P.ninv, P.ninv_sh, pf);
  };
  if constexpr (MODE == 1 || MODE == 6 || MODE == 7 || MODE == 8) {  // row r = w * nl + i of the ModDown conversion output
    const MdEpi& e = epi.md;
    const uint32_t r = rm.orow[by], w = r / e.nl, i = r - w * e.nl;
    const uint64_t* acc = e.acc + bz * e.acc_stride + (size_t(w * e.nx + i) << LOGN) + toff;
    uint64_t* o = e.out + bz * e.out_stride + (size_t(w * e.nl + i) << LOGN) + toff;
    if constexpr (MODE == 8) {
      const uint64_t* ad = (w == 0 ? e.add0 : e.add1) + bz * e.add_stride + (size_t(i) << LOGN) + toff;
      run(mk_ld<PlainLd>(gi), MdStore<AddRowScaled>{acc, o, P.q, e.pinv[i], e.pinv_sh[i],
                                                           AddRowScaled{ad, e.ascale[i], e.ascale_sh[i]}});
    } else if constexpr (MODE == 1) {
      const uint64_t* ad = w == 0 ? e.add0 : e.add1;
      run(mk_ld<PlainLd>(gi), MdStore<AddRow>{acc, o, P.q, e.pinv[i], e.pinv_sh[i],
                                         AddRow{ad ? ad + bz * e.add_stride + (size_t(i) << LOGN) + toff : nullptr}});
    } else if constexpr (MODE == 6) {
      const KsSrc& k = epi.ks;
      const uint64_t* a0 = k.a + bz * k.stride + (size_t(i) << LOGN) + toff;
      const uint64_t* b0 = k.b + bz * k.stride + (size_t(i) << LOGN) + toff;
      const size_t h = size_t(k.nl) << LOGN;
      run(mk_ld<PlainLd>(gi), MdStore<AddTensor>{acc, o, P.q, e.pinv[i], e.pinv_sh[i],
                                            AddTensor{a0, a0 + h, b0, b0 + h, P, int(w)}});
    } else {
      const KsSrc& k = epi.ks;
      const uint64_t* c0 = w == 0 ? k.a + bz * k.stride + (size_t(i) << LOGN) : nullptr;
      run(mk_ld<PlainLd>(gi), MdStore<AddPerm<LOGN>>{acc, o, P.q, e.pinv[i], e.pinv_sh[i],
                                                AddPerm<LOGN>{c0, k.g, uint32_t(toff)}});
    }
  } else if constexpr (MODE == 4 || MODE == 5) {  // inverse row pass of d = a1 b1 / sigma(c1), limb irow
    const KsSrc& k = epi.ks;
    const uint32_t i = rm.irow[by];
    const uint64_t* r1 = k.a + bz * k.stride + (size_t(k.nl + i) << LOGN);
    if constexpr (MODE == 4)
      run(TnLoad{r1 + toff, k.b + bz * k.stride + (size_t(k.nl + i) << LOGN) + toff, P}, PlainStore{go});
    else
      run(PermLoad<LOGN>{r1, k.g, uint32_t(toff)}, PlainStore{go});
  } else if constexpr (MODE == 2) {  // row r = p * level + i: [last_p]_{q_i}
    const RsEpi& e = epi.rs;
    const uint32_t r = rm.orow[by], p = r / e.level;
    run(RsLoad{e.last + bz * e.last_stride + (size_t(p) << LOGN) + toff, P, e.kon, e.kk(bz, e.level),
               e.kk_sh(bz, e.level), pcs[e.level].q},
        PlainStore{go});
  } else if constexpr (MODE == 3) {
    const RsEpi& e = epi.rs;
    const uint32_t r = rm.orow[by], p = r / e.level, i = r - p * e.level;
    const RsStore st{e.in + bz * e.in_stride + (size_t(p * (e.level + 1) + i) << LOGN) + toff,
                     e.out + bz * e.out_stride + (size_t(p * e.level + i) << LOGN) + toff, P.q, e.qinv[i],
                     e.qinv_sh[i], e.kon, e.kk(bz, i), e.kk_sh(bz, i),
                     (e.aitems && p == 0) ? e.aitems[size_t(bz) * e.level + i] : 0};
    run(mk_ld<PlainLd>(gi), st);
  } else {
    run(mk_ld<PlainLd>(gi), PlainStore{go});
  }
}

// Build switch HS_ROW_TW=1: row-pass twiddles (a distinct run per row) staged in shared
// memory at block start instead of read through L1/L2.  Off: measured slower (HMult+relin
// 198 against 184 us per ciphertext): the staging phase and the doubled shared memory per
// block cost more than the twiddle loads they replace.
#ifndef HS_ROW_TW
#define HS_ROW_TW 0
#endif
constexpr bool row_tw_on = HS_ROW_TW != 0;

template <bool INV, bool ROWS, int LOGN, int MODE = 0>
__global__ void __launch_bounds__(kNT, HS_NTT_MINB) k_ntt_pass(const uint64_t* in, size_t in_stride, uint64_t* out,
                                                  size_t out_stride, const __grid_constant__ RowMap rm,
                                                  const PrimeC* pcs, const uint64_t* tw, const double* twd,
                                                  const __grid_constant__ PassEpi epi) {
  __shared__ uint64_t sm[kNTile + (ROWS && row_tw_on ? RowTw<LOGN>::words : 0)];
  ntt_pass_dev<INV, ROWS, LOGN, MODE, 0>(blockIdx.x, blockIdx.y, blockIdx.z, sm, in, in_stride, out, out_stride, rm,
                                             pcs, tw, twd, epi, row_tw_on);
}

template <bool INV, bool ROWS, int LOGN, int MODE>
void launch_pass(const uint64_t* in, size_t in_stride, uint64_t* out, size_t out_stride, const RowMap& rm,
                 uint32_t n, uint32_t batch, const PrimeC* pcs, const uint64_t* tw, const double* twd,
                 const PassEpi& ep, cudaStream_t s) {
  using G = NttGeom<LOGN, ROWS>;
  const uint32_t ntx = ROWS ? 1u << (G::logR1 - G::logTPB) : 1u << (G::logC - G::logTPB);
  k_ntt_pass<INV, ROWS, LOGN, MODE><<<dim3(ntx, n, batch), kNT, 0, s>>>(in, in_stride, out, out_stride, rm, pcs, tw,
                                                                        twd, ep);
}

template <int LOGN>
void launch_ntt(const uint64_t* in, size_t in_stride, uint64_t* out, size_t out_stride, const RowMap& rm,
                const RowMap& rm2, uint32_t n, uint32_t batch, bool inverse, const PrimeC* pcs, const uint64_t* tw,
                const double* twd, cudaStream_t s, const MdEpi* md, const RsEpi* rs, const KsSrc* ks) {
  using Gc = NttGeom<LOGN, false>;
  using Gr = NttGeom<LOGN, true>;
  const dim3 gc(1u << (Gc::logC - Gc::logTPB), n, batch), gr(1u << (Gr::logR1 - Gr::logTPB), n, batch);
  PassEpi none{}, ep{};
  if (md) ep.md = *md;
  if (rs) ep.rs = *rs;
  const int ksm = ks ? ks->mode : KS_PLAIN;
  if (ks) ep.ks = *ks;
  const PassEpi& E = ep;
  if (!inverse && md && ksm != KS_PLAIN) {
    launch_pass<false, false, LOGN, 0>(in, in_stride, out, out_stride, rm, n, batch, pcs, tw, twd, none, s);
    if (ksm == KS_TENSOR)
      launch_pass<false, true, LOGN, 6>(out, out_stride, out, out_stride, rm2, n, batch, pcs, tw, twd, E, s);
    else
      launch_pass<false, true, LOGN, 7>(out, out_stride, out, out_stride, rm2, n, batch, pcs, tw, twd, E, s);
    return;
  }
  if (inverse && ksm != KS_PLAIN) {
    if (ksm == KS_TENSOR)
      launch_pass<true, true, LOGN, 4>(in, in_stride, out, out_stride, rm, n, batch, pcs, tw, twd, E, s);
    else
      launch_pass<true, true, LOGN, 5>(in, in_stride, out, out_stride, rm, n, batch, pcs, tw, twd, E, s);
    launch_pass<true, false, LOGN, 0>(out, out_stride, out, out_stride, rm2, n, batch, pcs, tw, twd, none, s);
    return;
  }
  if (!inverse) {
    if (rs)
      launch_pass<false, false, LOGN, 2>(in, in_stride, out, out_stride, rm, n, batch, pcs, tw, twd, E, s);
    else
      launch_pass<false, false, LOGN, 0>(in, in_stride, out, out_stride, rm, n, batch, pcs, tw, twd, none, s);
    if (md && md->ascale)
      launch_pass<false, true, LOGN, 8>(out, out_stride, out, out_stride, rm2, n, batch, pcs, tw, twd, E, s);
    else if (md)
      launch_pass<false, true, LOGN, 1>(out, out_stride, out, out_stride, rm2, n, batch, pcs, tw, twd, E, s);
    else if (rs)
      launch_pass<false, true, LOGN, 3>(out, out_stride, out, out_stride, rm2, n, batch, pcs, tw, twd, E, s);
    else
      launch_pass<false, true, LOGN, 0>(out, out_stride, out, out_stride, rm2, n, batch, pcs, tw, twd, none, s);
  } else {
    launch_pass<true, true, LOGN, 0>(in, in_stride, out, out_stride, rm, n, batch, pcs, tw, twd, none, s);
    launch_pass<true, false, LOGN, 0>(out, out_stride, out, out_stride, rm2, n, batch, pcs, tw, twd, none, s);
  }
}

}  // namespace
}  // namespace rns
}  // namespace hsg


namespace hsg {
namespace rns {
namespace {

// ---------------------------------------------------------------- sampling / keys
__global__ void k_random_ct(uint64_t* out, const PrimeC* pcs, uint64_t seed, uint64_t tag, uint32_t nl,
                            uint32_t logN) {
  const size_t total = size_t(2 * nl) << logN;
  for (size_t x = blockIdx.x * size_t(blockDim.x) + threadIdx.x; x < total; x += size_t(gridDim.x) * blockDim.x) {
    const uint32_t n = x & ((1u << logN) - 1), r = x >> logN, p = r / nl, i = r - p * nl;
    out[x] = uniform_mod(hash64(seed, D_CT, tag * 1024 + p * 64 + i, n), pcs[i].q);
  }
}

// Symmetric RLWE encryption of integer coefficients m (rns_oracle.c rnso_encrypt_coeffs):
// c1 = a (uniform, NTT form), c0 = NTT(m + e) - a s.  This kernel writes [m + e]_{q_i}
// (coefficient form) into the c0 rows and a into the c1 rows.
__global__ void k_enc_me(const int64_t* coeffs, uint64_t* ct, const PrimeC* pcs, uint64_t seed, uint64_t tag,
                         uint32_t nl, uint32_t logN) {
  const size_t half = size_t(nl) << logN;
  for (size_t x = blockIdx.x * size_t(blockDim.x) + threadIdx.x; x < half; x += size_t(gridDim.x) * blockDim.x) {
    const uint32_t i = x >> logN, n = x & ((1u << logN) - 1);
    const uint64_t q = pcs[i].q;
    const int64_t h = static_cast<int64_t>(__popcll(hash64(seed, D_ENC_E, tag, n) & 0x1FFFFFULL)) -
                      static_cast<int64_t>(__popcll((hash64(seed, D_ENC_E, tag, n) >> 21) & 0x1FFFFFULL));
    ct[x] = lift(coeffs[n] + h, q);
    ct[half + x] = uniform_mod(hash64(seed, D_ENC_A, tag * 64 + i, n), q);
  }
}

// c0 rows (coefficient form) += e (CBD, stream D_ENC_E/tag); c1 rows = a (uniform, NTT form)
__global__ void k_enc_res(uint64_t* ct, const PrimeC* pcs, uint64_t seed, uint64_t tag, uint32_t nl, uint32_t logN) {
  const size_t half = size_t(nl) << logN;
  for (size_t x = blockIdx.x * size_t(blockDim.x) + threadIdx.x; x < half; x += size_t(gridDim.x) * blockDim.x) {
    const uint32_t i = x >> logN, n = x & ((1u << logN) - 1);
    const uint64_t q = pcs[i].q, h = hash64(seed, D_ENC_E, tag, n);
    const int64_t e = static_cast<int64_t>(__popcll(h & 0x1FFFFFULL)) - static_cast<int64_t>(__popcll((h >> 21) & 0x1FFFFFULL));
    ct[x] = add_mod(ct[x], lift(e, q), q);
    ct[half + x] = uniform_mod(hash64(seed, D_ENC_A, tag * 64 + i, n), q);
  }
}

// decryption on limbs 0..use-1: out[i] = c0_i + c1_i s_i (NTT form)
__global__ void k_dec(const uint64_t* ct, const uint64_t* sk, uint64_t* out, const PrimeC* pcs, uint32_t nl,
                      uint32_t use, uint32_t logN) {
  const size_t half = size_t(nl) << logN;
  for (size_t x = blockIdx.x * size_t(blockDim.x) + threadIdx.x; x < (size_t(use) << logN);
       x += size_t(gridDim.x) * blockDim.x) {
    const PrimeC& P = pcs[x >> logN];
    out[x] = add_mod(ct[x], mul_mod(ct[half + x], sk[x], P), P.q);
  }
}

// decryption (phase m through q_0, or q_0 q_1 with CRT) -> centred coefficients as doubles
// (the value nearest to the exact integer, as the host conversion of the same integer gives)
__global__ void k_center(const uint64_t* m, double* co, const PrimeC* pcs, uint64_t q0inv, uint64_t q0inv_sh,
                         uint32_t use, uint32_t logN) {
  const uint32_t N = 1u << logN;
  const uint64_t q0 = pcs[0].q;
  for (uint32_t n = blockIdx.x * blockDim.x + threadIdx.x; n < N; n += gridDim.x * blockDim.x) {
    if (use == 1) {
      const uint64_t h = m[n];
      co[n] = h > q0 / 2 ? -static_cast<double>(q0 - h) : static_cast<double>(h);
      continue;
    }
    const uint64_t q1 = pcs[1].q;
    const uint64_t a0 = m[n], a1 = m[N + n];
    const uint64_t t = mul_shoup(sub_mod(a1, a0 % q1, q1), q0inv, q0inv_sh, q1);
    const u128 r = static_cast<u128>(q0) * t + a0, Q = static_cast<u128>(q0) * q1;
    co[n] = r > Q / 2 ? -static_cast<double>(Q - r) : static_cast<double>(r);
  }
}

__global__ void k_scale_round(double* co, double r, uint32_t N) {  // refresh: co = rint(co * r)
  for (uint32_t n = blockIdx.x * blockDim.x + threadIdx.x; n < N; n += gridDim.x * blockDim.x)
    co[n] = rint(__dmul_rn(co[n], r));
}

__global__ void k_enc_as(uint64_t* ct, const uint64_t* sk, const PrimeC* pcs, uint32_t nl, uint32_t logN) {
  const size_t half = size_t(nl) << logN;
  for (size_t x = blockIdx.x * size_t(blockDim.x) + threadIdx.x; x < half; x += size_t(gridDim.x) * blockDim.x) {
    const PrimeC& P = pcs[x >> logN];
    ct[x] = sub_mod(ct[x], mul_mod(ct[half + x], sk[x], P), P.q);
  }
}

__global__ void k_addsub(const uint64_t* a, const uint64_t* b, uint64_t* out, const PrimeC* pcs, uint32_t nl,
                         uint32_t logN, size_t total, bool sub) {
  for (size_t x = blockIdx.x * size_t(blockDim.x) + threadIdx.x; x < total; x += size_t(gridDim.x) * blockDim.x) {
    const uint32_t i = (x >> logN) % nl;
    const uint64_t q = pcs[i].q;
    out[x] = sub ? sub_mod(a[x], b[x], q) : add_mod(a[x], b[x], q);
  }
}

// kv[i] = [k]_{q_i}; add: c0 += kv (constant polynomial = constant in NTT form), mul: both polys *= kv
// per-prime constant residues and Shoup factors, passed by value (no upload, no sync)
struct ConstTab {
  uint64_t k[64], ks[64];
};

__global__ void k_constop(const uint64_t* a, const __grid_constant__ ConstTab kt, uint64_t* out, const PrimeC* pcs,
                          uint32_t nl, uint32_t logN, size_t total, bool mul) {
  for (size_t x = blockIdx.x * size_t(blockDim.x) + threadIdx.x; x < total; x += size_t(gridDim.x) * blockDim.x) {
    const size_t r = x >> logN;
    const uint32_t i = r % nl, poly = (r / nl) & 1;
    const uint64_t q = pcs[i].q;
    if (mul)
      out[x] = mul_shoup(a[x], kt.k[i], kt.ks[i], q);
    else
      out[x] = poly == 0 ? add_mod(a[x], kt.k[i], q) : a[x];
  }
}

// residues of integer-valued doubles (|v| < 2^127): pt[i][n] = [co[n]]_{q_i}
__global__ void k_residues(const double* co, uint64_t* pt, const PrimeC* pcs, uint32_t nl, uint32_t logN) {
  for (size_t x = blockIdx.x * size_t(blockDim.x) + threadIdx.x; x < (size_t(nl) << logN);
       x += size_t(gridDim.x) * blockDim.x) {
    const PrimeC& P = pcs[x >> logN];
    const double v = co[x & ((1u << logN) - 1)];
    const double m = fabs(v);
    const double hi = floor(__dmul_rn(m, 5.421010862427522e-20));  // * 2^-64 (exact)
    const double lo = __dsub_rn(m, __dmul_rn(hi, 18446744073709551616.0));
    const u128 w = (static_cast<u128>(static_cast<uint64_t>(hi)) << 64) + static_cast<uint64_t>(lo);
    const uint64_t r = reduce128(w, P);
    pt[x] = (v < 0 && r) ? P.q - r : r;
  }
}

// out = a * pt on both polynomials (NTT form)
__global__ void k_mul_plain(const uint64_t* a, const uint64_t* pt, uint64_t* out, const PrimeC* pcs, uint32_t nl,
                            uint32_t logN) {
  const size_t half = size_t(nl) << logN;
  for (size_t x = blockIdx.x * size_t(blockDim.x) + threadIdx.x; x < 2 * half; x += size_t(gridDim.x) * blockDim.x) {
    const size_t r = x < half ? x : x - half;
    const PrimeC& P = pcs[r >> logN];
    out[x] = mul_mod(a[x], pt[r], P);
  }
}

// decryption on limb 0: out = c0 + c1 s mod q_0 (NTT form; iNTT'd by the host after)
__global__ void k_dec0(const uint64_t* ct, const uint64_t* sk, uint64_t* out, const PrimeC* pcs, uint32_t nl,
                       uint32_t logN) {
  const PrimeC P = pcs[0];
  const size_t half = size_t(nl) << logN;
  for (uint32_t n = blockIdx.x * blockDim.x + threadIdx.x; n < (1u << logN); n += gridDim.x * blockDim.x)
    out[n] = add_mod(ct[n], mul_mod(ct[half + n], sk[n], P), P.q);
}

// dense ternary (h = 0) or sparse with ~h nonzeros (rns_oracle.c ternary)
__global__ void k_secret(uint64_t* sk, const PrimeC* pcs, uint64_t seed, uint32_t h, uint32_t np, uint32_t logN) {
  for (size_t x = blockIdx.x * size_t(blockDim.x) + threadIdx.x; x < (size_t(np) << logN);
       x += size_t(gridDim.x) * blockDim.x) {
    const uint32_t n = x & ((1u << logN) - 1), i = x >> logN;
    int64_t v;
    if (h == 0)
      v = static_cast<int64_t>(hash64(seed, D_SECRET, 0, n) % 3) - 1;
    else if (hash64(seed, D_SECRET, 1, n) >= (static_cast<uint64_t>(h) << (64 - logN)))
      v = 0;
    else
      v = (hash64(seed, D_SECRET, 2, n) & 1) ? -1 : 1;
    sk[x] = lift(v, pcs[i].q);
  }
}

__device__ inline int64_t cbd(uint64_t h) {
  return static_cast<int64_t>(__popcll(h & 0x1FFFFFULL)) - static_cast<int64_t>(__popcll((h >> 21) & 0x1FFFFFULL));
}

// key digit j: a uniform (NTT form), e small (coefficient form, NTT'd by the host after)
__global__ void k_key_ae(uint64_t* a, uint64_t* e, const PrimeC* pcs, uint64_t seed, uint64_t keyid, uint32_t j,
                         uint32_t np, uint32_t logN) {
  for (size_t x = blockIdx.x * size_t(blockDim.x) + threadIdx.x; x < (size_t(np) << logN);
       x += size_t(gridDim.x) * blockDim.x) {
    const uint32_t n = x & ((1u << logN) - 1), i = x >> logN;
    const uint64_t q = pcs[i].q;
    a[x] = uniform_mod(hash64(seed, D_KEY_A, keyid * 4096 + j * 64 + i, n), q);
    e[x] = lift(cbd(hash64(seed, D_KEY_E, keyid * 4096 + j, n)), q);
  }
}

// b = e - a s + [i in digit j] P_i s'
__global__ void k_key_b(uint64_t* b, const uint64_t* a, const uint64_t* e, const uint64_t* s, const uint64_t* sp,
                        const PrimeC* pcs, const uint64_t* Pmod, uint32_t j, uint32_t alpha, uint32_t nq,
                        uint32_t np, uint32_t logN) {
  for (size_t x = blockIdx.x * size_t(blockDim.x) + threadIdx.x; x < (size_t(np) << logN);
       x += size_t(gridDim.x) * blockDim.x) {
    const uint32_t i = x >> logN;
    const PrimeC& P = pcs[i];
    uint64_t v = sub_mod(e[x], mul_mod(a[x], s[x], P), P.q);
    if (i < nq && i / alpha == j) v = add_mod(v, mul_mod(Pmod[i], sp[x], P), P.q);
    b[x] = v;
  }
}

__global__ void k_square(uint64_t* out, const uint64_t* in, const PrimeC* pcs, uint32_t np, uint32_t logN) {
  for (size_t x = blockIdx.x * size_t(blockDim.x) + threadIdx.x; x < (size_t(np) << logN);
       x += size_t(gridDim.x) * blockDim.x)
    out[x] = mul_mod(in[x], in[x], pcs[x >> logN]);
}


// out[r][n] = in[r][src(n)] for `rows` rows per batch item
__global__ void k_automorph(uint64_t* out, const uint64_t* in, uint64_t g, uint32_t logN, uint32_t rows,
                            size_t gstride) {
  const uint64_t* src = in + blockIdx.z * gstride;
  uint64_t* dst = out + blockIdx.z * gstride;
  for (size_t x = blockIdx.x * size_t(blockDim.x) + threadIdx.x; x < (size_t(rows) << logN);
       x += size_t(gridDim.x) * blockDim.x) {
    const uint32_t n = x & ((1u << logN) - 1);
    dst[x] = src[(x - n) + galois_src(n, g, logN)];
  }
}

// ---------------------------------------------------------------- HMult / key switching
// tensor: d0 = a0 b0, d1 = a0 b1 + a1 b0, d2 = a1 b1 (NTT form, nl limbs)
__global__ void k_tensor(const uint64_t* a, const uint64_t* b, uint64_t* d, const PrimeC* pcs, uint32_t nl,
                         uint32_t logN, size_t ct_stride, size_t d_stride, size_t b_stride) {
  const uint64_t* A = a + blockIdx.z * ct_stride;
  const uint64_t* Bb = b + blockIdx.z * b_stride;
  uint64_t* D = d + blockIdx.z * d_stride;
  const size_t half = size_t(nl) << logN;
  for (size_t x = blockIdx.x * size_t(blockDim.x) + threadIdx.x; x < half; x += size_t(gridDim.x) * blockDim.x) {
    const PrimeC& P = pcs[x >> logN];
    const uint64_t a0 = A[x], a1 = A[half + x], b0 = Bb[x], b1 = Bb[half + x];
    D[x] = mul_mod(a0, b0, P);
    D[half + x] = reduce128(static_cast<u128>(a0) * b1 + static_cast<u128>(a1) * b0, P);
    D[2 * half + x] = mul_mod(a1, b1, P);
  }
}

// One base conversion job: y_i = [x_i * hinv_i]_{src_i};  out_t = sum_i y_i h[t][i] mod t.
constexpr int kMaxSrc = 32, kMaxTgt = 64;
struct ConvJob {
  uint32_t nsrc, ntgt;
  uint32_t in_row, out_row;  // first source row / row base of the outputs, per batch item
  uint32_t frag_off;  // B fragments of k_conv_mma (uint2 index into the plan's table)
  uint32_t img_off;   // B image of k_conv_tc (byte offset into the plan's image table)
  uint32_t nint;      // targets [0, nint) are >= 2^45 (integer reduction), the rest take the FP64 path
  uint8_t src[kMaxSrc], tgt[kMaxTgt], tgt_row[kMaxTgt];
  uint64_t hinv[kMaxSrc], hinv_sh[kMaxSrc];
  uint64_t h[kMaxTgt][kMaxSrc];
};

// A = nsrc (compile time, <= 15 so the 128-bit sums cannot overflow), or 0 for a
// run-time count (partial reductions every 15 terms).
// Targets are processed in groups: one through the 128-bit integer MAC (ALU / IMAD
// pipes) and, when they and every source prime are below 2^45, one or two through
// exact fp64 modular products (fp_mulmod, FP64 pipe), so the pipes work at once.
template <int A>
__global__ void __launch_bounds__(kT) k_conv(const uint64_t* in, size_t in_stride, uint64_t* out, size_t out_stride,
                                             const ConvJob* jobs, const PrimeC* pcs, uint32_t logN) {
  constexpr int AS = A ? A : kMaxSrc;
  __shared__ uint64_t h_s[kMaxTgt * AS];
  __shared__ double hd_s[A ? kMaxTgt * AS : 1];
  __shared__ PrimeC tq[kMaxTgt];
  __shared__ uint64_t hinv_s[AS], hinvsh_s[AS], qs_s[AS];
  __shared__ uint32_t orow_s[kMaxTgt];
  __shared__ int src_fp;
  const ConvJob& J = jobs[blockIdx.y];
  const uint32_t nsrc = A ? A : J.nsrc, ntgt = J.ntgt;
  if (threadIdx.x == 0) src_fp = 1;
  for (uint32_t k = threadIdx.x; k < ntgt * nsrc; k += blockDim.x) {
    h_s[k] = J.h[k / nsrc][k % nsrc];
    if (A) hd_s[k] = static_cast<double>(h_s[k]);  // exact for targets below 2^45 (the only ones read)
  }
  for (uint32_t k = threadIdx.x; k < ntgt; k += blockDim.x) {
    tq[k] = pcs[J.tgt[k]];
    orow_s[k] = J.out_row + J.tgt_row[k];
  }
  __syncthreads();
  for (uint32_t k = threadIdx.x; k < nsrc; k += blockDim.x) {
    hinv_s[k] = J.hinv[k];
    hinvsh_s[k] = J.hinv_sh[k];
    qs_s[k] = pcs[J.src[k]].q;
    if (!pcs[J.src[k]].fp) src_fp = 0;
  }
  __syncthreads();
  const uint32_t n = blockIdx.x * blockDim.x + threadIdx.x;
  const uint64_t* I = in + blockIdx.z * in_stride + (size_t(J.in_row) << logN) + n;
  uint64_t* O = out + blockIdx.z * out_stride + n;
  uint64_t y[AS];
#pragma unroll
  for (int i = 0; i < AS; ++i)
    if (A || i < int(nsrc)) y[i] = mul_shoup(I[size_t(i) << logN], hinv_s[i], hinvsh_s[i], qs_s[i]);
  if constexpr (A != 0) {
    double yd[A];
#pragma unroll
    for (int i = 0; i < A; ++i) yd[i] = u2d(y[i]);  // exact when the sources are < 2^45 (no XU convert)
    const bool sfp = src_fp != 0;
    uint32_t t = 0;
    // groups of three targets: one integer MAC + two fp64 chains when eligible
    for (; sfp && t + 2 < ntgt; t += 3) {
      if (!tq[t + 1].fp || !tq[t + 2].fp) break;
      const uint64_t* h0 = h_s + t * A;
      const double *h1 = hd_s + (t + 1) * A, *h2 = hd_s + (t + 2) * A;
      const double q1 = tq[t + 1].qd, q1inv = tq[t + 1].qinvd, q2 = tq[t + 2].qd, q2inv = tq[t + 2].qinvd;
      u128 acc0 = 0;
      double r1 = 0.0, r2 = 0.0;
#pragma unroll
      for (int i = 0; i < A; ++i) {
        acc0 += static_cast<u128>(y[i]) * h0[i];
        r1 = __dadd_rn(r1, fp_mulmod(yd[i], h1[i], q1, q1inv));
        r2 = __dadd_rn(r2, fp_mulmod(yd[i], h2[i], q2, q2inv));
      }
      O[size_t(orow_s[t]) << logN] = reduce128(acc0, tq[t]);
      O[size_t(orow_s[t + 1]) << logN] = fp_canon(r1, q1, q1inv);
      O[size_t(orow_s[t + 2]) << logN] = fp_canon(r2, q2, q2inv);
    }
    for (; t < ntgt; t += 2) {
      const uint64_t* h0 = h_s + t * A;
      u128 acc0 = 0;
      if (t + 1 < ntgt && sfp && tq[t + 1].fp) {
        const double* h1 = hd_s + (t + 1) * A;
        const double q1 = tq[t + 1].qd, q1inv = tq[t + 1].qinvd;
        double r1 = 0.0;
#pragma unroll
        for (int i = 0; i < A; ++i) {
          acc0 += static_cast<u128>(y[i]) * h0[i];
          r1 = __dadd_rn(r1, fp_mulmod(yd[i], h1[i], q1, q1inv));
        }
        O[size_t(orow_s[t]) << logN] = reduce128(acc0, tq[t]);
        O[size_t(orow_s[t + 1]) << logN] = fp_canon(r1, q1, q1inv);
      } else if (t + 1 < ntgt) {
        const uint64_t* h1 = h0 + A;
        u128 acc1 = 0;
#pragma unroll
        for (int i = 0; i < A; ++i) {
          acc0 += static_cast<u128>(y[i]) * h0[i];
          acc1 += static_cast<u128>(y[i]) * h1[i];
        }
        O[size_t(orow_s[t]) << logN] = reduce128(acc0, tq[t]);
        O[size_t(orow_s[t + 1]) << logN] = reduce128(acc1, tq[t + 1]);
      } else {
#pragma unroll
        for (int i = 0; i < A; ++i) acc0 += static_cast<u128>(y[i]) * h0[i];
        O[size_t(orow_s[t]) << logN] = reduce128(acc0, tq[t]);
      }
    }
  } else {
    for (uint32_t t = 0; t < ntgt; ++t) {
      const uint64_t* ht = h_s + t * nsrc;
      u128 acc = 0;
      for (uint32_t i = 0; i < nsrc; ++i) {
        acc += static_cast<u128>(y[i]) * ht[i];
        if (i % 15 == 14) acc = reduce128(acc, tq[t]);
      }
      O[size_t(orow_s[t]) << logN] = reduce128(acc, tq[t]);
    }
  }
}

// ---- base conversion on the tensor cores (IMMA u8 m16n8k32) ----------------------------
// out_t[n] = sum_i y_i[n] h[t][i] mod q_t as an exact integer GEMM over bytes:
//   A[n][8i + a] = byte a of y_i[n]                      (the u64 residues as they lie)
//   B[8i + a][b] = byte b of (h[t][i] 2^(8a) mod q_t)    (host-built per job, in
//                                                         fragment order: conv_frags)
//   C[n][b] = sum_k A[n][k] B[k][b] < 8 nsrc 255^2 < 2^23   (exact in s32)
//   out_t[n] = sum_b C[n][b] 2^(8b) mod q_t: lo/hi 4-byte halves (< 2^47 each), one
//              reduce128 of hi 2^32 + lo.
// The result is congruent to sum_i y_i h[t][i] and canonical, so it equals k_conv's
// word for word.  A block converts 128 coefficients (4 warps x 2 m16 tiles) of one job;
// per target a warp issues 2 KS IMMAs, parks C in shared memory and every lane finishes
// one coefficient (coalesced row store).  The u128 MAC chain of k_conv (~90 ALU
// instructions per output) becomes ~30.
constexpr int kConvMmaRows = 128;

__device__ __forceinline__ void imma_u8(int (&c)[4], const uint32_t (&a)[4], uint2 b) {
  asm("mma.sync.aligned.m16n8k32.row.col.s32.u8.u8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
      : "+r"(c[0]), "+r"(c[1]), "+r"(c[2]), "+r"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b.x), "r"(b.y));
}

#ifndef HS_CONV_TPR
#define HS_CONV_TPR 2
#endif
constexpr int kConvTpr = HS_CONV_TPR;  // targets per round of k_conv_mma (IMMA/epilogue chains interleaved)

template <int KS>
constexpr size_t conv_mma_smem() {
  return size_t(kConvMmaRows) * (KS * 8 + 4) * 4 + 4 * kConvTpr * 256 * 4;
}

struct ConvTgt {
  double qd, qinvd, c32d;  // fp targets: q, 1/q, 2^32 mod q
  uint32_t orow, fp;
};

template <int KS>  // k-steps of 32 bytes: nsrc <= 4 KS
__global__ void __launch_bounds__(kConvMmaRows, 6) k_conv_mma(const uint64_t* in, size_t in_stride, uint64_t* out,
                                                           size_t out_stride, const ConvJob* jobs, const uint2* frags,
                                                           const PrimeC* pcs, uint32_t logN) {
  constexpr int RSW = KS * 8 + 4;  // A row stride in words: fragment loads hit 32 distinct banks
  extern __shared__ uint4 dyn_smem[];
  uint32_t* As = reinterpret_cast<uint32_t*>(dyn_smem);       // [128][RSW]
  int* stg = reinterpret_cast<int*>(As + kConvMmaRows * RSW);  // [4 warps][2][32][8]
  __shared__ PrimeC tq[kMaxTgt];
  __shared__ ConvTgt tc[kMaxTgt];
  __shared__ uint64_t hinv_s[4 * KS], hinvsh_s[4 * KS], qs_s[4 * KS];
  const ConvJob& J = jobs[blockIdx.y];
  const uint32_t nsrc = J.nsrc, ntgt = J.ntgt;
  for (uint32_t k = threadIdx.x; k < ntgt; k += kConvMmaRows) {
    const PrimeC P = pcs[J.tgt[k]];
    tq[k] = P;
    const uint64_t c32 = (uint64_t(1) << 32) % P.q;
    tc[k] = ConvTgt{P.qd, P.qinvd, static_cast<double>(c32), J.out_row + J.tgt_row[k], P.fp};
  }
  if (threadIdx.x < nsrc) {
    hinv_s[threadIdx.x] = J.hinv[threadIdx.x];
    hinvsh_s[threadIdx.x] = J.hinv_sh[threadIdx.x];
    qs_s[threadIdx.x] = pcs[J.src[threadIdx.x]].q;
  }
  __syncthreads();
  const uint32_t n0 = blockIdx.x * kConvMmaRows;
  {  // y_i = [x_i hinv_i]_{q_i}: thread = coefficient, the u64 words are the A row's bytes
    const uint64_t* I = in + blockIdx.z * in_stride + (size_t(J.in_row) << logN) + n0 + threadIdx.x;
    uint2* row = reinterpret_cast<uint2*>(As + threadIdx.x * RSW);
    uint64_t x[4 * KS];
#pragma unroll
    for (int i = 0; i < 4 * KS; ++i) x[i] = uint32_t(i) < nsrc ? __ldcs(I + (size_t(i) << logN)) : 0;  // all loads in flight
#pragma unroll
    for (int i = 0; i < 4 * KS; ++i) {
      const uint64_t y = uint32_t(i) < nsrc ? mul_shoup(x[i], hinv_s[i], hinvsh_s[i], qs_s[i]) : 0;
      row[i] = make_uint2(static_cast<uint32_t>(y), static_cast<uint32_t>(y >> 32));
    }
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, t4 = lane & 3;
  uint32_t a[2][KS][4];
#pragma unroll
  for (int m = 0; m < 2; ++m)
#pragma unroll
    for (int ks = 0; ks < KS; ++ks) {
      const uint32_t* r0 = As + (warp * 32 + m * 16 + g) * RSW + ks * 8 + t4;
      const uint32_t* r1 = r0 + 8 * RSW;
      a[m][ks][0] = r0[0];
      a[m][ks][1] = r1[0];
      a[m][ks][2] = r0[4];
      a[m][ks][3] = r1[4];
    }
  uint64_t* O = out + blockIdx.z * out_stride + n0 + warp * 32 + lane;
  int* const S0 = stg + warp * (256 * kConvTpr);
  int2* const W0 = reinterpret_cast<int2*>(S0 + g * 8 + 2 * t4);  // this lane's C slots (rows g, g+8, 16+g, 24+g)
  const uint4* const R0 = reinterpret_cast<const uint4*>(S0 + lane * 8);  // this lane's coefficient row
  const uint2* F = frags + J.frag_off + lane;
  // one target: KS x 2 IMMAs -> C parked in buffer `buf` (256 ints) -> the lane's row
  auto mma_park = [&](uint32_t t, int buf) {
    uint2 b[KS];
#pragma unroll
    for (int ks = 0; ks < KS; ++ks) b[ks] = __ldg(F + (t * KS + ks) * 32);  // same 256 B for every warp: L1
    int c[2][4] = {{0, 0, 0, 0}, {0, 0, 0, 0}};
#pragma unroll
    for (int ks = 0; ks < KS; ++ks) {
      imma_u8(c[0], a[0][ks], b[ks]);
      imma_u8(c[1], a[1][ks], b[ks]);
    }
    int2* W = W0 + buf * 128;
    W[0] = make_int2(c[0][0], c[0][1]);
    W[32] = make_int2(c[0][2], c[0][3]);
    W[64] = make_int2(c[1][0], c[1][1]);
    W[96] = make_int2(c[1][2], c[1][3]);
  };
  auto finish = [&](uint32_t t, int buf) {
    const uint4 u = R0[buf * 64], v = R0[buf * 64 + 1];
    const uint64_t lo = uint64_t(u.x) + (uint64_t(u.y) << 8) + (uint64_t(u.z) << 16) + (uint64_t(u.w) << 24);
    const uint64_t hi = uint64_t(v.x) + (uint64_t(v.y) << 8) + (uint64_t(v.z) << 16) + (uint64_t(v.w) << 24);
    const ConvTgt T = tc[t];
    uint64_t r;
    if (T.fp) {  // lo + hi (2^32 mod q) on the FP64 pipe: lo, hi < 2^47, every step exact
      const double h = fp_mulmod(u2d(hi), T.c32d, T.qd, T.qinvd);
      r = fp_canon(__dadd_rn(h, u2d(lo)), T.qd, T.qinvd);
    } else {
      r = reduce128((static_cast<u128>(hi) << 32) + lo, tq[t]);
    }
    O[size_t(T.orow) << logN] = r;
  };
  uint32_t t = 0;
#pragma unroll 1
  for (; t + kConvTpr <= ntgt; t += kConvTpr) {  // kConvTpr targets per round: IMMA and epilogue chains interleave
#pragma unroll
    for (int u = 0; u < kConvTpr; ++u) mma_park(t + u, u);
    __syncwarp();
#pragma unroll
    for (int u = 0; u < kConvTpr; ++u) finish(t + u, u);
    __syncwarp();
  }
#pragma unroll 1
  for (; t < ntgt; ++t) {
    mma_park(t, 0);
    __syncwarp();
    finish(t, 0);
    __syncwarp();
  }
}

#include "conv_tc.cuh"

// acc_w[x] = sum_j e_j[x] * key_w[j][prime(x)] over the nx extended rows, w = 0 (b), 1 (a);
// e_j[x] = d[x] on digit j's own rows (NTT form, never converted), ext_j[x] elsewhere.
// Each thread holds its key words and walks the whole batch.
constexpr int kMaxDigits = 15;
#ifndef HS_INNER_MINB
#define HS_INNER_MINB 4  // 64 registers, 4 blocks per SM (3 at 80 registers: 5 % slower HMult)
#endif
#ifndef HS_INNER_UNROLL
#define HS_INNER_UNROLL 2
#endif
constexpr int kInnerUnroll = HS_INNER_UNROLL;  // batch items in flight per thread
template <int ND>
__global__ void __launch_bounds__(kT, HS_INNER_MINB) k_ks_inner(const uint64_t* ext, size_t ext_stride, const uint64_t* d,
                                                 size_t d_stride, uint64_t* acc, size_t acc_stride,
                                                 const uint64_t* kb, const uint64_t* ka, const PrimeC* pcs,
                                                 uint32_t nx, uint32_t nl, uint32_t np, uint32_t nq, uint32_t alpha,
                                                 uint32_t logN, uint32_t batch, const KsSrc src) {
  // two adjacent coefficients per thread: 16-byte loads and stores (twice the bytes in flight per
  // instruction; the kernel streams ext/acc once per batch item)
  const size_t x = 2 * (blockIdx.x * size_t(blockDim.x) + threadIdx.x);
  const uint32_t row = x >> logN, n = x & ((1u << logN) - 1);
  if (row >= nx) return;
  const uint32_t gi = row < nl ? row : nq + (row - nl);
  const PrimeC P = pcs[gi];
  ulonglong2 kbr[ND], kar[ND];
#pragma unroll
  for (int j = 0; j < ND; ++j) {
    const size_t kx = (size_t(j * np + gi) << logN) + n;
    kbr[j] = __ldg(reinterpret_cast<const ulonglong2*>(kb + kx));
    kar[j] = __ldg(reinterpret_cast<const ulonglong2*>(ka + kx));
  }
  const uint32_t own = row < nl ? row / alpha : 0xFFFFFFFFu;
  const size_t rowsN = size_t(nx) << logN;
  // d on the digit's own rows: materialised, or the tensor / automorphism of the inputs
  auto own_word = [&](uint32_t b) -> ulonglong2 {
    if (src.mode == KS_TENSOR) {
      const size_t o = b * src.stride + (size_t(nl + row) << logN) + n;
      const ulonglong2 u = *reinterpret_cast<const ulonglong2*>(src.a + o);
      const ulonglong2 v = *reinterpret_cast<const ulonglong2*>(src.b + o);
      return make_ulonglong2(mul_mod(u.x, v.x, P), mul_mod(u.y, v.y, P));
    }
    if (src.mode == KS_PERM) {
      const uint64_t* r = src.a + b * src.stride + (size_t(nl + row) << logN);
      return make_ulonglong2(r[galois_src(n, src.g, logN)], r[galois_src(n + 1, src.g, logN)]);
    }
    return *reinterpret_cast<const ulonglong2*>(d + b * d_stride + x);
  };
#pragma unroll(kInnerUnroll)
  for (uint32_t b = 0; b < batch; ++b) {
    const uint64_t* E = ext + b * ext_stride + x;
    ulonglong2 e[ND];
#pragma unroll
    for (int j = 0; j < ND; ++j)
      e[j] = uint32_t(j) == own ? own_word(b) : *reinterpret_cast<const ulonglong2*>(E + j * rowsN);
    u128 s0 = 0, s1 = 0, t0 = 0, t1 = 0;
#pragma unroll
    for (int j = 0; j < ND; ++j) {
      s0 += static_cast<u128>(e[j].x) * kbr[j].x;
      s1 += static_cast<u128>(e[j].x) * kar[j].x;
      t0 += static_cast<u128>(e[j].y) * kbr[j].y;
      t1 += static_cast<u128>(e[j].y) * kar[j].y;
    }
    uint64_t* Ac = acc + b * acc_stride + x;
    *reinterpret_cast<ulonglong2*>(Ac) = make_ulonglong2(reduce128(s0, P), reduce128(t0, P));
    *reinterpret_cast<ulonglong2*>(Ac + rowsN) = make_ulonglong2(reduce128(s1, P), reduce128(t1, P));
  }
}

// ---------------------------------------------------------------- rescale
// host helpers -----------------------------------------------------------------------
uint64_t h_mulmod(uint64_t a, uint64_t b, uint64_t q) { return static_cast<uint64_t>(static_cast<u128>(a) * b % q); }
uint64_t h_pow(uint64_t a, uint64_t e, uint64_t q) {
  uint64_t r = 1 % q;
  a %= q;
  while (e) {
    if (e & 1) r = h_mulmod(r, a, q);
    a = h_mulmod(a, a, q);
    e >>= 1;
  }
  return r;
}
uint64_t h_inv(uint64_t a, uint64_t q) { return h_pow(a, q - 2, q); }
bool h_prime(uint64_t n) {
  static const uint64_t bases[] = {2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37};
  if (n < 2) return false;
  for (uint64_t b : bases)
    if (n % b == 0) return n == b;
  uint64_t d = n - 1;
  int r = 0;
  while ((d & 1) == 0) {
    d >>= 1;
    ++r;
  }
  for (uint64_t b : bases) {
    uint64_t x = h_pow(b, d, n);
    if (x == 1 || x == n - 1) continue;
    bool comp = true;
    for (int j = 1; j < r; ++j) {
      x = h_mulmod(x, x, n);
      if (x == n - 1) {
        comp = false;
        break;
      }
    }
    if (comp) return false;
  }
  return true;
}
uint32_t h_bitrev(uint32_t x, uint32_t bits) {
  uint32_t r = 0;
  for (uint32_t i = 0; i < bits; ++i) r |= ((x >> i) & 1u) << (bits - 1 - i);
  return r;
}

unsigned grid_of(size_t n) {
  const size_t g = (n + kT - 1) / kT;
  return static_cast<unsigned>(std::min<size_t>(std::max<size_t>(g, 1), size_t(Runtime::get().sm_count()) * 16));
}

template <class T>
DevBuf upload(const std::vector<T>& v) {
  Runtime& rt = Runtime::get();
  const size_t words = (v.size() * sizeof(T) + 7) / 8;
  DevBuf d = rt.alloc(std::max<size_t>(words, 1));
  cuda_ok(cudaMemcpyAsync(d.get(), v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice, rt.stream()), "upload");
  rt.sync();
  return d;
}

template <class T>
T* dptr(const DevBuf& b) {
  return reinterpret_cast<T*>(b.get());
}

std::vector<uint32_t> iota_rows(uint32_t n, uint32_t first = 0) {
  std::vector<uint32_t> v(n);
  for (uint32_t i = 0; i < n; ++i) v[i] = first + i;
  return v;
}

}  // namespace

// ================================================================== NTT launch
namespace {
}  // namespace

void ntt_rows(const Ctx& c, const uint64_t* in, size_t in_stride, uint64_t* out, size_t out_stride,
              const std::vector<uint32_t>& irows, const std::vector<uint32_t>& orows,
              const std::vector<uint32_t>& primes, uint32_t batch, bool inverse, const void* epilogue,
              const void* rescale_epi, const void* ks_src) {
  const MdEpi* epi = static_cast<const MdEpi*>(epilogue);
  const RsEpi* rs = static_cast<const RsEpi*>(rescale_epi);
  const KsSrc* ks = static_cast<const KsSrc*>(ks_src);
  if (irows.empty() || batch == 0) return;
  if (irows.size() != orows.size() || irows.size() != primes.size()) fail(HS_E_INVALID_ARG, "ntt_rows: size mismatch");
  Runtime& rt = Runtime::get();
  cudaStream_t s = rt.stream();
  const uint32_t logN = c.spec.logN;
  const uint64_t* tw = dptr<const uint64_t>(c.d_tw);
  const double* twd = dptr<const double>(c.d_twd);
  for (size_t base = 0; base < irows.size(); base += kMaxRows) {
    const uint32_t n = static_cast<uint32_t>(std::min<size_t>(kMaxRows, irows.size() - base));
    RowMap rm{}, rm2{};
    for (uint32_t i = 0; i < n; ++i) {
      rm.irow[i] = static_cast<uint16_t>(irows[base + i]);
      rm.orow[i] = rm2.irow[i] = rm2.orow[i] = static_cast<uint16_t>(orows[base + i]);
      rm.prime[i] = rm2.prime[i] = static_cast<uint8_t>(primes[base + i]);
    }
    switch (logN) {
#define HS_NTT_CASE(L) \
  case L:              \
    launch_ntt<L>(in, in_stride, out, out_stride, rm, rm2, n, batch, inverse, c.dpc(), tw, twd, s, epi, rs, ks); \
    break;
      HS_NTT_CASE(9) HS_NTT_CASE(10) HS_NTT_CASE(11) HS_NTT_CASE(12) HS_NTT_CASE(13) HS_NTT_CASE(14)
      HS_NTT_CASE(15) HS_NTT_CASE(16) HS_NTT_CASE(17)
#undef HS_NTT_CASE
      default:
        fail(HS_E_INVALID_ARG, "ntt: unsupported ring degree");
    }
    cuda_ok(cudaGetLastError(), "ntt launch");
    rt.note_launch(2);
  }
}

void ntt(const Ctx& c, uint64_t* data, const std::vector<uint32_t>& prime_of, uint32_t batch, size_t gstride,
         bool inverse) {
  const auto rows = iota_rows(static_cast<uint32_t>(prime_of.size()));
  ntt_rows(c, data, gstride, data, gstride, rows, rows, prime_of, batch, inverse);
}

// ================================================================== context
uint64_t Ctx::galois_elt(int64_t k, uint32_t logN) {
  const uint64_t twoN = 2ULL << logN, half = 1ULL << (logN - 1);
  int64_t kk = k % static_cast<int64_t>(half);
  if (kk < 0) kk += static_cast<int64_t>(half);
  uint64_t g = 1;
  for (int64_t i = 0; i < kk; ++i) g = g * 5 % twoN;
  return g;
}

Ctx::Ctx(const Spec& s) : spec(s) {
  if (s.logN < 9 || s.logN > 17) fail(HS_E_INVALID_ARG, "rns: logN must be in [9, 17]");
  if (s.dnum < 1 || s.K < 1 || s.L + 1 + s.K > 64) fail(HS_E_INVALID_ARG, "rns: bad prime counts");
  if (s.dnum > s.L + 1) fail(HS_E_INVALID_ARG, "rns: dnum larger than the number of q primes");
  if (s.h >= (1u << s.logN)) fail(HS_E_INVALID_ARG, "rns: secret Hamming weight must be below N");
  if (s.logq0 > 61 || s.logq > 61 || s.logp > 61 || s.logq < 20) fail(HS_E_INVALID_ARG, "rns: primes must be 20..61 bits");
  N = 1u << s.logN;
  nq = s.L + 1;
  np = nq + s.K;
  alpha = (nq + s.dnum - 1) / s.dnum;
  if (alpha > kMaxSrc || s.K > kMaxSrc) fail(HS_E_INVALID_ARG, "rns: digits / special primes wider than 32 primes");
  if ((nq + alpha - 1) / alpha > kMaxDigits) fail(HS_E_INVALID_ARG, "rns: more than 15 digits");
  // primes (rns_oracle.c rnso_primes)
  const uint64_t twoN = 2ULL << s.logN;
  const uint32_t bits[3] = {s.logq0, s.logq, s.logp}, cnt[3] = {1, s.L, s.K};
  for (int g = 0; g < 3; ++g) {
    uint64_t c = ((1ULL << bits[g]) / twoN) * twoN + 1;
    if (c >= (1ULL << bits[g])) c -= twoN;
    for (uint32_t taken = 0; taken < cnt[g];) {
      if (c < twoN) fail(HS_E_INVALID_ARG, "rns: ran out of NTT primes");
      if (std::find(primes.begin(), primes.end(), c) == primes.end() && h_prime(c)) {
        primes.push_back(c);
        ++taken;
      }
      c -= twoN;
    }
  }
  // Hybrid key switching is only correct when P = prod p_j exceeds every digit modulus
  // Q_j = prod_{i in digit j} q_i: ModDown divides the digit's ModUp error (~ Q_j) by P.  An
  // undersized P decrypts to garbage without any other symptom, so it is refused here.
  {
    long double logP = 0.0L, worst = 0.0L;
    for (uint32_t k = 0; k < s.K; ++k) logP += std::log2(static_cast<long double>(primes[nq + k]));
    for (uint32_t lo = 0; lo < nq; lo += alpha) {
      long double lq = 0.0L;
      for (uint32_t i = lo; i < std::min(lo + alpha, nq); ++i) lq += std::log2(static_cast<long double>(primes[i]));
      worst = std::max(worst, lq);
    }
    if (!(logP > worst))
      fail(HS_E_INVALID_ARG, "rns: the special modulus P (" + std::to_string(static_cast<double>(logP)) +
                                 " bits) must exceed every key-switching digit modulus (" +
                                 std::to_string(static_cast<double>(worst)) + " bits): raise K or logp");
  }
  // per-prime constants and twiddle tables
  std::vector<uint64_t> tw(size_t(np) * 4 * N);
  std::vector<double> twd(size_t(np) * 2 * N);
  for (uint32_t i = 0; i < np; ++i) {
    const uint64_t q = primes[i];
    PrimeC p{};
    p.q = q;
    p.k = 64 - __builtin_clzll(q);
    p.mu = static_cast<uint64_t>((static_cast<u128>(1) << (2 * p.k)) / q);
    p.m64 = static_cast<uint64_t>((static_cast<u128>(1) << 64) / q);
    p.r64 = static_cast<uint64_t>((static_cast<u128>(1) << 64) % q);
    p.r64_sh = shoup_of(p.r64, q);
    p.ninv = h_inv(N % q, q);
    p.ninv_sh = shoup_of(p.ninv, q);
    p.fp = q < (1ULL << 45) ? 1u : 0u;
    p.qd = static_cast<double>(q);
    p.qinvd = 1.0 / static_cast<double>(q);
    pc.push_back(p);
    uint64_t psi = 0;
    for (uint64_t x = 2;; ++x) {
      psi = h_pow(x, (q - 1) / twoN, q);
      if (h_pow(psi, N, q) == q - 1) break;
    }
    const uint64_t ipsi = h_inv(psi, q);
    uint64_t* t = tw.data() + size_t(i) * 4 * N;
    for (uint32_t k = 0; k < N; ++k) {
      const uint32_t r = h_bitrev(k, s.logN);
      t[k] = h_pow(psi, r, q);
      t[N + k] = shoup_of(t[k], q);
      t[2 * N + k] = h_pow(ipsi, r, q);
      t[3 * N + k] = shoup_of(t[2 * N + k], q);
      twd[size_t(i) * 2 * N + k] = static_cast<double>(t[k]);
      twd[size_t(i) * 2 * N + N + k] = static_cast<double>(t[2 * N + k]);
    }
  }
  d_pc = upload(pc);
  d_tw = upload(tw);
  d_twd = upload(twd);
  // secret key (NTT form over every prime)
  Runtime& rt = Runtime::get();
  d_sk = rt.alloc(size_t(np) * N);
  k_secret<<<grid_of(size_t(np) * N), kT, 0, rt.stream()>>>(dptr<uint64_t>(d_sk), dpc(), s.seed, s.h, np, s.logN);
  cuda_ok(cudaGetLastError(), "secret");
  ntt(*this, dptr<uint64_t>(d_sk), iota_rows(np), 1, 0, false);
  rt.sync();
}

void Ctx::make_key(uint64_t keyid, const uint64_t* sprime, Key* out) {
  Runtime& rt = Runtime::get();
  const size_t kw = size_t(spec.dnum) * np * N;
  out->b = rt.alloc(kw);
  out->a = rt.alloc(kw);
  DevBuf e = rt.alloc(size_t(np) * N);
  std::vector<uint64_t> Pm(np);
  for (uint32_t i = 0; i < np; ++i) {
    uint64_t v = 1;
    for (uint32_t k = 0; k < spec.K; ++k) v = h_mulmod(v, primes[nq + k] % primes[i], primes[i]);
    Pm[i] = v;
  }
  DevBuf dP = upload(Pm);
  const auto all = iota_rows(np);
  uint64_t* B = dptr<uint64_t>(out->b);
  uint64_t* A = dptr<uint64_t>(out->a);
  uint64_t* E = dptr<uint64_t>(e);
  for (uint32_t j = 0; j < spec.dnum; ++j) {
    uint64_t* aj = A + size_t(j) * np * N;
    uint64_t* bj = B + size_t(j) * np * N;
    k_key_ae<<<grid_of(size_t(np) * N), kT, 0, rt.stream()>>>(aj, E, dpc(), spec.seed, keyid, j, np, spec.logN);
    ntt(*this, E, all, 1, 0, false);
    k_key_b<<<grid_of(size_t(np) * N), kT, 0, rt.stream()>>>(bj, aj, E, dptr<const uint64_t>(d_sk), sprime, dpc(),
                                                             dptr<const uint64_t>(dP), j, alpha, nq, np, spec.logN);
    cuda_ok(cudaGetLastError(), "keygen");
  }
  rt.sync();
}

const Ctx::Key& Ctx::relin_key() {
  std::lock_guard<std::mutex> g(key_mu);
  if (!relin_) {
    Runtime& rt = Runtime::get();
    DevBuf s2 = rt.alloc(size_t(np) * N);
    k_square<<<grid_of(size_t(np) * N), kT, 0, rt.stream()>>>(dptr<uint64_t>(s2), dptr<const uint64_t>(d_sk), dpc(),
                                                              np, spec.logN);
    relin_ = std::make_unique<Key>();
    make_key(0, dptr<const uint64_t>(s2), relin_.get());
  }
  return *relin_;
}

const Ctx::Key& Ctx::galois_key(uint64_t g) {
  std::lock_guard<std::mutex> lk(key_mu);
  auto it = gal_.find(g);
  if (it != gal_.end()) return *it->second;
  Runtime& rt = Runtime::get();
  DevBuf sg = rt.alloc(size_t(np) * N);
  k_automorph<<<dim3(grid_of(size_t(np) * N), 1, 1), kT, 0, rt.stream()>>>(dptr<uint64_t>(sg),
                                                                          dptr<const uint64_t>(d_sk), g, spec.logN, np, 0);
  auto k = std::make_unique<Key>();
  make_key(1 + g, dptr<const uint64_t>(sg), k.get());
  return *gal_.emplace(g, std::move(k)).first->second;
}

// ================================================================== device ops
void encrypt_coeffs(const Ctx& c, uint32_t level, const int64_t* coeffs, uint64_t tag, uint64_t* out) {
  if (level > c.spec.L) fail(HS_E_INVALID_ARG, "rns encrypt: level > L");
  Runtime& rt = Runtime::get();
  const uint32_t nl = level + 1, logN = c.spec.logN;
  DevBuf dco = rt.alloc(c.N);
  cuda_ok(cudaMemcpyAsync(dco.get(), coeffs, size_t(c.N) * 8, cudaMemcpyHostToDevice, rt.stream()), "encrypt upload");
  k_enc_me<<<grid_of(size_t(nl) * c.N), kT, 0, rt.stream()>>>(dptr<const int64_t>(dco), out, c.dpc(), c.spec.seed, tag,
                                                              nl, logN);
  ntt(c, out, iota_rows(nl), 1, 0, false);
  k_enc_as<<<grid_of(size_t(nl) * c.N), kT, 0, rt.stream()>>>(out, dptr<const uint64_t>(c.d_sk), c.dpc(), nl, logN);
  cuda_ok(cudaGetLastError(), "encrypt");
  rt.note_launch(2);
  rt.sync();  // the host coefficient buffer may be released by the caller
}

void decrypt_coeffs(const Ctx& c, uint32_t level, const uint64_t* ct, int64_t* coeffs) {
  if (level > c.spec.L) fail(HS_E_INVALID_ARG, "rns decrypt: level > L");
  Runtime& rt = Runtime::get();
  DevBuf m = rt.alloc(c.N);
  k_dec0<<<grid_of(c.N), kT, 0, rt.stream()>>>(ct, dptr<const uint64_t>(c.d_sk), dptr<uint64_t>(m), c.dpc(),
                                               level + 1, c.spec.logN);
  ntt(c, dptr<uint64_t>(m), {0}, 1, 0, true);
  std::vector<uint64_t> h(c.N);
  cuda_ok(cudaMemcpyAsync(h.data(), m.get(), size_t(c.N) * 8, cudaMemcpyDeviceToHost, rt.stream()), "decrypt read");
  rt.sync();
  rt.note_launch();
  const uint64_t q = c.primes[0], half = q / 2;
  for (uint32_t n = 0; n < c.N; ++n)
    coeffs[n] = h[n] > half ? -static_cast<int64_t>(q - h[n]) : static_cast<int64_t>(h[n]);
}

void add_sub(const Ctx& c, uint32_t level, const uint64_t* a, const uint64_t* b, uint64_t* out, uint32_t batch,
             bool sub) {
  if (level > c.spec.L) fail(HS_E_INVALID_ARG, "rns add: level > L");
  Runtime& rt = Runtime::get();
  const size_t total = size_t(batch) * 2 * (level + 1) * c.N;
  k_addsub<<<grid_of(total), kT, 0, rt.stream()>>>(a, b, out, c.dpc(), level + 1, c.spec.logN, total, sub);
  cuda_ok(cudaGetLastError(), "add");
  rt.note_launch();
}

__int128 i128_of(double v) {
  if (!(std::fabs(v) < 8.5e37)) fail(HS_E_ERROR, "rns: encoded value out of the 127-bit range");
  const bool neg = v < 0;
  const double m = neg ? -v : v;
  const double two64 = 18446744073709551616.0;
  const double hi = std::floor(m / two64);
  const double lo = m - hi * two64;  // exact: m has 53 significant bits
  const unsigned __int128 r =
      (static_cast<unsigned __int128>(static_cast<uint64_t>(hi)) << 64) + static_cast<uint64_t>(lo);
  return neg ? -static_cast<__int128>(r) : static_cast<__int128>(r);
}

uint64_t residue(__int128 k, uint64_t q) {
  __int128 r = k % static_cast<__int128>(q);
  if (r < 0) r += q;
  return static_cast<uint64_t>(r);
}

// add_pt with a per-item constant (RnsB's batched BSGS leaves): out_b = a_b + k_b on poly 0
__global__ void k_addc_items(const uint64_t* a, const uint64_t* kt, uint64_t* out, const PrimeC* pcs, uint32_t nl,
                             uint32_t logN, size_t total) {
  const size_t per = size_t(2) * nl << logN;
  for (size_t x = blockIdx.x * size_t(blockDim.x) + threadIdx.x; x < total; x += size_t(gridDim.x) * blockDim.x) {
    const size_t b = x / per, w = x - b * per, r = w >> logN;
    const uint32_t i = r % nl;
    out[x] = r < nl ? add_mod(a[x], kt[b * nl + i], pcs[i].q) : a[x];
  }
}

void add_const_items(const Ctx& c, uint32_t level, const uint64_t* a, const std::vector<uint64_t>& kitems,
                     uint64_t* out, uint32_t batch) {
  if (level > c.spec.L) fail(HS_E_INVALID_ARG, "rns const op: level > L");
  const uint32_t nl = level + 1;
  if (kitems.size() < size_t(batch) * nl) fail(HS_E_INVALID_ARG, "rns add_const_items: item residues");
  Runtime& rt = Runtime::get();
  std::vector<uint64_t> tab(size_t(batch) * nl);
  for (uint32_t b = 0; b < batch; ++b)
    for (uint32_t i = 0; i < nl; ++i) tab[size_t(b) * nl + i] = kitems[size_t(b) * nl + i] % c.primes[i];
  DevBuf kdev = rt.alloc(tab.size());
  cuda_ok(cudaMemcpyAsync(kdev.get(), tab.data(), tab.size() * 8, cudaMemcpyHostToDevice, rt.stream()),
          "const items");
  const size_t total = size_t(batch) * 2 * nl * c.N;
  k_addc_items<<<grid_of(total), kT, 0, rt.stream()>>>(a, dptr<const uint64_t>(kdev), out, c.dpc(), nl, c.spec.logN,
                                                        total);
  cuda_ok(cudaGetLastError(), "const items");
  rt.note_launch();
}

void const_op_res(const Ctx& c, uint32_t level, const uint64_t* a, const std::vector<uint64_t>& res, uint64_t* out,
                  uint32_t batch, bool mul) {
  if (level > c.spec.L) fail(HS_E_INVALID_ARG, "rns const op: level > L");
  Runtime& rt = Runtime::get();
  const uint32_t nl = level + 1;
  ConstTab kt{};
  for (uint32_t i = 0; i < nl; ++i) {
    kt.k[i] = res[i];
    kt.ks[i] = shoup_of(res[i], c.primes[i]);
  }
  const size_t total = size_t(batch) * 2 * nl * c.N;
  k_constop<<<grid_of(total), kT, 0, rt.stream()>>>(a, kt, out, c.dpc(), nl, c.spec.logN, total, mul);
  cuda_ok(cudaGetLastError(), "const op");
  rt.note_launch();
}

void const_op(const Ctx& c, uint32_t level, const uint64_t* a, int64_t k, uint64_t* out, uint32_t batch, bool mul) {
  std::vector<uint64_t> res(level + 1);
  for (uint32_t i = 0; i <= level && i < c.primes.size(); ++i) res[i] = residue(k, c.primes[i]);
  const_op_res(c, level, a, res, out, batch, mul);
}

void residues_of(const Ctx& c, uint32_t level, double k, uint64_t* res) {
  const __int128 v = i128_of(std::nearbyint(k));
  for (uint32_t i = 0; i <= level && i < c.primes.size(); ++i) res[i] = residue(v, c.primes[i]);
}

void rescale_mul_big(Ctx& c, uint32_t level, const uint64_t* a, double k, uint64_t* out, uint32_t batch) {
  const __int128 v = i128_of(std::nearbyint(k));
  std::vector<uint64_t> res(level + 1);
  for (uint32_t i = 0; i <= level && i < c.primes.size(); ++i) res[i] = residue(v, c.primes[i]);
  rescale_mul(c, level, a, &res, out, batch);
}

void const_op_big(const Ctx& c, uint32_t level, const uint64_t* a, double k, uint64_t* out, uint32_t batch,
                  bool mul) {
  const __int128 v = i128_of(std::nearbyint(k));
  std::vector<uint64_t> res(level + 1);
  for (uint32_t i = 0; i <= level && i < c.primes.size(); ++i) res[i] = residue(v, c.primes[i]);
  const_op_res(c, level, a, res, out, batch, mul);
}

void encrypt_real_dev(const Ctx& c, uint32_t level, const double* dco, uint64_t tag, uint64_t* out) {
  if (level > c.spec.L) fail(HS_E_INVALID_ARG, "rns encrypt: level > L");
  Runtime& rt = Runtime::get();
  const uint32_t nl = level + 1, logN = c.spec.logN;
  k_residues<<<grid_of(size_t(nl) * c.N), kT, 0, rt.stream()>>>(dco, out, c.dpc(), nl, logN);
  k_enc_res<<<grid_of(size_t(nl) * c.N), kT, 0, rt.stream()>>>(out, c.dpc(), c.spec.seed, tag, nl, logN);
  ntt(c, out, iota_rows(nl), 1, 0, false);
  k_enc_as<<<grid_of(size_t(nl) * c.N), kT, 0, rt.stream()>>>(out, dptr<const uint64_t>(c.d_sk), c.dpc(), nl, logN);
  cuda_ok(cudaGetLastError(), "encrypt");
  rt.note_launch(3);
}

void encrypt_real(const Ctx& c, uint32_t level, const double* co, uint64_t tag, uint64_t* out) {
  Runtime& rt = Runtime::get();
  DevBuf d = rt.alloc(c.N);
  cuda_ok(cudaMemcpyAsync(d.get(), co, size_t(c.N) * 8, cudaMemcpyHostToDevice, rt.stream()), "encrypt upload");
  encrypt_real_dev(c, level, dptr<const double>(d), tag, out);
  rt.sync();  // the caller's coefficient buffer may be released on return
}

void mul_plain_real_dev(const Ctx& c, uint32_t level, const uint64_t* a, const double* dco, uint64_t* out) {
  Runtime& rt = Runtime::get();
  const uint32_t nl = level + 1, logN = c.spec.logN;
  DevBuf pt = rt.alloc(size_t(nl) * c.N);
  k_residues<<<grid_of(size_t(nl) * c.N), kT, 0, rt.stream()>>>(dco, dptr<uint64_t>(pt), c.dpc(), nl, logN);
  ntt(c, dptr<uint64_t>(pt), iota_rows(nl), 1, 0, false);
  k_mul_plain<<<grid_of(size_t(2) * nl * c.N), kT, 0, rt.stream()>>>(a, dptr<const uint64_t>(pt), out, c.dpc(), nl,
                                                                     logN);
  cuda_ok(cudaGetLastError(), "mul_plain");
  rt.note_launch(2);
}

void mul_plain_real(const Ctx& c, uint32_t level, const uint64_t* a, const double* co, uint64_t* out) {
  Runtime& rt = Runtime::get();
  DevBuf d = rt.alloc(c.N);
  cuda_ok(cudaMemcpyAsync(d.get(), co, size_t(c.N) * 8, cudaMemcpyHostToDevice, rt.stream()), "pt upload");
  mul_plain_real_dev(c, level, a, dptr<const double>(d), out);
  rt.sync();
}

void decrypt_crt_dev(const Ctx& c, uint32_t level, const uint64_t* ct, double* dco) {
  if (level > c.spec.L) fail(HS_E_INVALID_ARG, "rns decrypt: level > L");
  Runtime& rt = Runtime::get();
  const uint32_t nl = level + 1, use = level >= 1 ? 2 : 1;
  DevBuf m = rt.alloc(size_t(use) * c.N);
  k_dec<<<grid_of(size_t(use) * c.N), kT, 0, rt.stream()>>>(ct, dptr<const uint64_t>(c.d_sk), dptr<uint64_t>(m),
                                                             c.dpc(), nl, use, c.spec.logN);
  ntt(c, dptr<uint64_t>(m), iota_rows(use), 1, 0, true);
  uint64_t q0inv = 0, q0inv_sh = 0;
  if (use == 2) {
    q0inv = h_inv(c.primes[0] % c.primes[1], c.primes[1]);
    q0inv_sh = shoup_of(q0inv, c.primes[1]);
  }
  k_center<<<grid_of(c.N), kT, 0, rt.stream()>>>(dptr<const uint64_t>(m), dco, c.dpc(), q0inv, q0inv_sh, use,
                                                  c.spec.logN);
  cuda_ok(cudaGetLastError(), "decrypt");
  rt.note_launch(2);
}

void decrypt_crt(const Ctx& c, uint32_t level, const uint64_t* ct, double* coeffs) {
  Runtime& rt = Runtime::get();
  DevBuf d = rt.alloc(c.N);
  decrypt_crt_dev(c, level, ct, dptr<double>(d));
  cuda_ok(cudaMemcpyAsync(coeffs, d.get(), size_t(c.N) * 8, cudaMemcpyDeviceToHost, rt.stream()), "decrypt read");
  rt.sync();
}

void scale_round_dev(const Ctx& c, double* dco, double r) {
  Runtime& rt = Runtime::get();
  k_scale_round<<<grid_of(c.N), kT, 0, rt.stream()>>>(dco, r, c.N);
  cuda_ok(cudaGetLastError(), "refresh scale");
  rt.note_launch();
}

void random_ct(const Ctx& c, uint32_t level, uint64_t tag, uint64_t* out) {
  Runtime& rt = Runtime::get();
  k_random_ct<<<grid_of(size_t(2) * (level + 1) * c.N), kT, 0, rt.stream()>>>(out, c.dpc(), c.spec.seed, tag, level + 1,
                                                                             c.spec.logN);
  cuda_ok(cudaGetLastError(), "random_ct");
  rt.note_launch();
}

namespace {

void fill_conv(const Ctx& c, const std::vector<uint32_t>& src, const std::vector<uint32_t>& tgt_in,
               const std::vector<uint32_t>& tgt_row_in, uint32_t in_row, uint32_t out_row, ConvJob* cv) {
  std::memset(cv, 0, sizeof *cv);
  // targets >= 2^45 first (k_conv_tc's epilogue runs the two reductions as separate
  // branch-free loops); tgt_row keeps every output where it belongs
  std::vector<uint32_t> tgt, tgt_row;
  for (int pass = 0; pass < 2; ++pass)
    for (size_t t = 0; t < tgt_in.size(); ++t)
      if ((c.pc[tgt_in[t]].fp == 0) == (pass == 0)) {
        tgt.push_back(tgt_in[t]);
        tgt_row.push_back(tgt_row_in[t]);
        if (pass == 0) ++cv->nint;
      }
  cv->nsrc = static_cast<uint32_t>(src.size());
  cv->ntgt = static_cast<uint32_t>(tgt.size());
  cv->in_row = in_row;
  cv->out_row = out_row;
  for (size_t i = 0; i < src.size(); ++i) {
    const uint64_t qi = c.primes[src[i]];
    uint64_t v = 1;
    for (size_t m = 0; m < src.size(); ++m)
      if (m != i) v = h_mulmod(v, c.primes[src[m]] % qi, qi);
    cv->src[i] = static_cast<uint8_t>(src[i]);
    cv->hinv[i] = h_inv(v, qi);
    cv->hinv_sh[i] = shoup_of(cv->hinv[i], qi);
  }
  for (size_t t = 0; t < tgt.size(); ++t) {
    const uint64_t qt = c.primes[tgt[t]];
    cv->tgt[t] = static_cast<uint8_t>(tgt[t]);
    cv->tgt_row[t] = static_cast<uint8_t>(tgt_row[t]);
    for (size_t i = 0; i < src.size(); ++i) {
      uint64_t v = 1;
      for (size_t m = 0; m < src.size(); ++m)
        if (m != i) v = h_mulmod(v, c.primes[src[m]] % qt, qt);
      cv->h[t][i] = v;
    }
  }
}

// k_conv_mma's B operand for one job, in mma fragment order: [target][k-step][lane] ->
// (b0, b1) = bytes B[32 ks + 4 (lane & 3) + 0..3][lane >> 2] and the same at k + 16, where
// B[8i + a][b] = byte b of (h[t][i] 2^(8a) mod q_t).
uint32_t conv_ks(uint32_t nsrc) { return (nsrc + 3) / 4; }

void conv_frags(const Ctx& c, const ConvJob& J, std::vector<uint2>* f) {
  const uint32_t KS = conv_ks(J.nsrc), K = 32 * KS;
  std::vector<uint8_t> hb(size_t(8) * K);
  for (uint32_t t = 0; t < J.ntgt; ++t) {
    const uint64_t qt = c.primes[J.tgt[t]];
    std::fill(hb.begin(), hb.end(), 0);
    for (uint32_t i = 0; i < J.nsrc; ++i)
      for (uint32_t a = 0; a < 8; ++a) {
        const uint64_t v = h_mulmod(J.h[t][i] % qt, h_pow(2, 8 * a, qt), qt);
        for (uint32_t b = 0; b < 8; ++b) hb[size_t(b) * K + 8 * i + a] = static_cast<uint8_t>(v >> (8 * b));
      }
    for (uint32_t ks = 0; ks < KS; ++ks)
      for (uint32_t lane = 0; lane < 32; ++lane) {
        const uint8_t* col = hb.data() + size_t(lane >> 2) * K + 32 * ks + 4 * (lane & 3);
        auto pack = [](const uint8_t* p) {
          return uint32_t(p[0]) | uint32_t(p[1]) << 8 | uint32_t(p[2]) << 16 | uint32_t(p[3]) << 24;
        };
        f->push_back(make_uint2(pack(col), pack(col + 16)));
      }
  }
}

// k_conv_tc's B operand for one job: the shared-memory image [KC][NR][16] (K-major,
// SWIZZLE_NONE core matrices) of B[8t + b][8i + a] = byte b of (h[t][i] 2^(8a) mod q_t);
// chunk kc holds K bytes 16 kc .. 16 kc + 15 (sources 2 kc, 2 kc + 1), rows past 8 ntgt
// and sources past nsrc are zero.
void conv_tc_image(const Ctx& c, const ConvJob& J, std::vector<uint8_t>* img) {
  const uint32_t KC = 2 * conv_ks(J.nsrc), NR = tc_rows(J.ntgt);
  const size_t base = img->size();
  img->resize(base + size_t(KC) * NR * 16, 0);
  for (uint32_t t = 0; t < J.ntgt; ++t) {
    const uint64_t qt = c.primes[J.tgt[t]];
    for (uint32_t i = 0; i < J.nsrc; ++i)
      for (uint32_t a = 0; a < 8; ++a) {
        const uint64_t v = h_mulmod(J.h[t][i] % qt, h_pow(2, 8 * a, qt), qt);
        const uint32_t k = 8 * i + a, kc = k / 16, j = k % 16;
        for (uint32_t b = 0; b < 8; ++b)
          (*img)[base + (size_t(kc) * NR + 8 * t + b) * 16 + j] = static_cast<uint8_t>(v >> (8 * b));
      }
  }
}

void attach_frags(const Ctx& c, std::vector<ConvJob>* jobs, std::vector<uint2>* f, std::vector<uint8_t>* img) {
  for (ConvJob& J : *jobs) {
    J.frag_off = static_cast<uint32_t>(f->size());
    conv_frags(c, J, f);
    J.img_off = static_cast<uint32_t>(img->size());
    conv_tc_image(c, J, img);
  }
}

// Per-level plan: conversion jobs, NTT row lists and scalar tables (device resident).
struct KsPlan {
  uint32_t nl, nx, nd;
  std::vector<uint32_t> ext_primes;   // extended basis row -> prime
  DevBuf up_jobs;                     // ConvJob[nd]: digit j -> ext rows of block j
  uint32_t n_full = 0;                // digits [0, n_full) have alpha sources; the rest fewer
  std::vector<uint32_t> up_rows, up_primes;  // ext rows (j*nx + x) to NTT after ModUp
  DevBuf down_jobs;                   // ConvJob[2]: acc_w P rows -> conv rows w*nl..
  std::vector<uint32_t> p_rows, p_primes;    // acc P rows (both halves) for the iNTT
  std::vector<uint32_t> cv_rows, cv_primes;  // conv rows (both halves) for the NTT
  DevBuf frags;                       // k_conv_mma B fragments of every job above
  DevBuf tc_img;                      // k_conv_tc B images of every job above
  DevBuf pinv, pinv_sh;               // [nl] P^-1 mod q_i
  DevBuf qinv, qinv_sh;               // [level] q_level^-1 mod q_i (rescale)
  // ModDown by P q_level (HMult's rescale merged into the key switch), level >= 1:
  DevBuf rd_jobs;                      // ConvJob[2]: acc_w rows level..level+K -> conv rows w*level..
  std::vector<uint32_t> r_rows, r_primes;    // acc rows q_level + P (both halves) for the iNTT
  std::vector<uint32_t> cv2_rows, cv2_primes;  // conv rows (both halves, level limbs) for the NTT
  DevBuf pqinv, pqinv_sh;             // [level] (P q_level)^-1 mod q_i
  uint64_t pql = 0, pql_sh = 0;       // [P]_{q_level}
};

std::mutex g_plan_mu;
std::map<std::pair<const Ctx*, uint32_t>, std::unique_ptr<KsPlan>> g_plans;

std::unique_ptr<KsPlan> build_plan(const Ctx& c, uint32_t level) {
  auto p = std::make_unique<KsPlan>();
  const uint32_t nl = level + 1, K = c.spec.K;
  p->nl = nl;
  p->nx = nl + K;
  p->nd = (nl + c.alpha - 1) / c.alpha;
  for (uint32_t i = 0; i < nl; ++i) p->ext_primes.push_back(i);
  for (uint32_t k = 0; k < K; ++k) p->ext_primes.push_back(c.nq + k);
  std::vector<ConvJob> up(p->nd);
  for (uint32_t j = 0; j < p->nd; ++j) {
    const uint32_t lo = j * c.alpha, hi = std::min(lo + c.alpha, nl);
    if (hi - lo == c.alpha) p->n_full = j + 1;
    std::vector<uint32_t> src, tgt, row;
    for (uint32_t i = lo; i < hi; ++i) src.push_back(i);
    for (uint32_t x = 0; x < p->nx; ++x)
      if (x < lo || x >= hi) {
        tgt.push_back(p->ext_primes[x]);
        row.push_back(x);
        p->up_rows.push_back(j * p->nx + x);
        p->up_primes.push_back(p->ext_primes[x]);
      }
    fill_conv(c, src, tgt, row, lo, j * p->nx, &up[j]);
  }
  std::vector<uint2> frags;
  std::vector<uint8_t> img;
  attach_frags(c, &up, &frags, &img);
  std::vector<ConvJob> down(2);
  std::vector<uint32_t> src, tgt, row;
  for (uint32_t k = 0; k < K; ++k) src.push_back(c.nq + k);
  for (uint32_t i = 0; i < nl; ++i) {
    tgt.push_back(i);
    row.push_back(i);
  }
  for (uint32_t w = 0; w < 2; ++w) {
    fill_conv(c, src, tgt, row, w * p->nx + nl, w * nl, &down[w]);
    for (uint32_t k = 0; k < K; ++k) {
      p->p_rows.push_back(w * p->nx + nl + k);
      p->p_primes.push_back(c.nq + k);
    }
    for (uint32_t i = 0; i < nl; ++i) {
      p->cv_rows.push_back(w * nl + i);
      p->cv_primes.push_back(i);
    }
  }
  attach_frags(c, &down, &frags, &img);
  std::vector<ConvJob> rdown;
  if (level >= 1) {
    rdown.resize(2);
    std::vector<uint32_t> rsrc{level}, rtgt, rrow;
    for (uint32_t k = 0; k < K; ++k) rsrc.push_back(c.nq + k);
    for (uint32_t i = 0; i < level; ++i) {
      rtgt.push_back(i);
      rrow.push_back(i);
    }
    for (uint32_t w = 0; w < 2; ++w) {
      fill_conv(c, rsrc, rtgt, rrow, w * p->nx + level, w * level, &rdown[w]);
      for (uint32_t k = 0; k <= K; ++k) {
        p->r_rows.push_back(w * p->nx + level + k);
        p->r_primes.push_back(rsrc[k]);
      }
      for (uint32_t i = 0; i < level; ++i) {
        p->cv2_rows.push_back(w * level + i);
        p->cv2_primes.push_back(i);
      }
    }
    attach_frags(c, &rdown, &frags, &img);
    const uint64_t ql = c.primes[level];
    uint64_t v = 1;
    for (uint32_t k = 0; k < K; ++k) v = h_mulmod(v, c.primes[c.nq + k] % ql, ql);
    p->pql = v;
    p->pql_sh = shoup_of(v, ql);
    std::vector<uint64_t> pq(level), pq_sh(level);
    for (uint32_t i = 0; i < level; ++i) {
      const uint64_t q = c.primes[i];
      uint64_t u = ql % q;
      for (uint32_t k = 0; k < K; ++k) u = h_mulmod(u, c.primes[c.nq + k] % q, q);
      pq[i] = h_inv(u, q);
      pq_sh[i] = shoup_of(pq[i], q);
    }
    p->pqinv = upload(pq);
    p->pqinv_sh = upload(pq_sh);
    p->rd_jobs = upload(rdown);
  }
  p->up_jobs = upload(up);
  p->down_jobs = upload(down);
  p->frags = upload(frags);
  p->tc_img = upload(img);
  std::vector<uint64_t> pinv(nl), pinv_sh(nl);
  for (uint32_t i = 0; i < nl; ++i) {
    const uint64_t q = c.primes[i];
    uint64_t v = 1;
    for (uint32_t k = 0; k < K; ++k) v = h_mulmod(v, c.primes[c.nq + k] % q, q);
    pinv[i] = h_inv(v, q);
    pinv_sh[i] = shoup_of(pinv[i], q);
  }
  p->pinv = upload(pinv);
  p->pinv_sh = upload(pinv_sh);
  std::vector<uint64_t> qinv(std::max<uint32_t>(level, 1)), qinv_sh(std::max<uint32_t>(level, 1));
  for (uint32_t i = 0; i < level; ++i) {
    qinv[i] = h_inv(c.primes[level] % c.primes[i], c.primes[i]);
    qinv_sh[i] = shoup_of(qinv[i], c.primes[i]);
  }
  p->qinv = upload(qinv);
  p->qinv_sh = upload(qinv_sh);
  return p;
}

const KsPlan& ks_plan(const Ctx& c, uint32_t level) {
  std::lock_guard<std::mutex> g(g_plan_mu);
  auto key = std::make_pair(&c, level);
  auto it = g_plans.find(key);
  if (it != g_plans.end()) return *it->second;
  return *g_plans.emplace(key, build_plan(c, level)).first->second;
}

template <int A>
void launch_conv_a(const uint64_t* in, size_t in_stride, uint64_t* out, size_t out_stride, const ConvJob* jobs,
                   uint32_t njobs, const Ctx& c, uint32_t batch, cudaStream_t s) {
  const dim3 g((c.N + kT - 1) / kT, njobs, batch);
  k_conv<A><<<g, kT, 0, s>>>(in, in_stride, out, out_stride, jobs, c.dpc(), c.spec.logN);
}

// HS_KS_FUSION bit 0: rotate's automorphism inside the key switch (default on: 184 -> 176 us
// per ciphertext at N=2^16, L=24); bit 1: mul_relin's tensor product inside it (default off:
// the extra loads and products in the register-capped ModDown pass cost more than k_tensor).
bool use_ks_fusion(int mode_bit) {
  static const int mode = [] {
    const char* e = std::getenv("HS_KS_FUSION");
    return e ? std::atoi(e) : 1;
  }();
  return (mode & mode_bit) != 0;
}

// HS_CONV_MMA: 2 (default) = k_conv_tc (tcgen05.mma, accumulators in TMEM), 1 = k_conv_mma
// (legacy warp-level mma.sync IMMA, C parked in shared memory per target), 0 = the ALU/FP64
// k_conv
int use_conv_mma() {
  static const int mode = [] {
    const char* e = std::getenv("HS_CONV_MMA");
    return e ? std::atoi(e) : 2;
  }();
  return mode;
}

template <int KS>
void launch_conv_mma(const uint64_t* in, size_t in_stride, uint64_t* out, size_t out_stride, const ConvJob* jobs,
                     const uint2* frags, uint32_t njobs, uint32_t ntgt, const Ctx& c, uint32_t batch, cudaStream_t s) {
  static const bool attr = [] {
    cuda_ok(cudaFuncSetAttribute(k_conv_mma<KS>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(conv_mma_smem<KS>())),
            "conv_mma smem");
    return true;
  }();
  (void)attr;
  const dim3 g(c.N / kConvMmaRows, njobs, batch);
  (void)ntgt;
  k_conv_mma<KS><<<g, kConvMmaRows, conv_mma_smem<KS>(), s>>>(in, in_stride, out, out_stride, jobs, frags,
                                                                   c.dpc(), c.spec.logN);
}

// k_conv_tc: persistent, one CTA per SM (the dynamic shared memory request keeps a second
// CTA off the SM, so no CTA waits in tcgen05.alloc); the SMs are split evenly between the
// jobs of the call, each CTA taking a contiguous run of its job's (batch item, tile) pairs.
template <int KS>
void launch_conv_tc(const uint64_t* in, size_t in_stride, uint64_t* out, size_t out_stride, const ConvJob* jobs,
                    const uint8_t* img, uint32_t njobs, uint32_t ntgt, const Ctx& c, uint32_t batch, cudaStream_t s) {
  static const bool attr = [] {
    cuda_ok(cudaFuncSetAttribute(k_conv_tc<KS>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024),
            "conv_tc smem");
    return true;
  }();
  (void)attr;
  const uint32_t NR = tc_rows(ntgt);
  const size_t smem = std::max<size_t>(2 * tc_smem_a<KS>() + size_t(2 * KS) * NR * 16, 120 * 1024);
  const uint32_t ntiles = batch * (c.N / kTcRows);
  const uint32_t sms = static_cast<uint32_t>(Runtime::get().sm_count());
  const uint32_t want = std::max<uint32_t>(1, sms / njobs);
  const uint32_t per = (ntiles + want - 1) / want, nblk = (ntiles + per - 1) / per;
  k_conv_tc<KS><<<dim3(nblk, njobs), kTcThreads, smem, s>>>(in, in_stride, out, out_stride, jobs, img, c.dpc(),
                                                              c.spec.logN, ntiles, per);
}

// nsrc sources per job (all jobs of a call alike), ntgt targets at most per job.
void launch_conv(uint32_t nsrc, uint32_t ntgt, const uint64_t* in, size_t in_stride, uint64_t* out,
                 size_t out_stride, const ConvJob* jobs, const KsPlan& P, uint32_t njobs, const Ctx& c,
                 uint32_t batch) {
  if (njobs == 0) return;
  cudaStream_t s = Runtime::get().stream();
  const uint2* frags = dptr<const uint2>(P.frags);
  if (use_conv_mma() == 2 && conv_ks(nsrc) <= 4 && ntgt <= 64 && c.N % kTcRows == 0) {
    const uint8_t* img = reinterpret_cast<const uint8_t*>(P.tc_img.get());
    switch (conv_ks(nsrc)) {
      case 1: launch_conv_tc<1>(in, in_stride, out, out_stride, jobs, img, njobs, ntgt, c, batch, s); break;
      case 2: launch_conv_tc<2>(in, in_stride, out, out_stride, jobs, img, njobs, ntgt, c, batch, s); break;
      case 3: launch_conv_tc<3>(in, in_stride, out, out_stride, jobs, img, njobs, ntgt, c, batch, s); break;
      default: launch_conv_tc<4>(in, in_stride, out, out_stride, jobs, img, njobs, ntgt, c, batch, s);
    }
    cuda_ok(cudaGetLastError(), "conv_tc launch");
    Runtime::get().note_launch();
    return;
  }
  if (use_conv_mma() != 0 && conv_ks(nsrc) <= 4 && c.N % kConvMmaRows == 0) {
    switch (conv_ks(nsrc)) {
      case 1: launch_conv_mma<1>(in, in_stride, out, out_stride, jobs, frags, njobs, ntgt, c, batch, s); break;
      case 2: launch_conv_mma<2>(in, in_stride, out, out_stride, jobs, frags, njobs, ntgt, c, batch, s); break;
      case 3: launch_conv_mma<3>(in, in_stride, out, out_stride, jobs, frags, njobs, ntgt, c, batch, s); break;
      default: launch_conv_mma<4>(in, in_stride, out, out_stride, jobs, frags, njobs, ntgt, c, batch, s);
    }
    cuda_ok(cudaGetLastError(), "conv_mma launch");
    Runtime::get().note_launch();
    return;
  }
  switch (nsrc) {
#define HS_CONV_CASE(a) \
  case a:               \
    launch_conv_a<a>(in, in_stride, out, out_stride, jobs, njobs, c, batch, s); \
    break;
    HS_CONV_CASE(1) HS_CONV_CASE(2) HS_CONV_CASE(3) HS_CONV_CASE(4) HS_CONV_CASE(5) HS_CONV_CASE(6)
    HS_CONV_CASE(7) HS_CONV_CASE(8) HS_CONV_CASE(9) HS_CONV_CASE(10) HS_CONV_CASE(11) HS_CONV_CASE(12)
#undef HS_CONV_CASE
    default:
      launch_conv_a<0>(in, in_stride, out, out_stride, jobs, njobs, c, batch, s);
  }
  cuda_ok(cudaGetLastError(), "conv launch");
  Runtime::get().note_launch();
}

// Key-switch `batch` polynomials d ([nl][N] each, NTT form, stride d_stride) with key
// kk; out_w = ModDown(acc_w) + add_w  ([2][nl][N] per batch item, stride out_stride).
// With src (mode KS_TENSOR / KS_PERM), d and add_w are not materialised: the first
// iNTT pass computes d from src and the ModDown store adds add_w from src.
// acc_w[q_level row] += [P]_{q_level} add_w[q_level row] (NTT form): the P d_w term of
// ModDown by P q_level on the one removed Q prime (on the P primes, P d_w = 0).
__global__ void k_acc_fold(uint64_t* acc, size_t acc_stride, const uint64_t* add0, const uint64_t* add1,
                           size_t add_stride, uint32_t nx, uint32_t level, uint32_t logN, uint64_t v, uint64_t v_sh,
                           uint64_t q) {
  const uint32_t N = 1u << logN;
  const uint32_t n = blockIdx.x * blockDim.x + threadIdx.x, w = blockIdx.y;
  if (n >= N) return;
  uint64_t* a = acc + blockIdx.z * acc_stride + (size_t(w * nx + level) << logN) + n;
  const uint64_t* d = (w == 0 ? add0 : add1) + blockIdx.z * add_stride + (size_t(level) << logN) + n;
  *a = add_mod(*a, mul_shoup(*d, v, v_sh, q), q);
}

// rescale = true (mul_relin_rescale, add_w required): HMult's rescale merged into ModDown --
// out_w = (acc_w + P add_w - Conv_{P q_l -> Q_{l-1}}) (P q_l)^-1 over q_0..q_{l-1}, one
// conversion from K + 1 removed primes instead of ModDown's K plus the rescale's iNTT/NTT of
// every limb.  Matches oracle/rns_oracle.c moddown_rescale word for word.
void key_switch(Ctx& c, uint32_t level, const uint64_t* d, size_t d_stride, const Ctx::Key& kk, const uint64_t* add0,
                const uint64_t* add1, size_t add_stride, uint64_t* out, size_t out_stride, uint32_t batch,
                const KsSrc* src = nullptr, bool rescale = false) {
  Runtime& rt = Runtime::get();
  cudaStream_t s = rt.stream();
  const KsPlan& P = ks_plan(c, level);
  const uint32_t N = c.N, logN = c.spec.logN, nl = P.nl, nx = P.nx, nd = P.nd;
  const size_t dc_stride = size_t(nl) * N, ext_stride = size_t(nd) * nx * N, acc_stride = size_t(2) * nx * N,
               cv_stride = size_t(2) * nl * N;
  DevBuf dc = rt.alloc(size_t(batch) * dc_stride);
  DevBuf ext = rt.alloc(size_t(batch) * ext_stride);
  DevBuf acc = rt.alloc(size_t(batch) * acc_stride);
  DevBuf conv = rt.alloc(size_t(batch) * cv_stride);
  uint64_t* DC = dptr<uint64_t>(dc);
  uint64_t* EXT = dptr<uint64_t>(ext);
  uint64_t* ACC = dptr<uint64_t>(acc);
  uint64_t* CV = dptr<uint64_t>(conv);
  const auto qrows = iota_rows(nl);
  // ModUp: d -> coefficient form (out of place), convert every digit, NTT the new rows
  ntt_rows(c, d, d_stride, DC, dc_stride, qrows, qrows, qrows, batch, true, nullptr, nullptr, src);
  const ConvJob* up = dptr<const ConvJob>(P.up_jobs);
  launch_conv(c.alpha, nx - c.alpha, DC, dc_stride, EXT, ext_stride, up, P, P.n_full, c, batch);
  if (P.n_full < nd) {
    const uint32_t rest = nl - P.n_full * c.alpha;
    launch_conv(rest, nx - rest, DC, dc_stride, EXT, ext_stride, up + P.n_full, P, nd - P.n_full, c, batch);
  }
  const uint64_t *KB = dptr<const uint64_t>(kk.b), *KA = dptr<const uint64_t>(kk.a);
  ntt_rows(c, EXT, ext_stride, EXT, ext_stride, P.up_rows, P.up_rows, P.up_primes, batch, false);
  // inner product with the key (each key word read once per call)
  {
    const unsigned g = (unsigned)((size_t(nx) * N / 2 + kT - 1) / kT);  // two coefficients per thread
    const KsSrc ksrc = src ? *src : KsSrc{};
    switch (nd) {
#define HS_INNER_CASE(D)                                                                                          \
  case D:                                                                                                         \
    k_ks_inner<D><<<g, kT, 0, s>>>(EXT, ext_stride, d, d_stride, ACC, acc_stride, KB, KA, c.dpc(), nx, nl, c.np, \
                                   c.nq, c.alpha, logN, batch, ksrc);                                             \
    break;
      HS_INNER_CASE(1) HS_INNER_CASE(2) HS_INNER_CASE(3) HS_INNER_CASE(4) HS_INNER_CASE(5) HS_INNER_CASE(6)
      HS_INNER_CASE(7) HS_INNER_CASE(8) HS_INNER_CASE(9) HS_INNER_CASE(10) HS_INNER_CASE(11) HS_INNER_CASE(12)
      HS_INNER_CASE(13) HS_INNER_CASE(14) HS_INNER_CASE(15)
#undef HS_INNER_CASE
      default:
        fail(HS_E_INVALID_ARG, "key switch: more than 15 digits");
    }
  }
  if (rescale) {
    const uint32_t lv = level;
    k_acc_fold<<<dim3((N + kT - 1) / kT, 2, batch), kT, 0, s>>>(ACC, acc_stride, add0, add1, add_stride, nx, lv, logN,
                                                                 P.pql, P.pql_sh, c.primes[lv]);
    rt.note_launch();
    ntt_rows(c, ACC, acc_stride, ACC, acc_stride, P.r_rows, P.r_rows, P.r_primes, batch, true);
    launch_conv(c.spec.K + 1, lv, ACC, acc_stride, CV, cv_stride, dptr<const ConvJob>(P.rd_jobs), P, 2, c, batch);
    MdEpi epi{ACC, add0, add1, out, dptr<const uint64_t>(P.pqinv), dptr<const uint64_t>(P.pqinv_sh),
              acc_stride, add_stride, out_stride, lv, nx};
    epi.ascale = dptr<const uint64_t>(P.qinv);
    epi.ascale_sh = dptr<const uint64_t>(P.qinv_sh);
    ntt_rows(c, CV, cv_stride, CV, cv_stride, P.cv2_rows, P.cv2_rows, P.cv2_primes, batch, false, &epi);
    cuda_ok(cudaGetLastError(), "key switch (ModDown by P q_l)");
    return;
  }
  // ModDown: P rows -> coefficient form (in place), convert into Q_l, NTT, combine
  ntt_rows(c, ACC, acc_stride, ACC, acc_stride, P.p_rows, P.p_rows, P.p_primes, batch, true);
  launch_conv(c.spec.K, nl, ACC, acc_stride, CV, cv_stride, dptr<const ConvJob>(P.down_jobs), P, 2, c, batch);
  // NTT of the converted rows with the ModDown combine fused into its last pass:
  // out_w = (acc_w - conv_w) * P^-1 (+ add_w), conv_w never stored
  const MdEpi epi{ACC, add0, add1, out, dptr<const uint64_t>(P.pinv), dptr<const uint64_t>(P.pinv_sh),
                  acc_stride, add_stride, out_stride, nl, nx};
  ntt_rows(c, CV, cv_stride, CV, cv_stride, P.cv_rows, P.cv_rows, P.cv_primes, batch, false, &epi, nullptr, src);
  cuda_ok(cudaGetLastError(), "key switch");
}

}  // namespace

void mul_relin(Ctx& c, uint32_t level, const uint64_t* a, const uint64_t* b, uint64_t* out, uint32_t batch) {
  if (level > c.spec.L) fail(HS_E_INVALID_ARG, "rns mul_relin: level > L");
  if (batch == 0) return;
  Runtime& rt = Runtime::get();
  const uint32_t N = c.N, nl = level + 1;
  const size_t ct = size_t(2) * nl * N, half = size_t(nl) * N;
  const Ctx::Key& key = c.relin_key();
  if (use_ks_fusion(2)) {  // tensor product computed inside the key switch's first and last passes
    KsSrc src;
    src.mode = KS_TENSOR;
    src.a = a;
    src.b = b;
    src.stride = ct;
    src.nl = nl;
    key_switch(c, level, nullptr, 0, key, nullptr, nullptr, 0, out, ct, batch, &src);
    return;
  }
  DevBuf d = rt.alloc(size_t(batch) * 3 * half);
  uint64_t* D = dptr<uint64_t>(d);
  // layout per batch item: [d0 | d1 | d2], stride 3*half
  k_tensor<<<dim3(grid_of(half), 1, batch), kT, 0, rt.stream()>>>(a, b, D, c.dpc(), nl, c.spec.logN, ct, 3 * half,
                                                                   ct);
  rt.note_launch();
  key_switch(c, level, D + 2 * half, 3 * half, key, D, D + half, 3 * half, out, ct, batch);
}

// HS_MD_RESCALE (default 1): mul_relin_rescale merges the rescale into the key switch's
// ModDown (ModDown by P q_l); 0 = mul_relin followed by rescale.  The two give different
// limbs (one rounding instead of two); the oracle has both (rnso_mul_relin_rescale and
// rnso_rescale(rnso_mul_relin)).
static bool use_md_rescale() {
  static const int mode = [] {
    const char* e = std::getenv("HS_MD_RESCALE");
    return e ? std::atoi(e) : 1;
  }();
  return mode != 0;
}

void mul_relin_rescale(Ctx& c, uint32_t level, const uint64_t* a, const uint64_t* b, uint64_t* out, uint32_t batch,
                       bool b_shared) {
  if (level < 1 || level > c.spec.L) fail(HS_E_INVALID_ARG, "rns mul_relin_rescale: level must be in [1, L]");
  if (batch == 0) return;
  Runtime& rt = Runtime::get();
  if (b_shared || use_md_rescale()) {
    const uint32_t N = c.N, nl = level + 1;
    const size_t ct = size_t(2) * nl * N, half = size_t(nl) * N;
    DevBuf d = rt.alloc(size_t(batch) * 3 * half);
    uint64_t* D = dptr<uint64_t>(d);
    k_tensor<<<dim3(grid_of(half), 1, batch), kT, 0, rt.stream()>>>(a, b, D, c.dpc(), nl, c.spec.logN, ct, 3 * half,
                                                                     b_shared ? 0 : ct);
    rt.note_launch();
    key_switch(c, level, D + 2 * half, 3 * half, c.relin_key(), D, D + half, 3 * half, out, size_t(2) * level * N,
               batch, nullptr, true);
    return;
  }
  DevBuf t = rt.alloc(size_t(batch) * 2 * (level + 1) * c.N);
  mul_relin(c, level, a, b, dptr<uint64_t>(t), batch);
  rescale(c, level, dptr<const uint64_t>(t), out, batch);
}

void rescale(Ctx& c, uint32_t level, const uint64_t* in, uint64_t* out, uint32_t batch) {
  rescale_mul(c, level, in, nullptr, out, batch);
}

void rescale_mul(Ctx& c, uint32_t level, const uint64_t* in, const std::vector<uint64_t>* kres, uint64_t* out,
                 uint32_t batch) {
  rescale_mul_items(c, level, in, false, kres, nullptr, out, batch, nullptr);
}

// rescale(k_b * in_b) for every batch item b: kres = one constant for all items (or null = 1),
// kitems = per-item residues [batch][level + 1] (RnsB's batched BSGS leaves); shared_in: every
// item reads the same input ciphertext (its last limb goes to coefficient form once).
void rescale_mul_items(Ctx& c, uint32_t level, const uint64_t* in, bool shared_in, const std::vector<uint64_t>* kres,
                       const std::vector<uint64_t>* kitems, uint64_t* out, uint32_t batch,
                       const std::vector<uint64_t>* aitems) {
  if (level < 1 || level > c.spec.L) fail(HS_E_INVALID_ARG, "rns rescale: level must be in [1, L]");
  if (kres && (kres->size() < level + 1 || level + 1 > uint32_t(kRsMaxLimbs)))
    fail(HS_E_INVALID_ARG, "rns rescale_mul: constant residues");
  if (kitems && kitems->size() < size_t(batch) * (level + 1)) fail(HS_E_INVALID_ARG, "rns rescale_mul: item residues");
  if (batch == 0) return;
  Runtime& rt = Runtime::get();
  const uint32_t N = c.N, nl = level + 1;
  const size_t in_stride = shared_in ? 0 : size_t(2) * nl * N, out_stride = size_t(2) * level * N;
  const KsPlan& P = ks_plan(c, level);
  const uint32_t nlast = shared_in ? 1 : batch;
  DevBuf last = rt.alloc(size_t(nlast) * 2 * N);
  DevBuf t = rt.alloc(size_t(batch) * out_stride);
  uint64_t* LAST = dptr<uint64_t>(last);
  uint64_t* T = dptr<uint64_t>(t);
  DevBuf kdev;
  if (aitems && aitems->size() < size_t(batch) * level) fail(HS_E_INVALID_ARG, "rns rescale_mul: item addends");
  if (kitems || aitems) {  // [batch][2][nl]: residues then Shoup companions; then [batch][level] addends
    const size_t ka = kitems ? size_t(batch) * 2 * nl : 0;
    std::vector<uint64_t> tab(ka + (aitems ? size_t(batch) * level : 0));
    if (kitems)
      for (uint32_t b = 0; b < batch; ++b)
        for (uint32_t i = 0; i < nl; ++i) {
          const uint64_t v = (*kitems)[size_t(b) * nl + i] % c.primes[i];
          tab[size_t(b) * 2 * nl + i] = v;
          tab[size_t(b) * 2 * nl + nl + i] = shoup_of(v, c.primes[i]);
        }
    if (aitems)
      for (uint32_t b = 0; b < batch; ++b)
        for (uint32_t i = 0; i < level; ++i)
          tab[ka + size_t(b) * level + i] = (*aitems)[size_t(b) * level + i] % c.primes[i];
    kdev = rt.alloc(tab.size());
    cuda_ok(cudaMemcpyAsync(kdev.get(), tab.data(), tab.size() * 8, cudaMemcpyHostToDevice, rt.stream()),
            "rescale constants");
  }
  // last limb of both polys -> coefficient form (out of place)
  ntt_rows(c, in, size_t(2) * nl * N, LAST, size_t(2) * N, {level, nl + level}, {0, 1}, {level, level}, nlast, true);
  // NTT of [c_l]_{q_i} for every remaining limb: the spread is the column pass's load,
  // (c_i - t_i) q_l^-1 the row pass's store (t never materialised after the first pass)
  std::vector<uint32_t> rows(2 * level), primes(2 * level);
  for (uint32_t i = 0; i < 2 * level; ++i) {
    rows[i] = i;
    primes[i] = i % level;
  }
  RsEpi rse{LAST, in, out, dptr<const uint64_t>(P.qinv), dptr<const uint64_t>(P.qinv_sh),
            shared_in ? 0 : size_t(2) * N, in_stride, out_stride, level};
  if (aitems) rse.aitems = dptr<const uint64_t>(kdev) + (kitems ? size_t(batch) * 2 * nl : 0);
  if (kitems) {
    rse.kon = true;
    rse.kitems = dptr<const uint64_t>(kdev);
  } else if (kres) {
    rse.kon = true;
    for (uint32_t i = 0; i <= level; ++i) {
      rse.k[i] = (*kres)[i] % c.primes[i];
      rse.k_sh[i] = shoup_of(rse.k[i], c.primes[i]);
    }
  }
  ntt_rows(c, T, out_stride, T, out_stride, rows, rows, primes, batch, false, nullptr, &rse);
  cuda_ok(cudaGetLastError(), "rescale");
}

void rotate(Ctx& c, uint32_t level, int64_t k, const uint64_t* in, uint64_t* out, uint32_t batch) {
  if (level > c.spec.L) fail(HS_E_INVALID_ARG, "rns rotate: level > L");
  if (batch == 0) return;
  Runtime& rt = Runtime::get();
  const uint32_t N = c.N, nl = level + 1;
  const size_t ct = size_t(2) * nl * N;
  const uint64_t g = Ctx::galois_elt(k, c.spec.logN);
  const Ctx::Key& key = c.galois_key(g);
  if (use_ks_fusion(1)) {  // automorphism applied by the key switch's first-pass load and last-pass store
    KsSrc src;
    src.mode = KS_PERM;
    src.a = in;
    src.stride = ct;
    src.g = g;
    src.nl = nl;
    key_switch(c, level, nullptr, 0, key, nullptr, nullptr, 0, out, ct, batch, &src);
    return;
  }
  DevBuf perm = rt.alloc(size_t(batch) * ct);
  uint64_t* PM = dptr<uint64_t>(perm);
  k_automorph<<<dim3(grid_of(ct), 1, batch), kT, 0, rt.stream()>>>(PM, in, g, c.spec.logN, 2 * nl, ct);
  rt.note_launch();
  // out0 = sigma(c0) + ks0, out1 = ks1
  key_switch(c, level, PM + size_t(nl) * N, ct, key, PM, nullptr, ct, out, ct, batch);
}

void prepare_level(Ctx& c, uint32_t level) {
  if (level > c.spec.L) fail(HS_E_INVALID_ARG, "rns: level > L");
  ks_plan(c, level);
}

Ctx::~Ctx() {
  try {
    Runtime::get().sync();
  } catch (...) {
  }
  forget(*this);
}

void forget(const Ctx& c) {
  std::lock_guard<std::mutex> g(g_plan_mu);
  for (auto it = g_plans.begin(); it != g_plans.end();) it = it->first.first == &c ? g_plans.erase(it) : std::next(it);
}

}  // namespace rns
}  // namespace hsg
