// rns.h — Tier R: RNS-CKKS evaluator on B200 (north_star items 1-4).
//
// Polynomials are limb-major u64 residues resident in HBM: a ciphertext at level
// l is [2][l+1][N].  Keys (relinearisation and Galois) are [dnum][L+1+K][N]
// pairs in NTT form over the full basis q_0..q_L, p_0..p_{K-1}.  Conventions
// (primes, roots, NTT ordering, deterministic key/ciphertext sampling, digit
// decomposition, ModUp / ModDown, rescale, Galois index map) are exactly those
// of oracle/rns_oracle.c, so every kernel is checked limb-for-limb against it
// (tests/test_parity_rns.py).
//
// Modular arithmetic (q < 2^62, 64-bit words):
//   * Shoup multiply-by-constant: w' = floor(w 2^64 / q); hi = mulhi(a, w');
//     r = a w - hi q in [0, 2q) for ANY a < 2^64 (so base-conversion inputs need
//     no pre-reduction);
//   * Barrett for two variable operands < q: k = bitlen(q), mu = floor(2^2k / q);
//   * lazy (Harvey) NTT butterflies keep values in [0, 4q) between stages and
//     canonicalise at the end.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <map>
#include <memory>
#include <mutex>
#include <vector>

#include "core.h"

namespace hsg {
namespace rns {

typedef unsigned __int128 u128;

struct Spec {
  uint32_t logN = 16, L = 24, K = 9, dnum = 3;
  uint32_t logq0 = 60, logq = 40, logp = 61;
  uint32_t h = 0;  // secret Hamming weight: 0 dense ternary, else sparse (~h nonzeros)
  uint64_t seed = 0;
};

// per-prime constants (device)
struct PrimeC {
  uint64_t q;
  uint64_t mu;       // Barrett floor(2^(2k)/q)
  uint64_t m64;      // floor(2^64 / q) (reduce64)
  uint64_t r64, r64_sh;  // 2^64 mod q and its Shoup constant (128-bit reduction)
  uint64_t ninv, ninv_sh;
  double qd, qinvd;  // q and 1/q in fp64 (FP64 NTT path)
  uint32_t k;        // bitlen(q)
  uint32_t fp;       // 1: q < 2^45, NTT on the FP64 pipe (rns.cu)
};

__host__ __device__ inline uint64_t shoup_of(uint64_t w, uint64_t q) {
  return static_cast<uint64_t>((static_cast<u128>(w) << 64) / q);
}

__device__ __forceinline__ uint64_t add_mod(uint64_t a, uint64_t b, uint64_t q) {
  const uint64_t r = a + b;
  return r >= q ? r - q : r;
}
__device__ __forceinline__ uint64_t sub_mod(uint64_t a, uint64_t b, uint64_t q) { return a >= b ? a - b : a + q - b; }
// a * w mod q in [0, 2q), any a < 2^64
__device__ __forceinline__ uint64_t mul_shoup_lazy(uint64_t a, uint64_t w, uint64_t wp, uint64_t q) {
  const uint64_t hi = __umul64hi(a, wp);
  return a * w - hi * q;
}
__device__ __forceinline__ uint64_t mul_shoup(uint64_t a, uint64_t w, uint64_t wp, uint64_t q) {
  const uint64_t r = mul_shoup_lazy(a, w, wp, q);
  return r >= q ? r - q : r;
}
// x mod q for any x < 2^64
__device__ __forceinline__ uint64_t reduce64(uint64_t x, const PrimeC& p) {
  const uint64_t r = x - __umul64hi(x, p.m64) * p.q;
  return r >= p.q ? r - p.q : r;
}
// a * b mod q for a, b < q (Barrett)
__device__ __forceinline__ uint64_t mul_mod(uint64_t a, uint64_t b, const PrimeC& p) {
  const u128 z = static_cast<u128>(a) * b;
  const uint64_t x = static_cast<uint64_t>(z >> (p.k - 1));
  const uint64_t qh = static_cast<uint64_t>((static_cast<u128>(x) * p.mu) >> (p.k + 1));
  uint64_t r = static_cast<uint64_t>(z) - qh * p.q;
  if (r >= p.q) r -= p.q;
  if (r >= p.q) r -= p.q;
  return r;
}

// x mod q for any x < 2^128: hi * (2^64 mod q) (Shoup) + lo (reduce64), one fold
__device__ __forceinline__ uint64_t reduce128(u128 x, const PrimeC& p) {
  const uint64_t hi = static_cast<uint64_t>(x >> 64), lo = static_cast<uint64_t>(x);
  uint64_t r = mul_shoup_lazy(hi, p.r64, p.r64_sh, p.q);  // [0, 2q)
  r += lo - __umul64hi(lo, p.m64) * p.q;                 // + [0, 2q)
  const uint64_t q2 = 2 * p.q;
  r = r >= q2 ? r - q2 : r;
  return r >= p.q ? r - p.q : r;
}

// ---- host context -------------------------------------------------------------------
class Ctx {
 public:
  explicit Ctx(const Spec& s);
  ~Ctx();  // drops this context's cached key-switching plans
  Ctx(const Ctx&) = delete;
  Ctx& operator=(const Ctx&) = delete;
  const Spec spec;
  uint32_t N, nq, np, alpha;
  std::vector<uint64_t> primes;   // q_0..q_L, p_0..p_{K-1}
  std::vector<PrimeC> pc;         // host copy
  DevBuf d_pc;                    // PrimeC[np] (reinterpreted)
  DevBuf d_tw;                    // [np][4][N]: psi_rev, psi_rev', ipsi_rev, ipsi_rev'
  DevBuf d_twd;                   // [np][2][N]: psi_rev, ipsi_rev as fp64 (primes < 2^45)
  DevBuf d_sk;                    // [np][N] secret, NTT form
  std::mutex key_mu;

  const PrimeC* dpc() const { return reinterpret_cast<const PrimeC*>(d_pc.get()); }
  const uint64_t* tw(uint32_t prime) const { return reinterpret_cast<const uint64_t*>(d_tw.get()) + size_t(prime) * 4 * N; }
  // keys (generated on first use, on device)
  struct Key {
    DevBuf b, a;  // [dnum][np][N]
  };
  const Key& relin_key();
  const Key& galois_key(uint64_t g);
  static uint64_t galois_elt(int64_t k, uint32_t logN);

 private:
  std::unique_ptr<Key> relin_;
  std::map<uint64_t, std::unique_ptr<Key>> gal_;
  void make_key(uint64_t keyid, const uint64_t* sprime, Key* out);
};

// ---- device ops (all on the library stream; pointers are device u64 arrays) --------------
// In-place NTT of `nlimbs` consecutive limbs (limb l uses prime prime_of[l]); `batch`
// groups of nlimbs limbs, group stride `gstride` words.  prime_of: host list.
void ntt(const Ctx& c, uint64_t* data, const std::vector<uint32_t>& prime_of, uint32_t batch, size_t gstride,
         bool inverse);
// Batched NTT over an explicit row list: row irows[i] of each input batch item
// (stride in_stride words) -> row orows[i] of the output item, mod primes[i].
// `epilogue` / `rescale_epi` (forward only, internal): the ModDown combine or the
// rescale spread/combine fused into the passes (rns.cu MdEpi, RsEpi).
void ntt_rows(const Ctx& c, const uint64_t* in, size_t in_stride, uint64_t* out, size_t out_stride,
              const std::vector<uint32_t>& irows, const std::vector<uint32_t>& orows,
              const std::vector<uint32_t>& primes, uint32_t batch, bool inverse, const void* epilogue = nullptr,
              const void* rescale_epi = nullptr, const void* ks_src = nullptr);
// Symmetric RLWE encryption of N integer coefficients (host array) at `level`
// (c1 = a, c0 = NTT(m + e) - a s; seeded by spec.seed and `tag`), and decryption
// to centred integers mod q_0 (valid while |m| < q_0 / 2).
void encrypt_coeffs(const Ctx& c, uint32_t level, const int64_t* coeffs, uint64_t tag, uint64_t* out);
void decrypt_coeffs(const Ctx& c, uint32_t level, const uint64_t* ct, int64_t* coeffs);
void random_ct(const Ctx& c, uint32_t level, uint64_t tag, uint64_t* out);
// Big-constant / real-valued variants used by the statistics backend (rns_eval.cu):
// integer-valued doubles up to 2^126 are reduced exactly through 128-bit integers.
void const_op_big(const Ctx& c, uint32_t level, const uint64_t* a, double k, uint64_t* out, uint32_t batch,
                  bool mul);
// encryption of / multiplication by a plaintext given as N integer-valued double
// coefficients (host), reduced into the RNS limbs on the device
void encrypt_real(const Ctx& c, uint32_t level, const double* co, uint64_t tag, uint64_t* out);
void mul_plain_real(const Ctx& c, uint32_t level, const uint64_t* a, const double* co, uint64_t* out);
// decryption through q_0 q_1 (CRT; q_0 alone at level 0): centred coefficients as doubles
void decrypt_crt(const Ctx& c, uint32_t level, const uint64_t* ct, double* coeffs);
// device-resident forms (dco: N device doubles; no host round trip, no synchronisation)
void decrypt_crt_dev(const Ctx& c, uint32_t level, const uint64_t* ct, double* dco);
void encrypt_real_dev(const Ctx& c, uint32_t level, const double* dco, uint64_t tag, uint64_t* out);
void mul_plain_real_dev(const Ctx& c, uint32_t level, const uint64_t* a, const double* dco, uint64_t* out);
void scale_round_dev(const Ctx& c, double* dco, double r);  // dco = rint(dco * r)
// CKKS canonical-embedding codec on the device (codec_gpu.cu; bit-identical to rns_codec.cpp):
// encode: item k of `batch` takes z[k N/2 .. min(n, (k+1) N/2)) (device) -> co + k N (device)
void encode_dev(uint32_t logN, const double* z, size_t n, double scale, double* co, uint32_t batch);
// decode: item k's N coefficients co + k N at `scale` -> its first n slots at z + k z_stride (device)
void decode_dev(uint32_t logN, const double* co, double scale, double* z, size_t n, size_t z_stride, uint32_t batch);
// out = a +- b (limb-wise), batch ciphertexts at `level`
void add_sub(const Ctx& c, uint32_t level, const uint64_t* a, const uint64_t* b, uint64_t* out, uint32_t batch,
             bool sub);
// out = a + c (constant polynomial, c0 only) or a * c (both polys); c a signed integer
void const_op(const Ctx& c, uint32_t level, const uint64_t* a, int64_t k, uint64_t* out, uint32_t batch, bool mul);
void mul_relin(Ctx& c, uint32_t level, const uint64_t* a, const uint64_t* b, uint64_t* out, uint32_t batch);
void rescale(Ctx& c, uint32_t level, const uint64_t* in, uint64_t* out, uint32_t batch);
// rescale(k * in) without materialising k * in (kres: residues of the integer k, limbs 0..level;
// null = 1); the words equal const_op(mul) followed by rescale
void rescale_mul(Ctx& c, uint32_t level, const uint64_t* in, const std::vector<uint64_t>* kres, uint64_t* out,
                 uint32_t batch);
// the same for k = nearbyint(kd), |kd| < 2^127
void rescale_mul_big(Ctx& c, uint32_t level, const uint64_t* a, double kd, uint64_t* out, uint32_t batch);
// per-item constants kitems [batch][level + 1] (or one constant kres); shared_in: all items read `in`;
// aitems [batch][level]: a per-item constant added to polynomial 0 of the result (a fused add_pt)
void rescale_mul_items(Ctx& c, uint32_t level, const uint64_t* in, bool shared_in, const std::vector<uint64_t>* kres,
                       const std::vector<uint64_t>* kitems, uint64_t* out, uint32_t batch,
                       const std::vector<uint64_t>* aitems = nullptr);
// out_b = a_b + k_b (k_b residues [batch][level + 1], added to poly 0)
void add_const_items(const Ctx& c, uint32_t level, const uint64_t* a, const std::vector<uint64_t>& kitems,
                     uint64_t* out, uint32_t batch);
// residues of the integer nearbyint(k), limbs 0..level
void residues_of(const Ctx& c, uint32_t level, double k, uint64_t* res);
// HMult + relinearisation + rescale (out at level - 1): the composition of the two ops.
// b_shared: every batch item multiplies by the same b (stride 0)
void mul_relin_rescale(Ctx& c, uint32_t level, const uint64_t* a, const uint64_t* b, uint64_t* out, uint32_t batch,
                       bool b_shared = false);
void rotate(Ctx& c, uint32_t level, int64_t k, const uint64_t* in, uint64_t* out, uint32_t batch);
// Build (and upload) the per-level key-switching / rescale constants ahead of time,
// so that ops can be captured into a CUDA graph.
void prepare_level(Ctx& c, uint32_t level);
// Drop every cached plan of this context (before destroying it).
void forget(const Ctx& c);

}  // namespace rns
}  // namespace hsg
