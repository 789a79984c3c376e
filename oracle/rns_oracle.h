/* rns_oracle.h — TEST INFRASTRUCTURE ONLY.
 *
 * CPU oracle for the Tier-R RNS-CKKS evaluator kernels (NTT / iNTT, HMult with
 * relinearisation by hybrid key switching, rescale, Galois rotation + key
 * switch).  The reference (/root/reference) is a CKKS *emulator* with no RNS
 * limbs, keys or NTT, so limb-level parity against it is
 * UNPINNED; this builder-written oracle stands in for limb-exact self-parity of
 * the GPU kernels, and the algorithms follow the standard
 * RNS-CKKS literature (full-RNS HEAAN / hybrid key switching).  Every
 * deterministic input (primes, roots, keys, random ciphertexts) is derived from
 * the same counter-based hash on both sides, so GPU and oracle agree limb for
 * limb.  Plain C11 + unsigned __int128.
 */
#ifndef RNS_ORACLE_H
#define RNS_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define RNS_MAX_PRIMES 64

typedef struct {
  uint32_t logN;      /* N = 2^logN */
  uint32_t L;         /* ciphertext primes q_0..q_L (L+1 of them) */
  uint32_t K;         /* special primes p_0..p_{K-1} */
  uint32_t dnum;      /* key-switching digits; alpha = ceil((L+1)/dnum) primes per digit */
  uint32_t logq0, logq, logp;
  uint32_t h;         /* secret: 0 = dense ternary, else sparse with ~h nonzeros */
  uint64_t seed;
} rns_spec;

/* primes: q_0..q_L then p_0..p_{K-1} (L+1+K entries) */
int rnso_primes(const rns_spec* s, uint64_t* primes);
/* counter-based 64-bit hash (splitmix64 finaliser of a mixed counter) */
uint64_t rnso_hash(uint64_t seed, uint64_t domain, uint64_t a, uint64_t b);

/* negacyclic NTT of one limb (normal order in, bit-reversed out) and inverse */
void rnso_ntt(const rns_spec* s, uint32_t prime_idx, uint64_t* a);
void rnso_intt(const rns_spec* s, uint32_t prime_idx, uint64_t* a);

/* deterministic test ciphertext: 2 polys x (level+1) limbs, uniform residues,
 * layout [2][level+1][N] */
void rnso_random_ct(const rns_spec* s, uint32_t level, uint64_t tag, uint64_t* ct);

/* HMult + relinearisation (no rescale): a, b, out are [2][level+1][N] in NTT form */
void rnso_mul_relin(const rns_spec* s, uint32_t level, const uint64_t* a, const uint64_t* b, uint64_t* out);
/* the same for `count` consecutive ciphertext pairs, key generated once (CPU baseline timing) */
void rnso_mul_relin_many(const rns_spec* s, uint32_t level, uint32_t count, const uint64_t* a, const uint64_t* b,
                         uint64_t* out);
/* rescale by q_level: in [2][level+1][N] -> out [2][level][N], NTT form */
void rnso_rescale(const rns_spec* s, uint32_t level, const uint64_t* in, uint64_t* out);
/* HMult + relin + rescale, the rescale merged into ModDown (ModDown by P q_level): level limbs out */
void rnso_mul_relin_rescale(const rns_spec* s, uint32_t level, const uint64_t* a, const uint64_t* b, uint64_t* out);
/* rotation by k slots (Galois element 5^k mod 2N) + key switch, NTT form */
void rnso_rotate(const rns_spec* s, uint32_t level, int64_t k, const uint64_t* in, uint64_t* out);
/* symmetric RLWE encryption of N integer coefficients at `level`: c1 = a (uniform,
 * NTT form, stream D_ENC_A/tag), c0 = NTT(m + e) - a s (e: CBD, stream D_ENC_E/tag) */
void rnso_encrypt_coeffs(const rns_spec* s, uint32_t level, const int64_t* coeffs, uint64_t tag, uint64_t* ct);
/* decryption on q_0: centred c0 + c1 s (coefficient form) */
void rnso_decrypt_coeffs(const rns_spec* s, uint32_t level, const uint64_t* ct, int64_t* coeffs);
/* secret key (ternary) as residues over all L+1+K primes, NTT form: [L+1+K][N] */
void rnso_secret(const rns_spec* s, uint64_t* sk);

#ifdef __cplusplus
}
#endif
#endif
