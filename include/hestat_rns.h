/* hestat_rns.h — C ABI of the Tier-R RNS-CKKS kernels in libhestat_gpu.so.
 *
 * BASELINE.json north_star items (1)-(4): forward/inverse NTT, fused tensor
 * product + relinearisation key switching (ModUp, key inner product, ModDown),
 * rescale, and Galois rotation + key switch, over limb-major u64 RNS
 * polynomials resident in HBM.
 *
 * Reference boundary: the reference is a CKKS *emulator* — its
 * Evaluator ops (/root/reference/proj/include/hestat/ckks.hpp:149 mul_ct,
 * :193 rotate, and the implicit rescale inside q()) have no RNS limbs, so these
 * entry points have no reference counterpart to bind.  They are the limb-level
 * realisation of those ops (SURVEY.md §7 item 6, §8 "Tier-R realisation"
 * column) and are checked limb-for-limb against the CPU RNS oracle
 * (oracle/rns_oracle.c, tests/test_parity_rns.py).
 *
 * Layouts (all device pointers, u64 words):
 *   ciphertext at level l : [2][l+1][N], NTT form, limb i mod q_i;
 *   batch of B ciphertexts: B consecutive ciphertexts (stride 2(l+1)N words).
 * Primes: q_0 (logq0 bits), q_1..q_L (logq bits), p_0..p_{K-1} (logp bits).
 * Keys are derived on the device from spec.seed (same streams as the oracle)
 * the first time an op needs them, or ahead of time with hs_rns_prepare_*.
 * Status codes and hs_last_error() are those of hestat_gpu.h.
 */
#ifndef HESTAT_RNS_H
#define HESTAT_RNS_H

#include <stdint.h>

#include "hestat_gpu.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
  uint32_t logN, L, K, dnum; /* ring degree 2^logN; L+1 q-primes; K p-primes; dnum digits */
  uint32_t logq0, logq, logp;
  uint32_t h;                /* secret Hamming weight: 0 = dense ternary, else ~h nonzeros (sparse) */
  uint64_t seed;             /* secret/key/sample streams (rns_oracle.h) */
} hs_rns_spec;

typedef struct hs_rns hs_rns;

int hs_rns_create(const hs_rns_spec* spec, hs_rns** out);
int hs_rns_destroy(hs_rns* ctx);
int hs_rns_primes(const hs_rns* ctx, uint64_t* out, uint32_t cap); /* q_0..q_L, p_0..p_{K-1} */

/* device memory on the library stream */
int hs_rns_alloc(uint64_t words, uint64_t** dev);
int hs_rns_free(uint64_t* dev);
int hs_rns_upload(uint64_t* dev, const uint64_t* host, uint64_t words);
int hs_rns_download(uint64_t* host, const uint64_t* dev, uint64_t words);

/* key material (optional: ops generate their key on first use) */
int hs_rns_prepare_relin(hs_rns* ctx);
int hs_rns_prepare_rotation(hs_rns* ctx, int64_t k);
int hs_rns_secret(hs_rns* ctx, uint64_t* dev_out); /* [L+1+K][N] NTT form (tests) */

/* CKKS encoding (host, canonical embedding; slot j <-> zeta^(5^j), so hs_rns_rotate
 * by k is a left rotation of the slots by k, ckks.hpp:193-202):
 * n <= N/2 real values -> N coefficients round(scale * m_k), and back. */
int hs_rns_encode(uint32_t logN, const double* z, uint64_t n, double scale, int64_t* coeffs);
int hs_rns_decode(uint32_t logN, const int64_t* coeffs, double scale, double* z, uint64_t n);
/* the same transforms on the GPU (codec_gpu.cu; what RNS-backed EvalContexts use), host buffers
 * in and out, coefficients as integer-valued doubles; bit-identical to the host codec */
int hs_rns_encode_gpu(uint32_t logN, const double* z, uint64_t n, double scale, double* coeffs);
int hs_rns_decode_gpu(uint32_t logN, const double* coeffs, double scale, double* z, uint64_t n);
/* symmetric RLWE encryption at `level` (seeded by spec.seed and tag) of host
 * coefficients / of slot values; decryption through q_0 (|scale * value| < q_0/2) */
int hs_rns_encrypt_coeffs(hs_rns* ctx, uint32_t level, const int64_t* coeffs, uint64_t tag, uint64_t* dev_out);
int hs_rns_encrypt(hs_rns* ctx, uint32_t level, const double* z, uint64_t n, double scale, uint64_t tag,
                   uint64_t* dev_out);
int hs_rns_decrypt_coeffs(hs_rns* ctx, uint32_t level, const uint64_t* dev_ct, int64_t* coeffs);
int hs_rns_decrypt(hs_rns* ctx, uint32_t level, const uint64_t* dev_ct, double scale, double* z, uint64_t n);

/* ops; `batch` ciphertexts per call, consecutive in memory.  Device pointers are raw: a
 * ciphertext at level l is 2 (l+1) N words, so every input and output must cover
 * batch * 2 (l+1) N words (out of rescale / mul_relin_rescale: batch * 2 l N); the library does
 * not know the allocations behind the pointers (the Python binding, rns.py, checks its
 * DeviceBuffer sizes before every call).  Tier R is an evaluation / parity / benchmark engine:
 * keys and encryption randomness are a deterministic hash of spec.seed (so the device and the
 * oracle produce identical limbs) and hs_rns_secret exports the secret key for the tests. */
int hs_rns_random_ct(hs_rns* ctx, uint32_t level, uint64_t tag, uint64_t* dev_out);
/* in-place NTT (inverse != 0: iNTT) of `batch` groups of `nlimbs` limbs, limb i
 * of each group taken mod prime first_prime + i, groups `nlimbs*N` words apart */
int hs_rns_ntt(hs_rns* ctx, uint64_t* dev, uint32_t first_prime, uint32_t nlimbs, uint32_t batch, int inverse);
/* limb-wise ops (ckks.hpp add_ct/sub_ct :113-133; add_pt :137 with c = round(value * scale);
 * integer constant multiply, rescale separately for mul_pt :168) */
int hs_rns_add(hs_rns* ctx, uint32_t level, const uint64_t* a, const uint64_t* b, uint64_t* out, uint32_t batch);
int hs_rns_sub(hs_rns* ctx, uint32_t level, const uint64_t* a, const uint64_t* b, uint64_t* out, uint32_t batch);
int hs_rns_add_const(hs_rns* ctx, uint32_t level, const uint64_t* a, int64_t c, uint64_t* out, uint32_t batch);
int hs_rns_mul_const(hs_rns* ctx, uint32_t level, const uint64_t* a, int64_t c, uint64_t* out, uint32_t batch);
int hs_rns_mul_relin(hs_rns* ctx, uint32_t level, const uint64_t* a, const uint64_t* b, uint64_t* out,
                     uint32_t batch);
/* HMult + relin + rescale: out at level-1 ([2][level][N] per ciphertext) */
int hs_rns_mul_relin_rescale(hs_rns* ctx, uint32_t level, const uint64_t* a, const uint64_t* b, uint64_t* out,
                             uint32_t batch);
int hs_rns_rescale(hs_rns* ctx, uint32_t level, const uint64_t* in, uint64_t* out, uint32_t batch); /* out: level-1 */
/* rescale(c * in) in one pass pair, c * in never stored (RnsB's mul_pt and level alignment); replaces
   the reference evaluator's mul_pt + rescale (ckks.hpp:168-176 at the RNS level) */
int hs_rns_rescale_mul_const(hs_rns* ctx, uint32_t level, const uint64_t* in, int64_t c, uint64_t* out,
                             uint32_t batch);
int hs_rns_rotate(hs_rns* ctx, uint32_t level, int64_t k, const uint64_t* in, uint64_t* out, uint32_t batch);

/* ---- RNS-backed EvalContexts: the reference's operator surface on RNS-CKKS ----------
 * An hs_ctx created here (or by hs_ctx_create when the environment has HESTAT_BACKEND=rns)
 * runs every hestat_gpu.h entry point taking a context -- encrypt/decrypt, the EvalContext ops
 * (ckks.hpp:97-230), Chebyshev, the inverse-root primitives, columns and every statistic
 * (stats.hpp) -- on RNS-CKKS ciphertexts with the Tier-R kernels: the reference's control flow,
 * levels, CostMeter and errors unchanged, values encrypted under the context's keys (seeded by
 * rng_seed).  hs_ct handles it returns hold RNS ciphertexts; hs_ct_read (Ciphertext::slots())
 * decrypts them.  Handles from hs_ct_new (host slot vectors) are encrypted on first use.
 * spec = NULL derives the parameter set from the CkksParams (N = 2 slot_count, 61/60-bit primes,
 * dense ternary secret):
 *   HS_RNS_BOOT_REFRESH  bootstrap() (a level reset in the reference, ckks.hpp:207-213) refreshes
 *                        the ciphertext with the secret key (decrypt + re-encrypt at the top of the
 *                        chain); chain = max_level + 1 primes (logQP ~1150 bits at max_level 11,
 *                        inside the 128-bit budget at N = 2^16).  Trusted-refresh model.
 *   HS_RNS_BOOT_LOGICAL  bootstrap() resets only the logical level; the chain must cover the whole
 *                        DAG (HESTAT_RNS_DEPTH, default 28); no key material beyond the evaluation
 *                        keys is used during evaluation, but the chain exceeds the 128-bit budget.
 * Environment for hs_ctx_create: HESTAT_BACKEND=rns, HESTAT_RNS_BOOT=refresh|logical,
 * HESTAT_RNS_DEPTH=d. */
enum { HS_RNS_BOOT_REFRESH = 0, HS_RNS_BOOT_LOGICAL = 1 };
int hs_ctx_create_rns(const hs_params* p, uint64_t rng_seed, const hs_rns_spec* spec, int boot, hs_ctx** out);
int hs_ctx_backend(const hs_ctx* ctx);                                  /* 0 emulator (Tier E), 1 RNS */
int hs_ctx_rns_spec(const hs_ctx* ctx, hs_rns_spec* out, int* boot);    /* the RNS parameter set in use */
int hs_ct_backend(const hs_ct* ct);                                     /* 1: an RNS ciphertext */

/* ---- the reference's statistics over RNS ciphertexts -------------------------------
 * An EvalContext (hs_params: slot_count must be N/2) whose ops run on Tier-R
 * kernels: the reference's DAG (stats.hpp / primitives.hpp / chebyshev.hpp), level
 * ledger, CostMeter and errors, with bootstrap() a logical level reset over a deep
 * modulus chain (L >= the statistic's no-bootstrap depth).  Inputs are encrypted
 * (column.hpp:25-39 chunking), outputs decrypted: out receives the first out_n
 * slots of each result ciphertext (znorm: the n normalised values), out_levels
 * the results' logical levels. */
typedef struct hs_rns_eval hs_rns_eval;
enum {
  HS_RNS_INVSQRT = 0,   /* crypto_invsqrt(x, S = B)      primitives.hpp:186 */
  HS_RNS_MEAN = 1,      /* mean_scaled(x, B)             stats.hpp:97  */
  HS_RNS_VARIANCE = 2,  /* variance_scaled(x, B)         stats.hpp:130 */
  HS_RNS_MOMENTS = 3,   /* moments(x, B): mu, var        stats.hpp:138 */
  HS_RNS_ZNORM = 4,     /* znorm(x, B)                   stats.hpp:153 */
  HS_RNS_KURTOSIS = 5,  /* kurtosis(x, B)                stats.hpp:170 */
  HS_RNS_SKEWNESS = 6,  /* skewness(x, B)                stats.hpp:192 */
  HS_RNS_PEARSON = 7    /* pearson(x, y, B)              stats.hpp:239 */
};
int hs_rns_eval_create(hs_rns* ctx, const hs_params* p, hs_rns_eval** out);
int hs_rns_eval_destroy(hs_rns_eval* e);
int hs_rns_eval_meter(const hs_rns_eval* e, hs_meter* out);
int hs_rns_eval_set_meter(hs_rns_eval* e, const hs_meter* m);
int hs_rns_eval_stat(hs_rns_eval* e, int which, const double* x, uint64_t n, const double* y, uint64_t ny, double B,
                     const hs_invroot_cfg* cfg, double* out, uint64_t out_n, int32_t* out_levels);

#ifdef __cplusplus
}
#endif
#endif /* HESTAT_RNS_H */
