/* rns_oracle.c — TEST INFRASTRUCTURE ONLY (see rns_oracle.h).
 *
 * Plain-C restatement of the RNS-CKKS evaluator algorithms the GPU Tier-R
 * kernels implement.  Conventions (shared with paper_2508_12093_b200/csrc/rns*):
 *
 *   primes      q_0 (logq0 bits), q_1..q_L (logq bits), p_0..p_{K-1} (logp bits):
 *               the largest primes = 1 mod 2N below 2^bits, distinct, found by
 *               stepping down by 2N with deterministic Miller-Rabin.
 *   psi_i       x^((q-1)/2N) for the smallest x >= 2 with psi^N = -1 (mod q).
 *   NTT         negacyclic Cooley-Tukey, normal order in, bit-reversed out,
 *               twiddle psi^bitrev(m+i); inverse Gentleman-Sande + N^-1.
 *   hash        splitmix64 finaliser of seed ^ mixes of (domain, a, b).
 *   uniform     residue = (hash * q) >> 64.
 *   ternary s   h = 0: hash % 3 - 1 per coefficient; h > 0 (sparse): s_n = +-1 with
 *               probability h/N (hash(1, n) < h 2^64 / N), sign from hash(2, n) & 1;
 *               error e: centered binomial,
 *               popcount(h & 2^21-1) - popcount((h >> 21) & 2^21-1).
 *   digits      dnum digits of alpha = ceil((L+1)/dnum) consecutive q primes.
 *   key j       (b_j, a_j) over all L+1+K primes, NTT form:
 *               b_j = -a_j*s + e_j + g_j*s', g_j = [P]_{q_i} on digit j's primes,
 *               0 elsewhere (so sum_j ModUp(d_j) g_j = P d exactly).
 *   ModUp       fast base conversion of a digit's limbs (coefficient form).
 *   ModDown     (c - Conv_P->Q([c]_P)) * P^-1.
 *   rescale     (c_i - [c_l]_{q_i}) * q_l^-1, c_l taken in [0, q_l).
 *   rotate      Galois element 5^k mod 2N; NTT-domain index map (see below).
 */
#include "rns_oracle.h"

#include <stdlib.h>
#include <string.h>

typedef unsigned __int128 u128;

/* ---------------------------------------------------------------- arithmetic */
static uint64_t mulmod(uint64_t a, uint64_t b, uint64_t q) { return (uint64_t)(((u128)a * b) % q); }
static uint64_t addmod(uint64_t a, uint64_t b, uint64_t q) {
  uint64_t r = a + b;
  return r >= q ? r - q : r;
}
static uint64_t submod(uint64_t a, uint64_t b, uint64_t q) { return a >= b ? a - b : a + q - b; }
static uint64_t powmod(uint64_t a, uint64_t e, uint64_t q) {
  uint64_t r = 1 % q;
  a %= q;
  while (e) {
    if (e & 1) r = mulmod(r, a, q);
    a = mulmod(a, a, q);
    e >>= 1;
  }
  return r;
}
static uint64_t invmod(uint64_t a, uint64_t q) { return powmod(a, q - 2, q); } /* q prime */

static int is_prime(uint64_t n) {
  static const uint64_t bases[] = {2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37};
  if (n < 2) return 0;
  for (int i = 0; i < 12; ++i) {
    if (n == bases[i]) return 1;
    if (n % bases[i] == 0) return 0;
  }
  uint64_t d = n - 1;
  int r = 0;
  while ((d & 1) == 0) {
    d >>= 1;
    ++r;
  }
  for (int i = 0; i < 12; ++i) {
    uint64_t x = powmod(bases[i], d, n);
    if (x == 1 || x == n - 1) continue;
    int comp = 1;
    for (int j = 1; j < r; ++j) {
      x = mulmod(x, x, n);
      if (x == n - 1) {
        comp = 0;
        break;
      }
    }
    if (comp) return 0;
  }
  return 1;
}

uint64_t rnso_hash(uint64_t seed, uint64_t domain, uint64_t a, uint64_t b) {
  uint64_t z = seed ^ (domain * 0x9E3779B97F4A7C15ULL) ^ (a * 0xC2B2AE3D27D4EB4FULL) ^ (b * 0x165667B19E3779F9ULL);
  z += 0x9E3779B97F4A7C15ULL;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

enum { D_SECRET = 1, D_KEY_A = 2, D_KEY_E = 3, D_CT = 4, D_ENC_A = 5, D_ENC_E = 6 };

/* --------------------------------------------------------------------- primes */
int rnso_primes(const rns_spec* s, uint64_t* out) {
  const uint64_t twoN = 2ULL << s->logN;
  const uint32_t nq = s->L + 1, total = nq + s->K;
  if (total > RNS_MAX_PRIMES) return 1;
  uint32_t k = 0;
  const uint32_t bits[3] = {s->logq0, s->logq, s->logp};
  const uint32_t cnt[3] = {1, s->L, s->K};
  for (int g = 0; g < 3; ++g) {
    uint64_t c = ((1ULL << bits[g]) / twoN) * twoN + 1;
    if (c >= (1ULL << bits[g])) c -= twoN;
    for (uint32_t taken = 0; taken < cnt[g];) {
      if (c < twoN) return 2;
      int dup = 0;
      for (uint32_t i = 0; i < k; ++i) dup |= out[i] == c;
      if (!dup && is_prime(c)) {
        out[k++] = c;
        ++taken;
      }
      c -= twoN;
    }
  }
  return 0;
}

static uint64_t find_psi(uint64_t q, uint32_t logN) {
  const uint64_t N = 1ULL << logN;
  for (uint64_t x = 2;; ++x) {
    const uint64_t psi = powmod(x, (q - 1) / (2 * N), q);
    if (powmod(psi, N, q) == q - 1) return psi;
  }
}

static uint32_t bitrev(uint32_t x, uint32_t bits) {
  uint32_t r = 0;
  for (uint32_t i = 0; i < bits; ++i) r |= ((x >> i) & 1u) << (bits - 1 - i);
  return r;
}

/* ----------------------------------------------------------------------- NTT */
typedef struct {
  rns_spec s;
  uint64_t primes[RNS_MAX_PRIMES];
  uint64_t* psi_rev[RNS_MAX_PRIMES];
  uint64_t* ipsi_rev[RNS_MAX_PRIMES];
  uint64_t ninv[RNS_MAX_PRIMES];
} ctx_t;

static void ctx_init(ctx_t* c, const rns_spec* s) {
  memset(c, 0, sizeof *c);
  c->s = *s;
  rnso_primes(s, c->primes);
}
static void ctx_tables(ctx_t* c, uint32_t i) {
  if (c->psi_rev[i]) return;
  const uint32_t N = 1u << c->s.logN;
  const uint64_t q = c->primes[i];
  const uint64_t psi = find_psi(q, c->s.logN), ipsi = invmod(psi, q);
  c->psi_rev[i] = (uint64_t*)malloc(N * sizeof(uint64_t));
  c->ipsi_rev[i] = (uint64_t*)malloc(N * sizeof(uint64_t));
  for (uint32_t k = 0; k < N; ++k) {
    const uint32_t r = bitrev(k, c->s.logN);
    c->psi_rev[i][k] = powmod(psi, r, q);
    c->ipsi_rev[i][k] = powmod(ipsi, r, q);
  }
  c->ninv[i] = invmod(N, q);
}
static void ctx_free(ctx_t* c) {
  for (int i = 0; i < RNS_MAX_PRIMES; ++i) {
    free(c->psi_rev[i]);
    free(c->ipsi_rev[i]);
  }
}

static void ntt_fwd(ctx_t* c, uint32_t pi, uint64_t* a) {
  ctx_tables(c, pi);
  const uint32_t N = 1u << c->s.logN;
  const uint64_t q = c->primes[pi];
  uint32_t t = N;
  for (uint32_t m = 1; m < N; m <<= 1) {
    t >>= 1;
    for (uint32_t i = 0; i < m; ++i) {
      const uint32_t j1 = 2 * i * t;
      const uint64_t S = c->psi_rev[pi][m + i];
      for (uint32_t j = j1; j < j1 + t; ++j) {
        const uint64_t U = a[j], V = mulmod(a[j + t], S, q);
        a[j] = addmod(U, V, q);
        a[j + t] = submod(U, V, q);
      }
    }
  }
}

static void ntt_inv(ctx_t* c, uint32_t pi, uint64_t* a) {
  ctx_tables(c, pi);
  const uint32_t N = 1u << c->s.logN;
  const uint64_t q = c->primes[pi];
  uint32_t t = 1;
  for (uint32_t m = N; m > 1; m >>= 1) {
    const uint32_t h = m >> 1;
    uint32_t j1 = 0;
    for (uint32_t i = 0; i < h; ++i) {
      const uint64_t S = c->ipsi_rev[pi][h + i];
      for (uint32_t j = j1; j < j1 + t; ++j) {
        const uint64_t U = a[j], V = a[j + t];
        a[j] = addmod(U, V, q);
        a[j + t] = mulmod(submod(U, V, q), S, q);
      }
      j1 += 2 * t;
    }
    t <<= 1;
  }
  for (uint32_t j = 0; j < N; ++j) a[j] = mulmod(a[j], c->ninv[pi], q);
}

void rnso_ntt(const rns_spec* s, uint32_t pi, uint64_t* a) {
  ctx_t c;
  ctx_init(&c, s);
  ntt_fwd(&c, pi, a);
  ctx_free(&c);
}
void rnso_intt(const rns_spec* s, uint32_t pi, uint64_t* a) {
  ctx_t c;
  ctx_init(&c, s);
  ntt_inv(&c, pi, a);
  ctx_free(&c);
}

static uint64_t uniform(uint64_t h, uint64_t q) { return (uint64_t)(((u128)h * q) >> 64); }

void rnso_random_ct(const rns_spec* s, uint32_t level, uint64_t tag, uint64_t* ct) {
  uint64_t primes[RNS_MAX_PRIMES];
  rnso_primes(s, primes);
  const uint32_t N = 1u << s->logN;
  for (uint32_t p = 0; p < 2; ++p)
    for (uint32_t i = 0; i <= level; ++i)
      for (uint32_t n = 0; n < N; ++n)
        ct[((size_t)p * (level + 1) + i) * N + n] =
            uniform(rnso_hash(s->seed, D_CT, tag * 1024 + p * 64 + i, n), primes[i]);
}

/* ------------------------------------------------------------------ keys */
static int64_t ternary(const rns_spec* s, uint32_t n) {
  if (s->h == 0) return (int64_t)(rnso_hash(s->seed, D_SECRET, 0, n) % 3) - 1;
  const uint64_t thr = (uint64_t)s->h << (64 - s->logN);
  if (rnso_hash(s->seed, D_SECRET, 1, n) >= thr) return 0;
  return (rnso_hash(s->seed, D_SECRET, 2, n) & 1) ? -1 : 1;
}
static int64_t cbd(uint64_t h) {
  return (int64_t)__builtin_popcountll(h & 0x1FFFFFULL) - (int64_t)__builtin_popcountll((h >> 21) & 0x1FFFFFULL);
}
static uint64_t lift(int64_t v, uint64_t q) { return v >= 0 ? (uint64_t)v % q : q - ((uint64_t)(-v) % q); }

/* secret key over every prime, NTT form, [nprimes][N] */
static void secret_ntt(ctx_t* c, uint64_t* sk) {
  const uint32_t N = 1u << c->s.logN, np = c->s.L + 1 + c->s.K;
  for (uint32_t i = 0; i < np; ++i) {
    for (uint32_t n = 0; n < N; ++n) sk[(size_t)i * N + n] = lift(ternary(&c->s, n), c->primes[i]);
    ntt_fwd(c, i, sk + (size_t)i * N);
  }
}

void rnso_secret(const rns_spec* s, uint64_t* sk) {
  ctx_t c;
  ctx_init(&c, s);
  secret_ntt(&c, sk);
  ctx_free(&c);
}

static uint32_t alpha_of(const rns_spec* s) { return (s->L + 1 + s->dnum - 1) / s->dnum; }

/* NTT-domain automorphism index map for Galois element g (bit-reversed order) */
static uint32_t galois_src(uint32_t j, uint64_t g, uint32_t logN) {
  const uint64_t twoN = 2ULL << logN;
  const uint64_t e = (2ULL * bitrev(j, logN) + 1) * g % twoN;
  return bitrev((uint32_t)((e - 1) / 2), logN);
}
static uint64_t galois_elt(int64_t k, uint32_t logN) {
  const uint64_t twoN = 2ULL << logN, half = 1ULL << (logN - 1);
  int64_t kk = k % (int64_t)half;
  if (kk < 0) kk += (int64_t)half;
  uint64_t g = 1;
  for (int64_t i = 0; i < kk; ++i) g = g * 5 % twoN;
  return g;
}

/* key for s' (NTT form over all primes): key id selects the randomness stream */
static void make_key(ctx_t* c, uint64_t keyid, const uint64_t* s_ntt, const uint64_t* sprime_ntt, uint64_t* kb,
                     uint64_t* ka) {
  const uint32_t N = 1u << c->s.logN, nq = c->s.L + 1, np = nq + c->s.K, al = alpha_of(&c->s);
  uint64_t P[RNS_MAX_PRIMES];
  for (uint32_t i = 0; i < np; ++i) {
    uint64_t pm = 1;
    for (uint32_t k = 0; k < c->s.K; ++k) pm = mulmod(pm, c->primes[nq + k] % c->primes[i], c->primes[i]);
    P[i] = pm;
  }
  uint64_t* e = (uint64_t*)malloc((size_t)N * sizeof(uint64_t));
  for (uint32_t j = 0; j < c->s.dnum; ++j) {
    for (uint32_t i = 0; i < np; ++i) {
      const uint64_t q = c->primes[i];
      uint64_t* a = ka + ((size_t)j * np + i) * N;
      uint64_t* b = kb + ((size_t)j * np + i) * N;
      for (uint32_t n = 0; n < N; ++n) a[n] = uniform(rnso_hash(c->s.seed, D_KEY_A, keyid * 4096 + j * 64 + i, n), q);
      for (uint32_t n = 0; n < N; ++n) e[n] = lift(cbd(rnso_hash(c->s.seed, D_KEY_E, keyid * 4096 + j, n)), q);
      ntt_fwd(c, i, e);
      const int in_digit = i < nq && i / al == j;
      for (uint32_t n = 0; n < N; ++n) {
        uint64_t v = submod(e[n], mulmod(a[n], s_ntt[(size_t)i * N + n], q), q);
        if (in_digit) v = addmod(v, mulmod(P[i], sprime_ntt[(size_t)i * N + n], q), q);
        b[n] = v;
      }
    }
  }
  free(e);
}

/* ------------------------------------------------------------ key switching */
/* d: [level+1][N] NTT form.  out0/out1: [level+1][N] NTT form. */
static void moddown_rescale(ctx_t* c, uint32_t level, uint64_t* acc, const uint64_t* dt, uint64_t* out);

/* Hybrid key switching of d (NTT form, level+1 limbs).  dterm == NULL: out_w = ModDown_P(acc_w)
   (level+1 limbs).  dterm = {d0, d1}: HMult's rescale fused into ModDown, out_w =
   ModDown_{P q_level}(acc_w + P d_w) (level limbs), see moddown_rescale. */
static void key_switch_x(ctx_t* c, uint32_t level, const uint64_t* d, const uint64_t* kb, const uint64_t* ka,
                         uint64_t* out0, uint64_t* out1, const uint64_t* const* dterm) {
  const uint32_t N = 1u << c->s.logN, nq = c->s.L + 1, K = c->s.K, np = nq + K, al = alpha_of(&c->s);
  const uint32_t nl = level + 1, nx = nl + K; /* extended basis: q_0..q_level, p_0..p_{K-1} */
  uint32_t idx[RNS_MAX_PRIMES];              /* extended index -> global prime index */
  for (uint32_t i = 0; i < nl; ++i) idx[i] = i;
  for (uint32_t k = 0; k < K; ++k) idx[nl + k] = nq + k;

  uint64_t* dc = (uint64_t*)malloc((size_t)nl * N * sizeof(uint64_t)); /* d in coefficient form */
  memcpy(dc, d, (size_t)nl * N * sizeof(uint64_t));
  for (uint32_t i = 0; i < nl; ++i) ntt_inv(c, i, dc + (size_t)i * N);
  uint64_t* ext = (uint64_t*)malloc((size_t)nx * N * sizeof(uint64_t));
  uint64_t* acc0 = (uint64_t*)calloc((size_t)nx * N, sizeof(uint64_t));
  uint64_t* acc1 = (uint64_t*)calloc((size_t)nx * N, sizeof(uint64_t));
  const uint32_t ndig = (nl + al - 1) / al;
  for (uint32_t j = 0; j < ndig; ++j) {
    const uint32_t lo = j * al, hi = (lo + al < nl) ? lo + al : nl; /* digit primes [lo, hi) */
    /* ModUp: fast base conversion of the digit to every other extended prime */
    uint64_t qhat_inv[RNS_MAX_PRIMES];
    for (uint32_t i = lo; i < hi; ++i) {
      uint64_t v = 1;
      for (uint32_t m = lo; m < hi; ++m)
        if (m != i) v = mulmod(v, c->primes[m] % c->primes[i], c->primes[i]);
      qhat_inv[i] = invmod(v, c->primes[i]);
    }
    for (uint32_t x = 0; x < nx; ++x) {
      const uint32_t gi = idx[x];
      const uint64_t t = c->primes[gi];
      uint64_t* dst = ext + (size_t)x * N;
      if (x >= lo && x < hi) {
        memcpy(dst, d + (size_t)x * N, N * sizeof(uint64_t)); /* own limb: already NTT form */
        continue;
      }
      uint64_t qhat_t[RNS_MAX_PRIMES];
      for (uint32_t i = lo; i < hi; ++i) {
        uint64_t v = 1;
        for (uint32_t m = lo; m < hi; ++m)
          if (m != i) v = mulmod(v, c->primes[m] % t, t);
        qhat_t[i] = v;
      }
      for (uint32_t n = 0; n < N; ++n) {
        uint64_t sum = 0;
        for (uint32_t i = lo; i < hi; ++i) {
          const uint64_t xi = mulmod(dc[(size_t)i * N + n], qhat_inv[i], c->primes[i]);
          sum = addmod(sum, mulmod(xi % t, qhat_t[i], t), t);
        }
        dst[n] = sum;
      }
      ntt_fwd(c, gi, dst);
    }
    /* inner product with key digit j (restricted to the extended basis) */
    for (uint32_t x = 0; x < nx; ++x) {
      const uint32_t gi = idx[x];
      const uint64_t t = c->primes[gi];
      const uint64_t* b = kb + ((size_t)j * np + gi) * N;
      const uint64_t* a = ka + ((size_t)j * np + gi) * N;
      for (uint32_t n = 0; n < N; ++n) {
        const uint64_t e = ext[(size_t)x * N + n];
        acc0[(size_t)x * N + n] = addmod(acc0[(size_t)x * N + n], mulmod(e, b[n], t), t);
        acc1[(size_t)x * N + n] = addmod(acc1[(size_t)x * N + n], mulmod(e, a[n], t), t);
      }
    }
  }
  if (dterm) {
    moddown_rescale(c, level, acc0, dterm[0], out0);
    moddown_rescale(c, level, acc1, dterm[1], out1);
    free(dc);
    free(ext);
    free(acc0);
    free(acc1);
    return;
  }
  /* ModDown: (acc - Conv_P->Q(acc_P)) * P^-1 on q_0..q_level */
  uint64_t phat_inv[RNS_MAX_PRIMES];
  for (uint32_t k = 0; k < K; ++k) {
    const uint64_t pk = c->primes[nq + k];
    uint64_t v = 1;
    for (uint32_t m = 0; m < K; ++m)
      if (m != k) v = mulmod(v, c->primes[nq + m] % pk, pk);
    phat_inv[k] = invmod(v, pk);
  }
  uint64_t* pc = (uint64_t*)malloc((size_t)K * N * sizeof(uint64_t));
  uint64_t* conv = (uint64_t*)malloc((size_t)N * sizeof(uint64_t));
  for (int w = 0; w < 2; ++w) {
    uint64_t* acc = w ? acc1 : acc0;
    uint64_t* out = w ? out1 : out0;
    for (uint32_t k = 0; k < K; ++k) {
      memcpy(pc + (size_t)k * N, acc + (size_t)(nl + k) * N, N * sizeof(uint64_t));
      ntt_inv(c, nq + k, pc + (size_t)k * N);
    }
    for (uint32_t i = 0; i < nl; ++i) {
      const uint64_t q = c->primes[i];
      uint64_t phat_q[RNS_MAX_PRIMES], pinv = 1;
      for (uint32_t k = 0; k < K; ++k) {
        uint64_t v = 1;
        for (uint32_t m = 0; m < K; ++m)
          if (m != k) v = mulmod(v, c->primes[nq + m] % q, q);
        phat_q[k] = v;
        pinv = mulmod(pinv, c->primes[nq + k] % q, q);
      }
      pinv = invmod(pinv, q);
      for (uint32_t n = 0; n < N; ++n) {
        uint64_t sum = 0;
        for (uint32_t k = 0; k < K; ++k) {
          const uint64_t pk = c->primes[nq + k];
          const uint64_t xk = mulmod(pc[(size_t)k * N + n], phat_inv[k], pk);
          sum = addmod(sum, mulmod(xk % q, phat_q[k], q), q);
        }
        conv[n] = sum;
      }
      ntt_fwd(c, i, conv);
      for (uint32_t n = 0; n < N; ++n)
        out[(size_t)i * N + n] = mulmod(submod(acc[(size_t)i * N + n], conv[n], q), pinv, q);
    }
  }
  free(pc);
  free(conv);
  free(dc);
  free(ext);
  free(acc0);
  free(acc1);
}

static void key_switch(ctx_t* c, uint32_t level, const uint64_t* d, const uint64_t* kb, const uint64_t* ka,
                       uint64_t* out0, uint64_t* out1) {
  key_switch_x(c, level, d, kb, ka, out0, out1, NULL);
}

/* ModDown by P q_level with HMult's tensor term folded in (the rescale of HMult+relin+rescale
   merged into the key switch's ModDown): x = acc + P d over q_0..q_level (x = acc on the P
   primes); the removed primes R = {q_level, p_0..p_{K-1}} go to coefficient form, are converted
   to q_0..q_{level-1} (fast base conversion), and out_i = (x_i - conv_i) (P q_level)^-1.  One
   rounding instead of ModDown's and the rescale's: the limbs differ from mul_relin followed by
   rescale, the decrypted value is the same up to the (smaller) rounding error. */
static void moddown_rescale(ctx_t* c, uint32_t level, uint64_t* acc, const uint64_t* dt, uint64_t* out) {
  const uint32_t N = 1u << c->s.logN, nq = c->s.L + 1, K = c->s.K, nl = level + 1, nr = K + 1;
  uint32_t ridx[RNS_MAX_PRIMES]; /* removed primes, as acc rows level .. level + K */
  ridx[0] = level;
  for (uint32_t k = 0; k < K; ++k) ridx[1 + k] = nq + k;
  uint64_t Pql = 1; /* [P]_{q_level} */
  for (uint32_t k = 0; k < K; ++k) Pql = mulmod(Pql, c->primes[nq + k] % c->primes[level], c->primes[level]);
  uint64_t* rc = (uint64_t*)malloc((size_t)nr * N * sizeof(uint64_t));
  uint64_t* conv = (uint64_t*)malloc((size_t)N * sizeof(uint64_t));
  for (uint32_t r = 0; r < nr; ++r) {
    const uint64_t* src = acc + (size_t)(r == 0 ? level : nl + r - 1) * N;
    uint64_t* dst = rc + (size_t)r * N;
    for (uint32_t n = 0; n < N; ++n)
      dst[n] = r == 0 ? addmod(src[n], mulmod(dt[(size_t)level * N + n], Pql, c->primes[level]), c->primes[level])
                      : src[n];
    ntt_inv(c, ridx[r], dst);
  }
  uint64_t rhat_inv[RNS_MAX_PRIMES];
  for (uint32_t r = 0; r < nr; ++r) {
    const uint64_t pr = c->primes[ridx[r]];
    uint64_t v = 1;
    for (uint32_t m = 0; m < nr; ++m)
      if (m != r) v = mulmod(v, c->primes[ridx[m]] % pr, pr);
    rhat_inv[r] = invmod(v, pr);
  }
  for (uint32_t i = 0; i < level; ++i) {
    const uint64_t q = c->primes[i];
    uint64_t rhat_q[RNS_MAX_PRIMES], Rq = 1, Pq = 1;
    for (uint32_t r = 0; r < nr; ++r) {
      uint64_t v = 1;
      for (uint32_t m = 0; m < nr; ++m)
        if (m != r) v = mulmod(v, c->primes[ridx[m]] % q, q);
      rhat_q[r] = v;
      Rq = mulmod(Rq, c->primes[ridx[r]] % q, q);
    }
    for (uint32_t k = 0; k < K; ++k) Pq = mulmod(Pq, c->primes[nq + k] % q, q);
    const uint64_t rinv = invmod(Rq, q);
    for (uint32_t n = 0; n < N; ++n) {
      uint64_t sum = 0;
      for (uint32_t r = 0; r < nr; ++r) {
        const uint64_t pr = c->primes[ridx[r]];
        const uint64_t xr = mulmod(rc[(size_t)r * N + n], rhat_inv[r], pr);
        sum = addmod(sum, mulmod(xr % q, rhat_q[r], q), q);
      }
      conv[n] = sum;
    }
    ntt_fwd(c, i, conv);
    for (uint32_t n = 0; n < N; ++n) {
      const size_t x = (size_t)i * N + n;
      const uint64_t xi = addmod(acc[x], mulmod(dt[x], Pq, q), q);
      out[x] = mulmod(submod(xi, conv[n], q), rinv, q);
    }
  }
  free(rc);
  free(conv);
}

static size_t key_words(const ctx_t* c) {
  return (size_t)c->s.dnum * (c->s.L + 1 + c->s.K) * ((size_t)1 << c->s.logN);
}

void rnso_mul_relin_many(const rns_spec* s, uint32_t level, uint32_t count, const uint64_t* a, const uint64_t* b,
                         uint64_t* out) {
  ctx_t c;
  ctx_init(&c, s);
  const uint32_t N = 1u << s->logN, nl = level + 1, np = s->L + 1 + s->K;
  const size_t ct = (size_t)2 * nl * N;
  uint64_t* sk = (uint64_t*)malloc((size_t)np * N * sizeof(uint64_t));
  uint64_t* s2 = (uint64_t*)malloc((size_t)np * N * sizeof(uint64_t));
  secret_ntt(&c, sk);
  for (uint32_t i = 0; i < np; ++i)
    for (uint32_t n = 0; n < N; ++n)
      s2[(size_t)i * N + n] = mulmod(sk[(size_t)i * N + n], sk[(size_t)i * N + n], c.primes[i]);
  uint64_t* kb = (uint64_t*)malloc(key_words(&c) * sizeof(uint64_t));
  uint64_t* ka = (uint64_t*)malloc(key_words(&c) * sizeof(uint64_t));
  make_key(&c, 0, sk, s2, kb, ka);
  uint64_t* d2 = (uint64_t*)malloc((size_t)nl * N * sizeof(uint64_t));
  uint64_t* k0 = (uint64_t*)malloc((size_t)nl * N * sizeof(uint64_t));
  uint64_t* k1 = (uint64_t*)malloc((size_t)nl * N * sizeof(uint64_t));
  for (uint32_t m = 0; m < count; ++m) {
    const uint64_t *a0 = a + m * ct, *a1 = a0 + (size_t)nl * N, *b0 = b + m * ct, *b1 = b0 + (size_t)nl * N;
    uint64_t *o0 = out + m * ct, *o1 = o0 + (size_t)nl * N;
    for (uint32_t i = 0; i < nl; ++i) {
      const uint64_t q = c.primes[i];
      for (uint32_t n = 0; n < N; ++n) {
        const size_t x = (size_t)i * N + n;
        o0[x] = mulmod(a0[x], b0[x], q);
        o1[x] = addmod(mulmod(a0[x], b1[x], q), mulmod(a1[x], b0[x], q), q);
        d2[x] = mulmod(a1[x], b1[x], q);
      }
    }
    key_switch(&c, level, d2, kb, ka, k0, k1);
    for (uint32_t i = 0; i < nl; ++i)
      for (uint32_t n = 0; n < N; ++n) {
        const size_t x = (size_t)i * N + n;
        o0[x] = addmod(o0[x], k0[x], c.primes[i]);
        o1[x] = addmod(o1[x], k1[x], c.primes[i]);
      }
  }
  free(sk);
  free(s2);
  free(kb);
  free(ka);
  free(d2);
  free(k0);
  free(k1);
  ctx_free(&c);
}

void rnso_mul_relin(const rns_spec* s, uint32_t level, const uint64_t* a, const uint64_t* b, uint64_t* out) {
  rnso_mul_relin_many(s, level, 1, a, b, out);
}

/* HMult + relinearisation + rescale with the rescale merged into ModDown (moddown_rescale):
   out has level limbs per polynomial. */
void rnso_mul_relin_rescale(const rns_spec* s, uint32_t level, const uint64_t* a, const uint64_t* b, uint64_t* out) {
  ctx_t c;
  ctx_init(&c, s);
  const uint32_t N = 1u << s->logN, nl = level + 1, np = s->L + 1 + s->K;
  uint64_t* sk = (uint64_t*)malloc((size_t)np * N * sizeof(uint64_t));
  uint64_t* s2 = (uint64_t*)malloc((size_t)np * N * sizeof(uint64_t));
  secret_ntt(&c, sk);
  for (uint32_t i = 0; i < np; ++i)
    for (uint32_t n = 0; n < N; ++n)
      s2[(size_t)i * N + n] = mulmod(sk[(size_t)i * N + n], sk[(size_t)i * N + n], c.primes[i]);
  uint64_t* kb = (uint64_t*)malloc(key_words(&c) * sizeof(uint64_t));
  uint64_t* ka = (uint64_t*)malloc(key_words(&c) * sizeof(uint64_t));
  make_key(&c, 0, sk, s2, kb, ka);
  uint64_t* d0 = (uint64_t*)malloc((size_t)nl * N * sizeof(uint64_t));
  uint64_t* d1 = (uint64_t*)malloc((size_t)nl * N * sizeof(uint64_t));
  uint64_t* d2 = (uint64_t*)malloc((size_t)nl * N * sizeof(uint64_t));
  const uint64_t *a0 = a, *a1 = a + (size_t)nl * N, *b0 = b, *b1 = b + (size_t)nl * N;
  for (uint32_t i = 0; i < nl; ++i) {
    const uint64_t q = c.primes[i];
    for (uint32_t n = 0; n < N; ++n) {
      const size_t x = (size_t)i * N + n;
      d0[x] = mulmod(a0[x], b0[x], q);
      d1[x] = addmod(mulmod(a0[x], b1[x], q), mulmod(a1[x], b0[x], q), q);
      d2[x] = mulmod(a1[x], b1[x], q);
    }
  }
  const uint64_t* dt[2] = {d0, d1};
  key_switch_x(&c, level, d2, kb, ka, out, out + (size_t)level * N, dt);
  free(sk);
  free(s2);
  free(kb);
  free(ka);
  free(d0);
  free(d1);
  free(d2);
  ctx_free(&c);
}

void rnso_rescale(const rns_spec* s, uint32_t level, const uint64_t* in, uint64_t* out) {
  ctx_t c;
  ctx_init(&c, s);
  const uint32_t N = 1u << s->logN;
  uint64_t* last = (uint64_t*)malloc((size_t)N * sizeof(uint64_t));
  uint64_t* t = (uint64_t*)malloc((size_t)N * sizeof(uint64_t));
  const uint64_t ql = c.primes[level];
  for (uint32_t p = 0; p < 2; ++p) {
    const uint64_t* ci = in + (size_t)p * (level + 1) * N;
    uint64_t* co = out + (size_t)p * level * N;
    memcpy(last, ci + (size_t)level * N, N * sizeof(uint64_t));
    ntt_inv(&c, level, last);
    for (uint32_t i = 0; i < level; ++i) {
      const uint64_t q = c.primes[i], qinv = invmod(ql % q, q);
      for (uint32_t n = 0; n < N; ++n) t[n] = last[n] % q;
      ntt_fwd(&c, i, t);
      for (uint32_t n = 0; n < N; ++n)
        co[(size_t)i * N + n] = mulmod(submod(ci[(size_t)i * N + n], t[n], q), qinv, q);
    }
  }
  free(last);
  free(t);
  ctx_free(&c);
}

void rnso_rotate(const rns_spec* s, uint32_t level, int64_t k, const uint64_t* in, uint64_t* out) {
  ctx_t c;
  ctx_init(&c, s);
  const uint32_t N = 1u << s->logN, nl = level + 1, np = s->L + 1 + s->K;
  const uint64_t g = galois_elt(k, s->logN);
  uint64_t* sk = (uint64_t*)malloc((size_t)np * N * sizeof(uint64_t));
  uint64_t* sg = (uint64_t*)malloc((size_t)np * N * sizeof(uint64_t));
  secret_ntt(&c, sk);
  for (uint32_t i = 0; i < np; ++i)
    for (uint32_t n = 0; n < N; ++n) sg[(size_t)i * N + n] = sk[(size_t)i * N + galois_src(n, g, s->logN)];
  uint64_t* kb = (uint64_t*)malloc(key_words(&c) * sizeof(uint64_t));
  uint64_t* ka = (uint64_t*)malloc(key_words(&c) * sizeof(uint64_t));
  make_key(&c, 1 + g, sk, sg, kb, ka);
  uint64_t* c0 = (uint64_t*)malloc((size_t)nl * N * sizeof(uint64_t));
  uint64_t* c1 = (uint64_t*)malloc((size_t)nl * N * sizeof(uint64_t));
  for (uint32_t i = 0; i < nl; ++i)
    for (uint32_t n = 0; n < N; ++n) {
      const uint32_t src = galois_src(n, g, s->logN);
      c0[(size_t)i * N + n] = in[(size_t)i * N + src];
      c1[(size_t)i * N + n] = in[((size_t)nl + i) * N + src];
    }
  uint64_t *o0 = out, *o1 = out + (size_t)nl * N;
  key_switch(&c, level, c1, kb, ka, o0, o1);
  for (uint32_t i = 0; i < nl; ++i)
    for (uint32_t n = 0; n < N; ++n) {
      const size_t x = (size_t)i * N + n;
      o0[x] = addmod(o0[x], c0[x], c.primes[i]);
    }
  free(sk);
  free(sg);
  free(kb);
  free(ka);
  free(c0);
  free(c1);
  ctx_free(&c);
}

/* ------------------------------------------------------------ encryption */
/* symmetric RLWE: c1 = a (uniform, NTT form), c0 = NTT(m + e) - a s */
void rnso_encrypt_coeffs(const rns_spec* s, uint32_t level, const int64_t* coeffs, uint64_t tag, uint64_t* ct) {
  ctx_t c;
  ctx_init(&c, s);
  const uint32_t N = 1u << s->logN, nl = level + 1, np = s->L + 1 + s->K;
  uint64_t* sk = (uint64_t*)malloc((size_t)np * N * sizeof(uint64_t));
  secret_ntt(&c, sk);
  for (uint32_t i = 0; i < nl; ++i) {
    const uint64_t q = c.primes[i];
    uint64_t* c0 = ct + (size_t)i * N;
    uint64_t* c1 = ct + ((size_t)nl + i) * N;
    for (uint32_t n = 0; n < N; ++n) {
      c0[n] = lift(coeffs[n] + cbd(rnso_hash(s->seed, D_ENC_E, tag, n)), q);
      c1[n] = uniform(rnso_hash(s->seed, D_ENC_A, tag * 64 + i, n), q);
    }
    ntt_fwd(&c, i, c0);
    for (uint32_t n = 0; n < N; ++n) c0[n] = submod(c0[n], mulmod(c1[n], sk[(size_t)i * N + n], q), q);
  }
  free(sk);
  ctx_free(&c);
}

/* m = c0 + c1 s on limb 0, centred mod q_0 */
void rnso_decrypt_coeffs(const rns_spec* s, uint32_t level, const uint64_t* ct, int64_t* coeffs) {
  ctx_t c;
  ctx_init(&c, s);
  const uint32_t N = 1u << s->logN, nl = level + 1, np = s->L + 1 + s->K;
  uint64_t* sk = (uint64_t*)malloc((size_t)np * N * sizeof(uint64_t));
  uint64_t* m = (uint64_t*)malloc((size_t)N * sizeof(uint64_t));
  secret_ntt(&c, sk);
  const uint64_t q = c.primes[0];
  for (uint32_t n = 0; n < N; ++n) m[n] = addmod(ct[n], mulmod(ct[(size_t)nl * N + n], sk[n], q), q);
  ntt_inv(&c, 0, m);
  for (uint32_t n = 0; n < N; ++n) coeffs[n] = m[n] > q / 2 ? -(int64_t)(q - m[n]) : (int64_t)m[n];
  free(sk);
  free(m);
  ctx_free(&c);
}
