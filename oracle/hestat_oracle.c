/* hestat_oracle.c — TEST INFRASTRUCTURE ONLY (see hestat_oracle.h).
 *
 * A from-scratch C11 restatement of the reference CKKS-emulator evaluation
 * path.  Every function names the reference file:line it follows
 * (paths relative to /root/reference/proj/include/hestat/).  Errors that the
 * reference raises as C++ exceptions unwind here via longjmp to the ABI entry
 * point, which returns the shared error code (include/hestat_gpu.h) and leaves
 * the meter exactly as the reference would leave it at the throw.
 *
 * Memory: every ciphertext of one ABI call lives in a per-call arena released
 * at exit, so unwinding never leaks.
 *
 * Build: gcc -std=c11 -O2 -ffp-contract=off (oracle/Makefile).  Contraction
 * would change bits.
 */
#define _GNU_SOURCE
#include "hestat_oracle.h"

#include <math.h>
#include <setjmp.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------------ */
/* error codes (== hestat_gpu.h HS_E_*)                                      */
enum {
  E_ERROR = 1, E_TOO_MANY_VALUES, E_LEVEL_EXHAUSTED, E_LENGTH_MISMATCH, E_DIRTY_PADDING,
  E_NON_FINITE_TARGET, E_DOMAIN_VIOLATION, E_DIVERGENCE, E_EMPTY_COLUMN,
  E_DEGENERATE_VARIANCE, E_NEAR_ZERO_MEAN, E_IO_ERROR, E_MISSING_COLUMN,
  E_UNPARSABLE_CELL, E_NON_FINITE_VALUE, E_ZERO_REFERENCE
};

static _Thread_local char g_msg[256];
const char* ora_last_error(void) { return g_msg; }

/* ------------------------------------------------------------------------ */
/* per-call arena + unwinding                                                */
typedef struct blk { struct blk* next; } blk;

typedef struct {
  orc_params p;
  orc_meter m;
  jmp_buf jb;
  blk* arena;
} ctx_t;

static void* amalloc(ctx_t* c, size_t bytes) {
  blk* b = (blk*)malloc(sizeof(blk) + bytes + 16);
  if (!b) abort();
  b->next = c->arena;
  c->arena = b;
  return (void*)((char*)b + sizeof(blk) + (16 - sizeof(blk) % 16) % 16);
}

static void arena_free(ctx_t* c) {
  while (c->arena) {
    blk* n = c->arena->next;
    free(c->arena);
    c->arena = n;
  }
}

static _Noreturn void raise_err(ctx_t* c, int code, const char* msg) {
  snprintf(g_msg, sizeof g_msg, "%s", msg);
  longjmp(c->jb, code);
}

/* CkksParams::validate, ckks.hpp:34-39 */
static void params_validate(ctx_t* c) {
  uint64_t s = c->p.slot_count;
  if (s == 0 || (s & (s - 1)) != 0)
    raise_err(c, E_ERROR, "CkksParams: slot_count must be a power of two");
  if (c->p.max_level < 1) raise_err(c, E_ERROR, "CkksParams: max_level must be >= 1");
  if (c->p.scale_bits < 1) raise_err(c, E_ERROR, "CkksParams: scale_bits must be >= 1");
}

static void ctx_init(ctx_t* c, const orc_params* p) {
  memset(c, 0, sizeof *c);
  c->p = *p;
}

/* ------------------------------------------------------------------------ */
/* ciphertext: slot vector + level (ckks.hpp:64-78)                          */
typedef struct {
  double* v;
  size_t n;
  int level;
} ct_t;

static ct_t ct_new(ctx_t* c, size_t n, int level) {
  ct_t r;
  r.v = (double*)amalloc(c, (n ? n : 1) * sizeof(double));
  r.n = n;
  r.level = level;
  return r;
}

static ct_t ct_from(ctx_t* c, const double* v, size_t n, int level) {
  ct_t r = ct_new(c, n, level);
  if (n) memcpy(r.v, v, n * sizeof(double));
  return r;
}

static size_t S_of(const ctx_t* c) { return (size_t)c->p.slot_count; }

/* quantize_inplace, ckks.hpp:247-252 */
static void quantize(const ctx_t* c, double* v, size_t n) {
  if (!c->p.quantize) return;
  const double s = ldexp(1.0, c->p.scale_bits);
  const double inv = ldexp(1.0, -c->p.scale_bits);
  for (size_t i = 0; i < n; ++i) v[i] = nearbyint(v[i] * s) * inv;
}

/* check_shape, ckks.hpp:242-245 */
static void check_shape(ctx_t* c, const ct_t* a) {
  if (a->n != S_of(c))
    raise_err(c, E_LENGTH_MISMATCH, "ciphertext slot count does not match context");
}

static int imin(int a, int b) { return a < b ? a : b; }

/* encrypt, ckks.hpp:97-104 */
static ct_t op_encrypt(ctx_t* c, const double* v, size_t n) {
  if (n > S_of(c)) raise_err(c, E_TOO_MANY_VALUES, "encrypt: more values than slots");
  ct_t r = ct_new(c, S_of(c), c->p.max_level);
  for (size_t i = 0; i < r.n; ++i) r.v[i] = i < n ? v[i] : 0.0;
  quantize(c, r.v, r.n);
  return r;
}

/* add_ct / sub_ct, ckks.hpp:113-133 */
static ct_t op_addsub(ctx_t* c, const ct_t* a, const ct_t* b, int sub) {
  check_shape(c, a);
  check_shape(c, b);
  ct_t r = ct_new(c, S_of(c), imin(a->level, b->level));
  for (size_t i = 0; i < r.n; ++i) r.v[i] = sub ? a->v[i] - b->v[i] : a->v[i] + b->v[i];
  quantize(c, r.v, r.n);
  ++c->m.add;
  return r;
}
static ct_t op_add(ctx_t* c, ct_t a, ct_t b) { return op_addsub(c, &a, &b, 0); }
static ct_t op_sub(ctx_t* c, ct_t a, ct_t b) { return op_addsub(c, &a, &b, 1); }

/* add_pt, ckks.hpp:137-144 */
static ct_t op_add_pt(ctx_t* c, ct_t a, double k) {
  check_shape(c, &a);
  ct_t r = ct_new(c, S_of(c), a.level);
  for (size_t i = 0; i < r.n; ++i) r.v[i] = a.v[i] + k;
  quantize(c, r.v, r.n);
  ++c->m.add;
  return r;
}

/* bootstrap, ckks.hpp:207-213 */
static ct_t op_bootstrap(ctx_t* c, ct_t a) {
  check_shape(c, &a);
  ct_t r = ct_from(c, a.v, a.n, c->p.max_level);
  quantize(c, r.v, r.n);
  ++c->m.bootstrap;
  return r;
}

/* mul_ct, ckks.hpp:149-164 (inputs by value; lazy auto-bootstrap of each
 * exhausted operand, a first) */
static ct_t op_mul_ct(ctx_t* c, ct_t a, ct_t b) {
  check_shape(c, &a);
  check_shape(c, &b);
  if (imin(a.level, b.level) < 1) {
    if (!c->p.auto_bootstrap)
      raise_err(c, E_LEVEL_EXHAUSTED, "mul_ct: no multiplicative level left");
    if (a.level < 1) a = op_bootstrap(c, a);
    if (b.level < 1) b = op_bootstrap(c, b);
  }
  ct_t r = ct_new(c, S_of(c), imin(a.level, b.level) - 1);
  for (size_t i = 0; i < r.n; ++i) r.v[i] = a.v[i] * b.v[i];
  quantize(c, r.v, r.n);
  ++c->m.mul_ct;
  return r;
}

/* prepare_mul_pt, ckks.hpp:233-240 */
static ct_t prepare_mul_pt(ctx_t* c, ct_t a) {
  if (a.level < 1) {
    if (!c->p.auto_bootstrap)
      raise_err(c, E_LEVEL_EXHAUSTED, "mul_pt: no multiplicative level left");
    a = op_bootstrap(c, a);
  }
  return a;
}

/* mul_pt (scalar), ckks.hpp:168-176 */
static ct_t op_mul_pt(ctx_t* c, ct_t a, double k) {
  check_shape(c, &a);
  a = prepare_mul_pt(c, a);
  ct_t r = ct_new(c, S_of(c), a.level - 1);
  for (size_t i = 0; i < r.n; ++i) r.v[i] = a.v[i] * k;
  quantize(c, r.v, r.n);
  ++c->m.mul_pt;
  return r;
}

/* mul_pt (vector), ckks.hpp:179-189 */
static ct_t op_mul_pt_vec(ctx_t* c, ct_t a, const double* p, size_t np) {
  check_shape(c, &a);
  if (np != S_of(c))
    raise_err(c, E_LENGTH_MISMATCH, "mul_pt: plaintext vector length != slot count");
  a = prepare_mul_pt(c, a);
  ct_t r = ct_new(c, S_of(c), a.level - 1);
  for (size_t i = 0; i < r.n; ++i) r.v[i] = a.v[i] * p[i];
  quantize(c, r.v, r.n);
  ++c->m.mul_pt;
  return r;
}

/* rotate, ckks.hpp:193-202 (left cyclic shift, no quantisation) */
static ct_t op_rotate(ctx_t* c, ct_t a, long k) {
  check_shape(c, &a);
  const long n = (long)S_of(c);
  const long shift = ((k % n) + n) % n;
  ct_t r = ct_new(c, S_of(c), a.level);
  for (size_t i = 0; i < r.n; ++i) r.v[i] = a.v[(i + (size_t)shift) % r.n];
  ++c->m.rotate;
  return r;
}

/* sum_all_slots, ckks.hpp:218-230 */
static ct_t op_sum_all(ctx_t* c, ct_t a, size_t n_valid) {
  check_shape(c, &a);
  if (c->p.debug_checks) {
    const double eps = ldexp(1.0, -(c->p.scale_bits - 1));
    for (size_t i = n_valid; i < S_of(c); ++i)
      if (fabs(a.v[i]) > eps) raise_err(c, E_DIRTY_PADDING, "sum_all_slots: nonzero padding slot");
  }
  ct_t acc = a;
  for (size_t step = 1; step < S_of(c); step <<= 1)
    acc = op_add(c, acc, op_rotate(c, acc, (long)step));
  return acc;
}

/* ------------------------------------------------------------------------ */
/* Chebyshev (chebyshev.hpp)                                                 */
typedef double (*target_fn)(double, const void*);

/* scaled_target, chebyshev.hpp:39-47 */
static double invsqrt_shifted(double t, const void* u) {
  const double S = *(const double*)u;
  return t > -1.0 ? 1.0 / (sqrt(S) * sqrt(t + 1.0)) : 0.0;
}
static double sqrt_shifted(double t, const void* u) {
  const double S = *(const double*)u;
  return t >= -1.0 ? sqrt(S) * sqrt(t + 1.0) : 0.0;
}
static double f_ident(double x, const void* u) { (void)u; return x; }
static double f_square(double x, const void* u) { (void)u; return x * x; }
static double f_exp(double x, const void* u) { (void)u; return exp(x); }
static double f_recip2(double x, const void* u) { (void)u; return 1.0 / (2.0 + x); }
static double f_cos2(double x, const void* u) { (void)u; return cos(2 * x); }
static double f_cos3(double x, const void* u) { (void)u; return cos(3.0 * x); }
static double f_one(double x, const void* u) { (void)u; (void)x; return 1.0; }
static double f_sqrt(double x, const void* u) { (void)u; return sqrt(x); }
static double f_zero(double x, const void* u) { (void)u; (void)x; return 0.0; }

static target_fn target_of(int kind) {
  switch (kind) {
    case 0: return invsqrt_shifted;
    case 1: return sqrt_shifted;
    case 2: return f_ident;
    case 3: return f_square;
    case 4: return f_exp;
    case 5: return f_recip2;
    case 6: return f_cos2;
    case 7: return f_cos3;
    case 8: return f_one;
    case 9: return f_sqrt;
    default: return f_zero;
  }
}

/* cheb_eval_depth, chebyshev.hpp:51-54: bit_width(degree) */
static int cheb_depth(int d) {
  if (d <= 0) return 0;
  int w = 0;
  for (unsigned u = (unsigned)d; u; u >>= 1) ++w;
  return w;
}

/* fit, chebyshev.hpp:59-85: DCT projection over degree+1 first-kind nodes */
static void cheb_fit(ctx_t* c, target_fn f, const void* u, int degree, double lo, double hi,
                     double* coeffs) {
  if (degree < 0) raise_err(c, E_ERROR, "fit: degree must be >= 0");
  const int n = degree + 1;
  double* theta = (double*)amalloc(c, (size_t)n * sizeof(double));
  double* samples = (double*)amalloc(c, (size_t)n * sizeof(double));
  for (int k = 0; k < n; ++k) {
    theta[k] = M_PI * (k + 0.5) / n;
    const double x = cos(theta[k]);
    const double arg = 0.5 * (lo + hi) + 0.5 * (hi - lo) * x;
    samples[k] = f(arg, u);
    if (!isfinite(samples[k]))
      raise_err(c, E_NON_FINITE_TARGET, "fit: target not finite at a Chebyshev node");
  }
  for (int j = 0; j < n; ++j) {
    double acc = 0.0;
    for (int k = 0; k < n; ++k) acc += samples[k] * cos(j * theta[k]);
    coeffs[j] = 2.0 * acc / n;
  }
  coeffs[0] *= 0.5;
}

/* eval_plain (Clenshaw), chebyshev.hpp:90-105 */
static double cheb_plain(const double* cf, int ncoef, double lo, double hi, double x) {
  const int native = lo == -1.0 && hi == 1.0;
  const double u = native ? x : (2.0 * x - (lo + hi)) / (hi - lo);
  double b1 = 0.0, b2 = 0.0;
  for (int k = ncoef - 1; k >= 1; --k) {
    const double next = cf[k] + 2.0 * u * b1 - b2;
    b2 = b1;
    b1 = next;
  }
  return cf[0] + u * b1 - b2;
}

/* ChebEncryptedEval, chebyshev.hpp:113-163 */
typedef struct {
  ctx_t* c;
  ct_t x;
  ct_t pw[32]; /* pw[j] = T_{2^j}; pw[0] unused (x) */
  int have[32];
} bsgs_t;

static int ilog2(int g) {
  int j = 0;
  while ((1 << j) < g) ++j;
  return j;
}

/* build_powers, chebyshev.hpp:130-138 */
static void bsgs_build_powers(bsgs_t* e, int depth) {
  int g = 1;
  while (2 * g < (1 << depth)) {
    const ct_t tg = g == 1 ? e->x : e->pw[ilog2(g)];
    const ct_t sq = op_mul_ct(e->c, tg, tg);
    e->pw[ilog2(2 * g)] = op_add_pt(e->c, op_add(e->c, sq, sq), -1.0);
    e->have[ilog2(2 * g)] = 1;
    g *= 2;
  }
}

/* eval, chebyshev.hpp:140-158: p = q*T_g + r with T_i T_g = (T_{i+g}+T_{g-i})/2 */
static ct_t bsgs_eval(bsgs_t* e, const double* cf, int ncoef) {
  ctx_t* c = e->c;
  const int d = ncoef - 1;
  if (d <= 1) {
    const ct_t r = op_mul_pt(c, e->x, d == 1 ? cf[1] : 0.0);
    return op_add_pt(c, r, cf[0]);
  }
  const int g = 1 << (cheb_depth(d) - 1);
  const int nq = d - g + 1;
  double* q = (double*)amalloc(c, (size_t)nq * sizeof(double));
  double* r = (double*)amalloc(c, (size_t)g * sizeof(double));
  q[0] = cf[g];
  for (int j = 1; j <= d - g; ++j) q[j] = 2.0 * cf[g + j];
  for (int j = 0; j < g; ++j) r[j] = cf[j];
  for (int j = 1; j <= d - g; ++j) r[g - j] -= cf[g + j];
  if (!e->have[ilog2(g)]) raise_err(c, E_ERROR, "map::at");
  const ct_t tg = e->pw[ilog2(g)];
  const ct_t head = nq == 1 ? op_mul_pt(c, tg, q[0]) : op_mul_ct(c, bsgs_eval(e, q, nq), tg);
  const ct_t rest = bsgs_eval(e, r, g);
  return op_add(c, head, rest);
}

/* ChebEncryptedEval::run, chebyshev.hpp:117-125 */
static ct_t bsgs_run(ctx_t* c, ct_t x, const double* cf, int ncoef) {
  const int d = ncoef - 1;
  if (d <= 0) return op_add_pt(c, op_sub(c, x, x), ncoef == 0 ? 0.0 : cf[0]);
  bsgs_t e;
  memset(&e, 0, sizeof e);
  e.c = c;
  e.x = x;
  bsgs_build_powers(&e, cheb_depth(d));
  return bsgs_eval(&e, cf, ncoef);
}

/* eval_encrypted, chebyshev.hpp:171-189 */
static ct_t eval_encrypted(ctx_t* c, const double* cf, int ncoef, double lo, double hi,
                           ct_t ct) {
  if (ncoef == 0) raise_err(c, E_ERROR, "eval_encrypted: empty series");
  if (c->p.debug_checks) {
    const double eps = 1e-9;
    for (size_t i = 0; i < ct.n; ++i)
      if (ct.v[i] < lo - eps || ct.v[i] > hi + eps)
        raise_err(c, E_DOMAIN_VIOLATION, "eval_encrypted: slot outside series domain");
  }
  const int native = lo == -1.0 && hi == 1.0;
  const int need = cheb_depth(ncoef - 1) + (native ? 0 : 1);
  ct_t x = ct;
  if (x.level < need && c->p.auto_bootstrap) x = op_bootstrap(c, x);
  if (!native) {
    const double span = hi - lo;
    x = op_add_pt(c, op_mul_pt(c, x, 2.0 / span), -(lo + hi) / span);
  }
  return bsgs_run(c, x, cf, ncoef);
}

/* ------------------------------------------------------------------------ */
/* inverse-root primitives (primitives.hpp)                                  */
#define ALL_SLOTS ((uint64_t)-1)

static size_t zmin(size_t a, size_t b) { return a < b ? a : b; }

/* check_divergence, primitives.hpp:89-96 */
static void check_divergence(ctx_t* c, const ct_t* y, size_t n_valid) {
  if (!c->p.debug_checks) return;
  const size_t n = zmin(n_valid, y->n);
  for (size_t i = 0; i < n; ++i)
    if (!(fabs(y->v[i]) <= 1e6))
      raise_err(c, E_DIVERGENCE, "newton iterate exceeded the divergence guard");
}

/* newton_loop, primitives.hpp:105-132: y <- ((n+1)/n) y - x_op * y^(n+1),
 * product as a balanced pairwise tree */
static ct_t newton_loop(ctx_t* c, ct_t x_op, ct_t y, int n, int iters, size_t n_valid) {
  const int per_iter = cheb_depth(n + 1);
  ct_t x = x_op;
  if (x.level < per_iter && c->p.auto_bootstrap) x = op_bootstrap(c, x);
  ct_t* f = (ct_t*)amalloc(c, (size_t)(n + 2) * sizeof(ct_t));
  for (int i = 0; i < iters; ++i) {
    if (y.level < per_iter && c->p.auto_bootstrap) y = op_bootstrap(c, y);
    int nf = 0;
    f[nf++] = x;
    for (int j = 0; j < n + 1; ++j) f[nf++] = y;
    while (nf > 1) {
      int m = 0;
      int k = 0;
      for (; k + 1 < nf; k += 2) f[m++] = op_mul_ct(c, f[k], f[k + 1]);
      if (nf % 2 == 1) f[m++] = f[nf - 1];
      nf = m;
    }
    const ct_t linear = op_mul_pt(c, y, (n + 1.0) / n);
    y = op_sub(c, linear, f[0]);
    check_divergence(c, &y, n_valid);
  }
  return y;
}

/* check_open_domain, primitives.hpp:134-144 */
static void check_open_domain(ctx_t* c, const ct_t* ct, size_t n_valid, double lo, double hi,
                              const char* who) {
  if (!c->p.debug_checks) return;
  const size_t n = zmin(n_valid, ct->n);
  for (size_t i = 0; i < n; ++i) {
    const double t = ct->v[i];
    if (!(t > lo) || !(t <= hi)) {
      char buf[128];
      snprintf(buf, sizeof buf, "%s: scaled slot outside domain", who);
      raise_err(c, E_DOMAIN_VIOLATION, buf);
    }
  }
}

typedef struct {
  int n, cheb_degree, newton_iters, baseline_mode, baseline_iters;
} cfg_t;

static cfg_t cfg_of(const orc_invroot* r) {
  cfg_t c = {2, 511, 6, 0, 0}; /* InvRootConfig defaults, primitives.hpp:23-28 */
  if (r) {
    c.n = r->n;
    c.cheb_degree = r->cheb_degree;
    c.newton_iters = r->newton_iters;
    c.baseline_mode = r->baseline_mode;
    c.baseline_iters = r->baseline_iters;
  }
  return c;
}

/* InvRootConfig::validate / effective_baseline_iters, primitives.hpp:30-40 */
static void cfg_validate(ctx_t* c, const cfg_t* k) {
  if (k->n != 1 && k->n != 2) raise_err(c, E_ERROR, "InvRootConfig: n must be 1 or 2");
  if (k->newton_iters < 0) raise_err(c, E_ERROR, "InvRootConfig: newton_iters < 0");
  if (k->cheb_degree < 0) raise_err(c, E_ERROR, "InvRootConfig: cheb_degree < 0");
}
static int cfg_baseline_iters(const cfg_t* k) {
  if (k->baseline_iters > 0) return k->baseline_iters;
  return k->n == 1 ? 25 : 21;
}

/* newton_refine, primitives.hpp:152-158 */
static ct_t newton_refine(ctx_t* c, ct_t x, ct_t y0, int n, int iters, size_t n_valid) {
  if (n < 1) raise_err(c, E_ERROR, "newton_refine: n must be >= 1");
  const ct_t x_op = n >= 2 ? op_mul_pt(c, x, 1.0 / n) : x;
  return newton_loop(c, x_op, y0, n, iters, n_valid);
}

/* baseline_invsqrt, primitives.hpp:173-184 */
static ct_t baseline_invsqrt(ctx_t* c, ct_t ct, double S, int iters, size_t n_valid) {
  check_open_domain(c, &ct, n_valid, 0.0, 1.0, "baseline_invsqrt");
  double* ones = (double*)amalloc(c, S_of(c) * sizeof(double));
  for (size_t i = 0; i < S_of(c); ++i) ones[i] = 1.0;
  ct_t y = op_encrypt(c, ones, S_of(c));
  if (iters > 0) {
    const ct_t x_op = op_mul_pt(c, ct, 0.5);
    y = newton_loop(c, x_op, y, 2, iters, n_valid);
  }
  return op_mul_pt(c, y, 1.0 / sqrt(S));
}

/* crypto_invsqrt, primitives.hpp:186-208 */
static ct_t crypto_invsqrt(ctx_t* c, ct_t ct, double S, const cfg_t* k, size_t n_valid) {
  cfg_validate(c, k);
  if (S <= 0.0) raise_err(c, E_ERROR, "crypto_invsqrt: scale must be positive");
  if (k->baseline_mode) return baseline_invsqrt(c, ct, S, cfg_baseline_iters(k), n_valid);
  check_open_domain(c, &ct, n_valid, 0.0, 2.0, "crypto_invsqrt");
  double* cf = (double*)amalloc(c, (size_t)(k->cheb_degree + 1) * sizeof(double));
  cheb_fit(c, invsqrt_shifted, &S, k->cheb_degree, -1.0, 1.0, cf);
  const ct_t arg = op_add_pt(c, ct, -1.0);
  ct_t y = eval_encrypted(c, cf, k->cheb_degree + 1, -1.0, 1.0, arg);
  y = op_bootstrap(c, y);
  if (k->newton_iters > 0) {
    const ct_t x_op = op_mul_pt(c, ct, S / 2.0);
    y = newton_loop(c, x_op, y, 2, k->newton_iters, n_valid);
  }
  return y;
}

/* crypto_inv, primitives.hpp:211-217 */
static ct_t crypto_inv(ctx_t* c, ct_t ct, double S, const cfg_t* k, size_t n_valid) {
  ct_t y = crypto_invsqrt(c, ct, S, k, n_valid);
  if (y.level < 1 && c->p.auto_bootstrap) y = op_bootstrap(c, y);
  return op_mul_ct(c, y, y);
}

/* crypto_sqrt, primitives.hpp:222-238 */
static ct_t crypto_sqrt(ctx_t* c, ct_t ct, double S, int degree, size_t n_valid) {
  if (S <= 0.0) raise_err(c, E_ERROR, "crypto_sqrt: scale must be positive");
  if (c->p.debug_checks) {
    const size_t n = zmin(n_valid, ct.n);
    for (size_t i = 0; i < n; ++i) {
      const double t = ct.v[i];
      if (t < -1e-9 || t > 2.0 + 1e-9)
        raise_err(c, E_DOMAIN_VIOLATION, "crypto_sqrt: scaled slot outside [0, 2]");
    }
  }
  if (degree < 0) raise_err(c, E_ERROR, "fit: degree must be >= 0");
  double* cf = (double*)amalloc(c, (size_t)(degree + 1) * sizeof(double));
  cheb_fit(c, sqrt_shifted, &S, degree, -1.0, 1.0, cf);
  return eval_encrypted(c, cf, degree + 1, -1.0, 1.0, op_add_pt(c, ct, -1.0));
}

/* g3_series, primitives.hpp:243-249 */
static const double G3[8] = {0.0, 1225.0 / 1024.0, 0.0, -245.0 / 1024.0,
                             0.0, 49.0 / 1024.0,   0.0, -5.0 / 1024.0};

typedef struct {
  const double* p;
  size_t n;
} poly_t;
static double f_horner(double x, const void* u) {
  const poly_t* pp = (const poly_t*)u;
  double acc = 0.0;
  for (size_t i = pp->n; i-- > 0;) acc = acc * x + pp->p[i];
  return acc;
}

/* odd_poly_series, primitives.hpp:255-272 */
static double* odd_poly_series(ctx_t* c, const double* power, size_t np) {
  if (np == 0) raise_err(c, E_ERROR, "sign: empty component polynomial");
  for (size_t i = 0; i < np; i += 2)
    if (power[i] != 0.0) raise_err(c, E_ERROR, "sign: component polynomial must be odd");
  const int d = (int)np - 1;
  poly_t pp = {power, np};
  double* cf = (double*)amalloc(c, np * sizeof(double));
  cheb_fit(c, f_horner, &pp, d, -1.0, 1.0, cf);
  for (size_t i = 0; i < np; i += 2) {
    if (fabs(cf[i]) > 1e-9) raise_err(c, E_ERROR, "sign: conversion produced a non-odd series");
    cf[i] = 0.0;
  }
  return cf;
}

/* crypto_sign, primitives.hpp:279-300 */
static ct_t crypto_sign(ctx_t* c, ct_t ct, int mode, int folds, const double* polys,
                        const uint64_t* plen, size_t npolys) {
  if (folds < 1) raise_err(c, E_ERROR, "crypto_sign: folds must be >= 1");
  if (c->p.debug_checks) {
    for (size_t i = 0; i < ct.n; ++i)
      if (ct.v[i] < -1.0 - 1e-9 || ct.v[i] > 1.0 + 1e-9)
        raise_err(c, E_DOMAIN_VIOLATION, "crypto_sign: slot outside [-1, 1]");
  }
  const double** st = (const double**)amalloc(c, (npolys + 1) * sizeof(double*));
  int* sn = (int*)amalloc(c, (npolys + 1) * sizeof(int));
  size_t nst = 0;
  if (mode == 0) {
    st[0] = G3;
    sn[0] = 8;
    nst = 1;
  } else {
    if (npolys == 0) raise_err(c, E_ERROR, "crypto_sign: custom mode needs component polynomials");
    size_t off = 0;
    for (size_t i = 0; i < npolys; ++i) {
      st[nst] = odd_poly_series(c, polys + off, (size_t)plen[i]);
      sn[nst++] = (int)plen[i];
      off += (size_t)plen[i];
    }
  }
  ct_t y = ct;
  for (int f = 0; f < folds; ++f)
    y = eval_encrypted(c, st[(size_t)f % nst], sn[(size_t)f % nst], -1.0, 1.0, y);
  return y;
}

/* ------------------------------------------------------------------------ */
/* columns (column.hpp) and statistics (stats.hpp)                           */
typedef struct {
  ct_t* chunks;
  size_t nchunks;
  size_t n_valid;
} col_t;

/* encode_column, column.hpp:25-39 */
static col_t encode_column(ctx_t* c, const double* v, size_t n) {
  for (size_t i = 0; i < n; ++i)
    if (!isfinite(v[i])) raise_err(c, E_NON_FINITE_VALUE, "encode_column: non-finite value in x");
  col_t col;
  const size_t sc = S_of(c);
  col.n_valid = n;
  col.nchunks = (n + sc - 1) / sc;
  col.chunks = (ct_t*)amalloc(c, (col.nchunks + 1) * sizeof(ct_t));
  size_t k = 0;
  for (size_t off = 0; off < n; off += sc) col.chunks[k++] = op_encrypt(c, v + off, zmin(sc, n - off));
  return col;
}

/* decode_column, column.hpp:41-56 */
static void decode_column(ctx_t* c, const col_t* col, double* out) {
  const size_t sc = S_of(c);
  if (col->n_valid > col->nchunks * sc)
    raise_err(c, E_LENGTH_MISMATCH, "decode_column: n_valid exceeds packed capacity");
  size_t remaining = col->n_valid, o = 0;
  for (size_t i = 0; i < col->nchunks; ++i) {
    const size_t take = zmin(sc, remaining);
    memcpy(out + o, col->chunks[i].v, take * sizeof(double));
    o += take;
    remaining -= take;
  }
}

/* require_nonempty / chunk_valid, stats.hpp:26-37 */
static void require_nonempty(ctx_t* c, const col_t* col) {
  if (col->n_valid == 0 || col->nchunks == 0) raise_err(c, E_EMPTY_COLUMN, "statistic on an empty column");
}
static size_t chunk_valid(const ctx_t* c, const col_t* col, size_t i) {
  const size_t sc = S_of(c);
  const size_t off = i * sc;
  return off >= col->n_valid ? 0 : zmin(sc, col->n_valid - off);
}

/* scaled_slot_sum, stats.hpp:41-51 */
static ct_t scaled_slot_sum(ctx_t* c, const col_t* col, double k) {
  ct_t acc = {0};
  for (size_t i = 0; i < col->nchunks; ++i) {
    const ct_t term = op_mul_pt(c, col->chunks[i], k);
    acc = i == 0 ? term : op_add(c, acc, term);
  }
  return op_sum_all(c, acc, S_of(c));
}

/* centered_chunks, stats.hpp:56-75 */
static ct_t* centered_chunks(ctx_t* c, const col_t* col, ct_t mu, int mask_padding) {
  const size_t sc = S_of(c);
  ct_t* out = (ct_t*)amalloc(c, (col->nchunks + 1) * sizeof(ct_t));
  for (size_t i = 0; i < col->nchunks; ++i) {
    const size_t valid = chunk_valid(c, col, i);
    if (mask_padding && valid < sc) {
      double* mask = (double*)amalloc(c, sc * sizeof(double));
      for (size_t k = 0; k < sc; ++k) mask[k] = k < valid ? 1.0 : 0.0;
      const ct_t mu_masked = op_mul_pt_vec(c, mu, mask, sc);
      out[i] = op_sub(c, col->chunks[i], mu_masked);
    } else {
      out[i] = op_sub(c, col->chunks[i], mu);
    }
  }
  return out;
}

/* mean_of_chunks, stats.hpp:78-87 */
static ct_t mean_of_chunks(ctx_t* c, const ct_t* ch, size_t nch, size_t n_valid) {
  ct_t acc = {0};
  for (size_t i = 0; i < nch; ++i) {
    const ct_t term = op_mul_pt(c, ch[i], 1.0 / (double)n_valid);
    acc = i == 0 ? term : op_add(c, acc, term);
  }
  return op_sum_all(c, acc, S_of(c));
}

/* replicated_value, stats.hpp:89-91 */
static double first_slot(const ct_t* ct) { return ct->v[0]; }

/* mean_scaled, stats.hpp:97-103 */
static ct_t mean_scaled(ctx_t* c, const col_t* col, double B) {
  require_nonempty(c, col);
  if (B <= 0.0) raise_err(c, E_ERROR, "mean_scaled: B must be positive");
  return scaled_slot_sum(c, col, 1.0 / (B * (double)col->n_valid));
}

/* variance_to_scale, stats.hpp:110-126 */
static ct_t variance_to_scale(ctx_t* c, const col_t* col, double S) {
  require_nonempty(c, col);
  if (S <= 0.0) raise_err(c, E_ERROR, "variance_to_scale: scale must be positive");
  const double n = (double)col->n_valid;
  ct_t sq_sum = {0};
  for (size_t i = 0; i < col->nchunks; ++i) {
    const ct_t a = op_mul_pt(c, col->chunks[i], 1.0 / sqrt(S * n));
    const ct_t sq = op_mul_ct(c, a, a);
    sq_sum = i == 0 ? sq : op_add(c, sq_sum, sq);
  }
  sq_sum = op_sum_all(c, sq_sum, S_of(c));
  const ct_t mean_part = scaled_slot_sum(c, col, 1.0 / (n * sqrt(S)));
  const ct_t mean_sq = op_mul_ct(c, mean_part, mean_part);
  return op_sub(c, sq_sum, mean_sq);
}

/* variance_scaled, stats.hpp:130-134 */
static ct_t variance_scaled(ctx_t* c, const col_t* col, double B) {
  if (B <= 0.0) raise_err(c, E_ERROR, "variance_scaled: B must be positive");
  return variance_to_scale(c, col, B * B);
}

/* moments, stats.hpp:138-148 */
static void moments(ctx_t* c, const col_t* col, double B, ct_t* mu, ct_t* var) {
  *mu = mean_scaled(c, col, 1.0);
  *var = variance_scaled(c, col, B);
  if (c->p.debug_checks && first_slot(var) < -1e-9)
    raise_err(c, E_DEGENERATE_VARIANCE, "moments: negative scaled variance");
}

/* znorm, stats.hpp:153-166 */
static col_t znorm(ctx_t* c, const col_t* col, double B, const cfg_t* k) {
  ct_t mu, var;
  moments(c, col, B, &mu, &var);
  if (c->p.debug_checks && first_slot(&var) * B * B < 1e-9)
    raise_err(c, E_DEGENERATE_VARIANCE, "znorm: variance below 1e-9");
  const ct_t inv = crypto_invsqrt(c, var, B * B, k, ALL_SLOTS);
  col_t out;
  out.n_valid = col->n_valid;
  out.nchunks = col->nchunks;
  out.chunks = (ct_t*)amalloc(c, (col->nchunks + 1) * sizeof(ct_t));
  for (size_t i = 0; i < col->nchunks; ++i)
    out.chunks[i] = op_mul_ct(c, op_sub(c, col->chunks[i], mu), inv);
  return out;
}

/* kurtosis (power 4) / skewness (power 3), stats.hpp:170-210 */
static ct_t std_moment(ctx_t* c, const col_t* col, double B, const cfg_t* k, int power) {
  ct_t mu, var;
  moments(c, col, B, &mu, &var);
  if (c->p.debug_checks && first_slot(&var) * B * B < 1e-9)
    raise_err(c, E_DEGENERATE_VARIANCE,
              power == 4 ? "kurtosis: variance below 1e-9" : "skewness: variance below 1e-9");
  ct_t* cen = centered_chunks(c, col, mu, 1);
  ct_t* pw = (ct_t*)amalloc(c, (col->nchunks + 1) * sizeof(ct_t));
  for (size_t i = 0; i < col->nchunks; ++i) {
    const ct_t sq = op_mul_ct(c, cen[i], cen[i]);
    pw[i] = power == 4 ? op_mul_ct(c, sq, sq) : op_mul_ct(c, sq, cen[i]);
  }
  const ct_t numerator = mean_of_chunks(c, pw, col->nchunks, col->n_valid);
  const ct_t inv = crypto_invsqrt(c, var, B * B, k, ALL_SLOTS);
  const ct_t inv2 = op_mul_ct(c, inv, inv);
  const ct_t invp = power == 4 ? op_mul_ct(c, inv2, inv2) : op_mul_ct(c, inv2, inv);
  return op_mul_ct(c, numerator, invp);
}

/* coeff_variation, stats.hpp:216-233 (default SignConfig) */
static ct_t coeff_variation(ctx_t* c, const col_t* col, double B, const cfg_t* k) {
  require_nonempty(c, col);
  const ct_t mu_b = mean_scaled(c, col, B);
  if (c->p.debug_checks && fabs(first_slot(&mu_b)) < 0.01)
    raise_err(c, E_NEAR_ZERO_MEAN, "coeff_variation: |mean| < 0.01 B");
  const ct_t sgn = crypto_sign(c, mu_b, 0, 7, NULL, NULL, 0);
  const ct_t mu_pos = op_mul_ct(c, mu_b, sgn);
  const ct_t inv_mu = crypto_inv(c, mu_pos, B, k, ALL_SLOTS);
  const ct_t var_b = variance_scaled(c, col, B);
  ct_t sigma = crypto_sqrt(c, var_b, B * B, k->cheb_degree, ALL_SLOTS);
  if (sigma.level < 1 && c->p.auto_bootstrap) sigma = op_bootstrap(c, sigma);
  const ct_t ratio = op_mul_ct(c, sigma, inv_mu);
  return op_mul_ct(c, ratio, sgn);
}

/* pearson, stats.hpp:239-265 */
static ct_t pearson(ctx_t* c, const col_t* x, const col_t* y, double B, const cfg_t* k) {
  require_nonempty(c, x);
  require_nonempty(c, y);
  if (x->n_valid != y->n_valid)
    raise_err(c, E_LENGTH_MISMATCH, "pearson: columns differ in element count");
  ct_t mux, varx, muy, vary;
  moments(c, x, B, &mux, &varx);
  moments(c, y, B, &muy, &vary);
  if (c->p.debug_checks) {
    if (first_slot(&varx) * B * B < 1e-9 || first_slot(&vary) * B * B < 1e-9)
      raise_err(c, E_DEGENERATE_VARIANCE, "pearson: degenerate column variance");
  }
  const ct_t inv_x = crypto_invsqrt(c, varx, B * B, k, ALL_SLOTS);
  const ct_t inv_y = crypto_invsqrt(c, vary, B * B, k, ALL_SLOTS);
  ct_t* cx = centered_chunks(c, x, mux, 1);
  ct_t* cy = centered_chunks(c, y, muy, 0);
  ct_t* prods = (ct_t*)amalloc(c, (x->nchunks + 1) * sizeof(ct_t));
  for (size_t i = 0; i < x->nchunks; ++i) prods[i] = op_mul_ct(c, cx[i], cy[i]);
  const ct_t cov = mean_of_chunks(c, prods, x->nchunks, x->n_valid);
  const ct_t r = op_mul_ct(c, cov, inv_x);
  return op_mul_ct(c, r, inv_y);
}

/* ------------------------------------------------------------------------ */
/* ABI entry points                                                          */
static void put_ct(const ct_t* c, double* out, int32_t* lvl) {
  if (out && c->n) memcpy(out, c->v, c->n * sizeof(double));
  if (lvl) *lvl = c->level;
}
static void put_meter(const ctx_t* c, orc_meter* m) {
  if (m) *m = c->m;
}

#define ENTER(ctxv, p)                    \
  ctx_t ctxv;                             \
  ctx_init(&ctxv, p);                     \
  {                                       \
    int _code = setjmp(ctxv.jb);          \
    if (_code) {                          \
      put_meter(&ctxv, meter);            \
      arena_free(&ctxv);                  \
      return _code;                       \
    }                                     \
  }                                       \
  params_validate(&ctxv)

#define LEAVE(ctxv)     \
  put_meter(&ctxv, meter); \
  arena_free(&ctxv);    \
  return 0

int ora_encrypt(const orc_params* p, const double* v, uint64_t n, double* out, int32_t* lvl) {
  orc_meter* meter = NULL;
  ENTER(c, p);
  ct_t r = op_encrypt(&c, v, (size_t)n);
  put_ct(&r, out, lvl);
  LEAVE(c);
}

int ora_op(const orc_params* p, int op, const double* a, uint64_t na, int32_t la,
           const double* b, uint64_t nb, int32_t lb, double k, const double* vec,
           uint64_t nvec, int64_t rot, uint64_t n_valid, double* out, int32_t* lout,
           orc_meter* meter) {
  ENTER(c, p);
  ct_t A = ct_from(&c, a, (size_t)na, la);
  ct_t B = b ? ct_from(&c, b, (size_t)nb, lb) : ct_new(&c, 0, 0);
  ct_t r;
  switch (op) {
    case ORC_OP_ADD: r = op_add(&c, A, B); break;
    case ORC_OP_SUB: r = op_sub(&c, A, B); break;
    case ORC_OP_ADD_PT: r = op_add_pt(&c, A, k); break;
    case ORC_OP_MUL_CT: r = op_mul_ct(&c, A, B); break;
    case ORC_OP_MUL_PT: r = op_mul_pt(&c, A, k); break;
    case ORC_OP_MUL_PT_VEC: r = op_mul_pt_vec(&c, A, vec, (size_t)nvec); break;
    case ORC_OP_ROTATE: r = op_rotate(&c, A, (long)rot); break;
    case ORC_OP_BOOTSTRAP: r = op_bootstrap(&c, A); break;
    case ORC_OP_SUM_ALL: r = op_sum_all(&c, A, (size_t)n_valid); break;
    default: raise_err(&c, E_ERROR, "ora_op: bad op");
  }
  put_ct(&r, out, lout);
  LEAVE(c);
}

int ora_fit(int kind, double S, int32_t degree, double lo, double hi, double* coeffs) {
  orc_meter* meter = NULL;
  orc_params dummy = {1, 1, 1, 0, 0, 0, 0};
  ENTER(c, &dummy);
  cheb_fit(&c, target_of(kind), &S, degree, lo, hi, coeffs);
  LEAVE(c);
}

double ora_eval_plain(const double* coeffs, uint64_t ncoef, double lo, double hi, double x,
                      int32_t* extrapolated) {
  if (extrapolated) *extrapolated = (x < lo || x > hi) ? 1 : 0;
  return cheb_plain(coeffs, (int)ncoef, lo, hi, x);
}

int ora_eval_encrypted(const orc_params* p, const double* coeffs, uint64_t ncoef, double lo,
                       double hi, const double* x, int32_t lx, double* out, int32_t* lout,
                       orc_meter* meter) {
  ENTER(c, p);
  ct_t X = ct_from(&c, x, S_of(&c), lx);
  ct_t r = eval_encrypted(&c, coeffs, (int)ncoef, lo, hi, X);
  put_ct(&r, out, lout);
  LEAVE(c);
}

int ora_newton_refine(const orc_params* p, const double* x, int32_t lx, const double* y0,
                      int32_t ly, int32_t n, int32_t iters, uint64_t n_valid, double* out,
                      int32_t* lout, orc_meter* meter) {
  ENTER(c, p);
  ct_t X = ct_from(&c, x, S_of(&c), lx);
  ct_t Y = ct_from(&c, y0, S_of(&c), ly);
  ct_t r = newton_refine(&c, X, Y, n, iters, (size_t)n_valid);
  put_ct(&r, out, lout);
  LEAVE(c);
}

int ora_invroot(const orc_params* p, int which, const double* x, int32_t lx, double S,
                const orc_invroot* cfg, uint64_t n_valid, double* out, int32_t* lout,
                orc_meter* meter) {
  ENTER(c, p);
  const cfg_t k = cfg_of(cfg);
  ct_t X = ct_from(&c, x, S_of(&c), lx);
  ct_t r;
  switch (which) {
    case 0: r = crypto_invsqrt(&c, X, S, &k, (size_t)n_valid); break;
    case 1: r = crypto_inv(&c, X, S, &k, (size_t)n_valid); break;
    case 2: r = baseline_invsqrt(&c, X, S, cfg ? cfg->newton_iters : 21, (size_t)n_valid); break;
    case 3: r = crypto_sqrt(&c, X, S, cfg ? cfg->cheb_degree : 511, (size_t)n_valid); break;
    default: raise_err(&c, E_ERROR, "ora_invroot: bad which");
  }
  put_ct(&r, out, lout);
  LEAVE(c);
}

int ora_crypto_sign(const orc_params* p, const double* x, int32_t lx, int32_t mode,
                    int32_t folds, const double* polys, const uint64_t* poly_len,
                    uint64_t npolys, double* out, int32_t* lout, orc_meter* meter) {
  ENTER(c, p);
  ct_t X = ct_from(&c, x, S_of(&c), lx);
  ct_t r = crypto_sign(&c, X, mode, folds, polys, poly_len, (size_t)npolys);
  put_ct(&r, out, lout);
  LEAVE(c);
}

int ora_stat(const orc_params* p, int which, const double* x, uint64_t n, const double* y,
             uint64_t ny, double B, const orc_invroot* cfg, double* out, int32_t* lout,
             orc_meter* meter) {
  ENTER(c, p);
  const cfg_t k = cfg_of(cfg);
  const size_t S = S_of(&c);
  col_t cx = encode_column(&c, x, (size_t)n);
  switch (which) {
    case 0: { ct_t r = mean_scaled(&c, &cx, B); put_ct(&r, out, lout); break; }
    case 1: { ct_t r = variance_scaled(&c, &cx, B); put_ct(&r, out, lout); break; }
    case 2: { ct_t r = variance_to_scale(&c, &cx, B); put_ct(&r, out, lout); break; }
    case 3: {
      ct_t mu, var;
      moments(&c, &cx, B, &mu, &var);
      put_ct(&mu, out, lout);
      put_ct(&var, out ? out + S : NULL, lout ? lout + 1 : NULL);
      break;
    }
    case 4: {
      col_t z = znorm(&c, &cx, B, &k);
      if (out) decode_column(&c, &z, out);
      if (lout) *lout = z.nchunks ? z.chunks[0].level : 0;
      break;
    }
    case 5: { ct_t r = std_moment(&c, &cx, B, &k, 4); put_ct(&r, out, lout); break; }
    case 6: { ct_t r = std_moment(&c, &cx, B, &k, 3); put_ct(&r, out, lout); break; }
    case 7: { ct_t r = coeff_variation(&c, &cx, B, &k); put_ct(&r, out, lout); break; }
    case 8: {
      col_t cy = encode_column(&c, y, (size_t)ny);
      ct_t r = pearson(&c, &cx, &cy, B, &k);
      put_ct(&r, out, lout);
      break;
    }
    default: raise_err(&c, E_ERROR, "ora_stat: bad which");
  }
  LEAVE(c);
}

static int znorm_once(const orc_params* p, const double* x, uint64_t n, double B, double* out,
                      orc_meter* meter) {
  const cfg_t k = cfg_of(NULL);
  ENTER(c, p);
  col_t cx = encode_column(&c, x, (size_t)n);
  col_t z = znorm(&c, &cx, B, &k);
  if (out) decode_column(&c, &z, out);
  LEAVE(c);
}

int ora_znorm_reps(const orc_params* p, const double* x, uint64_t n, double B, int32_t reps,
                   double* out, orc_meter* meter) {
  for (int r = 0; r < reps; ++r) {
    const int rc = znorm_once(p, x, n, B, r == reps - 1 ? out : NULL, meter);
    if (rc) return rc;
  }
  return 0;
}

/* ------------------------------------------------------------------------ */
/* data.hpp:148-208 generators; std::mt19937_64 restated                     */
typedef struct {
  uint64_t mt[312];
  int idx;
} mt64_t;

static void mt64_seed(mt64_t* s, uint64_t seed) {
  s->mt[0] = seed;
  for (int i = 1; i < 312; ++i)
    s->mt[i] = 6364136223846793005ULL * (s->mt[i - 1] ^ (s->mt[i - 1] >> 62)) + (uint64_t)i;
  s->idx = 312;
}

static uint64_t mt64_next(mt64_t* s) {
  if (s->idx >= 312) {
    for (int i = 0; i < 312; ++i) {
      const uint64_t x = (s->mt[i] & 0xFFFFFFFF80000000ULL) | (s->mt[(i + 1) % 312] & 0x7FFFFFFFULL);
      uint64_t xa = x >> 1;
      if (x & 1ULL) xa ^= 0xB5026F5AA96619E9ULL;
      s->mt[i] = s->mt[(i + 156) % 312] ^ xa;
    }
    s->idx = 0;
  }
  uint64_t y = s->mt[s->idx++];
  y ^= (y >> 29) & 0x5555555555555555ULL;
  y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
  y ^= (y << 37) & 0xFFF7EEE000000000ULL;
  y ^= y >> 43;
  return y;
}

/* synthetic_uniform, data.hpp:148-160 */
int ora_synthetic_uniform(uint64_t seed, uint64_t n, double lo, double hi, double* out) {
  if (n < 1) { snprintf(g_msg, sizeof g_msg, "synthetic_uniform: n must be >= 1"); return E_ERROR; }
  if (!(lo < hi)) { snprintf(g_msg, sizeof g_msg, "synthetic_uniform: lo must be < hi"); return E_ERROR; }
  mt64_t s;
  mt64_seed(&s, seed);
  for (uint64_t i = 0; i < n; ++i) {
    const double u = (double)(mt64_next(&s) >> 11) * 0x1.0p-53;
    out[i] = lo + u * (hi - lo);
  }
  return 0;
}

/* synthetic_grid, data.hpp:163-173 */
int ora_synthetic_grid(uint64_t n, double lo, double hi, double* out) {
  if (n < 2) { snprintf(g_msg, sizeof g_msg, "synthetic_grid: n must be >= 2"); return E_ERROR; }
  if (!(lo < hi)) { snprintf(g_msg, sizeof g_msg, "synthetic_grid: lo must be < hi"); return E_ERROR; }
  const double step = (hi - lo) / (double)(n - 1);
  for (uint64_t i = 0; i < n; ++i) out[i] = lo + step * (double)i;
  out[n - 1] = hi;
  return 0;
}

/* two_subrange_grid, data.hpp:178-186 */
int ora_two_subrange_grid(uint64_t n, double lo, double hi, double* out) {
  if (!(lo < 1.0 && 1.0 < hi)) return ora_synthetic_grid(n, lo, hi, out);
  int rc = ora_synthetic_grid(n / 2, lo, 1.0, out);
  if (rc) return rc;
  return ora_synthetic_grid(n - n / 2, 1.0, hi, out + n / 2);
}

/* plain.hpp:18-92 */
static double p_mean(const double* x, size_t n) {
  double acc = 0.0;
  for (size_t i = 0; i < n; ++i) acc += x[i];
  return acc / (double)n;
}
static double p_var(const double* x, size_t n) {
  const double mu = p_mean(x, n);
  double acc = 0.0;
  for (size_t i = 0; i < n; ++i) acc += (x[i] - mu) * (x[i] - mu);
  return acc / (double)n;
}

int ora_plain(int which, const double* x, uint64_t n, const double* y, double* out) {
  if (n == 0) { snprintf(g_msg, sizeof g_msg, "plain::mean: empty input"); return E_EMPTY_COLUMN; }
  const size_t N = (size_t)n;
  switch (which) {
    case 0: *out = p_mean(x, N); return 0;
    case 1: *out = p_var(x, N); return 0;
    case 2: {
      const double mu = p_mean(x, N);
      double m2 = 0.0, m3 = 0.0;
      for (size_t i = 0; i < N; ++i) {
        const double d = x[i] - mu;
        m2 += d * d;
        m3 += d * d * d;
      }
      m2 /= (double)N;
      m3 /= (double)N;
      *out = m3 / pow(m2, 1.5);
      return 0;
    }
    case 3: {
      const double mu = p_mean(x, N);
      double m2 = 0.0, m4 = 0.0;
      for (size_t i = 0; i < N; ++i) {
        const double d = x[i] - mu;
        m2 += d * d;
        m4 += d * d * d * d;
      }
      m2 /= (double)N;
      m4 /= (double)N;
      *out = m4 / (m2 * m2);
      return 0;
    }
    case 4: {
      const double mu = p_mean(x, N);
      if (mu == 0.0) { snprintf(g_msg, sizeof g_msg, "plain::coeff_variation: zero mean"); return E_NEAR_ZERO_MEAN; }
      *out = sqrt(p_var(x, N)) * (mu > 0 ? 1.0 : -1.0) / fabs(mu);
      return 0;
    }
    case 5: {
      const double mx = p_mean(x, N), my = p_mean(y, N);
      double cv = 0.0, vx = 0.0, vy = 0.0;
      for (size_t i = 0; i < N; ++i) {
        cv += (x[i] - mx) * (y[i] - my);
        vx += (x[i] - mx) * (x[i] - mx);
        vy += (y[i] - my) * (y[i] - my);
      }
      if (vx == 0.0 || vy == 0.0) { snprintf(g_msg, sizeof g_msg, "plain::pearson: constant column"); return E_DEGENERATE_VARIANCE; }
      *out = cv / sqrt(vx * vy);
      return 0;
    }
    case 6: {
      const double mu = p_mean(x, N);
      const double sd = sqrt(p_var(x, N));
      if (sd == 0.0) { snprintf(g_msg, sizeof g_msg, "plain::znorm: zero variance"); return E_DEGENERATE_VARIANCE; }
      for (size_t i = 0; i < N; ++i) out[i] = (x[i] - mu) / sd;
      return 0;
    }
    default: snprintf(g_msg, sizeof g_msg, "ora_plain: bad which"); return E_ERROR;
  }
}
