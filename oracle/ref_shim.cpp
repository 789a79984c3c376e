/* ref_shim.cpp — TEST INFRASTRUCTURE ONLY (oracle/).
 *
 * A C-ABI face over the *unmodified* reference headers
 * (/root/reference/proj/include/hestat/*.hpp), compiled by oracle/Makefile into
 * oracle/_ref/libhestat_ref.so.  Nothing here re-implements the reference: every
 * entry point constructs the reference's own objects and calls the reference's own
 * functions, then copies slot vectors / levels / meters out through plain pointers.
 *
 * Used by: tests/ (golden-vector generation, pinning oracle/hestat_oracle.c bit-for-bit)
 * and bench.py's cpu_baseline / `--impl reference` legs.  Never linked into the product.
 *
 * The ABI is shared with oracle/hestat_oracle.c (prefix `ora_` there, `ref_` here)
 * so the same Python harness (tests/oracle_abi.py) drives either.
 */
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>
#include <vector>

#include "hestat/hestat.hpp"

using namespace hestat;

extern "C" {

struct orc_params {
  uint64_t slot_count;
  int32_t max_level;
  int32_t scale_bits;
  int32_t quantize;
  int32_t auto_bootstrap;
  int32_t debug_checks;
  int32_t _pad;
};
struct orc_meter {
  uint64_t mul_ct, mul_pt, add, rotate, bootstrap;
};
struct orc_invroot {
  int32_t n, cheb_degree, newton_iters, baseline_mode, baseline_iters, _pad;
};

}  // extern "C"

namespace {

thread_local std::string g_msg;

CkksParams to_params(const orc_params* p) {
  CkksParams c;
  c.slot_count = static_cast<std::size_t>(p->slot_count);
  c.max_level = p->max_level;
  c.scale_bits = p->scale_bits;
  c.quantize = p->quantize != 0;
  c.auto_bootstrap = p->auto_bootstrap != 0;
  c.debug_checks = p->debug_checks != 0;
  return c;
}

InvRootConfig to_cfg(const orc_invroot* c) {
  InvRootConfig r;
  if (!c) return r;
  r.n = c->n;
  r.cheb_degree = c->cheb_degree;
  r.newton_iters = c->newton_iters;
  r.baseline_mode = c->baseline_mode != 0;
  r.baseline_iters = c->baseline_iters;
  return r;
}

void put_meter(const EvalContext& ctx, orc_meter* m) {
  if (!m) return;
  m->mul_ct = ctx.meter().mul_ct;
  m->mul_pt = ctx.meter().mul_pt;
  m->add = ctx.meter().add;
  m->rotate = ctx.meter().rotate;
  m->bootstrap = ctx.meter().bootstrap;
}

void put_ct(const Ciphertext& c, double* out, int32_t* lvl) {
  if (out) std::memcpy(out, c.slots().data(), c.size() * sizeof(double));
  if (lvl) *lvl = c.level();
}

// Error codes shared by hs_*, ref_* and ora_* (see include/hestat_gpu.h).
int code_of(const std::exception& e) {
  g_msg = e.what();
  if (dynamic_cast<const too_many_values*>(&e)) return 2;
  if (dynamic_cast<const level_exhausted*>(&e)) return 3;
  if (dynamic_cast<const length_mismatch*>(&e)) return 4;
  if (dynamic_cast<const dirty_padding*>(&e)) return 5;
  if (dynamic_cast<const non_finite_target*>(&e)) return 6;
  if (dynamic_cast<const domain_violation*>(&e)) return 7;
  if (dynamic_cast<const divergence*>(&e)) return 8;
  if (dynamic_cast<const empty_column*>(&e)) return 9;
  if (dynamic_cast<const degenerate_variance*>(&e)) return 10;
  if (dynamic_cast<const near_zero_mean*>(&e)) return 11;
  if (dynamic_cast<const io_error*>(&e)) return 12;
  if (dynamic_cast<const missing_column*>(&e)) return 13;
  if (dynamic_cast<const unparsable_cell*>(&e)) return 14;
  if (dynamic_cast<const non_finite_value*>(&e)) return 15;
  if (dynamic_cast<const zero_reference*>(&e)) return 16;
  return 1;
}

Ciphertext make_ct(const double* v, std::size_t n, int level) {
  return Ciphertext(std::vector<double>(v, v + n), level);
}

EncryptedColumn make_col(EvalContext& ctx, const double* v, std::size_t n) {
  return encode_column(ctx, std::span<const double>(v, n), "x");
}

// Fixed fit targets (the reference's fit() takes a std::function; the C ABI
// enumerates the targets the tests and benchmarks use).
std::function<double(double)> target_of(int kind, double S) {
  switch (kind) {
    case 0: return [S](double t) { return scaled_target(ScaledTargetKind::InvSqrtShifted, S, t); };
    case 1: return [S](double t) { return scaled_target(ScaledTargetKind::SqrtShifted, S, t); };
    case 2: return [](double x) { return x; };
    case 3: return [](double x) { return x * x; };
    case 4: return [](double x) { return std::exp(x); };
    case 5: return [](double x) { return 1.0 / (2.0 + x); };
    case 6: return [](double x) { return std::cos(2 * x); };
    case 7: return [](double x) { return std::cos(3.0 * x); };
    case 8: return [](double) { return 1.0; };
    case 9: return [](double x) { return std::sqrt(x); };
    default: return [](double) { return 0.0; };
  }
}

}  // namespace

#define GUARD_BEGIN try {
#define GUARD_END(ctxp)                       \
  }                                           \
  catch (const std::exception& e) {           \
    if (ctxp) put_meter(*(ctxp), meter);      \
    return code_of(e);                        \
  }

extern "C" {

const char* ref_last_error(void) { return g_msg.c_str(); }

/* op codes for ref_op */
enum {
  OP_ADD = 0, OP_SUB, OP_ADD_PT, OP_MUL_CT, OP_MUL_PT, OP_MUL_PT_VEC, OP_ROTATE,
  OP_BOOTSTRAP, OP_SUM_ALL
};

int ref_encrypt(const orc_params* p, const double* v, uint64_t n, double* out, int32_t* lvl) {
  try {
    EvalContext ctx(to_params(p));
    put_ct(ctx.encrypt(std::span<const double>(v, n)), out, lvl);
    return 0;
  } catch (const std::exception& e) {
    return code_of(e);
  }
}

/* One EvalContext op. a/b are raw slot vectors of length na/nb at levels la/lb
 * (Ciphertext(vector, level) — no re-quantisation), c is the scalar, vec the
 * plaintext vector (length nvec), k the rotation, n_valid for sum_all_slots.
 * The meter is reset per call. */
int ref_op(const orc_params* p, int op, const double* a, uint64_t na, int32_t la,
           const double* b, uint64_t nb, int32_t lb, double c, const double* vec,
           uint64_t nvec, int64_t k, uint64_t n_valid, double* out, int32_t* lout,
           orc_meter* meter) {
  EvalContext* cp = nullptr;
  GUARD_BEGIN
  EvalContext ctx(to_params(p));
  cp = &ctx;
  Ciphertext A = make_ct(a, na, la);
  Ciphertext B = b ? make_ct(b, nb, lb) : Ciphertext();
  Ciphertext r;
  switch (op) {
    case OP_ADD: r = ctx.add_ct(A, B); break;
    case OP_SUB: r = ctx.sub_ct(A, B); break;
    case OP_ADD_PT: r = ctx.add_pt(A, c); break;
    case OP_MUL_CT: r = ctx.mul_ct(A, B); break;
    case OP_MUL_PT: r = ctx.mul_pt(A, c); break;
    case OP_MUL_PT_VEC: r = ctx.mul_pt(A, std::span<const double>(vec, nvec)); break;
    case OP_ROTATE: r = ctx.rotate(A, static_cast<long>(k)); break;
    case OP_BOOTSTRAP: r = ctx.bootstrap(A); break;
    case OP_SUM_ALL: r = ctx.sum_all_slots(A, static_cast<std::size_t>(n_valid)); break;
    default: throw error("ref_op: bad op");
  }
  put_ct(r, out, lout);
  put_meter(ctx, meter);
  cp = nullptr;
  return 0;
  GUARD_END(cp)
}

int ref_fit(int kind, double S, int32_t degree, double lo, double hi, double* coeffs) {
  try {
    ChebyshevSeries s = fit(target_of(kind, S), degree, lo, hi);
    std::memcpy(coeffs, s.coeffs.data(), s.coeffs.size() * sizeof(double));
    return 0;
  } catch (const std::exception& e) {
    return code_of(e);
  }
}

double ref_eval_plain(const double* coeffs, uint64_t ncoef, double lo, double hi, double x,
                      int32_t* extrapolated) {
  ChebyshevSeries s;
  s.coeffs.assign(coeffs, coeffs + ncoef);
  s.domain_lo = lo;
  s.domain_hi = hi;
  bool ex = false;
  const double r = eval_plain(s, x, &ex);
  if (extrapolated) *extrapolated = ex ? 1 : 0;
  return r;
}

int ref_eval_encrypted(const orc_params* p, const double* coeffs, uint64_t ncoef, double lo,
                       double hi, const double* x, int32_t lx, double* out, int32_t* lout,
                       orc_meter* meter) {
  EvalContext* cp = nullptr;
  GUARD_BEGIN
  EvalContext ctx(to_params(p));
  cp = &ctx;
  ChebyshevSeries s;
  s.coeffs.assign(coeffs, coeffs + ncoef);
  s.domain_lo = lo;
  s.domain_hi = hi;
  Ciphertext r = eval_encrypted(ctx, s, make_ct(x, ctx.params().slot_count, lx));
  put_ct(r, out, lout);
  put_meter(ctx, meter);
  cp = nullptr;
  return 0;
  GUARD_END(cp)
}

int ref_newton_refine(const orc_params* p, const double* x, int32_t lx, const double* y0,
                      int32_t ly, int32_t n, int32_t iters, uint64_t n_valid, double* out,
                      int32_t* lout, orc_meter* meter) {
  EvalContext* cp = nullptr;
  GUARD_BEGIN
  EvalContext ctx(to_params(p));
  cp = &ctx;
  const std::size_t S = ctx.params().slot_count;
  Ciphertext r = newton_refine(ctx, make_ct(x, S, lx), make_ct(y0, S, ly), n, iters,
                               static_cast<std::size_t>(n_valid));
  put_ct(r, out, lout);
  put_meter(ctx, meter);
  cp = nullptr;
  return 0;
  GUARD_END(cp)
}

/* which: 0 crypto_invsqrt, 1 crypto_inv, 2 baseline_invsqrt (iters = cfg->newton_iters),
 *        3 crypto_sqrt (degree = cfg->cheb_degree) */
int ref_invroot(const orc_params* p, int which, const double* x, int32_t lx, double S,
                const orc_invroot* cfg, uint64_t n_valid, double* out, int32_t* lout,
                orc_meter* meter) {
  EvalContext* cp = nullptr;
  GUARD_BEGIN
  EvalContext ctx(to_params(p));
  cp = &ctx;
  const std::size_t nv = static_cast<std::size_t>(n_valid);
  Ciphertext X = make_ct(x, ctx.params().slot_count, lx);
  Ciphertext r;
  switch (which) {
    case 0: r = crypto_invsqrt(ctx, X, S, to_cfg(cfg), nv); break;
    case 1: r = crypto_inv(ctx, X, S, to_cfg(cfg), nv); break;
    case 2: r = baseline_invsqrt(ctx, X, S, cfg ? cfg->newton_iters : 21, nv); break;
    case 3: r = crypto_sqrt(ctx, X, S, cfg ? cfg->cheb_degree : 511, nv); break;
    default: throw error("ref_invroot: bad which");
  }
  put_ct(r, out, lout);
  put_meter(ctx, meter);
  cp = nullptr;
  return 0;
  GUARD_END(cp)
}

/* crypto_sign: mode 0 = g3 composition, 1 = custom (polys packed: npolys arrays of
 * poly_len[i] power-basis coefficients, concatenated in `polys`). */
int ref_crypto_sign(const orc_params* p, const double* x, int32_t lx, int32_t mode,
                    int32_t folds, const double* polys, const uint64_t* poly_len,
                    uint64_t npolys, double* out, int32_t* lout, orc_meter* meter) {
  EvalContext* cp = nullptr;
  GUARD_BEGIN
  EvalContext ctx(to_params(p));
  cp = &ctx;
  SignConfig sc;
  sc.mode = mode == 0 ? SignConfig::Mode::G3Composition : SignConfig::Mode::CustomComposite;
  sc.folds = folds;
  std::size_t off = 0;
  for (uint64_t i = 0; i < npolys; ++i) {
    sc.custom_polys.emplace_back(polys + off, polys + off + poly_len[i]);
    off += poly_len[i];
  }
  Ciphertext r = crypto_sign(ctx, make_ct(x, ctx.params().slot_count, lx), sc);
  put_ct(r, out, lout);
  put_meter(ctx, meter);
  cp = nullptr;
  return 0;
  GUARD_END(cp)
}

/* Statistics over a column given as raw values (encode_column inside).
 * which: 0 mean_scaled, 1 variance_scaled, 2 variance_to_scale (B is S),
 *        3 moments (out = mu slots ++ var slots, lout[0..1]), 4 znorm (out = decoded
 *        column, n values; lout[0] = level of chunk 0), 5 kurtosis, 6 skewness,
 *        7 coeff_variation, 8 pearson (y required).
 * Ciphertext-valued results write all slot_count slots. */
int ref_stat(const orc_params* p, int which, const double* x, uint64_t n, const double* y,
             uint64_t ny, double B, const orc_invroot* cfg, double* out, int32_t* lout,
             orc_meter* meter) {
  EvalContext* cp = nullptr;
  GUARD_BEGIN
  EvalContext ctx(to_params(p));
  cp = &ctx;
  EncryptedColumn cx = make_col(ctx, x, n);
  const InvRootConfig c = to_cfg(cfg);
  const std::size_t S = ctx.params().slot_count;
  switch (which) {
    case 0: put_ct(mean_scaled(ctx, cx, B), out, lout); break;
    case 1: put_ct(variance_scaled(ctx, cx, B), out, lout); break;
    case 2: put_ct(variance_to_scale(ctx, cx, B), out, lout); break;
    case 3: {
      MomentSet m = moments(ctx, cx, B);
      put_ct(m.ct_mu, out, lout);
      put_ct(m.ct_var, out ? out + S : nullptr, lout ? lout + 1 : nullptr);
      break;
    }
    case 4: {
      EncryptedColumn z = znorm(ctx, cx, B, c);
      std::vector<double> d = decode_column(ctx, z);
      if (out) std::memcpy(out, d.data(), d.size() * sizeof(double));
      if (lout) *lout = z.chunks.empty() ? 0 : z.chunks[0].level();
      break;
    }
    case 5: put_ct(kurtosis(ctx, cx, B, c), out, lout); break;
    case 6: put_ct(skewness(ctx, cx, B, c), out, lout); break;
    case 7: put_ct(coeff_variation(ctx, cx, B, SignConfig{}, c), out, lout); break;
    case 8: {
      EncryptedColumn cy = make_col(ctx, y, ny);
      put_ct(pearson(ctx, cx, cy, B, c), out, lout);
      break;
    }
    default: throw error("ref_stat: bad which");
  }
  put_meter(ctx, meter);
  cp = nullptr;
  return 0;
  GUARD_END(cp)
}

/* Synthetic data generators of data.hpp (seeded mt19937_64, 53-bit). */
int ref_synthetic_uniform(uint64_t seed, uint64_t n, double lo, double hi, double* out) {
  try {
    auto v = synthetic_uniform(seed, n, lo, hi);
    std::memcpy(out, v.data(), v.size() * sizeof(double));
    return 0;
  } catch (const std::exception& e) {
    return code_of(e);
  }
}
int ref_synthetic_grid(uint64_t n, double lo, double hi, double* out) {
  try {
    auto v = synthetic_grid(n, lo, hi);
    std::memcpy(out, v.data(), v.size() * sizeof(double));
    return 0;
  } catch (const std::exception& e) {
    return code_of(e);
  }
}
int ref_two_subrange_grid(uint64_t n, double lo, double hi, double* out) {
  try {
    auto v = two_subrange_grid(n, lo, hi);
    std::memcpy(out, v.data(), v.size() * sizeof(double));
    return 0;
  } catch (const std::exception& e) {
    return code_of(e);
  }
}

/* Plain fp64 statistics (plain.hpp). which: 0 mean 1 variance 2 skewness
 * 3 kurtosis_ratio 4 coeff_variation 5 pearson; 6 znorm (writes n values). */
int ref_plain(int which, const double* x, uint64_t n, const double* y, double* out) {
  try {
    std::span<const double> X(x, n);
    switch (which) {
      case 0: *out = plain::mean(X); break;
      case 1: *out = plain::variance(X); break;
      case 2: *out = plain::skewness(X); break;
      case 3: *out = plain::kurtosis_ratio(X); break;
      case 4: *out = plain::coeff_variation(X); break;
      case 5: *out = plain::pearson(X, std::span<const double>(y, n)); break;
      case 6: {
        auto z = plain::znorm(X);
        std::memcpy(out, z.data(), z.size() * sizeof(double));
        break;
      }
      default: throw error("ref_plain: bad which");
    }
    return 0;
  } catch (const std::exception& e) {
    return code_of(e);
  }
}

/* CPU-baseline driver: `reps` independent ZNorm runs (one EvalContext each,
 * the reference's sanctioned concurrency model) over the same
 * column; returns the decoded output of the last run.  Used by bench.py. */
int ref_znorm_reps(const orc_params* p, const double* x, uint64_t n, double B, int32_t reps,
                   double* out, orc_meter* meter) {
  EvalContext* cp = nullptr;
  GUARD_BEGIN
  for (int r = 0; r < reps; ++r) {
    EvalContext ctx(to_params(p));
    cp = &ctx;
    EncryptedColumn z = znorm(ctx, make_col(ctx, x, n), B);
    if (r == reps - 1) {
      std::vector<double> d = decode_column(ctx, z);
      if (out) std::memcpy(out, d.data(), d.size() * sizeof(double));
      put_meter(ctx, meter);
    }
    cp = nullptr;
  }
  return 0;
  GUARD_END(cp)
}

}  // extern "C"
