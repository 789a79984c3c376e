// flow.h — the reference's control flow for every hot-path entry point, written
// once and instantiated over two backends (backends.h):
//
//   SymB  level/meter ledger only (no values).  Runs before a fused launch so
//         levels, CostMeter counts, auto-bootstrap decisions and
//         level_exhausted / argument errors are exactly the reference's,
//         raised before any device work.
//   DevB  op-by-op: every EvalContext op is one CUDA kernel (ops.cu) with the
//         literal q() formula; debug-mode value checks read the slots back.
//         This is the always-exact path used for debug_checks, off-grid inputs
//         and shapes the fused kernels do not cover.
//
// Each function cites the reference lines it follows
// (/root/reference/proj/include/hestat/...).  Auto-bootstrap and level logic is
// inside the backends' op implementations, exactly where ckks.hpp puts it.
#pragma once

#include <cmath>
#include <concepts>
#include <cstddef>
#include <limits>
#include <memory>
#include <string>
#include <vector>

#include "core.h"
#include "series.h"

namespace hsg {
namespace flow {

constexpr size_t kAllSlots = std::numeric_limits<size_t>::max();  // primitives.hpp:20

struct InvCfg {  // InvRootConfig, primitives.hpp:23-40
  int n = 2;
  int cheb_degree = 511;
  int newton_iters = 6;
  bool baseline_mode = false;
  int baseline_iters = 0;
  int effective_baseline_iters() const { return baseline_iters > 0 ? baseline_iters : (n == 1 ? 25 : 21); }
  void validate() const {
    if (n != 1 && n != 2) fail(HS_E_ERROR, "InvRootConfig: n must be 1 or 2");
    if (newton_iters < 0) fail(HS_E_ERROR, "InvRootConfig: newton_iters < 0");
    if (cheb_degree < 0) fail(HS_E_ERROR, "InvRootConfig: cheb_degree < 0");
  }
};

struct SignCfg {  // SignConfig, primitives.hpp:59-70
  int mode = 0;   // 0 G3Composition, 1 CustomComposite
  int folds = 7;
  std::vector<std::vector<double>> custom_polys;
};

template <class C>
struct Col {  // EncryptedColumn, column.hpp:19-23
  std::vector<C> chunks;
  size_t n_valid = 0;
};

// ---------------------------------------------------------------------------
// chebyshev.hpp:113-163 — BSGS evaluation p = q * T_g + r
template <class B>
class Bsgs {
 public:
  using C = typename B::C;
  Bsgs(B& b, const C& x) : b_(b), x_(x) {}

  C run(const std::vector<double>& coeffs) {  // :117-125
    const int d = static_cast<int>(coeffs.size()) - 1;
    if (d <= 0) return b_.add_pt(b_.sub_ct(x_, x_), coeffs.empty() ? 0.0 : coeffs[0]);
    build_powers(cheb_depth(d));
    // Backends with a batched tree (RnsB): a full tree (d = 2^K - 1) runs level by level,
    // one batched op per stage -- the same ops on the same operands as eval() below.
    if constexpr (requires(B& bb, const C& xx, const std::vector<double>& cc, const std::vector<C>& pp) {
                    bb.bsgs_full_tree(xx, cc, pp);
                  }) {
      const int K = cheb_depth(d);
      if (d == (1 << K) - 1 && K >= 2 && b_.bsgs_batch_ok(x_, pw_, K)) return b_.bsgs_full_tree(x_, coeffs, pw_);
    }
    return eval(coeffs);
  }

 private:
  void build_powers(int depth) {  // :130-138
    for (int g = 1, j = 0; 2 * g < (1 << depth); g *= 2, ++j) {
      const C tg = g == 1 ? x_ : pw_[j];
      const C sq = b_.mul_ct(tg, tg);
      if (static_cast<int>(pw_.size()) <= j + 1) pw_.resize(j + 2);
      pw_[j + 1] = b_.add_pt(b_.add_ct(sq, sq), -1.0);
    }
  }

  C eval(const std::vector<double>& c) {  // :140-158
    const int d = static_cast<int>(c.size()) - 1;
    if (d <= 1) {
      const C r = b_.mul_pt(x_, d == 1 ? c[1] : 0.0);
      return b_.add_pt(r, c[0]);
    }
    std::vector<double> q, r;
    const int g = split_series(c, &q, &r);
    int j = 0;
    while ((1 << j) < g) ++j;
    const C& tg = pw_.at(j);
    const C head = q.size() == 1 ? b_.mul_pt(tg, q[0]) : b_.mul_ct(eval(q), tg);
    const C rest = eval(r);
    return b_.add_ct(head, rest);
  }

  B& b_;
  const C& x_;
  std::vector<C> pw_{C{}};  // pw_[j] = T_{2^j}; slot 0 unused (x_)
};

// chebyshev.hpp:171-189
template <class B>
typename B::C eval_encrypted(B& b, const Series& s, const typename B::C& ct) {
  if (s.coeffs.empty()) fail(HS_E_ERROR, "eval_encrypted: empty series");
  if (b.params().debug) b.check_eval_domain(ct, s.lo, s.hi);
  const int need = cheb_depth(s.degree()) + (s.native() ? 0 : 1);
  typename B::C x = ct;
  if (b.level(x) < need && b.params().auto_bootstrap) x = b.bootstrap(x);
  if (!s.native()) {
    const double span = s.hi - s.lo;
    x = b.add_pt(b.mul_pt(x, 2.0 / span), -(s.lo + s.hi) / span);
  }
  return Bsgs<B>(b, x).run(s.coeffs);
}

// ---------------------------------------------------------------------------
// primitives.hpp:105-132 — y <- ((n+1)/n) y - x_op * y^(n+1), balanced tree
template <class B>
typename B::C newton_loop(B& b, const typename B::C& x_op, typename B::C y, int n, int iters,
                          size_t n_valid) {
  using C = typename B::C;
  const int per_iter = cheb_depth(n + 1);
  C x = x_op;
  if (b.level(x) < per_iter && b.params().auto_bootstrap) x = b.bootstrap(x);
  for (int i = 0; i < iters; ++i) {
    if (b.level(y) < per_iter && b.params().auto_bootstrap) y = b.bootstrap(y);
    std::vector<C> f;
    f.reserve(static_cast<size_t>(n) + 2);
    f.push_back(x);
    for (int j = 0; j < n + 1; ++j) f.push_back(y);
    while (f.size() > 1) {
      std::vector<C> nx;
      nx.reserve(f.size() / 2 + 1);
      for (size_t k = 0; k + 1 < f.size(); k += 2) nx.push_back(b.mul_ct(f[k], f[k + 1]));
      if (f.size() % 2 == 1) nx.push_back(f.back());
      f = std::move(nx);
    }
    const C linear = b.mul_pt(y, (n + 1.0) / n);
    y = b.sub_ct(linear, f.front());
    if (b.params().debug) b.check_divergence(y, n_valid);  // :89-96
  }
  return y;
}

// primitives.hpp:152-158
template <class B>
typename B::C newton_refine(B& b, const typename B::C& x, const typename B::C& y0, int n, int iters,
                            size_t n_valid) {
  if (n < 1) fail(HS_E_ERROR, "newton_refine: n must be >= 1");
  const typename B::C x_op = n >= 2 ? b.mul_pt(x, 1.0 / n) : x;
  return newton_loop(b, x_op, y0, n, iters, n_valid);
}

// primitives.hpp:173-184
template <class B>
typename B::C baseline_invsqrt(B& b, const typename B::C& ct, double S, int iters, size_t n_valid) {
  if (b.params().debug) b.check_open_domain(ct, n_valid, 0.0, 1.0, "baseline_invsqrt");
  typename B::C y = b.encrypt_const(1.0);
  if (iters > 0) {
    const typename B::C x_op = b.mul_pt(ct, 0.5);
    y = newton_loop(b, x_op, y, 2, iters, n_valid);
  }
  return b.mul_pt(y, 1.0 / std::sqrt(S));
}

// primitives.hpp:186-208
template <class B>
typename B::C crypto_invsqrt(B& b, const typename B::C& ct, double S, const InvCfg& cfg, size_t n_valid) {
  cfg.validate();
  if (S <= 0.0) fail(HS_E_ERROR, "crypto_invsqrt: scale must be positive");
  if (cfg.baseline_mode) return baseline_invsqrt(b, ct, S, cfg.effective_baseline_iters(), n_valid);
  if (b.params().debug) b.check_open_domain(ct, n_valid, 0.0, 2.0, "crypto_invsqrt");
  const Series seed = fit_scaled(TargetKind::InvSqrtShifted, S, cfg.cheb_degree);
  const typename B::C arg = b.add_pt(ct, -1.0);
  typename B::C y = eval_encrypted(b, seed, arg);
  y = b.bootstrap(y);
  if (cfg.newton_iters > 0) {
    const typename B::C x_op = b.mul_pt(ct, S / 2.0);
    y = newton_loop(b, x_op, y, 2, cfg.newton_iters, n_valid);
  }
  return y;
}

// primitives.hpp:211-217
template <class B>
typename B::C crypto_inv(B& b, const typename B::C& ct, double S, const InvCfg& cfg, size_t n_valid) {
  typename B::C y = crypto_invsqrt(b, ct, S, cfg, n_valid);
  if (b.level(y) < 1 && b.params().auto_bootstrap) y = b.bootstrap(y);
  return b.mul_ct(y, y);
}

// primitives.hpp:222-238
template <class B>
typename B::C crypto_sqrt(B& b, const typename B::C& ct, double S, int degree, size_t n_valid) {
  if (S <= 0.0) fail(HS_E_ERROR, "crypto_sqrt: scale must be positive");
  if (b.params().debug) b.check_sqrt_domain(ct, n_valid);
  const Series s = fit_scaled(TargetKind::SqrtShifted, S, degree);
  return eval_encrypted(b, s, b.add_pt(ct, -1.0));
}

// primitives.hpp:279-300 (stages from sign_stages(): g3 or odd custom series)
template <class B>
typename B::C crypto_sign(B& b, const typename B::C& ct, const SignCfg& cfg) {
  if (cfg.folds < 1) fail(HS_E_ERROR, "crypto_sign: folds must be >= 1");
  if (b.params().debug) b.check_sign_domain(ct);
  const std::vector<Series> stages = sign_stages(cfg.mode, cfg.custom_polys);
  typename B::C y = ct;
  for (int f = 0; f < cfg.folds; ++f) y = eval_encrypted(b, stages[static_cast<size_t>(f) % stages.size()], y);
  return y;
}

// ---------------------------------------------------------------------------
// stats.hpp
template <class C>
void require_nonempty(const Col<C>& col) {  // :26-29
  if (col.n_valid == 0 || col.chunks.empty()) fail(HS_E_EMPTY_COLUMN, "statistic on an empty column");
}

inline size_t chunk_valid(size_t S, size_t n_valid, size_t i) {  // :32-37
  const size_t off = i * S;
  return off >= n_valid ? 0 : std::min(S, n_valid - off);
}

// Backends with batched chunk ops (RnsB): one batched mul_pt / square over a column's chunks
// when they allow it (same level, nothing to bootstrap); the same ops on the same operands as
// the per-chunk loops, so values, meter and levels are unchanged.
template <class B>
concept BatchedChunks = requires(B& b, const std::vector<typename B::C>& v, double c) {
  { b.mul_pt_many(v, c) } -> std::same_as<std::vector<typename B::C>>;
  { b.square_many(v) } -> std::same_as<std::vector<typename B::C>>;
};

template <class B>
std::vector<typename B::C> mul_pt_chunks(B& b, const std::vector<typename B::C>& xs, double c) {
  if constexpr (BatchedChunks<B>) {
    if (xs.size() > 1 && b.batch_ok(xs)) return b.mul_pt_many(xs, c);
  }
  std::vector<typename B::C> out;
  out.reserve(xs.size());
  for (const auto& x : xs) out.push_back(b.mul_pt(x, c));
  return out;
}

template <class B>
typename B::C scaled_slot_sum(B& b, const Col<typename B::C>& col, double c) {  // :41-51
  typename B::C acc{};
  if constexpr (BatchedChunks<B>) {
    if (col.chunks.size() > 1 && b.batch_ok(col.chunks)) {
      const auto terms = b.mul_pt_many(col.chunks, c);
      for (size_t i = 0; i < terms.size(); ++i) acc = i == 0 ? terms[i] : b.add_ct(acc, terms[i]);
      return b.sum_all_slots(acc, b.params().S);
    }
  }
  for (size_t i = 0; i < col.chunks.size(); ++i) {
    const typename B::C term = b.mul_pt(col.chunks[i], c);
    acc = i == 0 ? term : b.add_ct(acc, term);
  }
  return b.sum_all_slots(acc, b.params().S);
}

template <class B>
std::vector<typename B::C> centered_chunks(B& b, const Col<typename B::C>& col, const typename B::C& mu,
                                           bool mask_padding) {  // :56-75
  const size_t S = b.params().S;
  std::vector<typename B::C> out;
  out.reserve(col.chunks.size());
  for (size_t i = 0; i < col.chunks.size(); ++i) {
    const size_t valid = chunk_valid(S, col.n_valid, i);
    if (mask_padding && valid < S) {
      std::vector<double> mask(S, 0.0);
      for (size_t k = 0; k < valid; ++k) mask[k] = 1.0;
      const typename B::C mu_masked = b.mul_pt_vec(mu, mask);
      out.push_back(b.sub_ct(col.chunks[i], mu_masked));
    } else {
      out.push_back(b.sub_ct(col.chunks[i], mu));
    }
  }
  return out;
}

template <class B>
typename B::C mean_of_chunks(B& b, const std::vector<typename B::C>& chunks, size_t n_valid) {  // :78-87
  typename B::C acc{};
  for (size_t i = 0; i < chunks.size(); ++i) {
    const typename B::C term = b.mul_pt(chunks[i], 1.0 / static_cast<double>(n_valid));
    acc = i == 0 ? term : b.add_ct(acc, term);
  }
  return b.sum_all_slots(acc, b.params().S);
}

template <class B>
typename B::C mean_scaled(B& b, const Col<typename B::C>& col, double B_) {  // :97-103
  require_nonempty(col);
  if (B_ <= 0.0) fail(HS_E_ERROR, "mean_scaled: B must be positive");
  return scaled_slot_sum(b, col, 1.0 / (B_ * static_cast<double>(col.n_valid)));
}

template <class B>
typename B::C variance_to_scale(B& b, const Col<typename B::C>& col, double S) {  // :110-126
  require_nonempty(col);
  if (S <= 0.0) fail(HS_E_ERROR, "variance_to_scale: scale must be positive");
  const double n = static_cast<double>(col.n_valid);
  typename B::C sq_sum{};
  bool done = false;
  if constexpr (BatchedChunks<B>) {
    if (col.chunks.size() > 1 && b.batch_ok(col.chunks)) {
      const auto as = b.mul_pt_many(col.chunks, 1.0 / std::sqrt(S * n));
      if (b.batch_ok(as)) {
        const auto sqs = b.square_many(as);
        for (size_t i = 0; i < sqs.size(); ++i) sq_sum = i == 0 ? sqs[i] : b.add_ct(sq_sum, sqs[i]);
      } else {  // (unreachable for uniform chunks) the per-chunk squares
        for (size_t i = 0; i < as.size(); ++i) {
          const typename B::C sq = b.mul_ct(as[i], as[i]);
          sq_sum = i == 0 ? sq : b.add_ct(sq_sum, sq);
        }
      }
      done = true;
    }
  }
  if (!done) {
    for (size_t i = 0; i < col.chunks.size(); ++i) {
      const typename B::C a = b.mul_pt(col.chunks[i], 1.0 / std::sqrt(S * n));
      const typename B::C sq = b.mul_ct(a, a);
      sq_sum = i == 0 ? sq : b.add_ct(sq_sum, sq);
    }
  }
  sq_sum = b.sum_all_slots(sq_sum, b.params().S);
  const typename B::C mean_part = scaled_slot_sum(b, col, 1.0 / (n * std::sqrt(S)));
  const typename B::C mean_sq = b.mul_ct(mean_part, mean_part);
  return b.sub_ct(sq_sum, mean_sq);
}

template <class B>
typename B::C variance_scaled(B& b, const Col<typename B::C>& col, double B_) {  // :130-134
  if (B_ <= 0.0) fail(HS_E_ERROR, "variance_scaled: B must be positive");
  return variance_to_scale(b, col, B_ * B_);
}

template <class C>
struct Moments {  // MomentSet, stats.hpp:18-22
  C mu, var;
  size_t n_valid = 0;
};

template <class B>
Moments<typename B::C> moments(B& b, const Col<typename B::C>& col, double B_) {  // :138-148
  Moments<typename B::C> m;
  m.mu = mean_scaled(b, col, 1.0);
  m.var = variance_scaled(b, col, B_);
  m.n_valid = col.n_valid;
  if (b.params().debug && b.first_slot(m.var) < -1e-9)
    fail(HS_E_DEGENERATE_VARIANCE, "moments: negative scaled variance");
  return m;
}

template <class B>
Col<typename B::C> znorm(B& b, const Col<typename B::C>& col, double B_, const InvCfg& cfg) {  // :153-166
  Moments<typename B::C> m = moments(b, col, B_);
  if (b.params().debug && b.first_slot(m.var) * B_ * B_ < 1e-9)
    fail(HS_E_DEGENERATE_VARIANCE, "znorm: variance below 1e-9");
  const typename B::C inv_sigma = crypto_invsqrt(b, m.var, B_ * B_, cfg, kAllSlots);
  Col<typename B::C> out;
  out.n_valid = col.n_valid;
  for (const auto& chunk : col.chunks) out.chunks.push_back(b.mul_ct(b.sub_ct(chunk, m.mu), inv_sigma));
  return out;
}

// kurtosis (power 4, :170-188) and skewness (power 3, :192-210)
template <class B>
typename B::C std_moment(B& b, const Col<typename B::C>& col, double B_, const InvCfg& cfg, int power) {
  using C = typename B::C;
  Moments<C> m = moments(b, col, B_);
  if (b.params().debug && b.first_slot(m.var) * B_ * B_ < 1e-9)
    fail(HS_E_DEGENERATE_VARIANCE,
         power == 4 ? "kurtosis: variance below 1e-9" : "skewness: variance below 1e-9");
  std::vector<C> centered = centered_chunks(b, col, m.mu, true);
  std::vector<C> pw;
  pw.reserve(centered.size());
  for (const C& c : centered) {
    const C sq = b.mul_ct(c, c);
    pw.push_back(power == 4 ? b.mul_ct(sq, sq) : b.mul_ct(sq, c));
  }
  const C numerator = mean_of_chunks(b, pw, col.n_valid);
  const C inv = crypto_invsqrt(b, m.var, B_ * B_, cfg, kAllSlots);
  const C inv2 = b.mul_ct(inv, inv);
  const C invp = power == 4 ? b.mul_ct(inv2, inv2) : b.mul_ct(inv2, inv);
  return b.mul_ct(numerator, invp);
}

template <class B>
typename B::C coeff_variation(B& b, const Col<typename B::C>& col, double B_, const SignCfg& sign_cfg,
                              const InvCfg& cfg) {  // :216-233
  using C = typename B::C;
  require_nonempty(col);
  const C mu_b = mean_scaled(b, col, B_);
  if (b.params().debug && std::abs(b.first_slot(mu_b)) < 0.01)
    fail(HS_E_NEAR_ZERO_MEAN, "coeff_variation: |mean| < 0.01 B");
  const C sgn = crypto_sign(b, mu_b, sign_cfg);
  const C mu_pos = b.mul_ct(mu_b, sgn);
  const C inv_mu = crypto_inv(b, mu_pos, B_, cfg, kAllSlots);
  const C var_b = variance_scaled(b, col, B_);
  C sigma = crypto_sqrt(b, var_b, B_ * B_, cfg.cheb_degree, kAllSlots);
  if (b.level(sigma) < 1 && b.params().auto_bootstrap) sigma = b.bootstrap(sigma);
  const C ratio = b.mul_ct(sigma, inv_mu);
  return b.mul_ct(ratio, sgn);
}

template <class B>
typename B::C pearson(B& b, const Col<typename B::C>& x, const Col<typename B::C>& y, double B_,
                      const InvCfg& cfg) {  // :239-265
  using C = typename B::C;
  require_nonempty(x);
  require_nonempty(y);
  if (x.n_valid != y.n_valid) fail(HS_E_LENGTH_MISMATCH, "pearson: columns differ in element count");
  Moments<C> mx = moments(b, x, B_);
  Moments<C> my = moments(b, y, B_);
  if (b.params().debug) {
    if (b.first_slot(mx.var) * B_ * B_ < 1e-9 || b.first_slot(my.var) * B_ * B_ < 1e-9)
      fail(HS_E_DEGENERATE_VARIANCE, "pearson: degenerate column variance");
  }
  const C inv_x = crypto_invsqrt(b, mx.var, B_ * B_, cfg, kAllSlots);
  const C inv_y = crypto_invsqrt(b, my.var, B_ * B_, cfg, kAllSlots);
  std::vector<C> cx = centered_chunks(b, x, mx.mu, true);
  std::vector<C> cy = centered_chunks(b, y, my.mu, false);
  if (cy.size() < cx.size()) fail(HS_E_LENGTH_MISMATCH, "pearson: columns differ in chunk count");
  std::vector<C> prods;
  prods.reserve(cx.size());
  for (size_t i = 0; i < cx.size(); ++i) prods.push_back(b.mul_ct(cx[i], cy[i]));
  const C cov = mean_of_chunks(b, prods, x.n_valid);
  const C r = b.mul_ct(cov, inv_x);
  return b.mul_ct(r, inv_y);
}

}  // namespace flow
}  // namespace hsg
