// hestat/stats.hpp — drop-in for the reference's statistics
// (/root/reference/proj/include/hestat/stats.hpp:18-265).  Each statistic is
// one cooperative GPU kernel (moments -> grid barrier -> per-slot program),
// with the reference's levels, meter and errors.
#pragma once

#include <cstddef>
#include <vector>

#include "hestat/column.hpp"
#include "hestat/errors.hpp"
#include "hestat/primitives.hpp"

namespace hestat {

struct MomentSet {  // :18-22
  Ciphertext ct_mu;
  Ciphertext ct_var;
  std::size_t n_valid = 0;
};

namespace detail {
inline void require_nonempty(const EncryptedColumn& col) {  // :26-29
  if (col.n_valid == 0 || col.chunks.empty()) throw empty_column("statistic on an empty column");
}
inline std::size_t chunk_valid(const EvalContext& ctx, const EncryptedColumn& col, std::size_t i) {  // :32-37
  const std::size_t sc = ctx.params().slot_count;
  const std::size_t off = i * sc;
  return off >= col.n_valid ? 0 : std::min(sc, col.n_valid - off);
}
inline double replicated_value(const EvalContext& ctx, const Ciphertext& ct) {  // :89-91
  return ctx.decrypt(ct, 1)[0];
}
template <class F>
Ciphertext col_call(EvalContext& ctx, const EncryptedColumn& col, F&& f) {
  const EncryptedColumn::CView v = col.to_c();
  return ctx.run([&](hs_ct** o) { return f(&v.c, o); });
}
}  // namespace detail

inline Ciphertext mean_scaled(EvalContext& ctx, const EncryptedColumn& col, double B) {  // :97-103
  return detail::col_call(ctx, col, [&](const hs_column* c, hs_ct** o) { return hs_mean_scaled(ctx.raw(), c, B, o); });
}

inline Ciphertext variance_to_scale(EvalContext& ctx, const EncryptedColumn& col, double S) {  // :110-126
  return detail::col_call(ctx, col,
                          [&](const hs_column* c, hs_ct** o) { return hs_variance_to_scale(ctx.raw(), c, S, o); });
}

inline Ciphertext variance_scaled(EvalContext& ctx, const EncryptedColumn& col, double B) {  // :130-134
  return detail::col_call(ctx, col,
                          [&](const hs_column* c, hs_ct** o) { return hs_variance_scaled(ctx.raw(), c, B, o); });
}

inline MomentSet moments(EvalContext& ctx, const EncryptedColumn& col, double B) {  // :138-148
  const EncryptedColumn::CView v = col.to_c();
  hs_ct* mu = nullptr;
  hs_ct* var = nullptr;
  ctx.call([&] { return hs_moments(ctx.raw(), &v.c, B, &mu, &var); });
  MomentSet m;
  m.ct_mu = Ciphertext::adopt(mu);
  m.ct_var = Ciphertext::adopt(var);
  m.n_valid = col.n_valid;
  return m;
}

inline EncryptedColumn znorm(EvalContext& ctx, const EncryptedColumn& col, double B,
                             const InvRootConfig& cfg = {}) {  // :153-166
  const EncryptedColumn::CView v = col.to_c();
  const hs_invroot_cfg c = cfg.to_c();
  std::vector<hs_ct*> out(col.chunks.size() + 1, nullptr);
  ctx.call([&] { return hs_znorm(ctx.raw(), &v.c, B, &c, out.data()); });
  EncryptedColumn z;
  z.n_valid = col.n_valid;
  z.name = col.name;
  for (std::size_t i = 0; i < col.chunks.size(); ++i) z.chunks.push_back(Ciphertext::adopt(out[i]));
  return z;
}

inline Ciphertext kurtosis(EvalContext& ctx, const EncryptedColumn& col, double B,
                           const InvRootConfig& cfg = {}) {  // :170-188
  const hs_invroot_cfg c = cfg.to_c();
  return detail::col_call(ctx, col,
                          [&](const hs_column* cc, hs_ct** o) { return hs_kurtosis(ctx.raw(), cc, B, &c, o); });
}

inline Ciphertext skewness(EvalContext& ctx, const EncryptedColumn& col, double B,
                           const InvRootConfig& cfg = {}) {  // :192-210
  const hs_invroot_cfg c = cfg.to_c();
  return detail::col_call(ctx, col,
                          [&](const hs_column* cc, hs_ct** o) { return hs_skewness(ctx.raw(), cc, B, &c, o); });
}

inline Ciphertext coeff_variation(EvalContext& ctx, const EncryptedColumn& col, double B,
                                  const SignConfig& sign_cfg = {}, const InvRootConfig& cfg = {}) {  // :216-233
  const SignConfig::CView sv = sign_cfg.to_c();
  const hs_invroot_cfg c = cfg.to_c();
  return detail::col_call(
      ctx, col, [&](const hs_column* cc, hs_ct** o) { return hs_coeff_variation(ctx.raw(), cc, B, &sv.c, &c, o); });
}

inline Ciphertext pearson(EvalContext& ctx, const EncryptedColumn& col_x, const EncryptedColumn& col_y, double B,
                          const InvRootConfig& cfg = {}) {  // :239-265
  const EncryptedColumn::CView vx = col_x.to_c(), vy = col_y.to_c();
  const hs_invroot_cfg c = cfg.to_c();
  return ctx.run([&](hs_ct** o) { return hs_pearson(ctx.raw(), &vx.c, &vy.c, B, &c, o); });
}

// Extension: znorm(cols[k], B) for every column, in order (hs_znorm_batch: one launch per 64
// single-chunk columns; same slots, levels and meter as the calls).
inline std::vector<EncryptedColumn> znorm_batch(EvalContext& ctx, const std::vector<EncryptedColumn>& cols, double B,
                                                const InvRootConfig& cfg = {}) {
  std::vector<EncryptedColumn::CView> views;
  views.reserve(cols.size());
  size_t total = 0;
  for (const EncryptedColumn& c : cols) {
    views.push_back(c.to_c());
    total += c.chunks.size();
  }
  std::vector<const hs_column*> ptrs;
  for (const auto& v : views) ptrs.push_back(&v.c);
  const hs_invroot_cfg c = cfg.to_c();
  std::vector<hs_ct*> hs(total ? total : 1, nullptr);
  gpu::check(hs_znorm_batch(ctx.raw(), ptrs.data(), static_cast<uint32_t>(cols.size()), B, &c, hs.data()));
  std::vector<EncryptedColumn> out;
  size_t off = 0;
  for (const EncryptedColumn& col : cols) {
    EncryptedColumn z;
    z.n_valid = col.n_valid;
    z.name = col.name;
    for (size_t i = 0; i < col.chunks.size(); ++i) z.chunks.push_back(Ciphertext::adopt(hs[off + i]));
    off += col.chunks.size();
    out.push_back(std::move(z));
  }
  return out;
}

// Extension: pearson(cols[i], cols[j]) for every pair i < j, in that order (hs_pearson_table).
inline std::vector<Ciphertext> pearson_table(EvalContext& ctx, const std::vector<EncryptedColumn>& cols, double B,
                                             const InvRootConfig& cfg = {}) {
  std::vector<EncryptedColumn::CView> views;
  views.reserve(cols.size());
  for (const EncryptedColumn& c : cols) views.push_back(c.to_c());
  std::vector<const hs_column*> ptrs;
  for (const auto& v : views) ptrs.push_back(&v.c);
  const hs_invroot_cfg c = cfg.to_c();
  const size_t np = cols.size() * (cols.empty() ? 0 : cols.size() - 1) / 2;
  std::vector<hs_ct*> hs(np ? np : 1, nullptr);
  gpu::check(hs_pearson_table(ctx.raw(), ptrs.data(), static_cast<uint32_t>(cols.size()), B, &c, hs.data()));
  std::vector<Ciphertext> out;
  for (size_t k = 0; k < np; ++k) out.push_back(Ciphertext::adopt(hs[k]));
  return out;
}

}  // namespace hestat
