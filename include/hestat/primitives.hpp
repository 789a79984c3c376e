// hestat/primitives.hpp — drop-in for the reference's inverse-root primitives
// (/root/reference/proj/include/hestat/primitives.hpp:20-300).  Every entry
// point is one fused GPU launch (or the exact op-by-op path in debug mode).
#pragma once

#include <cstddef>
#include <limits>
#include <string>
#include <vector>

#include "hestat/chebyshev.hpp"
#include "hestat/ckks.hpp"
#include "hestat/errors.hpp"

namespace hestat {

inline constexpr std::size_t all_slots = std::numeric_limits<std::size_t>::max();  // :20

struct InvRootConfig {  // :23-40
  int n = 2;
  int cheb_degree = 511;
  int newton_iters = 6;
  bool baseline_mode = false;
  int baseline_iters = 0;

  int effective_baseline_iters() const { return baseline_iters > 0 ? baseline_iters : (n == 1 ? 25 : 21); }
  void validate() const {
    if (n != 1 && n != 2) throw error("InvRootConfig: n must be 1 or 2");
    if (newton_iters < 0) throw error("InvRootConfig: newton_iters < 0");
    if (cheb_degree < 0) throw error("InvRootConfig: cheb_degree < 0");
  }
  hs_invroot_cfg to_c() const {
    return hs_invroot_cfg{n, cheb_degree, newton_iters, baseline_mode ? 1 : 0, baseline_iters, 0};
  }
};

struct SignConfig {  // :59-70
  enum class Mode { G3Composition, CustomComposite };
  Mode mode = Mode::G3Composition;
  int folds = 7;
  std::vector<std::vector<double>> custom_polys;

  std::string mode_name() const { return mode == Mode::G3Composition ? "g3_composition" : "custom_composite"; }

  // flattened view for the C ABI (buffers owned by the returned object)
  struct CView {
    std::vector<double> flat;
    std::vector<uint64_t> lens;
    hs_sign_cfg c;
  };
  CView to_c() const {
    CView v;
    for (const auto& p : custom_polys) {
      v.flat.insert(v.flat.end(), p.begin(), p.end());
      v.lens.push_back(p.size());
    }
    v.c = hs_sign_cfg{mode == Mode::G3Composition ? 0 : 1, folds, v.flat.data(), v.lens.data(), v.lens.size()};
    return v;
  }
};

#ifdef HESTAT_DROPIN_HAVE_JSON
inline void to_json(nlohmann::json& j, const InvRootConfig& c) {
  j = nlohmann::json{{"n", c.n},
                     {"cheb_degree", c.cheb_degree},
                     {"newton_iters", c.newton_iters},
                     {"baseline_mode", c.baseline_mode},
                     {"baseline_iters", c.baseline_iters}};
}
inline void from_json(const nlohmann::json& j, InvRootConfig& c) {
  j.at("n").get_to(c.n);
  j.at("cheb_degree").get_to(c.cheb_degree);
  j.at("newton_iters").get_to(c.newton_iters);
  j.at("baseline_mode").get_to(c.baseline_mode);
  j.at("baseline_iters").get_to(c.baseline_iters);
}
inline void to_json(nlohmann::json& j, const SignConfig& c) {
  j = nlohmann::json{{"mode", c.mode_name()}, {"folds", c.folds}, {"custom_polys", c.custom_polys}};
}
inline void from_json(const nlohmann::json& j, SignConfig& c) {
  const std::string m = j.at("mode").get<std::string>();
  if (m == "g3_composition") c.mode = SignConfig::Mode::G3Composition;
  else if (m == "custom_composite") c.mode = SignConfig::Mode::CustomComposite;
  else throw error("SignConfig: unknown mode " + m);
  j.at("folds").get_to(c.folds);
  j.at("custom_polys").get_to(c.custom_polys);
}
#endif

namespace detail {
inline Ciphertext newton_loop(EvalContext& ctx, const Ciphertext& x_op, Ciphertext y, int n, int iters,
                              std::size_t n_valid) {  // :105-132
  return ctx.run([&](hs_ct** o) { return hs_newton_loop(ctx.raw(), x_op.raw(), y.raw(), n, iters, n_valid, o); });
}

inline ChebyshevSeries g3_series() {  // :244-249
  ChebyshevSeries s;
  s.coeffs = {0.0, 1225.0 / 1024.0, 0.0, -245.0 / 1024.0, 0.0, 49.0 / 1024.0, 0.0, -5.0 / 1024.0};
  return s;
}
}  // namespace detail

inline Ciphertext newton_refine(EvalContext& ctx, const Ciphertext& ct_x, const Ciphertext& ct_y0, int n, int iters,
                                std::size_t n_valid = all_slots) {  // :152-158
  return ctx.run(
      [&](hs_ct** o) { return hs_newton_refine(ctx.raw(), ct_x.raw(), ct_y0.raw(), n, iters, n_valid, o); });
}

inline Ciphertext crypto_invsqrt(EvalContext& ctx, const Ciphertext& ct, double S, const InvRootConfig& cfg = {},
                                 std::size_t n_valid = all_slots) {  // :186-208
  const hs_invroot_cfg c = cfg.to_c();
  return ctx.run([&](hs_ct** o) { return hs_crypto_invsqrt(ctx.raw(), ct.raw(), S, &c, n_valid, o); });
}

inline Ciphertext baseline_invsqrt(EvalContext& ctx, const Ciphertext& ct, double S, int iters = 21,
                                   std::size_t n_valid = all_slots) {  // :173-184
  return ctx.run([&](hs_ct** o) { return hs_baseline_invsqrt(ctx.raw(), ct.raw(), S, iters, n_valid, o); });
}

inline Ciphertext crypto_inv(EvalContext& ctx, const Ciphertext& ct, double S, const InvRootConfig& cfg = {},
                             std::size_t n_valid = all_slots) {  // :211-217
  const hs_invroot_cfg c = cfg.to_c();
  return ctx.run([&](hs_ct** o) { return hs_crypto_inv(ctx.raw(), ct.raw(), S, &c, n_valid, o); });
}

inline Ciphertext crypto_sqrt(EvalContext& ctx, const Ciphertext& ct, double S, int degree = 511,
                              std::size_t n_valid = all_slots) {  // :222-238
  return ctx.run([&](hs_ct** o) { return hs_crypto_sqrt(ctx.raw(), ct.raw(), S, degree, n_valid, o); });
}

inline Ciphertext crypto_sign(EvalContext& ctx, const Ciphertext& ct, const SignConfig& cfg = {}) {  // :279-300
  const SignConfig::CView v = cfg.to_c();
  return ctx.run([&](hs_ct** o) { return hs_crypto_sign(ctx.raw(), ct.raw(), &v.c, o); });
}

}  // namespace hestat
