// hestat/chebyshev.hpp — drop-in for the reference's Chebyshev module
// (/root/reference/proj/include/hestat/chebyshev.hpp:24-207).  fit() and
// eval_plain() are host code in the library (bit-identical to the reference's);
// eval_encrypted() runs the fused BSGS kernel on the GPU.
#pragma once

#include <exception>
#include <functional>
#include <vector>

#if __has_include(<json.hpp>)
#include <json.hpp>
#define HESTAT_DROPIN_HAVE_JSON 1
#endif

#include "hestat/ckks.hpp"
#include "hestat/errors.hpp"

namespace hestat {

struct ChebyshevSeries {  // :24-31
  std::vector<double> coeffs;
  double domain_lo = -1.0;
  double domain_hi = 1.0;

  int degree() const { return static_cast<int>(coeffs.size()) - 1; }
  bool native_domain() const { return domain_lo == -1.0 && domain_hi == 1.0; }
};

enum class ScaledTargetKind { InvSqrtShifted, SqrtShifted };  // :37

inline double scaled_target(ScaledTargetKind kind, double S, double t) {  // :39-47
  return hs_scaled_target(kind == ScaledTargetKind::SqrtShifted ? HS_TARGET_SQRT_SHIFTED
                                                                : HS_TARGET_INVSQRT_SHIFTED,
                          S, t);
}

inline int cheb_eval_depth(int degree) { return hs_cheb_eval_depth(degree); }  // :51-54

namespace detail {
struct FitCall {
  const std::function<double(double)>* f;
  std::exception_ptr err;
};
inline double fit_trampoline(double x, void* user) {
  auto* fc = static_cast<FitCall*>(user);
  if (fc->err) return 0.0;
  try {
    return (*fc->f)(x);
  } catch (...) {
    fc->err = std::current_exception();
    return 0.0;
  }
}
}  // namespace detail

inline ChebyshevSeries fit(const std::function<double(double)>& target, int degree, double domain_lo = -1.0,
                           double domain_hi = 1.0) {  // :59-85
  ChebyshevSeries s;
  s.domain_lo = domain_lo;
  s.domain_hi = domain_hi;
  s.coeffs.assign(degree >= 0 ? static_cast<std::size_t>(degree) + 1 : 1, 0.0);
  detail::FitCall fc{&target, nullptr};
  const int rc = hs_fit(detail::fit_trampoline, &fc, degree, domain_lo, domain_hi, s.coeffs.data());
  if (fc.err) std::rethrow_exception(fc.err);
  gpu::check(rc);
  return s;
}

inline double eval_plain(const ChebyshevSeries& s, double x, bool* extrapolated = nullptr) {  // :90-105
  int32_t ex = 0;
  const double r = hs_eval_plain(s.coeffs.data(), s.coeffs.size(), s.domain_lo, s.domain_hi, x, &ex);
  if (extrapolated) *extrapolated = ex != 0;
  return r;
}

inline Ciphertext eval_encrypted(EvalContext& ctx, const ChebyshevSeries& s, const Ciphertext& ct) {  // :171-189
  return ctx.run([&](hs_ct** o) {
    return hs_eval_encrypted(ctx.raw(), s.coeffs.data(), s.coeffs.size(), s.domain_lo, s.domain_hi, ct.raw(), o);
  });
}

#ifdef HESTAT_DROPIN_HAVE_JSON
inline nlohmann::json to_json(const ChebyshevSeries& s) {  // :192-196
  return nlohmann::json{{"degree", s.degree()}, {"coeffs", s.coeffs}, {"domain", {s.domain_lo, s.domain_hi}}};
}

inline ChebyshevSeries series_from_json(const nlohmann::json& j) {  // :198-207
  ChebyshevSeries s;
  s.coeffs = j.at("coeffs").get<std::vector<double>>();
  s.domain_lo = j.at("domain").at(0).get<double>();
  s.domain_hi = j.at("domain").at(1).get<double>();
  if (s.coeffs.empty()) throw error("series_from_json: empty coefficients");
  if (j.contains("degree") && j.at("degree").get<int>() != s.degree())
    throw error("series_from_json: degree field disagrees with coeffs");
  return s;
}
#endif

}  // namespace hestat
