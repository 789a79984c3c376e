// series.cpp — see series.h.  Compiled with -ffp-contract=off: fit() bits must
// equal the reference's.
#include "series.h"

#include <bit>
#include <cmath>
#include <cstring>
#include <map>
#include <mutex>
#include <numbers>
#include <tuple>

namespace hsg {

int cheb_depth(int degree) {
  if (degree <= 0) return 0;
  return static_cast<int>(std::bit_width(static_cast<unsigned>(degree)));
}

double scaled_target(TargetKind k, double S, double t) {
  switch (k) {
    case TargetKind::InvSqrtShifted: return t > -1.0 ? 1.0 / (std::sqrt(S) * std::sqrt(t + 1.0)) : 0.0;
    case TargetKind::SqrtShifted: return t >= -1.0 ? std::sqrt(S) * std::sqrt(t + 1.0) : 0.0;
  }
  return 0.0;
}

// chebyshev.hpp:59-85: discrete cosine projection at degree+1 first-kind nodes.
Series fit(const std::function<double(double)>& f, int degree, double lo, double hi) {
  if (degree < 0) fail(HS_E_ERROR, "fit: degree must be >= 0");
  const int n = degree + 1;
  std::vector<double> ang(static_cast<size_t>(n)), val(static_cast<size_t>(n));
  for (int k = 0; k < n; ++k) {
    ang[k] = std::numbers::pi * (k + 0.5) / n;
    const double node = std::cos(ang[k]);
    val[k] = f(0.5 * (lo + hi) + 0.5 * (hi - lo) * node);
    if (!std::isfinite(val[k])) fail(HS_E_NON_FINITE_TARGET, "fit: target not finite at a Chebyshev node");
  }
  Series s;
  s.lo = lo;
  s.hi = hi;
  s.coeffs.resize(static_cast<size_t>(n));
  for (int j = 0; j < n; ++j) {
    double acc = 0.0;
    for (int k = 0; k < n; ++k) acc += val[k] * std::cos(j * ang[k]);
    s.coeffs[j] = 2.0 * acc / n;
  }
  s.coeffs[0] *= 0.5;
  return s;
}

Series fit_scaled(TargetKind k, double S, int degree) {
  static std::mutex mu;
  static std::map<std::tuple<int, uint64_t, int>, Series> cache;
  uint64_t sb;
  std::memcpy(&sb, &S, sizeof sb);
  const auto key = std::make_tuple(static_cast<int>(k), sb, degree);
  {
    std::lock_guard<std::mutex> g(mu);
    auto it = cache.find(key);
    if (it != cache.end()) return it->second;
  }
  Series s = fit([k, S](double t) { return scaled_target(k, S, t); }, degree);
  s.key = "fit/" + std::to_string(static_cast<int>(k)) + "/" + std::to_string(sb) + "/" + std::to_string(degree);
  std::lock_guard<std::mutex> g(mu);
  if (cache.size() > 256) cache.clear();
  cache.emplace(key, s);
  return s;
}

double eval_plain(const Series& s, double x, bool* extrapolated) {
  if (extrapolated) *extrapolated = (x < s.lo || x > s.hi);
  const double u = s.native() ? x : (2.0 * x - (s.lo + s.hi)) / (s.hi - s.lo);
  double b1 = 0.0, b2 = 0.0;
  for (int k = s.degree(); k >= 1; --k) {
    const double next = s.coeffs[k] + 2.0 * u * b1 - b2;
    b2 = b1;
    b1 = next;
  }
  return s.coeffs[0] + u * b1 - b2;
}

int split_series(const std::vector<double>& c, std::vector<double>* q, std::vector<double>* r) {
  const int d = static_cast<int>(c.size()) - 1;
  const int g = 1 << (cheb_depth(d) - 1);
  q->assign(static_cast<size_t>(d - g) + 1, 0.0);
  (*q)[0] = c[g];
  for (int j = 1; j <= d - g; ++j) (*q)[j] = 2.0 * c[g + j];
  r->assign(c.begin(), c.begin() + g);
  for (int j = 1; j <= d - g; ++j) (*r)[g - j] -= c[g + j];
  return g;
}

std::vector<Series> sign_stages(int mode, const std::vector<std::vector<double>>& polys) {
  std::vector<Series> st;
  if (mode == 0) {  // g3 in the T basis, primitives.hpp:244-249
    Series s;
    s.coeffs = {0.0, 1225.0 / 1024.0, 0.0, -245.0 / 1024.0, 0.0, 49.0 / 1024.0, 0.0, -5.0 / 1024.0};
    s.key = "g3";
    st.push_back(s);
    return st;
  }
  if (polys.empty()) fail(HS_E_ERROR, "crypto_sign: custom mode needs component polynomials");
  for (const auto& p : polys) {  // odd_poly_series, primitives.hpp:255-272
    if (p.empty()) fail(HS_E_ERROR, "sign: empty component polynomial");
    for (size_t i = 0; i < p.size(); i += 2)
      if (p[i] != 0.0) fail(HS_E_ERROR, "sign: component polynomial must be odd");
    const int d = static_cast<int>(p.size()) - 1;
    Series s = fit([&p](double x) {
      double acc = 0.0;
      for (size_t i = p.size(); i-- > 0;) acc = acc * x + p[i];
      return acc;
    }, d);
    for (size_t i = 0; i < s.coeffs.size(); i += 2) {
      if (std::abs(s.coeffs[i]) > 1e-9) fail(HS_E_ERROR, "sign: conversion produced a non-odd series");
      s.coeffs[i] = 0.0;
    }
    st.push_back(std::move(s));
  }
  return st;
}

namespace {
// F_k table of a full remainder (size 2^k, degree 2^k - 1; or size 1)
void emit_full(const std::vector<double>& c, double sc, std::vector<double>* out) {
  const int d = static_cast<int>(c.size()) - 1;
  if (d <= 1) {
    out->push_back(d == 1 ? c[1] : 0.0);  // mul_pt(x, c1)  (0.0 for a degree-0 leaf)
    out->push_back(c[0] * sc);            // add_pt(., c0)
    return;
  }
  std::vector<double> q, r;
  split_series(c, &q, &r);
  emit_full(q, sc, out);
  emit_full(r, sc, out);
}
}  // namespace

std::vector<double> cheb_table(const std::vector<double>& coeffs, QSpec qs) {
  const double sc = qs.mode == QMode::Grid ? std::ldexp(1.0, qs.bits) : 1.0;
  std::vector<double> t;
  const int d = static_cast<int>(coeffs.size()) - 1;
  if (d <= 0) {  // constant series: add_pt(sub_ct(x, x), c0)
    t.push_back((coeffs.empty() ? 0.0 : coeffs[0]) * sc);
    return t;
  }
  if (d == 1) {
    t.push_back(coeffs[1]);
    t.push_back(coeffs[0] * sc);
    return t;
  }
  std::vector<std::vector<double>> rem;  // remainders, outermost first
  std::vector<double> c = coeffs, q, r;
  bool pt = false;
  for (;;) {
    split_series(c, &q, &r);
    rem.push_back(r);
    if (q.size() == 1) {
      pt = true;
      break;
    }
    if (q.size() == 2) break;  // degree-1 leaf
    c = q;
  }
  if (pt) {
    t.push_back(q[0]);  // head = mul_pt(T_g, q0)
  } else {
    t.push_back(q[1]);
    t.push_back(q[0] * sc);
  }
  for (size_t i = rem.size(); i-- > 0;) emit_full(rem[i], sc, &t);
  return t;
}

std::vector<double> interleave(const std::vector<double>& t, int parts) {
  const size_t part = t.size() / static_cast<size_t>(parts);
  std::vector<double> o(t.size());
  for (int l = 0; l < parts; ++l)
    for (size_t e = 0; e < part; ++e) o[e * parts + l] = t[l * part + e];
  return o;
}

}  // namespace hsg
