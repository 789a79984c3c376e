// series.h — host-side Chebyshev machinery (chebyshev.hpp, primitives.hpp:240-272).
//
// fit() is host code in the reference and stays host code here: it is O(d^2)
// libm work done once per (target, S, degree) and cached, and its bits must
// match the reference's (same expressions, no contraction).  The device never
// sees the reference's recursive coefficient splitting; the host replays it
// (split_series) and emits a flat per-slot table (cheb_table) that the fused
// kernel walks in one pass.
#pragma once

#include <functional>
#include <string>
#include <memory>
#include <vector>

#include "core.h"
#include "kernels.h"

namespace hsg {

enum class TargetKind { InvSqrtShifted = 0, SqrtShifted = 1 };

struct Series {  // ChebyshevSeries, chebyshev.hpp:24-31
  std::vector<double> coeffs;
  double lo = -1.0, hi = 1.0;
  std::string key;  // cache identity of library-made series ("" = user series)
  int degree() const { return static_cast<int>(coeffs.size()) - 1; }
  bool native() const { return lo == -1.0 && hi == 1.0; }
};

int cheb_depth(int degree);                          // chebyshev.hpp:51-54
double scaled_target(TargetKind k, double S, double t);  // chebyshev.hpp:39-47
Series fit(const std::function<double(double)>& f, int degree, double lo = -1.0, double hi = 1.0);
Series fit_scaled(TargetKind k, double S, int degree);  // cached fit of a scaled target
double eval_plain(const Series& s, double x, bool* extrapolated);  // chebyshev.hpp:90-105

// One recursion step of ChebEncryptedEval::eval (chebyshev.hpp:146-152):
// p = q * T_g + r; returns g.
int split_series(const std::vector<double>& c, std::vector<double>* q, std::vector<double>* r);

// crypto_sign stages (primitives.hpp:244-272, 288-303)
std::vector<Series> sign_stages(int mode, const std::vector<std::vector<double>>& custom_polys);

// Flat device table of a series for the per-slot CHEB instruction (fused.cu):
// [terminal][F-table of each peeled remainder, innermost first].  Leaf
// constants are pre-scaled to grid units when mode == Grid.
std::vector<double> cheb_table(const std::vector<double>& coeffs, QSpec q);
// The same table with each of `parts` equal sub-tables interleaved (element e of
// part l at e * parts + l), for a full-degree series split across `parts` lanes.
std::vector<double> interleave(const std::vector<double>& t, int parts);

}  // namespace hsg
