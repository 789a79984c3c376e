// hestat/plain.hpp — drop-in plaintext statistics (reference: plain.hpp:16-92),
// served by the library's host implementation (hs_plain).
#pragma once

#include <span>
#include <vector>

#include "hestat/errors.hpp"

namespace hestat::plain {

namespace detail {
inline double one(int which, std::span<const double> x, const double* y = nullptr) {
  double out = 0.0;
  gpu::check(hs_plain(which, x.data(), x.size(), y, &out));
  return out;
}
}  // namespace detail

inline double mean(std::span<const double> x) { return detail::one(0, x); }
inline double variance(std::span<const double> x) { return detail::one(1, x); }
inline double stddev(std::span<const double> x) { return detail::one(7, x); }
inline double skewness(std::span<const double> x) { return detail::one(2, x); }
inline double kurtosis_ratio(std::span<const double> x) { return detail::one(3, x); }
inline double coeff_variation(std::span<const double> x) { return detail::one(4, x); }

inline std::vector<double> znorm(std::span<const double> x) {
  std::vector<double> out(x.size() ? x.size() : 1);
  gpu::check(hs_plain(6, x.data(), x.size(), nullptr, out.data()));
  out.resize(x.size());
  return out;
}

inline double pearson(std::span<const double> x, std::span<const double> y) {
  if (x.size() != y.size()) throw length_mismatch("plain::pearson: length mismatch");
  return detail::one(5, x, y.data());
}

}  // namespace hestat::plain
