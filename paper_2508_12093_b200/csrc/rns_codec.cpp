// rns_codec.cpp — CKKS canonical-embedding encode / decode for Tier R (host).
//
// Slot j of a plaintext m(X) in Z[X]/(X^N + 1) is m(zeta^{t_j}) with
// zeta = exp(i*pi/N) and t_j = 5^j mod 2N (j < S = N/2), so the Galois map
// X -> X^{5^k} (hs_rns_rotate) is a left rotation of the slots by k — the
// reference's rotate semantics (ckks.hpp:193-202).
//
//   decode: z_j = sum_k m_k zeta^{k t_j}         = one 2N-point FFT (+ sign) of m
//   encode: m_k = (2/N) Re sum_j z_j zeta^{-k t_j} = one 2N-point FFT (- sign) of z
//           placed at positions t_j; coefficients are round(scale * m_k).
// Both are O(N log N) in double precision; the integer coefficients feed the
// device RLWE encryption (rns.cu), decryption returns centred integers mod q_0.
#include "rns_codec.h"

#include <cmath>
#include <complex>
#include <cstdint>
#include <mutex>
#include <stdexcept>
#include <unordered_map>
#include <vector>

namespace hsg {
namespace rns {
namespace {

using cd = std::complex<double>;

struct FftPlan {
  uint32_t n = 0, logn = 0;
  std::vector<cd> w;           // w[k] = exp(2 pi i k / n), k < n/2
  std::vector<uint32_t> rev;   // bit reversal of log2(n) bits
  std::vector<uint32_t> t;     // slot j -> 5^j mod n  (n = 2N)
};

const FftPlan& plan(uint32_t logN) {
  static std::mutex mu;
  static std::unordered_map<uint32_t, FftPlan> plans;
  std::lock_guard<std::mutex> g(mu);
  auto it = plans.find(logN);
  if (it != plans.end()) return it->second;
  FftPlan p;
  p.logn = logN + 1;
  p.n = 1u << p.logn;
  p.w.resize(p.n / 2);
  for (uint32_t k = 0; k < p.n / 2; ++k) {
    const double a = 2.0 * M_PI * static_cast<double>(k) / static_cast<double>(p.n);
    p.w[k] = cd(std::cos(a), std::sin(a));
  }
  p.rev.resize(p.n);
  for (uint32_t k = 0; k < p.n; ++k) {
    uint32_t r = 0;
    for (uint32_t b = 0; b < p.logn; ++b) r |= ((k >> b) & 1u) << (p.logn - 1 - b);
    p.rev[k] = r;
  }
  const uint32_t S = 1u << (logN - 1);
  p.t.resize(S);
  uint64_t t = 1;
  for (uint32_t j = 0; j < S; ++j) {
    p.t[j] = static_cast<uint32_t>(t);
    t = (t * 5) % p.n;
  }
  return plans.emplace(logN, std::move(p)).first->second;
}

// in-place radix-2 FFT, X_t = sum_k x_k exp(sign * 2 pi i k t / n).  The complex product is
// written out (re = ar wr - ai wi, im = ar wi + ai wr): the same roundings as std::complex's
// operator* on finite values (no contraction: -ffp-contract=off), without its out-of-line
// NaN/Inf recovery call, which made this loop ~5x slower.
void fft(std::vector<cd>& a, const FftPlan& p, int sign) {
  const uint32_t n = p.n;
  for (uint32_t k = 0; k < n; ++k)
    if (k < p.rev[k]) std::swap(a[k], a[p.rev[k]]);
  double* x = reinterpret_cast<double*>(a.data());  // interleaved re, im (std::complex layout)
  const double* w = reinterpret_cast<const double*>(p.w.data());
  const double sg = sign < 0 ? -1.0 : 1.0;
  for (uint32_t len = 2; len <= n; len <<= 1) {
    const uint32_t half = len / 2, step = n / len;
    for (uint32_t i = 0; i < n; i += len)
      for (uint32_t k = 0; k < half; ++k) {
        const double wr = w[2 * size_t(k) * step], wi = sg * w[2 * size_t(k) * step + 1];
        double* u = x + 2 * size_t(i + k);
        double* v = x + 2 * size_t(i + k + half);
        const double vr = v[0] * wr - v[1] * wi, vi = v[0] * wi + v[1] * wr;
        const double ur = u[0], ui = u[1];
        u[0] = ur + vr;
        u[1] = ui + vi;
        v[0] = ur - vr;
        v[1] = ui - vi;
      }
  }
}

}  // namespace

void encode(uint32_t logN, const double* z, size_t n, double scale, int64_t* coeffs) {
  const FftPlan& p = plan(logN);
  const uint32_t N = 1u << logN, S = N / 2;
  if (n > S) throw std::invalid_argument("encode: more values than slots");
  std::vector<cd> a(p.n, cd(0.0, 0.0));
  for (size_t j = 0; j < n; ++j) a[p.t[j]] = cd(z[j], 0.0);
  fft(a, p, -1);
  const double f = 2.0 / static_cast<double>(N);
  for (uint32_t k = 0; k < N; ++k) {
    const double v = std::nearbyint(a[k].real() * f * scale);
    if (!(std::fabs(v) < 9.0e18)) throw std::invalid_argument("encode: coefficient out of int64 range");
    coeffs[k] = static_cast<int64_t>(v);
  }
}

void encode_real(uint32_t logN, const double* z, size_t n, double scale, double* coeffs) {
  const FftPlan& p = plan(logN);
  const uint32_t N = 1u << logN, S = N / 2;
  if (n > S) throw std::invalid_argument("encode: more values than slots");
  std::vector<cd> a(p.n, cd(0.0, 0.0));
  for (size_t j = 0; j < n; ++j) a[p.t[j]] = cd(z[j], 0.0);
  fft(a, p, -1);
  const double f = 2.0 / static_cast<double>(N);
  for (uint32_t k = 0; k < N; ++k) coeffs[k] = std::nearbyint(a[k].real() * f * scale);
}

void decode_real(uint32_t logN, const double* coeffs, double scale, double* z, size_t n) {
  const FftPlan& p = plan(logN);
  const uint32_t N = 1u << logN, S = N / 2;
  if (n > S) throw std::invalid_argument("decode: more values than slots");
  std::vector<cd> a(p.n, cd(0.0, 0.0));
  for (uint32_t k = 0; k < N; ++k) a[k] = cd(coeffs[k] / scale, 0.0);
  fft(a, p, +1);
  for (size_t j = 0; j < n; ++j) z[j] = a[p.t[j]].real();
}

void decode(uint32_t logN, const int64_t* coeffs, double scale, double* z, size_t n) {
  const FftPlan& p = plan(logN);
  const uint32_t N = 1u << logN, S = N / 2;
  if (n > S) throw std::invalid_argument("decode: more values than slots");
  std::vector<cd> a(p.n, cd(0.0, 0.0));
  for (uint32_t k = 0; k < N; ++k) a[k] = cd(static_cast<double>(coeffs[k]) / scale, 0.0);
  fft(a, p, +1);
  for (size_t j = 0; j < n; ++j) z[j] = a[p.t[j]].real();
}

}  // namespace rns
}  // namespace hsg
