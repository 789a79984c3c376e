// rns_eval.cu — RnsB: EvalContext ops (ckks.hpp:97-240) over RNS-CKKS ciphertexts.
// Ledger logic (shape checks, level min-rule, auto-bootstrap of exhausted operands,
// level_exhausted, meter) is the same as SymB/DevB (backends.h); the values live in
// Tier-R ciphertexts and every op is Tier-R kernels (rns.cu).  See rns_eval.h.
#include "rns_eval.h"

#include <cmath>
#include <cstring>
#include <string>

#include "rns_codec.h"

namespace hsg {
namespace rns {

RnsB::RnsB(Ctx& c, const Params& p, Meter& m) : LedgerBase(p, m), c_(c) {
  if (p.S != c.N / 2) fail(HS_E_INVALID_ARG, "rns eval: slot_count must be N/2 of the RNS context");
  sigma_.resize(c.spec.L + 1);
  sigma_[0] = std::ldexp(1.0, static_cast<int>(c.spec.logq));  // CKKS scale ~ the rescaling primes
  for (uint32_t l = 1; l <= c.spec.L; ++l) sigma_[l] = std::sqrt(sigma_[l - 1] * static_cast<double>(c.primes[l]));
}

RCt RnsB::make(DevBuf b, int phys, int level) const {
  auto d = std::make_shared<RCtData>();
  d->buf = std::move(b);
  d->phys = phys;
  d->level = level;
  d->n = p_.S;
  return d;
}

RCt RnsB::encrypt(const double* v, size_t n) {  // ckks.hpp:97-104
  if (n > p_.S) fail(HS_E_TOO_MANY_VALUES, "encrypt: more values than slots");
  const int L = static_cast<int>(c_.spec.L);
  std::vector<double> co(c_.N);
  encode_real(c_.spec.logN, v, n, sigma_[L], co.data());
  DevBuf b = Runtime::get().alloc(words(L));
  encrypt_real(c_, L, co.data(), tag_++, reinterpret_cast<uint64_t*>(b.get()));
  return make(b, L, p_.max_level);
}

std::vector<RCt> RnsB::encrypt_column(const double* v, size_t n) {  // column.hpp:25-39
  for (size_t i = 0; i < n; ++i)
    if (!std::isfinite(v[i])) fail(HS_E_NON_FINITE_VALUE, "encode_column: non-finite value in column");
  std::vector<RCt> out;
  for (size_t off = 0; off < n; off += p_.S) out.push_back(encrypt(v + off, std::min(p_.S, n - off)));
  return out;
}

RCt RnsB::encrypt_const(double c) {
  std::vector<double> v(p_.S, c);
  return encrypt(v.data(), v.size());
}

RCt RnsB::align(const RCt& x, int p) {
  if (x->phys == p) return x;
  Runtime& rt = Runtime::get();
  const uint64_t* src = reinterpret_cast<const uint64_t*>(x->buf.get());
  const int k = p + 1;  // drop limbs down to level p+1, then one scaled rescale to p
  DevBuf t;
  const uint64_t* at = src;
  if (x->phys > k) {
    t = rt.alloc(words(k));
    const size_t row = c_.N * sizeof(uint64_t), keep = size_t(k + 1) * row;
    uint64_t* dst = reinterpret_cast<uint64_t*>(t.get());
    cuda_ok(cudaMemcpyAsync(dst, src, keep, cudaMemcpyDeviceToDevice, rt.stream()), "drop limbs");
    cuda_ok(cudaMemcpyAsync(reinterpret_cast<char*>(dst) + keep,
                            reinterpret_cast<const char*>(src) + size_t(x->phys + 1) * row, keep,
                            cudaMemcpyDeviceToDevice, rt.stream()),
            "drop limbs");
    at = dst;
  }
  // scale sigma_k * C / q_k = sigma_p  =>  C = sigma_p q_k / sigma_k
  const double C = sigma_[p] * static_cast<double>(c_.primes[k]) / sigma_[k];
  DevBuf o = rt.alloc(words(p));
  rescale_mul_big(c_, k, at, C, reinterpret_cast<uint64_t*>(o.get()), 1);  // rescale(C x), C x never stored
  return make(o, p, x->level);
}

RCt RnsB::addsub(const RCt& a, const RCt& b, bool sub) {  // ckks.hpp:113-133
  check_shape(sz(a));
  check_shape(sz(b));
  const int p = std::min(a->phys, b->phys);
  const RCt x = align(a, p), y = align(b, p);
  DevBuf o = Runtime::get().alloc(words(p));
  add_sub(c_, p, reinterpret_cast<const uint64_t*>(x->buf.get()), reinterpret_cast<const uint64_t*>(y->buf.get()),
          reinterpret_cast<uint64_t*>(o.get()), 1, sub);
  ++m_.add;
  return make(o, p, std::min(a->level, b->level));
}

RCt RnsB::add_pt(const RCt& a, double c) {  // ckks.hpp:137-144
  check_shape(sz(a));
  DevBuf o = Runtime::get().alloc(words(a->phys));
  const_op_big(c_, a->phys, reinterpret_cast<const uint64_t*>(a->buf.get()), c * sigma_[a->phys],
               reinterpret_cast<uint64_t*>(o.get()), 1, false);
  ++m_.add;
  return make(o, a->phys, a->level);
}

RCt RnsB::bootstrap(const RCt& a) {  // ckks.hpp:207-213: logical level reset (deep chain)
  check_shape(sz(a));
  ++m_.bootstrap;
  return make(a->buf, a->phys, p_.max_level);
}

RCt RnsB::mul_ct(RCt a, RCt b) {  // ckks.hpp:149-164
  check_shape(sz(a));
  check_shape(sz(b));
  if (std::min(a->level, b->level) < 1) {
    if (!p_.auto_bootstrap) fail(HS_E_LEVEL_EXHAUSTED, "mul_ct: no multiplicative level left");
    if (a->level < 1) a = bootstrap(a);
    if (b->level < 1) b = bootstrap(b);
  }
  const int p = std::min(a->phys, b->phys);
  if (p < 1) fail(HS_E_LEVEL_EXHAUSTED, "mul_ct: RNS modulus chain exhausted (deep chain too short)");
  const RCt x = align(a, p), y = a == b ? x : align(b, p);
  DevBuf o = Runtime::get().alloc(words(p - 1));
  mul_relin_rescale(c_, p, reinterpret_cast<const uint64_t*>(x->buf.get()),
                    reinterpret_cast<const uint64_t*>(y->buf.get()), reinterpret_cast<uint64_t*>(o.get()), 1);
  ++m_.mul_ct;
  return make(o, p - 1, std::min(a->level, b->level) - 1);
}

RCt RnsB::prepare_mul_pt(RCt a) {  // ckks.hpp:233-240
  if (a->level < 1) {
    if (!p_.auto_bootstrap) fail(HS_E_LEVEL_EXHAUSTED, "mul_pt: no multiplicative level left");
    a = bootstrap(a);
  }
  return a;
}

RCt RnsB::mul_pt(RCt a, double c) {  // ckks.hpp:168-176
  check_shape(sz(a));
  a = prepare_mul_pt(a);
  const int p = a->phys;
  if (p < 1) fail(HS_E_LEVEL_EXHAUSTED, "mul_pt: RNS modulus chain exhausted (deep chain too short)");
  // constant at sigma_{p-1} q_p / sigma_p: the product rescales onto sigma_{p-1} exactly
  const double C = c * sigma_[p - 1] * static_cast<double>(c_.primes[p]) / sigma_[p];
  DevBuf o = Runtime::get().alloc(words(p - 1));
  rescale_mul_big(c_, p, reinterpret_cast<const uint64_t*>(a->buf.get()), C, reinterpret_cast<uint64_t*>(o.get()), 1);
  ++m_.mul_pt;
  return make(o, p - 1, a->level - 1);
}

RCt RnsB::mul_pt_vec(RCt a, const std::vector<double>& v) {  // ckks.hpp:179-189
  check_shape(sz(a));
  if (v.size() != p_.S) fail(HS_E_LENGTH_MISMATCH, "mul_pt: plaintext vector length != slot count");
  a = prepare_mul_pt(a);
  const int p = a->phys;
  if (p < 1) fail(HS_E_LEVEL_EXHAUSTED, "mul_pt: RNS modulus chain exhausted (deep chain too short)");
  std::vector<double> co(c_.N);
  encode_real(c_.spec.logN, v.data(), v.size(), sigma_[p - 1] * static_cast<double>(c_.primes[p]) / sigma_[p],
              co.data());
  Runtime& rt = Runtime::get();
  DevBuf m = rt.alloc(words(p));
  mul_plain_real(c_, p, reinterpret_cast<const uint64_t*>(a->buf.get()), co.data(), reinterpret_cast<uint64_t*>(m.get()));
  DevBuf o = rt.alloc(words(p - 1));
  rescale(c_, p, reinterpret_cast<const uint64_t*>(m.get()), reinterpret_cast<uint64_t*>(o.get()), 1);
  ++m_.mul_pt;
  return make(o, p - 1, a->level - 1);
}

RCt RnsB::rotate(const RCt& a, long kk) {  // ckks.hpp:193-202
  check_shape(sz(a));
  const long n = static_cast<long>(p_.S);
  const long shift = ((kk % n) + n) % n;
  DevBuf o = Runtime::get().alloc(words(a->phys));
  rns::rotate(c_, a->phys, shift, reinterpret_cast<const uint64_t*>(a->buf.get()),
              reinterpret_cast<uint64_t*>(o.get()), 1);
  ++m_.rotate;
  return make(o, a->phys, a->level);
}

RCt RnsB::sum_all_slots(const RCt& a, size_t n_valid) {  // ckks.hpp:218-230
  check_shape(sz(a));
  if (p_.debug && n_valid < p_.S) {
    const double eps = std::ldexp(1.0, -(p_.scale_bits - 1));
    const std::vector<double> h = decrypt(a, p_.S);
    for (size_t i = n_valid; i < p_.S; ++i)
      if (std::abs(h[i]) > eps) fail(HS_E_DIRTY_PADDING, "sum_all_slots: nonzero padding slot");
  }
  RCt acc = a;
  for (size_t step = 1; step < p_.S; step <<= 1) acc = add_ct(acc, rotate(acc, static_cast<long>(step)));
  return acc;
}

std::vector<double> RnsB::decrypt(const RCt& c, size_t n) {
  // q_0 alone cannot hold sigma_0 * value for |value| >= 2^(log q_0 - log sigma_0 - 1): decrypt through two limbs
  if (c->phys < 1)
    fail(HS_E_LEVEL_EXHAUSTED, "rns decrypt: result at the last RNS limb (chain must exceed the statistic's depth)");
  std::vector<double> co(c_.N);
  decrypt_crt(c_, c->phys, reinterpret_cast<const uint64_t*>(c->buf.get()), co.data());
  std::vector<double> z(n);
  decode_real(c_.spec.logN, co.data(), sigma_[c->phys], z.data(), n);
  return z;
}

// ---- debug-mode value checks (decrypt on the diagnostics path) ----
double RnsB::first_slot(const RCt& c) { return decrypt(c, 1)[0]; }

void RnsB::check_open_domain(const RCt& c, size_t n_valid, double lo, double hi, const char* who) {
  const std::vector<double> h = decrypt(c, std::min(n_valid, c->n));
  for (double t : h)
    if (!(t > lo) || !(t <= hi)) fail(HS_E_DOMAIN_VIOLATION, std::string(who) + ": scaled slot outside domain");
}

void RnsB::check_eval_domain(const RCt& c, double lo, double hi) {
  for (double v : decrypt(c, c->n))
    if (v < lo - 1e-9 || v > hi + 1e-9) fail(HS_E_DOMAIN_VIOLATION, "eval_encrypted: slot outside series domain");
}

void RnsB::check_divergence(const RCt& c, size_t n_valid) {
  for (double v : decrypt(c, std::min(n_valid, c->n)))
    if (!(std::abs(v) <= 1e6)) fail(HS_E_DIVERGENCE, "newton iterate exceeded the divergence guard");
}

void RnsB::check_sqrt_domain(const RCt& c, size_t n_valid) {
  for (double v : decrypt(c, std::min(n_valid, c->n)))
    if (v < -1e-9 || v > 2.0 + 1e-9) fail(HS_E_DOMAIN_VIOLATION, "crypto_sqrt: scaled slot outside [0, 2]");
}

void RnsB::check_sign_domain(const RCt& c) {
  for (double v : decrypt(c, c->n))
    if (v < -1.0 - 1e-9 || v > 1.0 + 1e-9) fail(HS_E_DOMAIN_VIOLATION, "crypto_sign: slot outside [-1, 1]");
}

}  // namespace rns
}  // namespace hsg
