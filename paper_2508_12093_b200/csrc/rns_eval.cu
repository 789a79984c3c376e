// rns_eval.cu — RnsB: EvalContext ops (ckks.hpp:97-240) over RNS-CKKS ciphertexts.
// Ledger logic (shape checks, level min-rule, auto-bootstrap of exhausted operands,
// level_exhausted, meter) is the same as SymB/DevB (backends.h); the values live in
// Tier-R ciphertexts and every op is Tier-R kernels (rns.cu).  See rns_eval.h.
#include "rns_eval.h"

#include <cmath>
#include <algorithm>
#include <thread>
#include <mutex>
#include <exception>
#include <atomic>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <string>

#include "rns_codec.h"
#include "series.h"

namespace hsg {
namespace rns {

RnsB::RnsB(Ctx& c, const Params& p, Meter& m, Boot boot) : LedgerBase(p, m), c_(c), boot_(boot) {
  if (boot == Boot::Refresh && static_cast<int>(c.spec.L) < p.max_level + 1)
    fail(HS_E_INVALID_ARG, "rns eval: refresh bootstrapping needs a chain of at least max_level + 1 primes");
  if (p.S != c.N / 2) fail(HS_E_INVALID_ARG, "rns eval: slot_count must be N/2 of the RNS context");
  sigma_.resize(c.spec.L + 1);
  sigma_[0] = std::ldexp(1.0, static_cast<int>(c.spec.logq));  // CKKS scale ~ the rescaling primes
  for (uint32_t l = 1; l <= c.spec.L; ++l) sigma_[l] = std::sqrt(sigma_[l - 1] * static_cast<double>(c.primes[l]));
}

RCt RnsB::make(DevBuf b, int phys, int level, size_t off) const {
  auto d = std::make_shared<RCtData>();
  d->buf = std::move(b);
  d->off = off;
  d->phys = phys;
  d->level = level;
  d->n = p_.S;
  return d;
}

// host slot values -> device (the canonical-embedding encoding runs on the device, codec_gpu.cu)
static DevBuf upload_values(const double* v, size_t n) {
  Runtime& rt = Runtime::get();
  DevBuf d = rt.alloc(std::max<size_t>(n, 1));
  if (n) cuda_ok(cudaMemcpyAsync(d.get(), v, n * 8, cudaMemcpyHostToDevice, rt.stream()), "encode upload");
  return d;
}

RCt RnsB::encrypt(const double* v, size_t n) {  // ckks.hpp:97-104
  if (n > p_.S) fail(HS_E_TOO_MANY_VALUES, "encrypt: more values than slots");
  const int L = static_cast<int>(c_.spec.L);
  Runtime& rt = Runtime::get();
  DevBuf z = upload_values(v, n), co = rt.alloc(c_.N);
  encode_dev(c_.spec.logN, reinterpret_cast<const double*>(z.get()), n, sigma_[L], co.get(), 1);
  DevBuf b = rt.alloc(words(L));
  encrypt_real_dev(c_, L, co.get(), tag_++, reinterpret_cast<uint64_t*>(b.get()));
  return make(b, L, p_.max_level);
}

std::vector<RCt> RnsB::encrypt_column(const double* v, size_t n) {  // column.hpp:25-39
  for (size_t i = 0; i < n; ++i)
    if (!std::isfinite(v[i])) fail(HS_E_NON_FINITE_VALUE, "encode_column: non-finite value in column");
  // one upload, the chunks' canonical-embedding encodings as one batched device transform, then
  // the encryptions in order (the per-chunk randomness tags follow the chunk order, as in encrypt())
  const size_t nch = (n + p_.S - 1) / p_.S;
  const int L = static_cast<int>(c_.spec.L);
  Runtime& rt = Runtime::get();
  DevBuf z = upload_values(v, n), co = rt.alloc(nch * c_.N);
  encode_dev(c_.spec.logN, reinterpret_cast<const double*>(z.get()), n, sigma_[L], co.get(),
             static_cast<uint32_t>(nch));
  std::vector<RCt> out;
  DevBuf b = rt.alloc(nch * words(L));  // one contiguous buffer: chunk ops batch without copies
  for (size_t k = 0; k < nch; ++k) {
    encrypt_real_dev(c_, L, co.get() + k * c_.N, tag_++, reinterpret_cast<uint64_t*>(b.get()) + k * words(L));
    out.push_back(make(b, L, p_.max_level, k * words(L)));
  }
  rt.sync();  // the caller's values may be released on return
  return out;
}

std::vector<std::vector<double>> RnsB::decrypt_many(const std::vector<RCt>& cts, const std::vector<size_t>& ns) {
  std::vector<std::vector<double>> out(cts.size());
  for (size_t k = 0; k < cts.size(); ++k) out[k] = decrypt(cts[k], ns[k]);
  return out;
}

RCt RnsB::encrypt_const(double c) {
  std::vector<double> v(p_.S, c);
  return encrypt(v.data(), v.size());
}

RCt RnsB::align(const RCt& x, int p) {
  if (x->phys == p) return x;
  Runtime& rt = Runtime::get();
  const uint64_t* src = x->ptr();
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
  add_sub(c_, p, x->ptr(), y->ptr(),
          reinterpret_cast<uint64_t*>(o.get()), 1, sub);
  ++m_.add;
  return make(o, p, std::min(a->level, b->level));
}

RCt RnsB::add_pt(const RCt& a, double c) {  // ckks.hpp:137-144
  check_shape(sz(a));
  DevBuf o = Runtime::get().alloc(words(a->phys));
  const_op_big(c_, a->phys, a->ptr(), c * sigma_[a->phys],
               reinterpret_cast<uint64_t*>(o.get()), 1, false);
  ++m_.add;
  return make(o, a->phys, a->level);
}

RCt RnsB::bootstrap(const RCt& a) {  // ckks.hpp:207-213
  check_shape(sz(a));
  ++m_.bootstrap;
  if (boot_ == Boot::Refresh) return refresh(a);
  return make(a->buf, a->phys, p_.max_level, a->off);  // logical level reset (deep chain)
}

// decrypt (CRT through q_0 q_1) -> coefficients at sigma_phys -> rescaled to sigma_L -> encrypted
// at the top of the chain with a fresh tag: same slots, fresh noise, logical level max_level
RCt RnsB::refresh(const RCt& a) {
  if (a->phys < 1) fail(HS_E_LEVEL_EXHAUSTED, "rns refresh: ciphertext at the last RNS limb");
  const int L = static_cast<int>(c_.spec.L);
  Runtime& rt = Runtime::get();
  DevBuf co = rt.alloc(c_.N);  // the refresh stays on the device: decrypt, rescale, re-encrypt
  decrypt_crt_dev(c_, a->phys, a->ptr(), co.get());
  scale_round_dev(c_, co.get(), sigma_[L] / sigma_[a->phys]);
  DevBuf b = rt.alloc(words(L));
  encrypt_real_dev(c_, L, co.get(), tag_++, reinterpret_cast<uint64_t*>(b.get()));
  RCt o = make(b, L, p_.max_level);
  const_cast<RCtData*>(o.get())->n = a->n;
  return o;
}

RCt Home::adopt(const Ct& x) {
  if (!x || x->n == 0) return nullptr;  // Ciphertext(): the reference's empty accumulator (size 0, level 0)
  const std::vector<double>& v = x->host_slots();
  std::vector<double> pad(p.S, 0.0);
  std::copy(v.begin(), v.begin() + std::min(v.size(), p.S), pad.begin());
  RCt e = b->encrypt(pad.data(), pad.size());
  auto d = std::make_shared<RCtData>(*e);
  d->level = x->level;
  d->n = x->n;  // a size other than slot_count keeps failing shape checks, as in the reference
  return d;
}

Spec default_spec(const Params& p, Boot boot, uint32_t depth, uint64_t seed) {
  Spec s;
  uint32_t logN = 1;
  while ((size_t(1) << logN) < 2 * p.S) ++logN;
  if ((size_t(1) << logN) != 2 * p.S) fail(HS_E_INVALID_ARG, "rns: slot_count must be a power of two");
  s.logN = logN;
  s.L = boot == Boot::Refresh ? static_cast<uint32_t>(p.max_level) + 1 : depth + 1;
  s.logq0 = 61;
  s.logq = 60;
  s.logp = 61;
  s.dnum = std::min<uint32_t>(3, s.L + 1);
  const uint32_t alpha = (s.L + 1 + s.dnum - 1) / s.dnum;
  s.K = (s.logq0 + (alpha - 1) * s.logq + 1 + s.logp - 1) / s.logp;  // P above every digit modulus
  s.h = 0;
  s.seed = seed;
  return s;
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
  mul_relin_rescale(c_, p, x->ptr(),
                    y->ptr(), reinterpret_cast<uint64_t*>(o.get()), 1);
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
  rescale_mul_big(c_, p, a->ptr(), C, reinterpret_cast<uint64_t*>(o.get()), 1);
  ++m_.mul_pt;
  return make(o, p - 1, a->level - 1);
}

RCt RnsB::mul_pt_vec(RCt a, const std::vector<double>& v) {  // ckks.hpp:179-189
  check_shape(sz(a));
  if (v.size() != p_.S) fail(HS_E_LENGTH_MISMATCH, "mul_pt: plaintext vector length != slot count");
  a = prepare_mul_pt(a);
  const int p = a->phys;
  if (p < 1) fail(HS_E_LEVEL_EXHAUSTED, "mul_pt: RNS modulus chain exhausted (deep chain too short)");
  Runtime& rt = Runtime::get();
  DevBuf z = upload_values(v.data(), v.size()), co = rt.alloc(c_.N);
  encode_dev(c_.spec.logN, reinterpret_cast<const double*>(z.get()), v.size(),
             sigma_[p - 1] * static_cast<double>(c_.primes[p]) / sigma_[p], co.get(), 1);
  DevBuf m = rt.alloc(words(p));
  mul_plain_real_dev(c_, p, a->ptr(), co.get(), reinterpret_cast<uint64_t*>(m.get()));
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
  rns::rotate(c_, a->phys, shift, a->ptr(),
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

// ---- batched BSGS ---------------------------------------------------------------------
RnsB::Batch RnsB::slice(const Batch& b, uint32_t first, uint32_t count) const {
  Batch r = b;
  r.off = b.off + size_t(first) * words(b.phys);
  r.n = count;
  return r;
}

// RnsB::align for n ciphertexts at once (same constant, same rescale): words identical
RnsB::Batch RnsB::align_batch(const Batch& b, int p) {
  if (b.phys == p) return b;
  Runtime& rt = Runtime::get();
  const int k = p + 1;
  const uint64_t* at = b.ptr();
  DevBuf t;
  if (b.phys > k) {  // drop limbs: rows 0..k of every polynomial of every item
    t = rt.alloc(size_t(b.n) * words(k));
    const size_t row = c_.N * sizeof(uint64_t);
    cuda_ok(cudaMemcpy2DAsync(t.get(), size_t(k + 1) * row, at, size_t(b.phys + 1) * row, size_t(k + 1) * row,
                              size_t(2) * b.n, cudaMemcpyDeviceToDevice, rt.stream()),
            "drop limbs (batch)");
    at = reinterpret_cast<const uint64_t*>(t.get());
  }
  const double C = sigma_[p] * static_cast<double>(c_.primes[k]) / sigma_[k];
  std::vector<uint64_t> res(k + 1);
  residues_of(c_, k, C, res.data());
  Batch o;
  o.buf = rt.alloc(size_t(b.n) * words(p));
  o.phys = p;
  o.level = b.level;
  o.n = b.n;
  rescale_mul_items(c_, k, at, false, &res, nullptr, reinterpret_cast<uint64_t*>(o.buf.get()), b.n);
  return o;
}

// HS_RNS_BSGS=0: always the op-by-op recursion (A/B and parity switch)
static bool bsgs_batch_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("HS_RNS_BSGS");
    return !e || std::atoi(e) != 0;
  }();
  return on;
}

bool RnsB::batch_ok(const std::vector<RCt>& xs) const {
  if (!bsgs_batch_enabled() || xs.empty() || !xs[0]) return false;
  for (const RCt& x : xs)
    if (!x || x->phys != xs[0]->phys || x->level != xs[0]->level || x->n != xs[0]->n) return false;
  return xs[0]->phys >= 1 && xs[0]->level >= 1;
}

RnsB::Batch RnsB::gather(const std::vector<RCt>& xs) {
  Batch b;
  b.phys = xs[0]->phys;
  b.level = xs[0]->level;
  b.n = static_cast<uint32_t>(xs.size());
  const size_t w = words(b.phys);
  bool contiguous = true;
  for (size_t i = 1; i < xs.size() && contiguous; ++i)
    contiguous = xs[i]->buf == xs[0]->buf && xs[i]->off == xs[0]->off + i * w;
  if (contiguous) {
    b.buf = xs[0]->buf;
    b.off = xs[0]->off;
    return b;
  }
  Runtime& rt = Runtime::get();
  b.buf = rt.alloc(size_t(b.n) * w);
  for (size_t i = 0; i < xs.size(); ++i)
    cuda_ok(cudaMemcpyAsync(reinterpret_cast<uint64_t*>(b.buf.get()) + i * w, xs[i]->ptr(), w * 8,
                            cudaMemcpyDeviceToDevice, rt.stream()),
            "gather chunks");
  return b;
}

std::vector<RCt> RnsB::split(const Batch& b) {
  std::vector<RCt> out;
  for (uint32_t i = 0; i < b.n; ++i) out.push_back(make(b.buf, b.phys, b.level, b.off + size_t(i) * words(b.phys)));
  return out;
}

std::vector<RCt> RnsB::mul_pt_many(const std::vector<RCt>& xs, double c) {  // mul_pt (ckks.hpp:168-176) per chunk
  for (const RCt& x : xs) check_shape(sz(x));
  const Batch X = gather(xs);
  const int p = X.phys;
  const double C = c * sigma_[p - 1] * static_cast<double>(c_.primes[p]) / sigma_[p];  // exactly as mul_pt
  std::vector<uint64_t> res(p + 1);
  residues_of(c_, p, C, res.data());
  Batch o;
  o.phys = p - 1;
  o.level = X.level - 1;
  o.n = X.n;
  o.buf = Runtime::get().alloc(size_t(o.n) * words(o.phys));
  rescale_mul_items(c_, p, X.ptr(), false, &res, nullptr, reinterpret_cast<uint64_t*>(o.buf.get()), X.n);
  m_.mul_pt += X.n;
  return split(o);
}

std::vector<RCt> RnsB::square_many(const std::vector<RCt>& xs) {  // mul_ct(a, a) (ckks.hpp:149-164) per chunk
  for (const RCt& x : xs) check_shape(sz(x));
  const Batch X = gather(xs);
  const int p = X.phys;
  Batch o;
  o.phys = p - 1;
  o.level = X.level - 1;
  o.n = X.n;
  o.buf = Runtime::get().alloc(size_t(o.n) * words(o.phys));
  mul_relin_rescale(c_, p, X.ptr(), X.ptr(), reinterpret_cast<uint64_t*>(o.buf.get()), X.n);
  m_.mul_ct += X.n;
  return split(o);
}

bool RnsB::bsgs_batch_ok(const RCt& x, const std::vector<RCt>& pw, int K) const {
  if (!bsgs_batch_enabled() || !x || K < 2 || static_cast<int>(pw.size()) < K) return false;
  int lv = x->level, ph = x->phys;
  if (lv < 1 || ph < 1) return false;
  --lv, --ph;  // leaves: mul_pt then add_pt
  for (int h = 1; h < K; ++h) {
    const RCt& T = pw[h];
    if (!T || lv < 1 || T->level < 1) return false;
    const int p = std::min(ph, T->phys);
    if (p < 1) return false;
    const int hl = std::min(lv, T->level) - 1, hp = p - 1;
    lv = std::min(hl, lv);
    ph = std::min(hp, ph);
  }
  return true;
}

RCt RnsB::bsgs_full_tree(const RCt& x, const std::vector<double>& coeffs, const std::vector<RCt>& pw) {
  int K = 0;
  while ((size_t(1) << K) < coeffs.size()) ++K;
  // leaf coefficients through the reference's own split (chebyshev.hpp:140-158), placed in
  // the storage order that makes every stage's q- and r-children contiguous halves
  std::vector<std::vector<uint32_t>> order(K);
  order[K - 1] = {0};
  for (int h = K - 1; h >= 1; --h) {
    for (uint32_t v : order[h]) order[h - 1].push_back(2 * v + 1);  // q-children first
    for (uint32_t v : order[h]) order[h - 1].push_back(2 * v);      // then r-children
  }
  const uint32_t n0 = 1u << (K - 1);
  std::vector<double> c0(n0), c1(n0);
  std::vector<uint32_t> pos(n0);
  for (uint32_t i = 0; i < n0; ++i) pos[order[0][i]] = i;
  std::function<void(const std::vector<double>&, int, uint32_t)> collect =
      [&](const std::vector<double>& c, int h, uint32_t j) {
        if (h == 0) {
          c0[pos[j]] = c[0];
          c1[pos[j]] = c.size() > 1 ? c[1] : 0.0;
          return;
        }
        std::vector<double> q, r;
        split_series(c, &q, &r);
        collect(q, h - 1, 2 * j + 1);
        collect(r, h - 1, 2 * j);
      };
  collect(coeffs, K - 1, 0);

  Runtime& rt = Runtime::get();
  // leaves: mul_pt(x, c1) (rescale of c1' x, x shared), then add_pt(., c0)
  const int p0 = x->phys;
  Batch R;
  R.phys = p0 - 1;
  R.level = x->level - 1;
  R.n = n0;
  R.buf = rt.alloc(size_t(n0) * words(R.phys));
  {
    std::vector<uint64_t> km(size_t(n0) * (p0 + 1)), ka(size_t(n0) * p0);
    for (uint32_t i = 0; i < n0; ++i) {  // the constants exactly as mul_pt / add_pt compute them
      residues_of(c_, p0, c1[i] * sigma_[p0 - 1] * static_cast<double>(c_.primes[p0]) / sigma_[p0],
                  &km[size_t(i) * (p0 + 1)]);
      residues_of(c_, p0 - 1, c0[i] * sigma_[p0 - 1], &ka[size_t(i) * p0]);
    }
    uint64_t* o = reinterpret_cast<uint64_t*>(R.buf.get());
    rescale_mul_items(c_, p0, x->ptr(), true, nullptr, &km, o, n0, &ka);  // add_pt fused into the store
    m_.mul_pt += n0;
    m_.add += n0;
  }
  // height h: head = mul_ct(q-child, T_{2^h}); node = add_ct(head, r-child)
  for (int h = 1; h < K; ++h) {
    const uint32_t nh = R.n / 2;
    Batch Q = slice(R, 0, nh), Rr = slice(R, nh, nh);
    const RCt& T = pw[h];
    const int p = std::min(Q.phys, T->phys);
    Q = align_batch(Q, p);
    const RCt Ta = align(T, p);
    Batch H;
    H.phys = p - 1;
    H.level = std::min(Q.level, T->level) - 1;
    H.n = nh;
    H.buf = rt.alloc(size_t(nh) * words(H.phys));
    mul_relin_rescale(c_, p, Q.ptr(), Ta->ptr(), reinterpret_cast<uint64_t*>(H.buf.get()), nh, true);
    m_.mul_ct += nh;
    const int p2 = std::min(H.phys, Rr.phys);
    const Batch Ha = align_batch(H, p2), Ra = align_batch(Rr, p2);
    Batch S;
    S.phys = p2;
    S.level = std::min(H.level, Rr.level);
    S.n = nh;
    S.buf = rt.alloc(size_t(nh) * words(p2));
    add_sub(c_, p2, Ha.ptr(), Ra.ptr(), reinterpret_cast<uint64_t*>(S.buf.get()), nh, false);
    m_.add += nh;
    R = S;
  }
  return make(R.buf, R.phys, R.level, R.off);
}

std::vector<double> RnsB::decrypt(const RCt& c, size_t n) {
  // q_0 alone cannot hold sigma_0 * value for |value| >= 2^(log q_0 - log sigma_0 - 1): decrypt through two limbs
  if (c->phys < 1)
    fail(HS_E_LEVEL_EXHAUSTED, "rns decrypt: result at the last RNS limb (chain must exceed the statistic's depth)");
  Runtime& rt = Runtime::get();
  DevBuf co = rt.alloc(c_.N), zd = rt.alloc(std::max<size_t>(n, 1));
  decrypt_crt_dev(c_, c->phys, c->ptr(), co.get());
  decode_dev(c_.spec.logN, co.get(), sigma_[c->phys], zd.get(), n, n, 1);
  std::vector<double> z(n);
  if (n) cuda_ok(cudaMemcpyAsync(z.data(), zd.get(), n * 8, cudaMemcpyDeviceToHost, rt.stream()), "decode read");
  rt.sync();
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
