// hestat/ckks.hpp — drop-in for the reference's emulator core
// (/root/reference/proj/include/hestat/ckks.hpp:19-257) backed by libhestat_gpu.
//
// Same types, names and signatures; slot vectors live in B200 HBM behind
// reference-counted hs_ct handles and every op is a CUDA kernel.  Levels, the
// CostMeter and auto-bootstrap decisions are kept exactly as the reference
// keeps them.  Build: -I<repo>/include, link -lhestat_gpu.
#pragma once

#include <cmath>
#include <cstdint>
#include <memory>
#include <mutex>
#include <span>
#include <utility>
#include <vector>

#include "hestat/errors.hpp"
#include "hestat_gpu.h"
#include "hestat_rns.h"

namespace hestat {

// Backend choice at context creation (an extension; the reference has only the emulator).
// EvalContext(params, seed) is the emulator-semantics GPU backend (Tier E) unless the process
// runs with HESTAT_BACKEND=rns; EvalContext(params, seed, RnsBackend{}) is always RNS-CKKS: the
// same operator surface over real RLWE ciphertexts (hestat_rns.h, "RNS-backed EvalContexts").
struct RnsBackend {
  int boot = HS_RNS_BOOT_REFRESH;  // or HS_RNS_BOOT_LOGICAL (deep chain, `depth`-deep)
  bool has_spec = false;           // false: parameters derived from the CkksParams
  hs_rns_spec spec{};
};

struct CkksParams {  // ckks.hpp:19-42
  std::size_t slot_count = 32768;
  int max_level = 11;
  int scale_bits = 40;
  bool quantize = true;
  bool auto_bootstrap = true;
  bool debug_checks = false;

  hs_params to_c() const {
    hs_params p{};
    p.slot_count = slot_count;
    p.max_level = max_level;
    p.scale_bits = scale_bits;
    p.quantize = quantize;
    p.auto_bootstrap = auto_bootstrap;
    p.debug_checks = debug_checks;
    return p;
  }
  void validate() const {
    const hs_params p = to_c();
    gpu::check(hs_params_validate(&p));
  }
  double quantum() const { return std::ldexp(1.0, -scale_bits); }
};

struct CostMeter {  // ckks.hpp:46-60
  std::uint64_t mul_ct = 0;
  std::uint64_t mul_pt = 0;
  std::uint64_t add = 0;
  std::uint64_t rotate = 0;
  std::uint64_t bootstrap = 0;

  void merge(const CostMeter& o) {
    mul_ct += o.mul_ct;
    mul_pt += o.mul_pt;
    add += o.add;
    rotate += o.rotate;
    bootstrap += o.bootstrap;
  }
};

// Immutable ciphertext handle (ckks.hpp:64-78).  Copies share the device buffer.
class Ciphertext {
 public:
  Ciphertext() = default;
  Ciphertext(std::vector<double> slots, int level) {
    hs_ct* h = nullptr;
    gpu::check(hs_ct_new(slots.data(), slots.size(), level, &h));
    h_ = std::shared_ptr<hs_ct>(h, hs_ct_release);
    cache_ = std::make_shared<Cache>();
    cache_->v = std::move(slots);
    cache_->ready = true;
  }

  const std::vector<double>& slots() const {
    if (!h_) return empty_slots();
    std::lock_guard<std::mutex> g(cache_->mu);
    if (!cache_->ready) {
      cache_->v.resize(hs_ct_size(h_.get()));
      gpu::check(hs_ct_read(h_.get(), cache_->v.data(), cache_->v.size()));
      cache_->ready = true;
    }
    return cache_->v;
  }
  int level() const { return h_ ? hs_ct_level(h_.get()) : 0; }
  std::size_t size() const { return h_ ? static_cast<std::size_t>(hs_ct_size(h_.get())) : 0; }

  // ---- backend plumbing (not part of the reference surface) ----
  hs_ct* raw() const {
    if (!h_) {  // default-constructed: an empty ciphertext at level 0
      hs_ct* h = nullptr;
      gpu::check(hs_ct_new(nullptr, 0, 0, &h));
      h_ = std::shared_ptr<hs_ct>(h, hs_ct_release);
      cache_ = std::make_shared<Cache>();
      cache_->ready = true;
    }
    return h_.get();
  }
  static Ciphertext adopt(hs_ct* h) {
    Ciphertext c;
    c.h_ = std::shared_ptr<hs_ct>(h, hs_ct_release);
    c.cache_ = std::make_shared<Cache>();
    return c;
  }

 private:
  struct Cache {
    std::mutex mu;
    std::vector<double> v;
    bool ready = false;
  };
  static const std::vector<double>& empty_slots() {
    static const std::vector<double> e;
    return e;
  }
  mutable std::shared_ptr<hs_ct> h_;
  mutable std::shared_ptr<Cache> cache_;
};

// ckks.hpp:83-257.  The meter is mirrored host-side so meter() can hand out a
// mutable reference exactly like the reference; it is pushed to / pulled from
// the library around every call.
class EvalContext {
 public:
  explicit EvalContext(CkksParams params = {}, std::uint64_t rng_seed = 0) : params_(params), seed_(rng_seed) {
    const hs_params p = params_.to_c();
    hs_ctx* h = nullptr;
    gpu::check(hs_ctx_create(&p, rng_seed, &h));
    h_ = std::shared_ptr<hs_ctx>(h, hs_ctx_destroy);
  }
  EvalContext(CkksParams params, std::uint64_t rng_seed, const RnsBackend& rns) : params_(params), seed_(rng_seed) {
    const hs_params p = params_.to_c();
    hs_ctx* h = nullptr;
    gpu::check(hs_ctx_create_rns(&p, rng_seed, rns.has_spec ? &rns.spec : nullptr, rns.boot, &h));
    h_ = std::shared_ptr<hs_ctx>(h, hs_ctx_destroy);
  }
  EvalContext(const EvalContext& o) : params_(o.params_), meter_(o.meter_), seed_(o.seed_) {
    hs_ctx* h = nullptr;
    gpu::check(hs_ctx_clone(o.h_.get(), &h));
    h_ = std::shared_ptr<hs_ctx>(h, hs_ctx_destroy);
  }
  EvalContext& operator=(const EvalContext& o) {
    if (this != &o) {
      EvalContext t(o);
      std::swap(h_, t.h_);
      params_ = o.params_;
      seed_ = o.seed_;
      meter_ = o.meter_;
    }
    return *this;
  }

  const CkksParams& params() const { return params_; }
  bool rns_backed() const { return hs_ctx_backend(h_.get()) == 1; }  // extension: which backend runs
  CostMeter& meter() { return meter_; }
  const CostMeter& meter() const { return meter_; }
  std::uint64_t rng_seed() const { return seed_; }

  Ciphertext encrypt(std::span<const double> values) const {  // :97-104
    hs_ct* o = nullptr;
    gpu::check(hs_encrypt(h_.get(), values.data(), values.size(), &o));
    return Ciphertext::adopt(o);
  }
  std::vector<double> decrypt(const Ciphertext& ct, std::size_t n) const {  // :107-111
    std::vector<double> out(n);
    gpu::check(hs_decrypt(h_.get(), ct.raw(), n, out.data()));
    return out;
  }
  Ciphertext add_ct(const Ciphertext& a, const Ciphertext& b) {
    return run([&](hs_ct** o) { return hs_add_ct(h_.get(), a.raw(), b.raw(), o); });
  }
  Ciphertext sub_ct(const Ciphertext& a, const Ciphertext& b) {
    return run([&](hs_ct** o) { return hs_sub_ct(h_.get(), a.raw(), b.raw(), o); });
  }
  Ciphertext add_pt(const Ciphertext& a, double c) {
    return run([&](hs_ct** o) { return hs_add_pt(h_.get(), a.raw(), c, o); });
  }
  Ciphertext mul_ct(Ciphertext a, Ciphertext b) {
    return run([&](hs_ct** o) { return hs_mul_ct(h_.get(), a.raw(), b.raw(), o); });
  }
  Ciphertext mul_pt(Ciphertext a, double c) {
    return run([&](hs_ct** o) { return hs_mul_pt(h_.get(), a.raw(), c, o); });
  }
  Ciphertext mul_pt(Ciphertext a, std::span<const double> p) {
    return run([&](hs_ct** o) { return hs_mul_pt_vec(h_.get(), a.raw(), p.data(), p.size(), o); });
  }
  Ciphertext rotate(const Ciphertext& a, long k) {
    return run([&](hs_ct** o) { return hs_rotate(h_.get(), a.raw(), k, o); });
  }
  Ciphertext bootstrap(const Ciphertext& a) {
    return run([&](hs_ct** o) { return hs_bootstrap(h_.get(), a.raw(), o); });
  }
  Ciphertext sum_all_slots(const Ciphertext& a, std::size_t n_valid) {
    return run([&](hs_ct** o) { return hs_sum_all_slots(h_.get(), a.raw(), n_valid, o); });
  }

  // ---- backend plumbing: run a metered library call ----
  template <class F>
  Ciphertext run(F&& f) {
    hs_ct* o = nullptr;
    call([&] { return f(&o); });
    return Ciphertext::adopt(o);
  }
  template <class F>
  void call(F&& f) {
    const hs_meter in{meter_.mul_ct, meter_.mul_pt, meter_.add, meter_.rotate, meter_.bootstrap};
    hs_ctx_set_meter(h_.get(), &in);
    const int rc = f();
    hs_meter m{};
    hs_ctx_meter(h_.get(), &m);
    meter_ = CostMeter{m.mul_ct, m.mul_pt, m.add, m.rotate, m.bootstrap};
    gpu::check(rc);
  }
  hs_ctx* raw() const { return h_.get(); }

 private:
  CkksParams params_;
  CostMeter meter_;
  std::uint64_t seed_ = 0;
  std::shared_ptr<hs_ctx> h_;
};

}  // namespace hestat
