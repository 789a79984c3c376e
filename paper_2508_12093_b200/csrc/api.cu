// api.cu — the extern "C" ABI of include/hestat_gpu.h.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <random>
#include <string>
#include <vector>

#include "backends.h"
#include "core.h"
#include "pipelines.h"
#include "rns.h"
#include "rns_codec.h"
#include "rns_eval.h"
#include "flow.h"
#include "series.h"
#include "hestat_rns.h"

using namespace hsg;

namespace {

thread_local std::string g_err;

// Every entry point runs under one process-wide (recursive) lock: the library's device work
// shares one stream and process-wide scratch (statistics partials, grid-barrier words), and a
// call sequence like stat_args -> launch must not interleave with another thread's call that
// regrows that scratch.  hs_graph_begin takes the lock once more and hs_graph_end releases it,
// so while one thread captures a graph, other threads' calls wait instead of being recorded
// into it.  The reference's concurrency model (independent EvalContexts on worker threads,
// ckks.hpp:80-82, hestat_cli.cpp:77-111) stays valid: calls are serialised, not refused.
std::recursive_mutex g_api_mu;
thread_local int g_capture_depth = 0;

thread_local int g_guard_depth = 0;  // guard() nesting on this thread

// Runtime::wait: the blocking waits of hs_encode_column / hs_decode_column give the API lock up
// while they sleep (their enqueues are complete, what remains touches only the caller's state),
// unless this thread holds it more than once (a nested call, or a graph capture in progress).
void wait_unlocked(cudaStream_t s) {
  const bool drop = g_guard_depth == 1 && g_capture_depth == 0;
  if (drop) g_api_mu.unlock();
  const cudaError_t e = cudaStreamSynchronize(s);
  if (drop) g_api_mu.lock();
  cuda_ok(e, "cudaStreamSynchronize");
}
const bool g_wait_hook_set = (Runtime::set_wait_hook(&wait_unlocked), true);

template <class F>
int guard(F&& f) {
  std::lock_guard<std::recursive_mutex> lk(g_api_mu);
  struct Depth {
    Depth() { ++g_guard_depth; }
    ~Depth() { --g_guard_depth; }
  } depth;
  try {
    f();
    return HS_OK;
  } catch (const Error& e) {
    g_err = e.what();
    return e.code;
  } catch (const std::out_of_range& e) {  // map::at in the reference's BSGS
    g_err = e.what();
    return HS_E_ERROR;
  } catch (const std::exception& e) {
    g_err = e.what();
    return HS_E_ERROR;
  }
}

void need(const void* p, const char* what) {
  if (!p) fail(HS_E_INVALID_ARG, std::string("null argument: ") + what);
}

const Ct& get(const hs_ct* h) {
  need(h, "ciphertext");
  if (!h->p && h->r) fail(HS_E_INVALID_ARG, "an RNS ciphertext passed to a Tier-E (emulator) context");
  return h->p;
}

hs_ct* wrap(Ct c) {
  auto* h = new hs_ct;
  h->p = std::move(c);
  return h;
}

// ---- RNS-backed contexts (hs_ctx::rns) ----
rns::RCt rget(hs_ctx* c, const hs_ct* h) {
  need(h, "ciphertext");
  if (h->r) return h->r;
  return c->rns->adopt(h->p);  // a host-constructed (or Tier-E) handle: encrypted on first use
}
std::vector<rns::RCt> rgets(hs_ctx* c, const hs_ct* const* a, uint64_t n) {
  if (n) need(a, "ciphertext array");
  std::vector<rns::RCt> v;
  for (uint64_t i = 0; i < n; ++i) v.push_back(rget(c, a[i]));
  return v;
}
hs_ct* rwrap(hs_ctx* c, rns::RCt r) {
  auto* h = new hs_ct;
  h->r = std::move(r);
  h->home = c->rns;
  return h;
}
Meter& meter_of(hs_ctx* c) { return c->rns ? c->rns->m : c->m; }

hs_ctx* ctxp(hs_ctx* c) {
  need(c, "context");
  return c;
}
const hs_ctx* ctxp(const hs_ctx* c) {
  need(c, "context");
  return c;
}

flow::InvCfg cfg_of(const hs_invroot_cfg* c) {
  flow::InvCfg r;
  if (c) {
    r.n = c->n;
    r.cheb_degree = c->cheb_degree;
    r.newton_iters = c->newton_iters;
    r.baseline_mode = c->baseline_mode != 0;
    r.baseline_iters = c->baseline_iters;
  }
  return r;
}

flow::SignCfg sign_of(const hs_sign_cfg* c) {
  flow::SignCfg r;
  if (c) {
    r.mode = c->mode;
    r.folds = c->folds;
    size_t off = 0;
    for (uint64_t i = 0; i < c->npolys; ++i) {
      r.custom_polys.emplace_back(c->polys + off, c->polys + off + c->poly_len[i]);
      off += c->poly_len[i];
    }
  }
  return r;
}

pipe::ColC col_of(const hs_column* c) {
  need(c, "column");
  pipe::ColC r;
  r.n_valid = c->n_valid;
  for (uint64_t i = 0; i < c->n_chunks; ++i) r.chunks.push_back(get(c->chunks[i]));
  return r;
}

size_t nv_of(uint64_t n) { return n == HS_ALL_SLOTS ? flow::kAllSlots : static_cast<size_t>(n); }

flow::Col<rns::RCt> rcol_of(hs_ctx* c, const hs_column* col) {
  need(col, "column");
  flow::Col<rns::RCt> r;
  r.n_valid = col->n_valid;
  for (uint64_t i = 0; i < col->n_chunks; ++i) r.chunks.push_back(rget(c, col->chunks[i]));
  return r;
}

rns::Spec spec_of(const hs_rns_spec& spec) {
  rns::Spec s;
  s.logN = spec.logN;
  s.L = spec.L;
  s.K = spec.K;
  s.dnum = spec.dnum;
  s.logq0 = spec.logq0;
  s.logq = spec.logq;
  s.logp = spec.logp;
  s.h = spec.h;
  s.seed = spec.seed;
  return s;
}

// An RNS-backed EvalContext: spec = null derives the parameter set from the CkksParams
// (rns::default_spec); boot = HS_RNS_BOOT_*.
hs_ctx* make_rns_ctx(const Params& q, uint64_t seed, const hs_rns_spec* spec, int boot, uint32_t depth) {
  if (boot != HS_RNS_BOOT_REFRESH && boot != HS_RNS_BOOT_LOGICAL)
    fail(HS_E_INVALID_ARG, "rns context: unknown bootstrap mode");
  const rns::Boot bm = boot == HS_RNS_BOOT_REFRESH ? rns::Boot::Refresh : rns::Boot::Logical;
  const rns::Spec s = spec ? spec_of(*spec) : rns::default_spec(q, bm, depth, seed);
  if ((size_t(1) << s.logN) != 2 * q.S) fail(HS_E_INVALID_ARG, "rns context: slot_count must be N/2");
  auto c = std::make_unique<hs_ctx>();
  c->p = q;
  c->seed = seed;
  c->rns = std::make_shared<rns::Home>(std::make_shared<rns::Ctx>(s), q, bm);
  return c.release();
}

// HESTAT_BACKEND=rns makes every EvalContext RNS-backed (reference programs run unmodified on
// RNS-CKKS ciphertexts); HESTAT_RNS_BOOT=logical + HESTAT_RNS_DEPTH=d selects the deep chain.
bool env_rns(int* boot, uint32_t* depth) {
  const char* e = std::getenv("HESTAT_BACKEND");
  if (!e || std::strcmp(e, "rns") != 0) return false;
  const char* b = std::getenv("HESTAT_RNS_BOOT");
  *boot = (b && std::strcmp(b, "logical") == 0) ? HS_RNS_BOOT_LOGICAL : HS_RNS_BOOT_REFRESH;
  const char* d = std::getenv("HESTAT_RNS_DEPTH");
  *depth = d ? static_cast<uint32_t>(std::atoi(d)) : 28;
  return true;
}

}  // namespace

extern "C" {

const char* hs_last_error(void) { return g_err.c_str(); }
const char* hs_version(void) { return "hestat-gpu 0.1 (sm_100a)"; }

int hs_init(int device) {
  return guard([&] {
    Runtime::init(device);
    Runtime::get();
  });
}

int hs_sync(void) {
  return guard([&] { Runtime::get().sync(); });
}

void* hs_stream(void) {
  void* s = nullptr;
  guard([&] { s = reinterpret_cast<void*>(Runtime::get().stream()); });
  return s;
}

int hs_set_fused(int enabled) {
  return guard([&] { Runtime::get().fused = enabled != 0; });
}

uint64_t hs_kernel_launches(void) {
  uint64_t n = 0;
  guard([&] { n = Runtime::get().launches(); });
  return n;
}

// ---- EvalContext ----------------------------------------------------------------------
int hs_params_validate(const hs_params* p) {
  return guard([&] {
    need(p, "params");
    Params::from(*p).validate();
  });
}

int hs_ctx_create(const hs_params* p, uint64_t seed, hs_ctx** out) {
  return guard([&] {
    need(p, "params");
    need(out, "out");
    Params q = Params::from(*p);
    q.validate();  // EvalContext ctor, ckks.hpp:85-88
    int boot = 0;
    uint32_t depth = 0;
    if (env_rns(&boot, &depth)) {
      *out = make_rns_ctx(q, seed, nullptr, boot, depth);
      return;
    }
    auto* c = new hs_ctx;
    c->p = q;
    c->seed = seed;
    *out = c;
  });
}

int hs_ctx_create_rns(const hs_params* p, uint64_t seed, const hs_rns_spec* spec, int boot, hs_ctx** out) {
  return guard([&] {
    need(p, "params");
    need(out, "out");
    Params q = Params::from(*p);
    q.validate();
    *out = make_rns_ctx(q, seed, spec, boot, 28);
  });
}

int hs_ctx_backend(const hs_ctx* c) { return c && c->rns ? 1 : 0; }

// EvalContext's copy (the reference copies params, meter and seed): an RNS-backed copy shares the
// RNS context (primes, keys) and gets its own meter and backend state.
int hs_ctx_clone(const hs_ctx* c, hs_ctx** out) {
  return guard([&] {
    need(out, "out");
    const hs_ctx* src = ctxp(c);
    auto d = std::make_unique<hs_ctx>();
    d->p = src->p;
    d->seed = src->seed;
    d->m = src->m;
    if (src->rns) {
      d->rns = std::make_shared<rns::Home>(src->rns->c, src->p, src->rns->b->boot_mode());
      d->rns->m = src->rns->m;
    }
    *out = d.release();
  });
}

int hs_ctx_rns_spec(const hs_ctx* c, hs_rns_spec* out, int* boot) {
  return guard([&] {
    need(out, "out");
    if (!ctxp(c)->rns) fail(HS_E_INVALID_ARG, "hs_ctx_rns_spec: not an RNS-backed context");
    const rns::Spec& s = c->rns->c->spec;
    *out = hs_rns_spec{s.logN, s.L, s.K, s.dnum, s.logq0, s.logq, s.logp, s.h, s.seed};
    if (boot) *boot = c->rns->b->boot_mode() == rns::Boot::Refresh ? HS_RNS_BOOT_REFRESH : HS_RNS_BOOT_LOGICAL;
  });
}

void hs_ctx_destroy(hs_ctx* c) {
  if (!c) return;
  std::lock_guard<std::recursive_mutex> lk(g_api_mu);
  delete c;
}

int hs_ctx_params(const hs_ctx* c, hs_params* out) {
  return guard([&] {
    need(out, "out");
    *out = ctxp(c)->p.to();
  });
}

int hs_ctx_meter(const hs_ctx* c, hs_meter* out) {
  return guard([&] {
    need(out, "out");
    const Meter& m = meter_of(const_cast<hs_ctx*>(ctxp(c)));
    *out = hs_meter{m.mul_ct, m.mul_pt, m.add, m.rotate, m.bootstrap};
  });
}

int hs_ctx_set_meter(hs_ctx* c, const hs_meter* m) {
  return guard([&] {
    need(m, "meter");
    meter_of(ctxp(c)) = Meter{m->mul_ct, m->mul_pt, m->add, m->rotate, m->bootstrap};
  });
}

uint64_t hs_ctx_rng_seed(const hs_ctx* c) { return c ? c->seed : 0; }

// ---- Ciphertext -------------------------------------------------------------------------
int hs_ct_new(const double* slots, uint64_t n, int32_t level, hs_ct** out) {
  return guard([&] {
    need(out, "out");
    if (n) need(slots, "slots");
    *out = wrap(ct_host(std::vector<double>(slots, slots + n), level));
  });
}

hs_ct* hs_ct_retain(hs_ct* ct) { return ct ? new hs_ct(*ct) : nullptr; }
void hs_ct_release(hs_ct* ct) {
  if (!ct) return;
  std::lock_guard<std::recursive_mutex> lk(g_api_mu);  // stream-ordered frees of shared buffers
  delete ct;
}
int32_t hs_ct_level(const hs_ct* ct) {
  if (ct && ct->r) return ct->r->level;
  return ct && ct->p ? ct->p->level : 0;
}
uint64_t hs_ct_size(const hs_ct* ct) {
  if (ct && ct->r) return ct->r->n;
  return ct && ct->p ? ct->p->n : 0;
}
int hs_ct_backend(const hs_ct* ct) { return ct && ct->r ? 1 : 0; }

int hs_ct_read(const hs_ct* ct, double* out, uint64_t n) {
  return guard([&] {
    need(ct, "ciphertext");
    if (ct->r) {  // Ciphertext::slots() of an RNS ciphertext: decrypted with its context's key
      if (n > ct->r->n) fail(HS_E_TOO_MANY_VALUES, "hs_ct_read: n exceeds ciphertext size");
      if (!n) return;
      need(out, "out");
      const std::vector<double> v = ct->home->b->decrypt(ct->r, static_cast<size_t>(n));
      std::copy(v.begin(), v.end(), out);
      return;
    }
    const Ct& c = get(ct);
    if (n > c->n) fail(HS_E_TOO_MANY_VALUES, "hs_ct_read: n exceeds ciphertext size");
    if (n) need(out, "out");
    c->read(out, static_cast<size_t>(n));
  });
}

// ---- EvalContext ops ------------------------------------------------------------------------
int hs_encrypt(const hs_ctx* c, const double* v, uint64_t n, hs_ct** out) {
  return guard([&] {
    need(out, "out");
    if (n) need(v, "values");
    hs_ctx* cc = const_cast<hs_ctx*>(ctxp(c));
    if (cc->rns) {  // RLWE encryption at the top of the chain (no meter update either)
      *out = rwrap(cc, cc->rns->b->encrypt(v, static_cast<size_t>(n)));
      return;
    }
    DevB db(cc->p, cc->m);  // encrypt is const: no meter update
    *out = wrap(db.encrypt(v, static_cast<size_t>(n)));
  });
}

int hs_decrypt(const hs_ctx* c, const hs_ct* ct, uint64_t n, double* out) {  // ckks.hpp:107-111
  return guard([&] {
    const hs_ctx* cc = ctxp(c);
    if (n > cc->p.S) fail(HS_E_TOO_MANY_VALUES, "decrypt: n exceeds slot count");
    need(ct, "ciphertext");
    if (ct->r) {
      if (n > ct->r->n) fail(HS_E_LENGTH_MISMATCH, "decrypt: ciphertext shorter than n");
      if (!n) return;
      need(out, "out");
      const std::vector<double> v = ct->home->b->decrypt(ct->r, static_cast<size_t>(n));
      std::copy(v.begin(), v.end(), out);
      return;
    }
    const Ct& x = get(ct);
    if (n > x->n) fail(HS_E_LENGTH_MISMATCH, "decrypt: ciphertext shorter than n");
    if (n) need(out, "out");
    x->read(out, static_cast<size_t>(n));
  });
}

// body: the Tier-E op on DevB `db`; rbody: the same op on the context's RNS backend `rb`
#define HS_OP2(body, rbody)               \
  return guard([&] {                      \
    need(out, "out");                     \
    hs_ctx* cc = ctxp(c);                 \
    if (cc->rns) {                        \
      rns::RnsB& rb = *cc->rns->b;        \
      (void)rb;                           \
      rbody;                              \
      return;                             \
    }                                     \
    DevB db(cc->p, cc->m);                \
    body;                                 \
  })
#define HS_OP(body) HS_OP2(body, fail(HS_E_INVALID_ARG, "not available on an RNS-backed context"))

int hs_add_ct(hs_ctx* c, const hs_ct* a, const hs_ct* b, hs_ct** out) {
  HS_OP2(*out = wrap(db.add_ct(get(a), get(b))), *out = rwrap(cc, rb.add_ct(rget(cc, a), rget(cc, b))));
}
int hs_sub_ct(hs_ctx* c, const hs_ct* a, const hs_ct* b, hs_ct** out) {
  HS_OP2(*out = wrap(db.sub_ct(get(a), get(b))), *out = rwrap(cc, rb.sub_ct(rget(cc, a), rget(cc, b))));
}
int hs_add_pt(hs_ctx* c, const hs_ct* a, double k, hs_ct** out) {
  HS_OP2(*out = wrap(db.add_pt(get(a), k)), *out = rwrap(cc, rb.add_pt(rget(cc, a), k)));
}
int hs_mul_ct(hs_ctx* c, const hs_ct* a, const hs_ct* b, hs_ct** out) {
  HS_OP2(*out = wrap(db.mul_ct(get(a), get(b))), *out = rwrap(cc, rb.mul_ct(rget(cc, a), rget(cc, b))));
}
int hs_mul_pt(hs_ctx* c, const hs_ct* a, double k, hs_ct** out) {
  HS_OP2(*out = wrap(db.mul_pt(get(a), k)), *out = rwrap(cc, rb.mul_pt(rget(cc, a), k)));
}
int hs_mul_pt_vec(hs_ctx* c, const hs_ct* a, const double* p, uint64_t n, hs_ct** out) {
  HS_OP2(
      {
        if (n) need(p, "plaintext");
        *out = wrap(db.mul_pt_vec(get(a), std::vector<double>(p, p + n)));
      },
      {
        if (n) need(p, "plaintext");
        *out = rwrap(cc, rb.mul_pt_vec(rget(cc, a), std::vector<double>(p, p + n)));
      });
}
int hs_rotate(hs_ctx* c, const hs_ct* a, int64_t k, hs_ct** out) {
  HS_OP2(*out = wrap(db.rotate(get(a), static_cast<long>(k))),
         *out = rwrap(cc, rb.rotate(rget(cc, a), static_cast<long>(k))));
}
int hs_bootstrap(hs_ctx* c, const hs_ct* a, hs_ct** out) {
  HS_OP2(*out = wrap(db.bootstrap(get(a))), *out = rwrap(cc, rb.bootstrap(rget(cc, a))));
}
int hs_sum_all_slots(hs_ctx* c, const hs_ct* a, uint64_t n_valid, hs_ct** out) {
  HS_OP2(*out = wrap(db.sum_all_slots(get(a), static_cast<size_t>(n_valid))),
         *out = rwrap(cc, rb.sum_all_slots(rget(cc, a), static_cast<size_t>(n_valid))));
}

// ---- batched ops (C5) ---------------------------------------------------------------------
namespace {
std::vector<Ct> gets(const hs_ct* const* a, uint64_t n) {
  if (n) need(a, "ciphertext array");
  std::vector<Ct> v;
  v.reserve(n);
  for (uint64_t i = 0; i < n; ++i) v.push_back(get(a[i]));
  return v;
}
void put_all(const std::vector<Ct>& v, hs_ct** out) {
  for (size_t i = 0; i < v.size(); ++i) out[i] = wrap(v[i]);
}
}  // namespace

// RNS-backed contexts: element by element, in element order (same ledger semantics)
#define HS_RBATCH2(expr)                                              \
  {                                                                   \
    const auto A = rgets(cc, a, n), Bv = rgets(cc, b, n);             \
    std::vector<rns::RCt> r;                                          \
    for (uint64_t i = 0; i < n; ++i) r.push_back(expr);               \
    for (uint64_t i = 0; i < n; ++i) out[i] = rwrap(cc, r[i]);        \
  }
#define HS_RBATCH1(expr)                                              \
  {                                                                   \
    const auto A = rgets(cc, a, n);                                   \
    std::vector<rns::RCt> r;                                          \
    for (uint64_t i = 0; i < n; ++i) r.push_back(expr);               \
    for (uint64_t i = 0; i < n; ++i) out[i] = rwrap(cc, r[i]);        \
  }
int hs_add_ct_batch(hs_ctx* c, const hs_ct* const* a, const hs_ct* const* b, uint64_t n, hs_ct** out) {
  HS_OP2(put_all(db.binary_batch(gets(a, n), gets(b, n), k::B_ADD), out), HS_RBATCH2(rb.add_ct(A[i], Bv[i])));
}
int hs_sub_ct_batch(hs_ctx* c, const hs_ct* const* a, const hs_ct* const* b, uint64_t n, hs_ct** out) {
  HS_OP2(put_all(db.binary_batch(gets(a, n), gets(b, n), k::B_SUB), out), HS_RBATCH2(rb.sub_ct(A[i], Bv[i])));
}
int hs_mul_ct_batch(hs_ctx* c, const hs_ct* const* a, const hs_ct* const* b, uint64_t n, hs_ct** out) {
  HS_OP2(put_all(db.binary_batch(gets(a, n), gets(b, n), k::B_MUL), out), HS_RBATCH2(rb.mul_ct(A[i], Bv[i])));
}
int hs_add_pt_batch(hs_ctx* c, const hs_ct* const* a, double k, uint64_t n, hs_ct** out) {
  HS_OP2(put_all(db.scalar_batch(gets(a, n), k, k::S_ADD), out), HS_RBATCH1(rb.add_pt(A[i], k)));
}
int hs_mul_pt_batch(hs_ctx* c, const hs_ct* const* a, double k, uint64_t n, hs_ct** out) {
  HS_OP2(put_all(db.scalar_batch(gets(a, n), k, k::S_MUL), out), HS_RBATCH1(rb.mul_pt(A[i], k)));
}
int hs_rotate_batch(hs_ctx* c, const hs_ct* const* a, int64_t k, uint64_t n, hs_ct** out) {
  HS_OP2(put_all(db.rotate_batch(gets(a, n), static_cast<long>(k)), out),
         HS_RBATCH1(rb.rotate(A[i], static_cast<long>(k))));
}

// Inside a guard: run `rexpr` on the context's RNS backend (rb, cc) when it has one.
#define HS_RNS_BRANCH(rexpr)              \
  if (ctxp(c)->rns) {                     \
    hs_ctx* cc = c;                       \
    rns::RnsB& rb = *cc->rns->b;          \
    rexpr;                                \
    return;                               \
  }

// ---- Chebyshev ------------------------------------------------------------------------------
double hs_scaled_target(int kind, double S, double t) {
  return scaled_target(kind == 1 ? TargetKind::SqrtShifted : TargetKind::InvSqrtShifted, S, t);
}

int32_t hs_cheb_eval_depth(int32_t degree) { return cheb_depth(degree); }

int hs_fit(hs_target_fn f, void* user, int32_t degree, double lo, double hi, double* coeffs) {
  return guard([&] {
    need(reinterpret_cast<void*>(f), "target");
    need(coeffs, "coeffs");
    Series s = fit([f, user](double x) { return f(x, user); }, degree, lo, hi);
    std::memcpy(coeffs, s.coeffs.data(), s.coeffs.size() * sizeof(double));
  });
}

int hs_fit_target(int kind, double S, int32_t degree, double lo, double hi, double* coeffs) {
  return guard([&] {
    need(coeffs, "coeffs");
    const TargetKind k = kind == 1 ? TargetKind::SqrtShifted : TargetKind::InvSqrtShifted;
    Series s = (lo == -1.0 && hi == 1.0) ? fit_scaled(k, S, degree)
                                         : fit([k, S](double t) { return scaled_target(k, S, t); }, degree, lo, hi);
    std::memcpy(coeffs, s.coeffs.data(), s.coeffs.size() * sizeof(double));
  });
}

double hs_eval_plain(const double* coeffs, uint64_t n, double lo, double hi, double x, int32_t* extrapolated) {
  Series s;
  s.coeffs.assign(coeffs, coeffs + n);
  s.lo = lo;
  s.hi = hi;
  bool ex = false;
  const double r = n ? eval_plain(s, x, &ex) : 0.0;
  if (extrapolated) *extrapolated = ex ? 1 : 0;
  return r;
}

int hs_eval_encrypted(hs_ctx* c, const double* coeffs, uint64_t n, double lo, double hi, const hs_ct* ct,
                      hs_ct** out) {
  return guard([&] {
    need(out, "out");
    if (n) need(coeffs, "coeffs");
    Series s;
    s.coeffs.assign(coeffs, coeffs + n);
    s.lo = lo;
    s.hi = hi;
    HS_RNS_BRANCH(*out = rwrap(cc, flow::eval_encrypted(rb, s, rget(cc, ct))));
    *out = wrap(pipe::eval_encrypted(ctxp(c), s, get(ct)));
  });
}

// ---- primitives -----------------------------------------------------------------------------
int hs_newton_loop(hs_ctx* c, const hs_ct* x_op, const hs_ct* y, int32_t n, int32_t iters, uint64_t n_valid,
                   hs_ct** out) {
  return guard([&] {
    need(out, "out");
    HS_RNS_BRANCH(*out = rwrap(cc, flow::newton_loop(rb, rget(cc, x_op), rget(cc, y), n, iters, nv_of(n_valid))));
    *out = wrap(pipe::newton_loop(ctxp(c), get(x_op), get(y), n, iters, nv_of(n_valid)));
  });
}

int hs_newton_refine(hs_ctx* c, const hs_ct* x, const hs_ct* y0, int32_t n, int32_t iters, uint64_t n_valid,
                     hs_ct** out) {
  return guard([&] {
    need(out, "out");
    HS_RNS_BRANCH(*out = rwrap(cc, flow::newton_refine(rb, rget(cc, x), rget(cc, y0), n, iters, nv_of(n_valid))));
    *out = wrap(pipe::newton_refine(ctxp(c), get(x), get(y0), n, iters, nv_of(n_valid)));
  });
}

int hs_crypto_invsqrt(hs_ctx* c, const hs_ct* ct, double S, const hs_invroot_cfg* cfg, uint64_t n_valid,
                      hs_ct** out) {
  return guard([&] {
    need(out, "out");
    HS_RNS_BRANCH(*out = rwrap(cc, flow::crypto_invsqrt(rb, rget(cc, ct), S, cfg_of(cfg), nv_of(n_valid))));
    *out = wrap(pipe::crypto_invsqrt(ctxp(c), get(ct), S, cfg_of(cfg), nv_of(n_valid)));
  });
}

int hs_baseline_invsqrt(hs_ctx* c, const hs_ct* ct, double S, int32_t iters, uint64_t n_valid, hs_ct** out) {
  return guard([&] {
    need(out, "out");
    HS_RNS_BRANCH(*out = rwrap(cc, flow::baseline_invsqrt(rb, rget(cc, ct), S, iters, nv_of(n_valid))));
    *out = wrap(pipe::baseline_invsqrt(ctxp(c), get(ct), S, iters, nv_of(n_valid)));
  });
}

int hs_crypto_inv(hs_ctx* c, const hs_ct* ct, double S, const hs_invroot_cfg* cfg, uint64_t n_valid,
                  hs_ct** out) {
  return guard([&] {
    need(out, "out");
    HS_RNS_BRANCH(*out = rwrap(cc, flow::crypto_inv(rb, rget(cc, ct), S, cfg_of(cfg), nv_of(n_valid))));
    *out = wrap(pipe::crypto_inv(ctxp(c), get(ct), S, cfg_of(cfg), nv_of(n_valid)));
  });
}

int hs_crypto_sqrt(hs_ctx* c, const hs_ct* ct, double S, int32_t degree, uint64_t n_valid, hs_ct** out) {
  return guard([&] {
    need(out, "out");
    HS_RNS_BRANCH(*out = rwrap(cc, flow::crypto_sqrt(rb, rget(cc, ct), S, degree, nv_of(n_valid))));
    *out = wrap(pipe::crypto_sqrt(ctxp(c), get(ct), S, degree, nv_of(n_valid)));
  });
}

int hs_crypto_sign(hs_ctx* c, const hs_ct* ct, const hs_sign_cfg* cfg, hs_ct** out) {
  return guard([&] {
    need(out, "out");
    HS_RNS_BRANCH(*out = rwrap(cc, flow::crypto_sign(rb, rget(cc, ct), sign_of(cfg))));
    *out = wrap(pipe::crypto_sign(ctxp(c), get(ct), sign_of(cfg)));
  });
}

// hs_decode_column's Tier-E body: enqueue the D2H copies of the column's chunks and either wait
// for them (releasing the API lock, Runtime::wait) or return the stream they were enqueued on.
// One copy per run of chunks that is contiguous on both sides (the outputs of hs_znorm_batch are
// slices of one allocation: a 64-chunk column is one 16 MiB copy).  Chunks that carry a completion
// event (fused statistics) are copied on the download stream after that event, beside whatever the
// compute stream runs next; anything else keeps the compute stream's order.
cudaStream_t decode_enqueue(size_t S, const hs_column* col, double* out, size_t remaining, bool wait) {
  Runtime& rt = Runtime::get();
  struct Run {
    const double* src;
    double* dst;
    size_t n;
    const DevBuf* owner;  // runs only grow inside one allocation (slices share its ownership)
  };
  std::vector<Run> runs;
  std::vector<cudaEvent_t> evs;
  bool all_ready = true, any_dev = false;
  size_t o = 0;
  for (uint64_t i = 0; i < col->n_chunks; ++i) {
    const size_t take = std::min(S, remaining);
    const Ct& x = get(col->chunks[i]);
    if (take > x->n) fail(HS_E_LENGTH_MISMATCH, "decode_column: chunk shorter than slot count");
    if (take) {
      bool on_host, filling;
      {
        std::lock_guard<std::mutex> g(x->mu);
        on_host = x->host_ok;
        filling = static_cast<bool>(x->filling);
      }
      if (on_host || !x->dev) {
        x->read_async(out + o, take, 0);  // host mirror: a memcpy
      } else {
        any_dev = true;
        if (filling) x->device();  // an asynchronous encode in flight: the compute stream waits for it
        if (x->ready && !filling) {
          if (evs.empty() || evs.back() != x->ready->e) evs.push_back(x->ready->e);
        } else {
          all_ready = false;
        }
        const double* src = x->dev.get();
        if (!runs.empty() && runs.back().src + runs.back().n == src && runs.back().dst + runs.back().n == out + o &&
            !runs.back().owner->owner_before(x->dev) && !x->dev.owner_before(*runs.back().owner))
          runs.back().n += take;
        else
          runs.push_back(Run{src, out + o, take, &x->dev});
      }
    }
    o += take;
    remaining -= take;
  }
  if (!any_dev) return nullptr;
  const bool side = all_ready && !rt.capturing();
  cudaStream_t st = side ? rt.download_stream() : rt.stream();
  if (side)
    for (cudaEvent_t e : evs) cuda_ok(cudaStreamWaitEvent(st, e, 0), "decode_column wait");
  for (const Run& r : runs)
    cuda_ok(cudaMemcpyAsync(r.dst, r.src, r.n * sizeof(double), cudaMemcpyDeviceToHost, st), "decode_column read");
  if (wait) rt.wait(st);
  return st;
}

// ---- columns ----------------------------------------------------------------------------------
int hs_encode_column(hs_ctx* c, const double* v, uint64_t n, hs_ct** chunks_out, uint64_t* n_chunks) {
  return guard([&] {  // column.hpp:25-39
    hs_ctx* cc = ctxp(c);
    need(n_chunks, "n_chunks");
    if (n) {
      need(v, "values");
      need(chunks_out, "chunks_out");
    }
    if (cc->rns) {  // column.hpp:25-39 over RLWE encryptions
      std::vector<rns::RCt> ch = cc->rns->b->encrypt_column(v, static_cast<size_t>(n));
      for (size_t i = 0; i < ch.size(); ++i) chunks_out[i] = rwrap(cc, ch[i]);
      *n_chunks = ch.size();
      return;
    }
    DevB db(cc->p, cc->m);
    std::vector<Ct> chunks = db.encrypt_column(v, static_cast<size_t>(n));
    for (size_t i = 0; i < chunks.size(); ++i) chunks_out[i] = wrap(chunks[i]);
    *n_chunks = chunks.size();
  });
}

int hs_decode_column(const hs_ctx* c, const hs_column* col, double* out) {
  return guard([&] {  // column.hpp:41-56
    const size_t S = ctxp(c)->p.S;
    need(col, "column");
    if (col->n_valid > col->n_chunks * S) fail(HS_E_LENGTH_MISMATCH, "decode_column: n_valid exceeds packed capacity");
    if (col->n_valid) need(out, "out");
    size_t remaining = col->n_valid, o = 0;
    if (ctxp(c)->rns) {  // decrypt the chunks (host FFTs on worker threads)
      std::vector<rns::RCt> cts;
      std::vector<size_t> ns;
      for (uint64_t i = 0; i < col->n_chunks && remaining; ++i) {
        const size_t take = std::min(S, remaining);
        cts.push_back(rget(const_cast<hs_ctx*>(c), col->chunks[i]));
        if (!cts.back() || take > cts.back()->n)
          fail(HS_E_LENGTH_MISMATCH, "decode_column: chunk shorter than slot count");
        ns.push_back(take);
        remaining -= take;
      }
      const auto vs = c->rns->b->decrypt_many(cts, ns);
      for (const auto& v : vs) {
        std::copy(v.begin(), v.end(), out + o);
        o += v.size();
      }
      return;
    }
    decode_enqueue(S, col, out, remaining, true);
  });
}

// ---- asynchronous column transfers (extension; the reference's encode_column / decode_column
// are the synchronous calls above) --------------------------------------------------------------
struct hs_pending {
  std::shared_ptr<ReadyEv> done;      // fires when the enqueued work has completed (null: nothing to wait for)
  std::unique_ptr<EncodePending> enc;  // encode: deferred finiteness verdict + staging buffer
  std::vector<Ct> reading;             // decode: the chunks being copied stay alive until the copy has completed
  bool settled = false;
  int rc = HS_OK;
  std::string err;
};

int hs_encode_column_async(hs_ctx* c, const double* v, uint64_t n, hs_ct** chunks_out, uint64_t* n_chunks,
                           hs_pending** pending) {
  return guard([&] {
    hs_ctx* cc = ctxp(c);
    need(n_chunks, "n_chunks");
    need(pending, "pending");
    if (n) {
      need(v, "values");
      need(chunks_out, "chunks_out");
    }
    auto p = std::make_unique<hs_pending>();
    if (cc->rns || n == 0) {  // RNS contexts (host-side encoding) and empty columns: the synchronous call
      const int rc = hs_encode_column(c, v, n, chunks_out, n_chunks);
      if (rc != HS_OK) throw Error(rc, g_err);
      p->settled = true;
      *pending = p.release();
      return;
    }
    p->enc = std::make_unique<EncodePending>();
    DevB db(cc->p, cc->m);
    std::vector<Ct> chunks = db.encrypt_column(v, static_cast<size_t>(n), p->enc.get());
    p->done = p->enc->done;
    for (size_t i = 0; i < chunks.size(); ++i) chunks_out[i] = wrap(chunks[i]);
    *n_chunks = chunks.size();
    *pending = p.release();
  });
}

int hs_decode_column_async(const hs_ctx* c, const hs_column* col, double* out, hs_pending** pending) {
  return guard([&] {
    need(pending, "pending");
    need(col, "column");
    auto p = std::make_unique<hs_pending>();
    if (ctxp(c)->rns) {
      const int rc = hs_decode_column(c, col, out);
      if (rc != HS_OK) throw Error(rc, g_err);
      p->settled = true;
      *pending = p.release();
      return;
    }
    const size_t S = ctxp(c)->p.S;
    if (col->n_valid > col->n_chunks * S) fail(HS_E_LENGTH_MISMATCH, "decode_column: n_valid exceeds packed capacity");
    if (col->n_valid) need(out, "out");
    for (uint64_t i = 0; i < col->n_chunks; ++i) p->reading.push_back(get(col->chunks[i]));
    cudaStream_t st = decode_enqueue(S, col, out, col->n_valid, false);
    if (st) {
      p->done = Runtime::get().mark_on(st);
    } else {
      p->settled = true;
      p->reading.clear();
    }
    *pending = p.release();
  });
}

// Blocks until the transfer has completed (the API lock is not held while waiting); returns the
// call's deferred status: HS_E_NON_FINITE_VALUE for an encode whose input held a NaN or infinity
// (its chunks must then be discarded), HS_OK otherwise.  Idempotent.
int hs_pending_wait(hs_pending* p) {
  if (!p) return HS_E_INVALID_ARG;
  if (!p->settled) {
    if (p->done) {
      const cudaError_t e = cudaEventSynchronize(p->done->e);
      if (e != cudaSuccess) {
        g_err = std::string("hs_pending_wait: ") + cudaGetErrorString(e);
        return HS_E_CUDA;
      }
    }
    p->rc = guard([&] {
      p->reading.clear();  // buffer frees are stream-ordered: under the API lock
      if (p->enc) p->enc->finish();
    });
    if (p->rc != HS_OK) p->err = g_err;
    p->settled = true;
  } else if (p->rc != HS_OK) {
    g_err = p->err;
  }
  return p->rc;
}

void hs_pending_release(hs_pending* p) {
  if (!p) return;
  if (!p->settled) hs_pending_wait(p);  // the staging buffer and the caller's buffers are in use until then
  std::lock_guard<std::recursive_mutex> lk(g_api_mu);
  delete p;
}

// ---- statistics ---------------------------------------------------------------------------------
int hs_mean_scaled(hs_ctx* c, const hs_column* col, double B, hs_ct** out) {
  return guard([&] {
    need(out, "out");
    HS_RNS_BRANCH(*out = rwrap(cc, flow::mean_scaled(rb, rcol_of(cc, col), B)));
    *out = wrap(pipe::mean_scaled(ctxp(c), col_of(col), B));
  });
}

int hs_variance_to_scale(hs_ctx* c, const hs_column* col, double S, hs_ct** out) {
  return guard([&] {
    need(out, "out");
    HS_RNS_BRANCH(*out = rwrap(cc, flow::variance_to_scale(rb, rcol_of(cc, col), S)));
    *out = wrap(pipe::variance_to_scale(ctxp(c), col_of(col), S));
  });
}

int hs_variance_scaled(hs_ctx* c, const hs_column* col, double B, hs_ct** out) {
  return guard([&] {
    need(out, "out");
    HS_RNS_BRANCH(*out = rwrap(cc, flow::variance_scaled(rb, rcol_of(cc, col), B)));
    *out = wrap(pipe::variance_scaled(ctxp(c), col_of(col), B));
  });
}

int hs_moments(hs_ctx* c, const hs_column* col, double B, hs_ct** mu, hs_ct** var) {
  return guard([&] {
    need(mu, "mu");
    need(var, "var");
    HS_RNS_BRANCH({
      auto m = flow::moments(rb, rcol_of(cc, col), B);
      *mu = rwrap(cc, m.mu);
      *var = rwrap(cc, m.var);
    });
    auto m = pipe::moments(ctxp(c), col_of(col), B);
    *mu = wrap(m.mu);
    *var = wrap(m.var);
  });
}

int hs_znorm(hs_ctx* c, const hs_column* col, double B, const hs_invroot_cfg* cfg, hs_ct** out_chunks) {
  return guard([&] {
    HS_RNS_BRANCH({
      auto z = flow::znorm(rb, rcol_of(cc, col), B, cfg_of(cfg));
      if (!z.chunks.empty()) need(out_chunks, "out_chunks");
      for (size_t i = 0; i < z.chunks.size(); ++i) out_chunks[i] = rwrap(cc, z.chunks[i]);
    });
    auto z = pipe::znorm(ctxp(c), col_of(col), B, cfg_of(cfg));
    if (!z.chunks.empty()) need(out_chunks, "out_chunks");
    for (size_t i = 0; i < z.chunks.size(); ++i) out_chunks[i] = wrap(z.chunks[i]);
  });
}

int hs_kurtosis(hs_ctx* c, const hs_column* col, double B, const hs_invroot_cfg* cfg, hs_ct** out) {
  return guard([&] {
    need(out, "out");
    HS_RNS_BRANCH(*out = rwrap(cc, flow::std_moment(rb, rcol_of(cc, col), B, cfg_of(cfg), 4)));
    *out = wrap(pipe::kurtosis(ctxp(c), col_of(col), B, cfg_of(cfg)));
  });
}

int hs_skewness(hs_ctx* c, const hs_column* col, double B, const hs_invroot_cfg* cfg, hs_ct** out) {
  return guard([&] {
    need(out, "out");
    HS_RNS_BRANCH(*out = rwrap(cc, flow::std_moment(rb, rcol_of(cc, col), B, cfg_of(cfg), 3)));
    *out = wrap(pipe::skewness(ctxp(c), col_of(col), B, cfg_of(cfg)));
  });
}

int hs_coeff_variation(hs_ctx* c, const hs_column* col, double B, const hs_sign_cfg* sc, const hs_invroot_cfg* cfg,
                       hs_ct** out) {
  return guard([&] {
    need(out, "out");
    HS_RNS_BRANCH(*out = rwrap(cc, flow::coeff_variation(rb, rcol_of(cc, col), B, sign_of(sc), cfg_of(cfg))));
    *out = wrap(pipe::coeff_variation(ctxp(c), col_of(col), B, sign_of(sc), cfg_of(cfg)));
  });
}

int hs_pearson(hs_ctx* c, const hs_column* x, const hs_column* y, double B, const hs_invroot_cfg* cfg,
               hs_ct** out) {
  return guard([&] {
    need(out, "out");
    HS_RNS_BRANCH(*out = rwrap(cc, flow::pearson(rb, rcol_of(cc, x), rcol_of(cc, y), B, cfg_of(cfg))));
    *out = wrap(pipe::pearson(ctxp(c), col_of(x), col_of(y), B, cfg_of(cfg)));
  });
}

int hs_znorm_batch(hs_ctx* c, const hs_column* const* cols, uint32_t ncols, double B, const hs_invroot_cfg* cfg,
                   hs_ct** out) {
  return guard([&] {
    if (ncols && !cols) fail(HS_E_INVALID_ARG, "hs_znorm_batch: null columns");
    std::vector<hs_ct*> res;
    try {
      if (ctxp(c)->rns) {
        hs_ctx* cc = c;
        rns::RnsB& rb = *cc->rns->b;
        for (uint32_t i = 0; i < ncols; ++i)
          for (auto& z : flow::znorm(rb, rcol_of(cc, cols[i]), B, cfg_of(cfg)).chunks) res.push_back(rwrap(cc, z));
      } else {
        std::vector<pipe::ColC> cs;
        for (uint32_t i = 0; i < ncols; ++i) cs.push_back(col_of(cols[i]));
        for (auto& z : pipe::znorm_batch(ctxp(c), cs, B, cfg_of(cfg)))
          for (Ct& ch : z.chunks) res.push_back(wrap(std::move(ch)));
      }
    } catch (...) {
      for (hs_ct* h : res) hs_ct_release(h);
      throw;
    }
    if (!res.empty()) need(out, "out_chunks");
    std::copy(res.begin(), res.end(), out);
  });
}

int hs_pearson_table(hs_ctx* c, const hs_column* const* cols, uint32_t ncols, double B, const hs_invroot_cfg* cfg,
                     hs_ct** out) {
  return guard([&] {
    need(out, "out");
    if (ncols && !cols) fail(HS_E_INVALID_ARG, "hs_pearson_table: null columns");
    const size_t np = size_t(ncols) * (ncols ? ncols - 1 : 0) / 2;
    std::vector<hs_ct*> res;
    auto release = [&] {
      for (hs_ct* h : res) hs_ct_release(h);
    };
    try {
      if (ctxp(c)->rns) {  // RNS-backed: the sequential calls (rns_eval batches inside each)
        hs_ctx* cc = c;
        rns::RnsB& rb = *cc->rns->b;
        for (uint32_t i = 0; i < ncols; ++i)
          for (uint32_t j = i + 1; j < ncols; ++j)
            res.push_back(rwrap(cc, flow::pearson(rb, rcol_of(cc, cols[i]), rcol_of(cc, cols[j]), B, cfg_of(cfg))));
      } else {
        std::vector<pipe::ColC> cs;
        for (uint32_t i = 0; i < ncols; ++i) cs.push_back(col_of(cols[i]));
        for (Ct& r : pipe::pearson_table(ctxp(c), cs, B, cfg_of(cfg))) res.push_back(wrap(std::move(r)));
      }
    } catch (...) {
      release();
      throw;
    }
    if (res.size() != np) fail(HS_E_ERROR, "hs_pearson_table: internal pair count");
    std::copy(res.begin(), res.end(), out);
  });
}

// ---- host-side data helpers (data.hpp:148-208, plain.hpp:18-92) -------------------------------
int hs_synthetic_uniform(uint64_t seed, uint64_t n, double lo, double hi, double* out) {
  return guard([&] {
    if (n < 1) fail(HS_E_ERROR, "synthetic_uniform: n must be >= 1");
    if (!(lo < hi)) fail(HS_E_ERROR, "synthetic_uniform: lo must be < hi");
    need(out, "out");
    std::mt19937_64 rng(seed);
    for (uint64_t i = 0; i < n; ++i) {
      const double u = static_cast<double>(rng() >> 11) * 0x1.0p-53;
      out[i] = lo + u * (hi - lo);
    }
  });
}

int hs_synthetic_grid(uint64_t n, double lo, double hi, double* out) {
  return guard([&] {
    if (n < 2) fail(HS_E_ERROR, "synthetic_grid: n must be >= 2");
    if (!(lo < hi)) fail(HS_E_ERROR, "synthetic_grid: lo must be < hi");
    need(out, "out");
    const double step = (hi - lo) / static_cast<double>(n - 1);
    for (uint64_t i = 0; i < n; ++i) out[i] = lo + step * static_cast<double>(i);
    out[n - 1] = hi;
  });
}

int hs_two_subrange_grid(uint64_t n, double lo, double hi, double* out) {
  if (!(lo < 1.0 && 1.0 < hi)) return hs_synthetic_grid(n, lo, hi, out);
  const int rc = hs_synthetic_grid(n / 2, lo, 1.0, out);
  if (rc) return rc;
  return hs_synthetic_grid(n - n / 2, 1.0, hi, out + n / 2);
}

int hs_mre(const double* a, const double* e, uint64_t n, double* out) {
  return guard([&] {
    need(out, "out");
    if (n == 0) fail(HS_E_ERROR, "mre: empty input");
    double acc = 0.0;
    for (uint64_t i = 0; i < n; ++i) {
      if (e[i] == 0.0) fail(HS_E_ZERO_REFERENCE, "mre: exact value is zero at index " + std::to_string(i));
      acc += std::abs(a[i] - e[i]) / std::abs(e[i]);
    }
    *out = acc / static_cast<double>(n);
  });
}

int hs_relative_error(double a, double e, double* out) {
  return guard([&] {
    need(out, "out");
    if (e == 0.0) fail(HS_E_ZERO_REFERENCE, "relative_error: zero reference");
    *out = std::abs(a - e) / std::abs(e);
  });
}

int hs_plain(int which, const double* x, uint64_t n, const double* y, double* out) {
  return guard([&] {
    need(out, "out");
    if (n == 0) fail(HS_E_EMPTY_COLUMN, "plain::mean: empty input");
    const size_t N = static_cast<size_t>(n);
    auto mean = [&](const double* v) {
      double acc = 0.0;
      for (size_t i = 0; i < N; ++i) acc += v[i];
      return acc / static_cast<double>(N);
    };
    auto var = [&](const double* v) {
      const double mu = mean(v);
      double acc = 0.0;
      for (size_t i = 0; i < N; ++i) acc += (v[i] - mu) * (v[i] - mu);
      return acc / static_cast<double>(N);
    };
    switch (which) {
      case 0: *out = mean(x); break;
      case 1: *out = var(x); break;
      case 2: {
        const double mu = mean(x);
        double m2 = 0.0, m3 = 0.0;
        for (size_t i = 0; i < N; ++i) {
          const double d = x[i] - mu;
          m2 += d * d;
          m3 += d * d * d;
        }
        m2 /= static_cast<double>(N);
        m3 /= static_cast<double>(N);
        *out = m3 / std::pow(m2, 1.5);
        break;
      }
      case 3: {
        const double mu = mean(x);
        double m2 = 0.0, m4 = 0.0;
        for (size_t i = 0; i < N; ++i) {
          const double d = x[i] - mu;
          m2 += d * d;
          m4 += d * d * d * d;
        }
        m2 /= static_cast<double>(N);
        m4 /= static_cast<double>(N);
        *out = m4 / (m2 * m2);
        break;
      }
      case 4: {
        const double mu = mean(x);
        if (mu == 0.0) fail(HS_E_NEAR_ZERO_MEAN, "plain::coeff_variation: zero mean");
        *out = std::sqrt(var(x)) * (mu > 0 ? 1.0 : -1.0) / std::abs(mu);
        break;
      }
      case 5: {
        need(y, "y");
        const double mx = mean(x), my = mean(y);
        double cv = 0.0, vx = 0.0, vy = 0.0;
        for (size_t i = 0; i < N; ++i) {
          cv += (x[i] - mx) * (y[i] - my);
          vx += (x[i] - mx) * (x[i] - mx);
          vy += (y[i] - my) * (y[i] - my);
        }
        if (vx == 0.0 || vy == 0.0) fail(HS_E_DEGENERATE_VARIANCE, "plain::pearson: constant column");
        *out = cv / std::sqrt(vx * vy);
        break;
      }
      case 6: {
        const double mu = mean(x), sd = std::sqrt(var(x));
        if (sd == 0.0) fail(HS_E_DEGENERATE_VARIANCE, "plain::znorm: zero variance");
        for (size_t i = 0; i < N; ++i) out[i] = (x[i] - mu) / sd;
        break;
      }
      case 7: *out = std::sqrt(var(x)); break;
      default: fail(HS_E_INVALID_ARG, "hs_plain: bad selector");
    }
  });
}

}  // extern "C"

// ---- CUDA graphs --------------------------------------------------------------------------------
struct hs_graph {
  cudaGraph_t g = nullptr;
  cudaGraphExec_t exec = nullptr;
};

extern "C" {

int hs_graph_begin(void) {
  const int rc = guard([&] {
    if (g_capture_depth) fail(HS_E_INVALID_ARG, "hs_graph_begin: this thread is already capturing");
    cuda_ok(cudaStreamBeginCapture(Runtime::get().stream(), cudaStreamCaptureModeRelaxed), "begin capture");
  });
  if (rc == HS_OK) {  // held until hs_graph_end on this thread
    g_api_mu.lock();
    ++g_capture_depth;
  }
  return rc;
}

int hs_graph_end(hs_graph** out) {
  struct Release {  // the capture's lock goes, whatever the outcome of ending it
    ~Release() {
      if (g_capture_depth) {
        --g_capture_depth;
        g_api_mu.unlock();
      }
    }
  } release;
  return guard([&] {
    need(out, "out");
    auto* h = new hs_graph;
    cudaError_t e = cudaStreamEndCapture(Runtime::get().stream(), &h->g);
    if (e != cudaSuccess) {
      delete h;
      cuda_ok(e, "end capture");
    }
    e = cudaGraphInstantiate(&h->exec, h->g, 0);
    if (e != cudaSuccess) {
      cudaGraphDestroy(h->g);
      delete h;
      cuda_ok(e, "graph instantiate");
    }
    *out = h;
  });
}

int hs_graph_launch(hs_graph* g) {
  return guard([&] {
    need(g, "graph");
    cuda_ok(cudaGraphLaunch(g->exec, Runtime::get().stream()), "graph launch");
  });
}

void hs_graph_destroy(hs_graph* g) {
  if (!g) return;
  if (g->exec) cudaGraphExecDestroy(g->exec);
  if (g->g) cudaGraphDestroy(g->g);
  delete g;
}

}  // extern "C"

// ---------------------------------------------------------------- Tier R (hestat_rns.h)
struct hs_rns {
  std::shared_ptr<rns::Ctx> c;
};
struct hs_rns_eval {  // EvalContext (params + meter) bound to an RNS context (kept alive by it)
  std::shared_ptr<rns::Ctx> r;
  Params p;
  Meter m;
};

namespace {
rns::Ctx& rctx(hs_rns* h) {
  need(h, "rns context");
  return *h->c;
}
}  // namespace

extern "C" {

int hs_rns_create(const hs_rns_spec* spec, hs_rns** out) {
  return guard([&] {
    need(spec, "spec");
    need(out, "out");
    auto h = std::make_unique<hs_rns>();
    h->c = std::make_shared<rns::Ctx>(spec_of(*spec));
    *out = h.release();
  });
}

int hs_rns_destroy(hs_rns* ctx) {
  return guard([&] {
    if (!ctx) return;
    Runtime::get().sync();
    delete ctx;  // the RNS context itself goes with its last user (EvalContexts, ciphertexts)
  });
}

int hs_rns_primes(const hs_rns* ctx, uint64_t* out, uint32_t cap) {
  return guard([&] {
    need(ctx, "rns context");
    need(out, "out");
    const auto& p = ctx->c->primes;
    if (cap < p.size()) fail(HS_E_INVALID_ARG, "hs_rns_primes: buffer too small");
    std::copy(p.begin(), p.end(), out);
  });
}

int hs_rns_alloc(uint64_t words, uint64_t** dev) {
  return guard([&] {
    need(dev, "out");
    Runtime& rt = Runtime::get();
    void* p = nullptr;
    cuda_ok(cudaMallocAsync(&p, std::max<uint64_t>(words, 1) * 8, rt.stream()), "cudaMallocAsync");
    *dev = static_cast<uint64_t*>(p);
  });
}

int hs_rns_free(uint64_t* dev) {
  return guard([&] {
    if (dev) cuda_ok(cudaFreeAsync(dev, Runtime::get().stream()), "cudaFreeAsync");
  });
}

int hs_rns_upload(uint64_t* dev, const uint64_t* host, uint64_t words) {
  return guard([&] {
    need(dev, "dev");
    need(host, "host");
    Runtime& rt = Runtime::get();
    cuda_ok(cudaMemcpyAsync(dev, host, words * 8, cudaMemcpyHostToDevice, rt.stream()), "upload");
    rt.sync();
  });
}

int hs_rns_download(uint64_t* host, const uint64_t* dev, uint64_t words) {
  return guard([&] {
    need(dev, "dev");
    need(host, "host");
    Runtime& rt = Runtime::get();
    cuda_ok(cudaMemcpyAsync(host, dev, words * 8, cudaMemcpyDeviceToHost, rt.stream()), "download");
    rt.sync();
  });
}

int hs_rns_prepare_relin(hs_rns* ctx) {
  return guard([&] {
    rns::Ctx& c = rctx(ctx);
    c.relin_key();
    for (uint32_t l = 0; l <= c.spec.L; ++l) rns::prepare_level(c, l);
  });
}

int hs_rns_prepare_rotation(hs_rns* ctx, int64_t k) {
  return guard([&] {
    rns::Ctx& c = rctx(ctx);
    c.galois_key(rns::Ctx::galois_elt(k, c.spec.logN));
    for (uint32_t l = 0; l <= c.spec.L; ++l) rns::prepare_level(c, l);
  });
}

int hs_rns_secret(hs_rns* ctx, uint64_t* dev_out) {
  return guard([&] {
    rns::Ctx& c = rctx(ctx);
    need(dev_out, "out");
    Runtime& rt = Runtime::get();
    cuda_ok(cudaMemcpyAsync(dev_out, c.d_sk.get(), size_t(c.np) * c.N * 8, cudaMemcpyDeviceToDevice, rt.stream()),
            "secret");
  });
}

int hs_rns_random_ct(hs_rns* ctx, uint32_t level, uint64_t tag, uint64_t* dev_out) {
  return guard([&] {
    rns::Ctx& c = rctx(ctx);
    need(dev_out, "out");
    if (level > c.spec.L) fail(HS_E_INVALID_ARG, "hs_rns_random_ct: level > L");
    rns::random_ct(c, level, tag, dev_out);
  });
}

int hs_rns_encode(uint32_t logN, const double* z, uint64_t n, double scale, int64_t* coeffs) {
  return guard([&] {
    need(coeffs, "coeffs");
    if (logN < 2 || logN > 17) fail(HS_E_INVALID_ARG, "hs_rns_encode: logN out of range");
    if (n && !z) fail(HS_E_INVALID_ARG, "null values");
    if (n > (1u << logN) / 2) fail(HS_E_TOO_MANY_VALUES, "hs_rns_encode: more values than slots");
    if (!(scale > 0.0) || !std::isfinite(scale)) fail(HS_E_INVALID_ARG, "hs_rns_encode: bad scale");
    for (uint64_t i = 0; i < n; ++i)
      if (!std::isfinite(z[i])) fail(HS_E_NON_FINITE_VALUE, "hs_rns_encode: non-finite value");
    rns::encode(logN, z, n, scale, coeffs);
  });
}

int hs_rns_decode(uint32_t logN, const int64_t* coeffs, double scale, double* z, uint64_t n) {
  return guard([&] {
    need(coeffs, "coeffs");
    if (logN < 2 || logN > 17) fail(HS_E_INVALID_ARG, "hs_rns_decode: logN out of range");
    if (n > (1u << logN) / 2) fail(HS_E_TOO_MANY_VALUES, "hs_rns_decode: more values than slots");
    if (n && !z) fail(HS_E_INVALID_ARG, "null output");
    if (!(scale > 0.0) || !std::isfinite(scale)) fail(HS_E_INVALID_ARG, "hs_rns_decode: bad scale");
    rns::decode(logN, coeffs, scale, z, n);
  });
}

int hs_rns_encode_gpu(uint32_t logN, const double* z, uint64_t n, double scale, double* coeffs) {
  return guard([&] {
    need(coeffs, "coeffs");
    if (logN < 2 || logN > 17) fail(HS_E_INVALID_ARG, "hs_rns_encode_gpu: logN out of range");
    if (n && !z) fail(HS_E_INVALID_ARG, "null values");
    if (n > (1u << logN) / 2) fail(HS_E_TOO_MANY_VALUES, "hs_rns_encode_gpu: more values than slots");
    if (!(scale > 0.0) || !std::isfinite(scale)) fail(HS_E_INVALID_ARG, "hs_rns_encode_gpu: bad scale");
    Runtime& rt = Runtime::get();
    const size_t N = size_t(1) << logN;
    DevBuf zd = rt.alloc(std::max<uint64_t>(n, 1)), cd = rt.alloc(N);
    if (n) cuda_ok(cudaMemcpyAsync(zd.get(), z, n * 8, cudaMemcpyHostToDevice, rt.stream()), "encode upload");
    rns::encode_dev(logN, zd.get(), n, scale, cd.get(), 1);
    cuda_ok(cudaMemcpyAsync(coeffs, cd.get(), N * 8, cudaMemcpyDeviceToHost, rt.stream()), "encode read");
    rt.sync();
  });
}

int hs_rns_decode_gpu(uint32_t logN, const double* coeffs, double scale, double* z, uint64_t n) {
  return guard([&] {
    need(coeffs, "coeffs");
    if (logN < 2 || logN > 17) fail(HS_E_INVALID_ARG, "hs_rns_decode_gpu: logN out of range");
    if (n > (1u << logN) / 2) fail(HS_E_TOO_MANY_VALUES, "hs_rns_decode_gpu: more values than slots");
    if (n && !z) fail(HS_E_INVALID_ARG, "null output");
    if (!(scale > 0.0) || !std::isfinite(scale)) fail(HS_E_INVALID_ARG, "hs_rns_decode_gpu: bad scale");
    Runtime& rt = Runtime::get();
    const size_t N = size_t(1) << logN;
    DevBuf cd = rt.alloc(N), zd = rt.alloc(std::max<uint64_t>(n, 1));
    cuda_ok(cudaMemcpyAsync(cd.get(), coeffs, N * 8, cudaMemcpyHostToDevice, rt.stream()), "decode upload");
    rns::decode_dev(logN, cd.get(), scale, zd.get(), n, n, 1);
    if (n) cuda_ok(cudaMemcpyAsync(z, zd.get(), n * 8, cudaMemcpyDeviceToHost, rt.stream()), "decode read");
    rt.sync();
  });
}

int hs_rns_encrypt_coeffs(hs_rns* ctx, uint32_t level, const int64_t* coeffs, uint64_t tag, uint64_t* dev_out) {
  return guard([&] {
    need(coeffs, "coeffs");
    need(dev_out, "out");
    rns::encrypt_coeffs(rctx(ctx), level, coeffs, tag, dev_out);
  });
}

int hs_rns_encrypt(hs_rns* ctx, uint32_t level, const double* z, uint64_t n, double scale, uint64_t tag,
                   uint64_t* dev_out) {
  std::vector<int64_t> co;
  int rc = guard([&] { co.resize(rctx(ctx).N); });
  if (rc) return rc;
  rc = hs_rns_encode(ctx->c->spec.logN, z, n, scale, co.data());
  if (rc) return rc;
  return hs_rns_encrypt_coeffs(ctx, level, co.data(), tag, dev_out);
}

int hs_rns_decrypt_coeffs(hs_rns* ctx, uint32_t level, const uint64_t* dev_ct, int64_t* coeffs) {
  return guard([&] {
    need(dev_ct, "ciphertext");
    need(coeffs, "coeffs");
    rns::decrypt_coeffs(rctx(ctx), level, dev_ct, coeffs);
  });
}

int hs_rns_decrypt(hs_rns* ctx, uint32_t level, const uint64_t* dev_ct, double scale, double* z, uint64_t n) {
  std::vector<int64_t> co;
  int rc = guard([&] { co.resize(rctx(ctx).N); });
  if (rc) return rc;
  rc = hs_rns_decrypt_coeffs(ctx, level, dev_ct, co.data());
  if (rc) return rc;
  return hs_rns_decode(ctx->c->spec.logN, co.data(), scale, z, n);
}

int hs_rns_ntt(hs_rns* ctx, uint64_t* dev, uint32_t first_prime, uint32_t nlimbs, uint32_t batch, int inverse) {
  return guard([&] {
    rns::Ctx& c = rctx(ctx);
    need(dev, "dev");
    if (first_prime + nlimbs > c.np) fail(HS_E_INVALID_ARG, "hs_rns_ntt: prime range out of the basis");
    std::vector<uint32_t> pm(nlimbs);
    for (uint32_t i = 0; i < nlimbs; ++i) pm[i] = first_prime + i;
    rns::ntt(c, dev, pm, batch, size_t(nlimbs) * c.N, inverse != 0);
  });
}

int hs_rns_add(hs_rns* ctx, uint32_t level, const uint64_t* a, const uint64_t* b, uint64_t* out, uint32_t batch) {
  return guard([&] {
    need(a, "a");
    need(b, "b");
    need(out, "out");
    rns::add_sub(rctx(ctx), level, a, b, out, batch, false);
  });
}

int hs_rns_sub(hs_rns* ctx, uint32_t level, const uint64_t* a, const uint64_t* b, uint64_t* out, uint32_t batch) {
  return guard([&] {
    need(a, "a");
    need(b, "b");
    need(out, "out");
    rns::add_sub(rctx(ctx), level, a, b, out, batch, true);
  });
}

int hs_rns_add_const(hs_rns* ctx, uint32_t level, const uint64_t* a, int64_t c, uint64_t* out, uint32_t batch) {
  return guard([&] {
    need(a, "a");
    need(out, "out");
    rns::const_op(rctx(ctx), level, a, c, out, batch, false);
  });
}

int hs_rns_mul_const(hs_rns* ctx, uint32_t level, const uint64_t* a, int64_t c, uint64_t* out, uint32_t batch) {
  return guard([&] {
    need(a, "a");
    need(out, "out");
    rns::const_op(rctx(ctx), level, a, c, out, batch, true);
  });
}

int hs_rns_mul_relin(hs_rns* ctx, uint32_t level, const uint64_t* a, const uint64_t* b, uint64_t* out,
                     uint32_t batch) {
  return guard([&] {
    need(a, "a");
    need(b, "b");
    need(out, "out");
    rns::mul_relin(rctx(ctx), level, a, b, out, batch);
  });
}

int hs_rns_mul_relin_rescale(hs_rns* ctx, uint32_t level, const uint64_t* a, const uint64_t* b, uint64_t* out,
                             uint32_t batch) {
  return guard([&] {
    need(a, "a");
    need(b, "b");
    need(out, "out");
    rns::mul_relin_rescale(rctx(ctx), level, a, b, out, batch);
  });
}

int hs_rns_rescale(hs_rns* ctx, uint32_t level, const uint64_t* in, uint64_t* out, uint32_t batch) {
  return guard([&] {
    need(in, "in");
    need(out, "out");
    rns::rescale(rctx(ctx), level, in, out, batch);
  });
}

int hs_rns_rescale_mul_const(hs_rns* ctx, uint32_t level, const uint64_t* in, int64_t c, uint64_t* out,
                             uint32_t batch) {
  return guard([&] {
    need(in, "in");
    need(out, "out");
    rns::rescale_mul_big(rctx(ctx), level, in, static_cast<double>(c), out, batch);
  });
}

int hs_rns_rotate(hs_rns* ctx, uint32_t level, int64_t k, const uint64_t* in, uint64_t* out, uint32_t batch) {
  return guard([&] {
    need(in, "in");
    need(out, "out");
    rns::rotate(rctx(ctx), level, k, in, out, batch);
  });
}

// ---- Tier R statistics: the reference's EvalContext over RNS ciphertexts (rns_eval.h)
int hs_rns_eval_create(hs_rns* r, const hs_params* p, hs_rns_eval** out) {
  return guard([&] {
    need(p, "params");
    need(out, "out");
    rns::Ctx& c = rctx(r);
    Params pp = Params::from(*p);
    pp.validate();
    if (pp.S != c.N / 2) fail(HS_E_INVALID_ARG, "hs_rns_eval_create: slot_count must be N/2");
    auto e = std::make_unique<hs_rns_eval>();
    e->r = r->c;
    e->p = pp;
    *out = e.release();
  });
}

int hs_rns_eval_destroy(hs_rns_eval* e) {
  return guard([&] { delete e; });
}

int hs_rns_eval_meter(const hs_rns_eval* e, hs_meter* out) {
  return guard([&] {
    need(e, "eval");
    need(out, "out");
    *out = hs_meter{e->m.mul_ct, e->m.mul_pt, e->m.add, e->m.rotate, e->m.bootstrap};
  });
}

int hs_rns_eval_set_meter(hs_rns_eval* e, const hs_meter* m) {
  return guard([&] {
    need(e, "eval");
    need(m, "meter");
    e->m = Meter{m->mul_ct, m->mul_pt, m->add, m->rotate, m->bootstrap};
  });
}

int hs_rns_eval_stat(hs_rns_eval* e, int which, const double* x, uint64_t n, const double* y, uint64_t ny, double B,
                     const hs_invroot_cfg* cfg, double* out, uint64_t out_n, int32_t* out_levels) {
  return guard([&] {
    need(e, "eval");
    need(out, "out");
    if (n && !x) fail(HS_E_INVALID_ARG, "null column");
    rns::RnsB b(*e->r, e->p, e->m);
    const flow::InvCfg ic = cfg_of(cfg);
    auto column = [&](const double* v, uint64_t len) {
      if (len && !v) fail(HS_E_INVALID_ARG, "null column");
      flow::Col<rns::RCt> col;
      col.chunks = b.encrypt_column(v, len);
      col.n_valid = len;
      return col;
    };
    std::vector<rns::RCt> res;
    switch (which) {
      case HS_RNS_INVSQRT: {  // t in one ciphertext, S = B
        if (n > e->p.S) fail(HS_E_TOO_MANY_VALUES, "invsqrt: more values than slots");
        res.push_back(flow::crypto_invsqrt(b, b.encrypt(x, n), B, ic, n));
        break;
      }
      case HS_RNS_MEAN: res.push_back(flow::mean_scaled(b, column(x, n), B)); break;
      case HS_RNS_VARIANCE: res.push_back(flow::variance_scaled(b, column(x, n), B)); break;
      case HS_RNS_MOMENTS: {
        auto m = flow::moments(b, column(x, n), B);
        res.push_back(m.mu);
        res.push_back(m.var);
        break;
      }
      case HS_RNS_ZNORM: {
        auto z = flow::znorm(b, column(x, n), B, ic);
        res = z.chunks;
        break;
      }
      case HS_RNS_KURTOSIS: res.push_back(flow::std_moment(b, column(x, n), B, ic, 4)); break;
      case HS_RNS_SKEWNESS: res.push_back(flow::std_moment(b, column(x, n), B, ic, 3)); break;
      case HS_RNS_PEARSON: {
        auto cx = column(x, n);
        auto cy = column(y, ny);
        res.push_back(flow::pearson(b, cx, cy, B, ic));
        break;
      }
      default:
        fail(HS_E_INVALID_ARG, "hs_rns_eval_stat: unknown statistic");
    }
    // znorm: the n values across chunks; others: the first out_n slots of each result
    size_t w = 0;
    if (which == HS_RNS_ZNORM) {
      std::vector<rns::RCt> cts;
      std::vector<size_t> ns;
      for (size_t i = 0, left = out_n; i < res.size() && left > 0; ++i) {
        const size_t take = std::min<size_t>(e->p.S, left);
        cts.push_back(res[i]);
        ns.push_back(take);
        left -= take;
      }
      const auto vs = b.decrypt_many(cts, ns);
      for (const auto& v : vs) {
        std::copy(v.begin(), v.end(), out + w);
        w += v.size();
      }
    } else {
      for (const auto& r : res) {
        const std::vector<double> v = b.decrypt(r, out_n);
        std::copy(v.begin(), v.end(), out + w);
        w += out_n;
      }
    }
    if (out_levels)
      for (size_t i = 0; i < res.size(); ++i) out_levels[i] = res[i]->level;
  });
}

}  // extern "C"
