// pipelines.cu — fused executors (see pipelines.h).
#include <chrono>
#include <cstdio>
#include "pipelines.h"

#include <cmath>
#include <cstdlib>
#include <type_traits>
#include <cstring>
#include <map>
#include <mutex>
#include <unordered_map>
#include <utility>
#include <string>
#include <vector>

#include "backends.h"
#include "kernels.h"

namespace hsg {
namespace pipe {
namespace {

using flow::InvCfg;
using flow::SignCfg;

QSpec fused_q(const Params& p) { return QSpec{p.quantize ? QMode::Grid : QMode::None, p.scale_bits}; }
int out_grid(const Params& p) { return p.quantize ? p.scale_bits : 0; }

// Grid-unit carriers (QGrid) form products A*B = ab 2^(2s): fused kernels only for scales whose
// square stays far inside the fp64 exponent range; larger scale_bits run the literal q() kernels.
constexpr int kMaxFusedScaleBits = 400;

bool ct_ok(const Params& p, const Ct& c) {
  return c && c->n == p.S && (!p.quantize || (c->grid == p.scale_bits && p.scale_bits <= kMaxFusedScaleBits));
}

// debug_checks (HS_DEBUG_FUSED, default 1): "checked fusion" -- the fused kernels evaluate the
// reference's value checks as device predicates (M_CHK, the Newton guard); when any fails, the
// call is replayed op by op (DevB), which raises the reference's error at the reference's op with
// the reference's meter.  The checks never steer the computation, so a clean run's outputs,
// levels and meter are exactly the op-by-op ones.  Graph capture cannot read the flags back: a
// debug call while capturing takes the op-by-op path as before.
bool debug_fused() {
  static const bool on = [] {
    const char* e = std::getenv("HS_DEBUG_FUSED");
    return !e || std::atoi(e) != 0;
  }();
  return on;
}
bool mode_ok(const Params& p) {
  Runtime& rt = Runtime::get();
  if (!rt.fused) return false;
  return !p.debug || (debug_fused() && !rt.capturing());
}

bool fusable(const hs_ctx* ctx, std::initializer_list<const Ct*> cts) {
  const Params& p = ctx->p;
  if (!mode_ok(p)) return false;
  if (p.S > (1u << 30)) return false;
  for (const Ct* c : cts)
    if (!ct_ok(p, *c)) return false;
  return true;
}

bool col_ok(const hs_ctx* ctx, const ColC& col) {
  const Params& p = ctx->p;
  if (!mode_ok(p)) return false;
  if (col.chunks.empty() || col.chunks.size() > static_cast<size_t>(k::kMaxChunks)) return false;
  if (p.S > (1u << 24)) return false;
  for (const Ct& c : col.chunks)
    if (!ct_ok(p, c)) return false;
  return true;
}

bool degree_ok(int d) { return d <= k::kMaxFusedDegree; }
bool const_tree_on() {  // HS_CONST_TREE=0: the shared-memory table walk for every series
  static const bool on = [] {
    const char* e = std::getenv("HS_CONST_TREE");
    return !e || std::atoi(e) != 0;
  }();
  return on;
}
bool cfg_ok(const InvCfg& c) {
  return c.baseline_mode ? true : degree_ok(c.cheb_degree);
}
bool sign_ok(const SignCfg& s) {
  if (s.mode == 0) return true;
  for (const auto& p : s.custom_polys)
    if (static_cast<int>(p.size()) - 1 > k::kMaxFusedDegree) return false;
  return true;
}

SymCt sym(const Ct& c) { return SymCt{c ? c->n : 0, c ? c->level : 0}; }
flow::Col<SymCt> sym(const ColC& c) {
  flow::Col<SymCt> s;
  s.n_valid = c.n_valid;
  for (const Ct& x : c.chunks) s.chunks.push_back(sym(x));
  return s;
}

// ---- ledger memo ----------------------------------------------------------------
// The ledger (levels, meter, auto-bootstrap decisions) is a pure function of the
// parameters, the input sizes/levels and the scalar arguments — never of slot
// values — so a successful symbolic run is memoised under a key of exactly
// those inputs: steady-state calls skip the host-side replay of ~1,200 ops.
// Runs that throw are never memoised (errors re-raise from a fresh replay).
class Key {
 public:
  explicit Key(const char* fn, const Params& p) : k_(fn) {
    add(p.S);
    add(p.max_level);
    add(p.scale_bits);
    add(static_cast<int>(p.quantize) | static_cast<int>(p.auto_bootstrap) << 1 | static_cast<int>(p.debug) << 2);
  }
  template <class T>
  Key& add(const T& v) {
    static_assert(std::is_trivially_copyable_v<T>);
    k_.append(reinterpret_cast<const char*>(&v), sizeof v);
    return *this;
  }
  Key& ct(const Ct& c) { return add(c ? c->n : size_t(0)).add(c ? c->level : 0); }
  Key& col(const ColC& c) {
    add(c.n_valid).add(c.chunks.size());
    for (const Ct& x : c.chunks) ct(x);
    return *this;
  }
  Key& cfg(const InvCfg& c) {
    return add(c.n).add(c.cheb_degree).add(c.newton_iters).add(c.baseline_mode).add(c.baseline_iters);
  }
  Key& sign(const SignCfg& c) {
    add(c.mode).add(c.folds).add(c.custom_polys.size());
    for (const auto& p : c.custom_polys) {
      add(p.size());
      k_.append(reinterpret_cast<const char*>(p.data()), p.size() * sizeof(double));
    }
    return *this;
  }
  const std::string& str() const { return k_; }

 private:
  std::string k_;
};

void put(std::vector<int>& v, const SymCt& c) { v.push_back(c.level); }
void put(std::vector<int>& v, const flow::Col<SymCt>& c) {
  for (const SymCt& x : c.chunks) v.push_back(x.level);
}
void put(std::vector<int>& v, const flow::Moments<SymCt>& m) {
  v.push_back(m.mu.level);
  v.push_back(m.var.level);
}
void get(const std::vector<int>& v, size_t S, SymCt* c) { *c = SymCt{S, v.at(0)}; }
void get(const std::vector<int>& v, size_t S, flow::Col<SymCt>* c) {
  c->chunks.clear();
  for (int l : v) c->chunks.push_back(SymCt{S, l});
}
void get(const std::vector<int>& v, size_t S, flow::Moments<SymCt>* m) {
  m->mu = SymCt{S, v.at(0)};
  m->var = SymCt{S, v.at(1)};
}

struct Memo {
  Meter delta;
  std::vector<int> levels;
};
std::mutex g_memo_mu;
std::unordered_map<std::string, Memo> g_memo;

// Run the reference ledger symbolically on a copy of the meter; commit the
// copy whether it returns or throws (the reference's meter state at its throw).
template <class F>
auto ledger(hs_ctx* ctx, const Key& key, F&& f) {
  using R = decltype(f(std::declval<SymB&>()));
  {
    std::lock_guard<std::mutex> g(g_memo_mu);
    auto it = g_memo.find(key.str());
    if (it != g_memo.end()) {
      R r{};
      get(it->second.levels, ctx->p.S, &r);
      Meter m = ctx->m;
      m.mul_ct += it->second.delta.mul_ct;
      m.mul_pt += it->second.delta.mul_pt;
      m.add += it->second.delta.add;
      m.rotate += it->second.delta.rotate;
      m.bootstrap += it->second.delta.bootstrap;
      return std::make_pair(r, m);
    }
  }
  Meter m = ctx->m;
  SymB sb(ctx->p, m);
  try {
    R r = f(sb);
    Memo e;
    e.delta = Meter{m.mul_ct - ctx->m.mul_ct, m.mul_pt - ctx->m.mul_pt, m.add - ctx->m.add,
                    m.rotate - ctx->m.rotate, m.bootstrap - ctx->m.bootstrap};
    put(e.levels, r);
    std::lock_guard<std::mutex> g(g_memo_mu);
    if (g_memo.size() > 4096) g_memo.clear();
    g_memo.emplace(key.str(), std::move(e));
    return std::make_pair(r, m);
  } catch (...) {
    ctx->m = m;
    throw;
  }
}

// ---- checked fusion (debug_checks) -------------------------------------------------
unsigned* debug_flag_word() { return reinterpret_cast<unsigned*>(Runtime::get().scratch(2, 1)); }

bool checks_failed() {
  Runtime& rt = Runtime::get();
  unsigned h = 0;
  cuda_ok(cudaMemcpyAsync(&h, debug_flag_word(), sizeof h, cudaMemcpyDeviceToHost, rt.stream()), "debug flags");
  cuda_ok(cudaStreamSynchronize(rt.stream()), "debug flags");
  return h != 0;
}

// Run the fused body; with debug_checks on, a failed device check (or a ledger error, whose
// place relative to the value checks only the op-by-op order decides) restores the meter and
// replays the call op by op, which raises exactly where the reference raises.
template <class Body, class Fallback>
auto checked(hs_ctx* ctx, Body&& body, Fallback&& fallback) -> decltype(body()) {
  if (!ctx->p.debug) return body();
  const Meter m0 = ctx->m;
  try {
    auto out = body();
    if (!checks_failed()) return out;
  } catch (const Error& e) {
    if (e.code == HS_E_CUDA) throw;
  }
  ctx->m = m0;
  return fallback();
}

// ---- per-slot program builder ---------------------------------------------------
class PB {
 public:
  explicit PB(const Params& p) : p_(p), q_(fused_q(p)) { prog_.S = static_cast<unsigned>(p.S); }

  int ld(const double* dev) {
    if (nin_ >= k::kMaxArr) fail(HS_E_ERROR, "fused program: too many inputs");
    prog_.in[nin_] = dev;
    return emit(k::M_LD, reg(), 0, 0, nin_++, 0, 0.0);
  }
  int ld(const Ct& c) { return ld(c->device()); }
  void st(int r, double* dev) {
    if (nout_ >= k::kMaxArr) fail(HS_E_ERROR, "fused program: too many outputs");
    prog_.out[nout_] = dev;
    emit(k::M_ST, -1, r, 0, nout_++, 0, 0.0);
  }
  int cnst(double v) {  // encrypt(v) broadcast: q(v) in policy units
    double u = v;
    if (p_.quantize) u = std::nearbyint(v * std::ldexp(1.0, p_.scale_bits));
    return emit(k::M_CONST, reg(), 0, 0, 0, 0, u);
  }
  int ldr(int k) { return emit(k::M_LDR, reg(), 0, 0, k, 0, 0.0); }  // per-slot statistic value
  // debug_checks: the reference's value check of register r on slots [0, n_valid) (no-op otherwise)
  void check(int r, k::ChkKind kind, size_t n_valid, double c, double c2 = 0.0) {
    if (p_.debug) emit(k::M_CHK, -1, r, 0, kind, lim(n_valid), c, 0, c2);
  }
  int add(int a, int b) { return emit(k::M_ADD, reg(), a, b, 0, 0, 0.0); }
  int sub(int a, int b) { return emit(k::M_SUB, reg(), a, b, 0, 0, 0.0); }
  int mul(int a, int b) { return emit(k::M_MUL, reg(), a, b, 0, 0, 0.0); }
  int mulc(int a, double c) { return emit(k::M_MULC, reg(), a, 0, 0, 0, c); }
  int addc(int a, double c) {
    return emit(k::M_ADDC, reg(), a, 0, 0, 0, p_.quantize ? c * std::ldexp(1.0, p_.scale_bits) : c);
  }

  // eval_encrypted (chebyshev.hpp:171-189); bootstraps are value-identities here.
  // The table offset (i0) and lane-split flag (b) are patched in launch().
  int cheb(int x, const Series& s) {
    check(x, k::CK_RANGE, p_.S, s.lo - 1e-9, s.hi + 1e-9);  // chebyshev.hpp:174-179 (every slot)
    if (!s.native()) {
      const double span = s.hi - s.lo;
      x = addc(mulc(x, 2.0 / span), -(s.lo + s.hi) / span);
    }
    if (s.degree() >= 63) big_cheb_ = true;
    chebs_.push_back(std::make_pair(prog_.n, s));
    return emit(k::M_CHEB, reg(), x, 0, 0, s.degree(), 0.0);
  }
  // newton_loop (primitives.hpp:105-132)
  int newton(int x, int y, int n, int iters, size_t n_valid = flow::kAllSlots) {
    if (iters <= 0) return y;
    return emit(k::M_NEWTON, reg(), x, y, n, iters, (n + 1.0) / n, p_.debug ? lim(n_valid) : 0);
  }
  void zapply(int mu, int inv, const std::vector<Ct>& in, const std::vector<DevBuf>& out) {
    prog_.nchunks = static_cast<int>(in.size());
    for (size_t c = 0; c < in.size(); ++c) {
      prog_.zin[c] = in[c]->device();
      prog_.zout[c] = out[c].get();
    }
    emit(k::M_ZAPPLY, -1, mu, inv, 0, 0, 0.0);
  }

  // ---- composite primitives -------------------------------------------------------
  int baseline(int t, double S, int iters, size_t nv = flow::kAllSlots) {  // primitives.hpp:173-184
    check(t, k::CK_OPEN, nv, 0.0, 1.0);
    int y = cnst(1.0);
    if (iters > 0) y = newton(mulc(t, 0.5), y, 2, iters, nv);
    return mulc(y, 1.0 / std::sqrt(S));
  }
  int invsqrt(int t, double S, const InvCfg& cfg, size_t nv = flow::kAllSlots) {  // primitives.hpp:186-208
    if (cfg.baseline_mode) return baseline(t, S, cfg.effective_baseline_iters(), nv);
    check(t, k::CK_OPEN, nv, 0.0, 2.0);
    const Series seed = fit_scaled(TargetKind::InvSqrtShifted, S, cfg.cheb_degree);
    int y = cheb(addc(t, -1.0), seed);
    if (cfg.newton_iters > 0) y = newton(mulc(t, S / 2.0), y, 2, cfg.newton_iters, nv);
    return y;
  }
  int inv(int t, double S, const InvCfg& cfg, size_t nv = flow::kAllSlots) {  // primitives.hpp:211-217
    const int y = invsqrt(t, S, cfg, nv);
    return mul(y, y);
  }
  int sqrt_(int t, double S, int degree, size_t nv = flow::kAllSlots) {  // primitives.hpp:222-238
    check(t, k::CK_RANGE, nv, -1e-9, 2.0 + 1e-9);
    const Series s = fit_scaled(TargetKind::SqrtShifted, S, degree);
    return cheb(addc(t, -1.0), s);
  }
  int sign(int x, const SignCfg& cfg) {  // primitives.hpp:279-300
    check(x, k::CK_RANGE, p_.S, -1.0 - 1e-9, 1.0 + 1e-9);
    const std::vector<Series> st = sign_stages(cfg.mode, cfg.custom_polys);
    int y = x;
    for (int f = 0; f < cfg.folds; ++f) y = cheb(y, st[static_cast<size_t>(f) % st.size()]);
    return y;
  }

  void launch() { finish(false, nullptr); }
  void launch_stat(const k::StatArgs& a) { finish(true, &a); }
  void launch_table(const k::PTableArgs& a) {
    table_ = &a;
    finish(false, nullptr);
  }
  void launch_zbatch(const k::ZBatchArgs& a) {
    zbatch_ = &a;
    finish(false, nullptr);
  }

 private:
  void finish(bool stat, const k::StatArgs* a) {
    Runtime& rt = Runtime::get();
    int lanes = !big_cheb_ ? 1 : ((zbatch_ || table_) ? rt.batch_lanes : rt.prog_lanes);
    if (big_cheb_ && (zbatch_ || table_) && lanes == 0) {
      const size_t ncols = zbatch_ ? zbatch_->ncols : table_->ncols;
      const size_t items = (p_.S + rt.sm_count() - 1) / rt.sm_count() * ncols;
      lanes = items >= 1024 ? 1 : (items >= 512 ? 2 : 4);  // one lane as soon as a block has one full round
    }
    int p = 0;
    while ((1 << p) < lanes) ++p;
    // one concatenated table per distinct series (deduplicated), cached on the
    // device by the series' identity so steady-state calls upload nothing
    std::string key = std::to_string(static_cast<int>(q_.mode)) + "/" + std::to_string(q_.bits) + "/" +
                      std::to_string(lanes);
    std::vector<std::string> ids;
    for (auto& [ins, s] : chebs_) {
      const int d = s.degree(), K = cheb_depth(d);
      const bool split = lanes > 1 && d >= 2 && d == (1 << K) - 1 && K - p >= 1;
      prog_.ins[ins].b = split ? 1 : 0;
      std::string id = s.key;
      if (id.empty()) {
        id = "u" + std::string(reinterpret_cast<const char*>(s.coeffs.data()), s.coeffs.size() * sizeof(double));
      }
      id += split ? "/s" : "/n";
      ids.push_back(id);
      key += "|" + id;
    }
    if (!chebs_.empty()) {
      const TableSet ts = tables(key, ids, lanes);
      for (size_t i = 0; i < chebs_.size(); ++i) {
        prog_.ins[chebs_[i].first].i0 = ts.off[i];
        prog_.ins[chebs_[i].first].c = ts.fast[i] ? 1.0 : 0.0;
      }
      prog_.tabs = ts.dev.get();
      prog_.ntab = ts.n;
    }
#ifdef HS_HOST_PROFILE
    static double tl = 0;
    static int nl = 0;
    auto l0 = std::chrono::steady_clock::now();
#endif
    if (p_.debug) {  // checked fusion: arm the flag word (read back by checks_failed())
      prog_.flags = debug_flag_word();
      cuda_ok(cudaMemsetAsync(prog_.flags, 0, sizeof(unsigned), rt.stream()), "debug flags");
    }
    if ((zbatch_ || table_) && lanes == 1 && const_tree_on()) {
      // a fast-path degree-511 series of a one-lane batch: its table also goes to the constant bank
      for (auto& [ins, s] : chebs_)
        if (s.degree() == 511 && prog_.ins[ins].c != 0.0 && prog_.ins[ins].b == 0) {
          k::upload_const_table(prog_.tabs + prog_.ins[ins].i0, rt.stream());
          prog_.ins[ins].i2 = 1;
          break;  // one table in the bank
        }
    }
    if (zbatch_) k::run_zbatch(q_, *zbatch_, prog_, lanes, rt.stream());
    else if (table_) k::run_ptable(q_, *table_, prog_, lanes, rt.stream());
    else if (stat) k::run_stat(q_, *a, prog_, lanes, rt.stream());
    else k::run_prog(q_, prog_, lanes, rt.stream());
#ifdef HS_HOST_PROFILE
    tl += std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - l0).count();
    if (++nl % 200 == 0) std::fprintf(stderr, "run_stat/run_prog host us/call %.2f (n=%d)\n", tl / nl, nl);
#endif
  }

  int reg() {
    if (nreg_ >= k::kRegs) fail(HS_E_ERROR, "fused program: register file exhausted");
    return nreg_++;
  }
  int emit(int op, int dst, int a, int b, int i0, int i1, double c, int i2 = 0, double c2 = 0.0) {
    if (prog_.n >= k::kMaxInst) fail(HS_E_ERROR, "fused program: too many instructions");
    prog_.ins[prog_.n++] = k::MInst{op, dst, a, b, i0, i1, c, i2, c2};
    return dst;
  }
  int lim(size_t n_valid) const { return static_cast<int>(std::min(n_valid, p_.S)); }

  struct TableSet {
    DevBuf dev;
    std::vector<int> off;
    std::vector<char> fast;  // magic-rounding range precondition holds (quant.cuh)
    int n = 0;
  };
  TableSet tables(const std::string& key, const std::vector<std::string>& ids, int lanes) {
    static std::mutex mu;
    static std::unordered_map<std::string, TableSet> cache;
    std::lock_guard<std::mutex> g(mu);
    auto it = cache.find(key);
    if (it != cache.end()) return it->second;
    TableSet ts;
    std::vector<double> all;
    std::map<std::string, int> seen;
    for (size_t i = 0; i < chebs_.size(); ++i) {
      // range precondition of the magic-rounding core (quant.cuh): every leaf, product and
      // partial sum below 2^51 grid units, i.e. 1.001 * sum|c| < 2^(51 - scale_bits) real units;
      // capped at 2^11 (the bound the |T_k| <= 1 + 2^-20 argument was made for, scale_bits = 40)
      double mag = 0.0;
      for (double c : cheb_table(chebs_[i].second.coeffs, QSpec{QMode::None, q_.bits})) mag += std::abs(c);
      const double lim = std::ldexp(1.0, std::min(11, 51 - q_.bits));
      ts.fast.push_back(std::isfinite(mag) && 1.001 * mag < lim ? 1 : 0);
      auto f = seen.find(ids[i]);
      if (f != seen.end()) {
        ts.off.push_back(f->second);
        continue;
      }
      std::vector<double> t = cheb_table(chebs_[i].second.coeffs, q_);
      if (prog_.ins[chebs_[i].first].b) t = interleave(t, lanes);
      const int off = static_cast<int>(all.size());
      all.insert(all.end(), t.begin(), t.end());
      seen.emplace(ids[i], off);
      ts.off.push_back(off);
    }
    ts.n = static_cast<int>(all.size());
    Runtime& rt = Runtime::get();
    // on the upload stream, waited for here: legal (and not recorded) while the compute stream
    // is being captured into a graph, so a series' first use may happen inside a capture
    cudaStream_t up = rt.upload_stream();
    ts.dev = rt.alloc_on(all.size(), up);
    cuda_ok(cudaMemcpyAsync(ts.dev.get(), all.data(), all.size() * sizeof(double), cudaMemcpyHostToDevice, up),
            "series table upload");
    cuda_ok(cudaStreamSynchronize(up), "series table upload");
    if (cache.size() > 512) cache.clear();  // in-flight users hold no reference: frees are stream-ordered
    return cache.emplace(key, std::move(ts)).first->second;
  }

  const Params& p_;
  QSpec q_;
  k::Prog prog_{};
  int nreg_ = 0, nin_ = 0, nout_ = 0;
  bool big_cheb_ = false;
  std::vector<std::pair<int, Series>> chebs_;
  const k::PTableArgs* table_ = nullptr;
  const k::ZBatchArgs* zbatch_ = nullptr;
};

// ---- statistics: one cooperative launch per call (stat.cu) ------------------------------
// StatArgs for phase A over one or two columns: mean_scaled(col, Bm) and/or
// variance_to_scale(col, Sv) terms (stats.hpp:97-126).
k::StatArgs stat_args(hs_ctx* ctx, const std::vector<const ColC*>& cols, int mode, double Bm, double Sv) {
  Runtime& rt = Runtime::get();
  const size_t S = ctx->p.S;
  k::StatArgs a{};
  a.ncols = static_cast<int>(cols.size());
  a.mom_mode = mode;
  a.nchunks = static_cast<int>(cols[0]->chunks.size());
  for (size_t i = 0; i < cols.size(); ++i) {
    const ColC& col = *cols[i];
    for (size_t c = 0; c < col.chunks.size(); ++c) (i == 0 ? a.x : a.y)[c] = col.chunks[c]->device();
    const double n = static_cast<double>(col.n_valid);
    a.cm[i] = 1.0 / (Bm * static_cast<double>(col.n_valid));  // stats.hpp:101
    a.ca[i] = 1.0 / std::sqrt(Sv * n);                         // stats.hpp:117
    a.cmp[i] = 1.0 / (n * std::sqrt(Sv));                      // stats.hpp:123
  }
  for (size_t c = 0; c < cols[0]->chunks.size(); ++c) a.valid[c] = flow::chunk_valid(S, cols[0]->n_valid, c);
  a.inv_n = 1.0 / static_cast<double>(cols[0]->n_valid);  // mean_of_chunks, stats.hpp:83
  a.partial = rt.scratch(0, k::stat_partial_doubles(), true);
  a.scratch = rt.scratch(1, 24 * S);
  return a;
}

Ct make_out(hs_ctx* ctx, const DevBuf& b, int level, std::shared_ptr<ReadyEv> ready = nullptr) {
  return ct_device(b, ctx->p.S, level, out_grid(ctx->p), std::move(ready));
}

}  // namespace

// =====================================================================================
// Every entry point: the op-by-op path `dev` when the call is not fusable, else the fused
// launch, wrapped by checked() (debug_checks: device predicates + op-by-op replay on failure).
Ct eval_encrypted(hs_ctx* ctx, const Series& s, const Ct& ct) {
  auto dev = [&] {
    DevB db(ctx->p, ctx->m);
    return flow::eval_encrypted(db, s, ct);
  };
  if (!fusable(ctx, {&ct}) || s.coeffs.empty() || !degree_ok(s.degree())) return dev();
  return checked(ctx, [&] {
    auto [r, m] = ledger(ctx, Key("eval", ctx->p).ct(ct).add(s.degree()).add(s.lo).add(s.hi),
                         [&](SymB& sb) { return flow::eval_encrypted(sb, s, sym(ct)); });
    PB pb(ctx->p);
    DevBuf out = Runtime::get().alloc(ctx->p.S);
    pb.st(pb.cheb(pb.ld(ct), s), out.get());
    pb.launch();
    ctx->m = m;
    return make_out(ctx, out, r.level);
  }, dev);
}

Ct newton_loop(hs_ctx* ctx, const Ct& x_op, const Ct& y, int n, int iters, size_t n_valid) {
  auto dev = [&] {
    DevB db(ctx->p, ctx->m);
    return flow::newton_loop(db, x_op, y, n, iters, n_valid);
  };
  if (!fusable(ctx, {&x_op, &y}) || n < 1 || n > k::kMaxFusedNewtonN) return dev();
  return checked(ctx, [&] {
    auto [r, m] = ledger(ctx, Key("newton_loop", ctx->p).ct(x_op).ct(y).add(n).add(iters).add(n_valid),
                         [&](SymB& sb) { return flow::newton_loop(sb, sym(x_op), sym(y), n, iters, n_valid); });
    PB pb(ctx->p);
    DevBuf out = Runtime::get().alloc(ctx->p.S);
    const int xr = pb.ld(x_op);
    pb.st(pb.newton(xr, pb.ld(y), n, iters, n_valid), out.get());
    pb.launch();
    ctx->m = m;
    return make_out(ctx, out, r.level);
  }, dev);
}

Ct newton_refine(hs_ctx* ctx, const Ct& x, const Ct& y0, int n, int iters, size_t n_valid) {
  auto dev = [&] {
    DevB db(ctx->p, ctx->m);
    return flow::newton_refine(db, x, y0, n, iters, n_valid);
  };
  if (!fusable(ctx, {&x, &y0}) || n < 1 || n > k::kMaxFusedNewtonN) return dev();
  return checked(ctx, [&] {
    auto [r, m] = ledger(ctx, Key("newton_refine", ctx->p).ct(x).ct(y0).add(n).add(iters).add(n_valid),
                         [&](SymB& sb) { return flow::newton_refine(sb, sym(x), sym(y0), n, iters, n_valid); });
    PB pb(ctx->p);
    DevBuf out = Runtime::get().alloc(ctx->p.S);
    int xr = pb.ld(x);
    const int yr = pb.ld(y0);
    if (n >= 2) xr = pb.mulc(xr, 1.0 / n);
    pb.st(pb.newton(xr, yr, n, iters, n_valid), out.get());
    pb.launch();
    ctx->m = m;
    return make_out(ctx, out, r.level);
  }, dev);
}

Ct crypto_invsqrt(hs_ctx* ctx, const Ct& ct, double S, const InvCfg& cfg, size_t n_valid) {
  auto dev = [&] {
    DevB db(ctx->p, ctx->m);
    return flow::crypto_invsqrt(db, ct, S, cfg, n_valid);
  };
  if (!fusable(ctx, {&ct}) || !cfg_ok(cfg)) return dev();
  return checked(ctx, [&] {
    auto [r, m] = ledger(ctx, Key("invsqrt", ctx->p).ct(ct).add(S).cfg(cfg).add(n_valid),
                         [&](SymB& sb) { return flow::crypto_invsqrt(sb, sym(ct), S, cfg, n_valid); });
    PB pb(ctx->p);
    DevBuf out = Runtime::get().alloc(ctx->p.S);
    pb.st(pb.invsqrt(pb.ld(ct), S, cfg, n_valid), out.get());
    pb.launch();
    ctx->m = m;
    return make_out(ctx, out, r.level);
  }, dev);
}

Ct baseline_invsqrt(hs_ctx* ctx, const Ct& ct, double S, int iters, size_t n_valid) {
  auto dev = [&] {
    DevB db(ctx->p, ctx->m);
    return flow::baseline_invsqrt(db, ct, S, iters, n_valid);
  };
  if (!fusable(ctx, {&ct})) return dev();
  return checked(ctx, [&] {
    auto [r, m] = ledger(ctx, Key("baseline", ctx->p).ct(ct).add(S).add(iters).add(n_valid),
                         [&](SymB& sb) { return flow::baseline_invsqrt(sb, sym(ct), S, iters, n_valid); });
    PB pb(ctx->p);
    DevBuf out = Runtime::get().alloc(ctx->p.S);
    pb.st(pb.baseline(pb.ld(ct), S, iters, n_valid), out.get());
    pb.launch();
    ctx->m = m;
    return make_out(ctx, out, r.level);
  }, dev);
}

Ct crypto_inv(hs_ctx* ctx, const Ct& ct, double S, const InvCfg& cfg, size_t n_valid) {
  auto dev = [&] {
    DevB db(ctx->p, ctx->m);
    return flow::crypto_inv(db, ct, S, cfg, n_valid);
  };
  if (!fusable(ctx, {&ct}) || !cfg_ok(cfg)) return dev();
  return checked(ctx, [&] {
    auto [r, m] = ledger(ctx, Key("inv", ctx->p).ct(ct).add(S).cfg(cfg).add(n_valid),
                         [&](SymB& sb) { return flow::crypto_inv(sb, sym(ct), S, cfg, n_valid); });
    PB pb(ctx->p);
    DevBuf out = Runtime::get().alloc(ctx->p.S);
    pb.st(pb.inv(pb.ld(ct), S, cfg, n_valid), out.get());
    pb.launch();
    ctx->m = m;
    return make_out(ctx, out, r.level);
  }, dev);
}

Ct crypto_sqrt(hs_ctx* ctx, const Ct& ct, double S, int degree, size_t n_valid) {
  auto dev = [&] {
    DevB db(ctx->p, ctx->m);
    return flow::crypto_sqrt(db, ct, S, degree, n_valid);
  };
  if (!fusable(ctx, {&ct}) || !degree_ok(degree)) return dev();
  return checked(ctx, [&] {
    auto [r, m] = ledger(ctx, Key("sqrt", ctx->p).ct(ct).add(S).add(degree).add(n_valid),
                         [&](SymB& sb) { return flow::crypto_sqrt(sb, sym(ct), S, degree, n_valid); });
    PB pb(ctx->p);
    DevBuf out = Runtime::get().alloc(ctx->p.S);
    pb.st(pb.sqrt_(pb.ld(ct), S, degree, n_valid), out.get());
    pb.launch();
    ctx->m = m;
    return make_out(ctx, out, r.level);
  }, dev);
}

Ct crypto_sign(hs_ctx* ctx, const Ct& ct, const SignCfg& cfg) {
  auto dev = [&] {
    DevB db(ctx->p, ctx->m);
    return flow::crypto_sign(db, ct, cfg);
  };
  if (!fusable(ctx, {&ct}) || !sign_ok(cfg) || cfg.folds > 24) return dev();
  return checked(ctx, [&] {
    auto [r, m] = ledger(ctx, Key("sign", ctx->p).ct(ct).sign(cfg),
                         [&](SymB& sb) { return flow::crypto_sign(sb, sym(ct), cfg); });
    PB pb(ctx->p);
    DevBuf out = Runtime::get().alloc(ctx->p.S);
    pb.st(pb.sign(pb.ld(ct), cfg), out.get());
    pb.launch();
    ctx->m = m;
    return make_out(ctx, out, r.level);
  }, dev);
}

// ---- statistics ---------------------------------------------------------------------------
// moments() debug checks (stats.hpp:144-146, 156-158, ...): slot 0 of the scaled variance
void check_var(PB& pb, int var, double B, bool scaled_check) {
  pb.check(var, k::CK_LT, 1, -1e-9);                        // moments: negative scaled variance
  if (scaled_check) pb.check(var, k::CK_SCALED_LT, 1, B, 1e-9);  // (var * B) * B < 1e-9
}

Ct mean_scaled(hs_ctx* ctx, const ColC& col, double B) {
  auto dev = [&] {
    DevB db(ctx->p, ctx->m);
    return flow::mean_scaled(db, col, B);
  };
  if (!col_ok(ctx, col)) return dev();
  return checked(ctx, [&] {
    auto [r, m] = ledger(ctx, Key("mean", ctx->p).col(col).add(B),
                         [&](SymB& sb) { return flow::mean_scaled(sb, sym(col), B); });
    DevBuf out = Runtime::get().alloc(ctx->p.S);
    PB pb(ctx->p);
    pb.st(pb.ldr(0), out.get());
    pb.launch_stat(stat_args(ctx, {&col}, k::MOM_MEAN, B, 1.0));
    ctx->m = m;
    return make_out(ctx, out, r.level);
  }, dev);
}

static Ct variance_impl(hs_ctx* ctx, const ColC& col, double S, const Key& key, bool scaled, double B) {
  auto [r, m] = ledger(ctx, key, [&](SymB& sb) {
    return scaled ? flow::variance_scaled(sb, sym(col), B) : flow::variance_to_scale(sb, sym(col), S);
  });
  DevBuf out = Runtime::get().alloc(ctx->p.S);
  PB pb(ctx->p);
  pb.st(pb.ldr(1), out.get());
  pb.launch_stat(stat_args(ctx, {&col}, k::MOM_VAR, 1.0, S));
  ctx->m = m;
  return make_out(ctx, out, r.level);
}

Ct variance_to_scale(hs_ctx* ctx, const ColC& col, double S) {
  auto dev = [&] {
    DevB db(ctx->p, ctx->m);
    return flow::variance_to_scale(db, col, S);
  };
  if (!col_ok(ctx, col)) return dev();
  return checked(ctx, [&] { return variance_impl(ctx, col, S, Key("var_to_scale", ctx->p).col(col).add(S), false, 0.0); },
                 dev);
}

Ct variance_scaled(hs_ctx* ctx, const ColC& col, double B) {
  auto dev = [&] {
    DevB db(ctx->p, ctx->m);
    return flow::variance_scaled(db, col, B);
  };
  if (!col_ok(ctx, col)) return dev();
  return checked(ctx, [&] { return variance_impl(ctx, col, B * B, Key("var_scaled", ctx->p).col(col).add(B), true, B); },
                 dev);
}

flow::Moments<Ct> moments(hs_ctx* ctx, const ColC& col, double B) {
  auto dev = [&] {
    DevB db(ctx->p, ctx->m);
    return flow::moments(db, col, B);
  };
  if (!col_ok(ctx, col)) return dev();
  return checked(ctx, [&] {
    auto [r, m] = ledger(ctx, Key("moments", ctx->p).col(col).add(B),
                         [&](SymB& sb) { return flow::moments(sb, sym(col), B); });
    Runtime& rt = Runtime::get();
    DevBuf mu = rt.alloc(ctx->p.S), var = rt.alloc(ctx->p.S);
    PB pb(ctx->p);
    pb.st(pb.ldr(0), mu.get());
    const int v = pb.ldr(1);
    check_var(pb, v, B, false);
    pb.st(v, var.get());
    pb.launch_stat(stat_args(ctx, {&col}, k::MOM_BOTH, 1.0, B * B));
    ctx->m = m;
    flow::Moments<Ct> out;
    out.mu = make_out(ctx, mu, r.mu.level);
    out.var = make_out(ctx, var, r.var.level);
    out.n_valid = col.n_valid;
    return out;
  }, dev);
}

ColC znorm(hs_ctx* ctx, const ColC& col, double B, const InvCfg& cfg) {
  auto dev = [&] {
    DevB db(ctx->p, ctx->m);
    return flow::znorm(db, col, B, cfg);
  };
  if (!col_ok(ctx, col) || !cfg_ok(cfg)) return dev();
  return checked(ctx, [&] {
    auto [r, m] = ledger(ctx, Key("znorm", ctx->p).col(col).add(B).cfg(cfg),
                         [&](SymB& sb) { return flow::znorm(sb, sym(col), B, cfg); });
    Runtime& rt = Runtime::get();
    std::vector<DevBuf> outs;
    for (size_t c = 0; c < col.chunks.size(); ++c) outs.push_back(rt.alloc(ctx->p.S));
    PB pb(ctx->p);
    const int var = pb.ldr(1);
    check_var(pb, var, B, true);
    const int inv = pb.invsqrt(var, B * B, cfg);  // crypto_invsqrt(var, B^2)
    pb.zapply(pb.ldr(0), inv, col.chunks, outs);  // mul_ct(sub_ct(chunk, mu), inv)
    pb.launch_stat(stat_args(ctx, {&col}, k::MOM_BOTH, 1.0, B * B));
    ctx->m = m;
    ColC z;
    z.n_valid = col.n_valid;
    const auto ready = rt.mark_ready();  // decode_column may fetch the result beside later compute work
    for (size_t c = 0; c < outs.size(); ++c)
      z.chunks.push_back(make_out(ctx, outs[c], r.chunks[c].level, ready));
    return z;
  }, dev);
}

static Ct std_moment(hs_ctx* ctx, const ColC& col, double B, const InvCfg& cfg, int power) {
  auto dev = [&] {
    DevB db(ctx->p, ctx->m);
    return flow::std_moment(db, col, B, cfg, power);
  };
  if (!col_ok(ctx, col) || !cfg_ok(cfg)) return dev();
  return checked(ctx, [&] {
    auto [r, m] = ledger(ctx, Key("std_moment", ctx->p).col(col).add(B).cfg(cfg).add(power),
                         [&](SymB& sb) { return flow::std_moment(sb, sym(col), B, cfg, power); });
    DevBuf out = Runtime::get().alloc(ctx->p.S);
    PB pb(ctx->p);
    const int var = pb.ldr(1);
    check_var(pb, var, B, true);
    const int inv = pb.invsqrt(var, B * B, cfg);
    const int inv2 = pb.mul(inv, inv);
    const int invp = power == 4 ? pb.mul(inv2, inv2) : pb.mul(inv2, inv);
    pb.st(pb.mul(pb.ldr(4), invp), out.get());  // mul_ct(numerator, inv^p)
    k::StatArgs a = stat_args(ctx, {&col}, k::MOM_BOTH, 1.0, B * B);
    a.power = power;
    pb.launch_stat(a);
    ctx->m = m;
    return make_out(ctx, out, r.level);
  }, dev);
}

Ct kurtosis(hs_ctx* ctx, const ColC& col, double B, const InvCfg& cfg) { return std_moment(ctx, col, B, cfg, 4); }
Ct skewness(hs_ctx* ctx, const ColC& col, double B, const InvCfg& cfg) { return std_moment(ctx, col, B, cfg, 3); }

Ct coeff_variation(hs_ctx* ctx, const ColC& col, double B, const SignCfg& sc, const InvCfg& cfg) {
  auto dev = [&] {
    DevB db(ctx->p, ctx->m);
    return flow::coeff_variation(db, col, B, sc, cfg);
  };
  if (!col_ok(ctx, col) || !cfg_ok(cfg) || !degree_ok(cfg.cheb_degree) || !sign_ok(sc) || sc.folds > 24) return dev();
  return checked(ctx, [&] {
    auto [r, m] = ledger(ctx, Key("cv", ctx->p).col(col).add(B).sign(sc).cfg(cfg),
                         [&](SymB& sb) { return flow::coeff_variation(sb, sym(col), B, sc, cfg); });
    DevBuf out = Runtime::get().alloc(ctx->p.S);
    PB pb(ctx->p);
    const int mu_b = pb.ldr(0);  // mean_scaled(col, B)
    pb.check(mu_b, k::CK_ABS_LT, 1, 0.01);  // stats.hpp:221-223
    const int sgn = pb.sign(mu_b, sc);
    const int inv_mu = pb.inv(pb.mul(mu_b, sgn), B, cfg);
    const int sigma = pb.sqrt_(pb.ldr(1), B * B, cfg.cheb_degree);  // variance_scaled(col, B)
    pb.st(pb.mul(pb.mul(sigma, inv_mu), sgn), out.get());
    pb.launch_stat(stat_args(ctx, {&col}, k::MOM_BOTH, B, B * B));
    ctx->m = m;
    return make_out(ctx, out, r.level);
  }, dev);
}

Ct pearson(hs_ctx* ctx, const ColC& x, const ColC& y, double B, const InvCfg& cfg) {
  auto dev = [&] {
    DevB db(ctx->p, ctx->m);
    return flow::pearson(db, x, y, B, cfg);
  };
  if (!col_ok(ctx, x) || !col_ok(ctx, y) || !cfg_ok(cfg) || x.chunks.size() != y.chunks.size()) return dev();
  return checked(ctx, [&] {
    auto [r, m] = ledger(ctx, Key("pearson", ctx->p).col(x).col(y).add(B).cfg(cfg),
                         [&](SymB& sb) { return flow::pearson(sb, sym(x), sym(y), B, cfg); });
    DevBuf out = Runtime::get().alloc(ctx->p.S);
    PB pb(ctx->p);
    const int vx = pb.ldr(1), vy = pb.ldr(3);
    check_var(pb, vx, B, true);
    check_var(pb, vy, B, true);
    const int ix = pb.invsqrt(vx, B * B, cfg);
    const int iy = pb.invsqrt(vy, B * B, cfg);
    pb.st(pb.mul(pb.mul(pb.ldr(4), ix), iy), out.get());  // mul_ct(mul_ct(cov, inv_x), inv_y)
    k::StatArgs a = stat_args(ctx, {&x, &y}, k::MOM_BOTH, 1.0, B * B);
    a.power = 2;
    pb.launch_stat(a);
    ctx->m = m;
    return make_out(ctx, out, r.level);
  }, dev);
}

// C4's table: pearson(cols[i], cols[j]) for every pair i < j, in that order, in one launch
// (kernels.h PTableArgs).  Reference semantics: the same values, levels and meter as the
// sequential calls (each pair's ledger replayed in order); one inverse square root per column
// instead of two per pair, since pearson(x, y) evaluates crypto_invsqrt of the same var_x ciphertext
// for every y (identical inputs, identical ops: identical slots).  Cases the kernel does not take
// (debug_checks, more than 8 or multi-chunk columns, unequal lengths, quantize off, a ledger error,
// or a sum that is not provably exact) run the pairs one by one.
std::vector<Ct> pearson_table(hs_ctx* ctx, const std::vector<ColC>& cols, double B, const InvCfg& cfg) {
  const size_t n = cols.size();
  auto sequential = [&] {
    std::vector<Ct> out;
    for (size_t i = 0; i < n; ++i)
      for (size_t j = i + 1; j < n; ++j) out.push_back(pearson(ctx, cols[i], cols[j], B, cfg));
    return out;
  };
  const Params& p = ctx->p;
  bool ok = n >= 2 && n <= static_cast<size_t>(k::kMaxTableCols) && !p.debug && p.quantize && cfg_ok(cfg) &&
            Runtime::get().fused;
  for (const ColC& c : cols) ok = ok && col_ok(ctx, c) && c.chunks.size() == 1 && c.n_valid == cols[0].n_valid;
  if (!ok) return sequential();
  const Meter m0 = ctx->m;
  std::vector<int> levels;
  try {
    for (size_t i = 0; i < n; ++i)
      for (size_t j = i + 1; j < n; ++j) {
        auto [r, m] = ledger(ctx, Key("pearson", ctx->p).col(cols[i]).col(cols[j]).add(B).cfg(cfg),
                             [&](SymB& sb) { return flow::pearson(sb, sym(cols[i]), sym(cols[j]), B, cfg); });
        ctx->m = m;
        levels.push_back(r.level);
      }
  } catch (const Error& e) {
    if (e.code == HS_E_CUDA) throw;
    ctx->m = m0;
    return sequential();
  }
  const Meter m_all = ctx->m;
  Runtime& rt = Runtime::get();
  const size_t S = p.S;
  k::PTableArgs a{};
  a.ncols = static_cast<int>(n);
  const double nv = static_cast<double>(cols[0].n_valid), Sv = B * B;
  a.valid = cols[0].n_valid;
  a.cm = 1.0 / (1.0 * nv);               // mean_scaled(col, 1), stats.hpp:101
  a.ca = 1.0 / std::sqrt(Sv * nv);       // variance_to_scale(col, B^2), stats.hpp:117
  a.cmp = 1.0 / (nv * std::sqrt(Sv));    // stats.hpp:123
  a.inv_n = 1.0 / nv;                    // mean_of_chunks, stats.hpp:83
  for (size_t c = 0; c < n; ++c) a.x[c] = cols[c].chunks[0]->device();
  std::vector<DevBuf> outs;
  const DevBuf block = rt.alloc(n * (n - 1) / 2 * S);  // one allocation; each output aliases its slice
  for (size_t i = 0; i < n; ++i)
    for (size_t j = i + 1; j < n; ++j) {
      a.pi[a.npairs] = static_cast<uint8_t>(i);
      a.pj[a.npairs] = static_cast<uint8_t>(j);
      outs.push_back(DevBuf(block, block.get() + a.npairs * S));
      a.out[a.npairs] = outs.back().get();
      ++a.npairs;
    }
  a.partial = rt.scratch(3, k::ptable_partial_doubles(), true);
  DevBuf inexact = rt.alloc(1);
  a.inexact = reinterpret_cast<unsigned*>(inexact.get());
  cuda_ok(cudaMemsetAsync(a.inexact, 0, sizeof(unsigned), rt.stream()), "pearson table flag");
  DevBuf inv = rt.alloc(n * S);
  PB pb(p);
  pb.st(pb.invsqrt(pb.ldr(1), B * B, cfg), inv.get());  // crypto_invsqrt(var, B^2), pearson's inv_x / inv_y
  pb.launch_table(a);
  unsigned flag = 0;
  cuda_ok(cudaMemcpyAsync(&flag, a.inexact, sizeof flag, cudaMemcpyDeviceToHost, rt.stream()), "pearson table flag");
  cuda_ok(cudaStreamSynchronize(rt.stream()), "pearson table flag");
  if (flag) {  // a sum beyond the exact-sum bound: the literal butterflies, pair by pair
    ctx->m = m0;
    return sequential();
  }
  ctx->m = m_all;
  std::vector<Ct> out;
  for (size_t k = 0; k < outs.size(); ++k) out.push_back(make_out(ctx, outs[k], levels[k]));
  return out;
}

// znorm of many independent columns in one launch (kernels.h ZBatchArgs): the same chunks,
// levels and meter as znorm(cols[0]), znorm(cols[1]), ... in order.  Columns must be single-chunk
// for the fused path (up to 64 per launch); debug_checks, quantize off, multi-chunk columns or a
// ledger error run the calls one by one.  No host synchronisation: capturable into a graph.
std::vector<ColC> znorm_batch(hs_ctx* ctx, const std::vector<ColC>& cols, double B, const InvCfg& cfg) {
  auto sequential = [&] {
    std::vector<ColC> out;
    for (const ColC& c : cols) out.push_back(znorm(ctx, c, B, cfg));
    return out;
  };
  const Params& p = ctx->p;
  bool ok = !cols.empty() && !p.debug && p.quantize && cfg_ok(cfg) && Runtime::get().fused;
  for (const ColC& c : cols) ok = ok && col_ok(ctx, c) && c.chunks.size() == 1;
  if (!ok) return sequential();
  std::vector<ColC> out;
  const Meter m0 = ctx->m;
  std::vector<int> levels;
  try {
    for (const ColC& c : cols) {
      auto [r, m] = ledger(ctx, Key("znorm", ctx->p).col(c).add(B).cfg(cfg),
                           [&](SymB& sb) { return flow::znorm(sb, sym(c), B, cfg); });
      ctx->m = m;
      levels.push_back(r.chunks.at(0).level);
    }
  } catch (const Error& e) {
    if (e.code == HS_E_CUDA) throw;
    ctx->m = m0;
    return sequential();
  }
  const Meter m_all = ctx->m;
  Runtime& rt = Runtime::get();
  const size_t S = p.S;
  const size_t nmax = std::min(cols.size(), size_t(k::kMaxZBatch));
  DevBuf inv = rt.alloc(nmax * S);
  for (size_t b0 = 0; b0 < cols.size(); b0 += k::kMaxZBatch) {
    const size_t nb = std::min(cols.size() - b0, size_t(k::kMaxZBatch));
    k::ZBatchArgs a{};
    a.ncols = static_cast<int>(nb);
    std::vector<DevBuf> zs;
    const DevBuf block = rt.alloc(nb * S);  // one allocation; each output aliases its slice
    for (size_t k = 0; k < nb; ++k) {
      const ColC& c = cols[b0 + k];
      const double nv = static_cast<double>(c.n_valid);
      a.x[k] = c.chunks[0]->device();
      zs.push_back(DevBuf(block, block.get() + k * S));
      a.z[k] = zs.back().get();
      a.cm[k] = 1.0 / (1.0 * nv);                 // mean_scaled(col, 1), stats.hpp:101
      a.ca[k] = 1.0 / std::sqrt(B * B * nv);      // variance_to_scale(col, B^2), stats.hpp:117
      a.cmp[k] = 1.0 / (nv * std::sqrt(B * B));   // stats.hpp:123
    }
    a.partial = rt.scratch(4, k::zbatch_partial_doubles(), true);
    a.scratch = rt.scratch(5, 2 * 3 * nmax * S);  // butterfly fallback (never read on the exact path)
    PB pb(p);
    pb.st(pb.invsqrt(pb.ldr(1), B * B, cfg), inv.get());  // crypto_invsqrt(var, B^2), stats.hpp:159
    pb.launch_zbatch(a);
    const auto ready = rt.mark_ready();
    for (size_t k = 0; k < nb; ++k) {
      ColC z;
      z.n_valid = cols[b0 + k].n_valid;
      z.chunks.push_back(make_out(ctx, zs[k], levels[b0 + k], ready));
      out.push_back(std::move(z));
    }
  }
  ctx->m = m_all;
  return out;
}

}  // namespace pipe
}  // namespace hsg
