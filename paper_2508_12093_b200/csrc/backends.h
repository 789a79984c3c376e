// backends.h — the two backends flow.h is instantiated over.
//
// Both implement the EvalContext op semantics of ckks.hpp:97-240 on the host
// side (shape checks, level min-rule, lazy auto-bootstrap of exhausted operands
// — each counted — level_exhausted when auto_bootstrap is off, meter updates).
// SymB carries only (size, level); DevB additionally launches one CUDA kernel
// per op on the library stream (ops.cu).
#pragma once

#include <algorithm>
#include <cmath>
#include <string>
#include <vector>

#include "core.h"
#include "kernels.h"

namespace hsg {

// Shared ledger logic (ckks.hpp:113-240), parameterised on the ciphertext type.
template <class Derived, class C>
class LedgerBase {
 public:
  LedgerBase(const Params& p, Meter& m) : p_(p), m_(m) {}
  const Params& params() const { return p_; }
  Meter& meter() { return m_; }

 protected:
  void check_shape(size_t n) const {  // ckks.hpp:242-245
    if (n != p_.S) fail(HS_E_LENGTH_MISMATCH, "ciphertext slot count does not match context");
  }
  const Params& p_;
  Meter& m_;
};

// ---------------------------------------------------------------------------
struct SymCt {
  size_t n = 0;
  int level = 0;
};

class SymB : public LedgerBase<SymB, SymCt> {
 public:
  using C = SymCt;
  using LedgerBase::LedgerBase;

  int level(const C& c) const { return c.level; }
  C encrypt_const(double) const { return C{p_.S, p_.max_level}; }
  C add_ct(const C& a, const C& b) {
    check_shape(a.n);
    check_shape(b.n);
    ++m_.add;
    return C{p_.S, std::min(a.level, b.level)};
  }
  C sub_ct(const C& a, const C& b) { return add_ct(a, b); }
  C add_pt(const C& a, double) {
    check_shape(a.n);
    ++m_.add;
    return C{p_.S, a.level};
  }
  C bootstrap(const C& a) {
    check_shape(a.n);
    ++m_.bootstrap;
    return C{p_.S, p_.max_level};
  }
  C mul_ct(C a, C b) {
    check_shape(a.n);
    check_shape(b.n);
    if (std::min(a.level, b.level) < 1) {
      if (!p_.auto_bootstrap) fail(HS_E_LEVEL_EXHAUSTED, "mul_ct: no multiplicative level left");
      if (a.level < 1) a = bootstrap(a);
      if (b.level < 1) b = bootstrap(b);
    }
    ++m_.mul_ct;
    return C{p_.S, std::min(a.level, b.level) - 1};
  }
  C mul_pt(C a, double) {
    check_shape(a.n);
    a = prepare_mul_pt(a);
    ++m_.mul_pt;
    return C{p_.S, a.level - 1};
  }
  C mul_pt_vec(C a, const std::vector<double>& v) {
    check_shape(a.n);
    if (v.size() != p_.S) fail(HS_E_LENGTH_MISMATCH, "mul_pt: plaintext vector length != slot count");
    a = prepare_mul_pt(a);
    ++m_.mul_pt;
    return C{p_.S, a.level - 1};
  }
  C rotate(const C& a, long) {
    check_shape(a.n);
    ++m_.rotate;
    return C{p_.S, a.level};
  }
  C sum_all_slots(const C& a, size_t) {  // debug padding check only on the DevB path
    check_shape(a.n);
    C acc = a;
    for (size_t step = 1; step < p_.S; step <<= 1) acc = add_ct(acc, rotate(acc, static_cast<long>(step)));
    return acc;
  }
  // value checks never run symbolically: with debug_checks the fused kernels evaluate them on
  // the device (pipelines.cu checked()); the ledger assumes they pass (1.0 passes every
  // first-slot predicate for B >= 2^-15; a failing one throws and the call replays op by op)
  double first_slot(const C&) { return 1.0; }
  void check_open_domain(const C&, size_t, double, double, const char*) {}
  void check_eval_domain(const C&, double, double) {}
  void check_divergence(const C&, size_t) {}
  void check_sqrt_domain(const C&, size_t) {}
  void check_sign_domain(const C&) {}

 private:
  C prepare_mul_pt(C a) {  // ckks.hpp:233-240
    if (a.level < 1) {
      if (!p_.auto_bootstrap) fail(HS_E_LEVEL_EXHAUSTED, "mul_pt: no multiplicative level left");
      a = bootstrap(a);
    }
    return a;
  }
};

// ---------------------------------------------------------------------------
// The unsettled part of an asynchronous encode_column: completion event of its upload-stream
// work, the finiteness flag that work writes, and the staging buffer it reads.
struct EncodePending {
  std::shared_ptr<ReadyEv> done;
  int* bad = nullptr;
  DevBuf stage;
  DevBuf block;  // the column's output allocation: kept until the upload has completed, whatever the
                 // caller does with the chunk handles meanwhile (its free is compute-stream ordered)
  void finish();  // after `done` has fired: returns the flag, frees the stage; throws non_finite_value
  ~EncodePending();
};

class DevB : public LedgerBase<DevB, Ct> {
 public:
  using C = Ct;
  DevB(const Params& p, Meter& m);

  int level(const C& c) const { return c ? c->level : 0; }
  C encrypt(const double* v, size_t n) const;  // ckks.hpp:97-104 (const: no meter)
  // encode_column's chunks (column.hpp:25-39) with the non-finite check on device
  // With `pend`, nothing is waited for: the chunks are marked `filling`, and the caller settles
  // the finiteness verdict later (EncodePending::finish).
  std::vector<C> encrypt_column(const double* v, size_t n, struct EncodePending* pend = nullptr) const;
  C encrypt_const(double c) const;
  C add_ct(const C& a, const C& b) { return addsub(a, b, k::B_ADD); }
  C sub_ct(const C& a, const C& b) { return addsub(a, b, k::B_SUB); }
  C add_pt(const C& a, double c);
  C bootstrap(const C& a);
  C mul_ct(C a, C b);
  C mul_pt(C a, double c);
  C mul_pt_vec(C a, const std::vector<double>& v);
  C rotate(const C& a, long k);
  C sum_all_slots(const C& a, size_t n_valid);

  // Batched ops (C5): element i has exactly the single op's semantics (ledger in
  // element order, per-element auto-bootstrap); one kernel per 64 ciphertexts,
  // outputs are views of one allocation.
  std::vector<C> binary_batch(const std::vector<C>& a, const std::vector<C>& b, k::BinOp op);
  std::vector<C> scalar_batch(const std::vector<C>& a, double c, k::ScalOp op);
  std::vector<C> rotate_batch(const std::vector<C>& a, long k);

  double first_slot(const C& c);
  void check_open_domain(const C& c, size_t n_valid, double lo, double hi, const char* who);
  void check_eval_domain(const C& c, double lo, double hi);
  void check_divergence(const C& c, size_t n_valid);
  void check_sqrt_domain(const C& c, size_t n_valid);
  void check_sign_domain(const C& c);

 private:
  C addsub(const C& a, const C& b, k::BinOp op);
  C prepare_mul_pt(C a);
  size_t sz(const C& c) const { return c ? c->n : 0; }
  QSpec qs_;
};

}  // namespace hsg
