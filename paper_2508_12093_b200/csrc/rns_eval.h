// rns_eval.h — the reference's EvalContext semantics over real RNS-CKKS ciphertexts.
//
// RnsB is a third backend for flow.h (next to SymB and DevB): the same control
// flow (levels, CostMeter, auto-bootstrap decisions, errors — ckks.hpp:113-240)
// drives Tier-R kernels instead of slot kernels, so every statistic of the
// reference runs on RNS ciphertexts with the reference's DAG.
//
//   logical level  the reference's level (ledger; bootstrap resets it);
//   physical level the RNS chain position (limbs q_0..q_p).  Every mul_ct /
//                  mul_pt consumes one physical level (rescale); bootstrap is a
//                  logical reset only ("deep chain"), so the chain
//                  must be at least the DAG's no-bootstrap depth.
//   scale          exact per physical level: sigma_0 = 2^logq (~ the rescaling primes),
//                  sigma_p = sqrt(sigma_{p-1} q_p).  Then HMult+rescale of two
//                  level-p ciphertexts lands exactly on sigma_{p-1}; plaintext
//                  constants are encoded at sigma_{p-1} q_p / sigma_p so mul_pt also
//                  lands on sigma_{p-1}; operands at different physical levels are
//                  aligned by dropping limbs and one constant-multiply + rescale.
#pragma once

#include <memory>
#include <vector>

#include "backends.h"
#include "core.h"
#include "rns.h"

namespace hsg {
namespace rns {

struct RCtData {
  DevBuf buf;      // u64 [2][phys+1][N], NTT form, at word offset `off` (a batched op's output slice)
  size_t off = 0;
  int phys = 0;
  int level = 0;
  size_t n = 0;
  const uint64_t* ptr() const { return reinterpret_cast<const uint64_t*>(buf.get()) + off; }
};
using RCt = std::shared_ptr<const RCtData>;

// How bootstrap() (ckks.hpp:207-213, a value-preserving level reset in the reference) is realised:
//   Logical  the logical level is reset, the physical chain is not: the chain must be at least the
//            statistic's whole no-bootstrap depth (deep chain, no secret key during evaluation);
//   Refresh  the ciphertext is refreshed to the top of the chain with the context's secret key
//            (decrypt + re-encrypt on the device, fresh noise): a trusted-refresh stand-in for CKKS
//            bootstrapping, which the reference does not implement either.  Physical level =
//            logical level + 1 at all times, so a chain of max_level + 1 primes suffices.
enum class Boot { Logical = 0, Refresh = 1 };

class RnsB : public LedgerBase<RnsB, RCt> {
 public:
  using C = RCt;
  RnsB(Ctx& c, const Params& p, Meter& m, Boot boot = Boot::Logical);
  Boot boot_mode() const { return boot_; }

  int level(const C& c) const { return c ? c->level : 0; }
  C encrypt(const double* v, size_t n);
  std::vector<C> encrypt_column(const double* v, size_t n);  // column.hpp:25-39
  C encrypt_const(double c);
  C add_ct(const C& a, const C& b) { return addsub(a, b, false); }
  C sub_ct(const C& a, const C& b) { return addsub(a, b, true); }
  C add_pt(const C& a, double c);
  C bootstrap(const C& a);
  C mul_ct(C a, C b);
  C mul_pt(C a, double c);
  C mul_pt_vec(C a, const std::vector<double>& v);
  C rotate(const C& a, long k);
  C sum_all_slots(const C& a, size_t n_valid);

  double first_slot(const C& c);
  void check_open_domain(const C& c, size_t n_valid, double lo, double hi, const char* who);
  void check_eval_domain(const C& c, double lo, double hi);
  void check_divergence(const C& c, size_t n_valid);
  void check_sqrt_domain(const C& c, size_t n_valid);
  void check_sign_domain(const C& c);

  std::vector<double> decrypt(const C& c, size_t n);
  // several results at once: the host side (CRT words -> coefficients -> FFT) on host threads
  std::vector<std::vector<double>> decrypt_many(const std::vector<C>& cts, const std::vector<size_t>& ns);
  double scale(int phys) const { return sigma_[static_cast<size_t>(phys)]; }

  // Batched BSGS (flow.h Bsgs::run): a full tree (2^K coefficients) evaluated level by level,
  // each stage one batched op over all its nodes -- the same ops on the same operands as the
  // recursion (identical limbs, meter and levels), ~K stages instead of ~2^K op calls.
  // bsgs_batch_ok: every multiplication of the tree has operands at level >= 1 and physical
  // level >= 1 (no auto-bootstrap, no level_exhausted inside), else the recursion runs.
  bool bsgs_batch_ok(const C& x, const std::vector<C>& pw, int K) const;
  // Batched chunk ops (flow.h BatchedChunks): every chunk at the same physical and logical level
  // >= 1 (nothing to bootstrap); one rescale / HMult launch set for the whole column.
  bool batch_ok(const std::vector<C>& xs) const;
  std::vector<C> mul_pt_many(const std::vector<C>& xs, double c);
  std::vector<C> square_many(const std::vector<C>& xs);
  C bsgs_full_tree(const C& x, const std::vector<double>& coeffs, const std::vector<C>& pw);

 private:
  struct Batch {  // n ciphertexts at one (phys, level), contiguous from ptr
    DevBuf buf;
    size_t off = 0;
    int phys = 0, level = 0;
    uint32_t n = 0;
    const uint64_t* ptr() const { return reinterpret_cast<const uint64_t*>(buf.get()) + off; }
  };
  Batch slice(const Batch& b, uint32_t first, uint32_t count) const;
  Batch gather(const std::vector<C>& xs);  // contiguous view (a copy unless they already are)
  std::vector<C> split(const Batch& b);   // one ciphertext handle per item (slices)
  Batch align_batch(const Batch& b, int p);
  C addsub(const C& a, const C& b, bool sub);
  C prepare_mul_pt(C a);
  C align(const C& x, int p);  // same value at physical level p (<= x->phys), scale sigma_p
  C make(DevBuf b, int phys, int level, size_t off = 0) const;
  C refresh(const C& a);  // Boot::Refresh: the same slots at the top of the chain, fresh noise
  size_t words(int phys) const { return size_t(2) * (phys + 1) * c_.N; }
  size_t sz(const C& c) const { return c ? c->n : 0; }
  Ctx& c_;
  Boot boot_ = Boot::Logical;
  std::vector<double> sigma_;
  uint64_t tag_ = 1;
};

// An RNS-backed EvalContext (hs_ctx::rns): the RNS context with its keys, the EvalContext's
// parameters and meter, and the backend bound to them.  Ciphertext handles share it, so
// Ciphertext::slots() can decrypt a handle that outlives its context.
struct Home {
  std::shared_ptr<Ctx> c;
  Params p;
  Meter m;
  std::unique_ptr<RnsB> b;
  Home(std::shared_ptr<Ctx> ctx, const Params& params, Boot boot) : c(std::move(ctx)), p(params) {
    b = std::make_unique<RnsB>(*c, p, m, boot);
  }
  // a Tier-E handle (Ciphertext(std::vector<double>, int) or another context's output) as an RNS
  // ciphertext of this context: its slots encrypted at the top of the chain, its level and size kept
  RCt adopt(const Ct& x);
};

// The RNS parameter set an RNS-backed EvalContext uses for CkksParams p (N = 2 slot_count):
//   Refresh: L = max_level + 1 (physical = logical + 1), logq0 = 61, logq = 60, dnum = 3, K so that
//            P exceeds every digit modulus, dense ternary secret (logQP ~1100 bits at max_level 11:
//            inside the 128-bit budget of N = 2^16, ~1760 bits);
//   Logical: L = depth + 1 for a caller-given depth (deep chain), same primes.
Spec default_spec(const Params& p, Boot boot, uint32_t depth, uint64_t seed);

}  // namespace rns
}  // namespace hsg
