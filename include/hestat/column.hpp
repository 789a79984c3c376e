// hestat/column.hpp — drop-in for /root/reference/proj/include/hestat/column.hpp:19-56.
#pragma once

#include <span>
#include <string>
#include <vector>

#include "hestat/ckks.hpp"
#include "hestat/errors.hpp"

namespace hestat {

struct EncryptedColumn {  // :19-23
  std::vector<Ciphertext> chunks;
  std::size_t n_valid = 0;
  std::string name;

  // C-ABI view (handles borrowed for the duration of one call)
  struct CView {
    std::vector<hs_ct*> h;
    hs_column c;
  };
  CView to_c() const {
    CView v;
    for (const Ciphertext& ct : chunks) v.h.push_back(ct.raw());
    v.c = hs_column{v.h.data(), v.h.size(), n_valid};
    return v;
  }
};

inline EncryptedColumn encode_column(EvalContext& ctx, std::span<const double> values,
                                     std::string name = {}) {  // :25-39
  const std::size_t S = ctx.params().slot_count;
  std::vector<hs_ct*> h((values.size() + S - 1) / S + 1, nullptr);
  uint64_t n = 0;
  const int rc = hs_encode_column(ctx.raw(), values.data(), values.size(), h.data(), &n);
  if (rc == HS_E_NON_FINITE_VALUE) throw non_finite_value("encode_column: non-finite value in " + name);
  gpu::check(rc);
  EncryptedColumn col;
  col.n_valid = values.size();
  col.name = std::move(name);
  for (uint64_t i = 0; i < n; ++i) col.chunks.push_back(Ciphertext::adopt(h[i]));
  return col;
}

inline std::vector<double> decode_column(const EvalContext& ctx, const EncryptedColumn& col) {  // :41-56
  const EncryptedColumn::CView v = col.to_c();
  std::vector<double> out(col.n_valid);
  gpu::check(hs_decode_column(ctx.raw(), &v.c, out.data()));
  return out;
}

// ---- extension: the same transfers without the wait (hs_*_async, hestat_gpu.h) -----------------
// A transfer in flight.  wait() blocks until it has completed and throws the call's deferred
// error (non_finite_value for an encode whose input held a NaN or infinity).  The host buffer
// handed to the call must stay untouched until then; pinned buffers (cudaHostAlloc) move by DMA
// at PCIe rate beside running kernels.
class Pending {
 public:
  Pending() = default;
  explicit Pending(hs_pending* p, std::string what = {}) : p_(p), what_(std::move(what)) {}
  Pending(Pending&& o) noexcept : p_(o.p_), what_(std::move(o.what_)) { o.p_ = nullptr; }
  Pending& operator=(Pending&& o) noexcept {
    if (this != &o) {
      hs_pending_release(p_);
      p_ = o.p_;
      what_ = std::move(o.what_);
      o.p_ = nullptr;
    }
    return *this;
  }
  Pending(const Pending&) = delete;
  Pending& operator=(const Pending&) = delete;
  ~Pending() { hs_pending_release(p_); }
  void wait() {
    if (!p_) return;
    const int rc = hs_pending_wait(p_);
    if (rc == HS_E_NON_FINITE_VALUE) throw non_finite_value("encode_column: non-finite value in " + what_);
    gpu::check(rc);
  }

 private:
  hs_pending* p_ = nullptr;
  std::string what_;
};

// encode_column without the wait: the column can be passed to any op at once (the library orders
// its streams behind the upload); `pending.wait()` delivers the finiteness verdict.
inline EncryptedColumn encode_column_async(EvalContext& ctx, std::span<const double> values, Pending& pending,
                                           std::string name = {}) {
  const std::size_t S = ctx.params().slot_count;
  std::vector<hs_ct*> h((values.size() + S - 1) / S + 1, nullptr);
  uint64_t n = 0;
  hs_pending* p = nullptr;
  gpu::check(hs_encode_column_async(ctx.raw(), values.data(), values.size(), h.data(), &n, &p));
  pending = Pending(p, name);
  EncryptedColumn col;
  col.n_valid = values.size();
  col.name = std::move(name);
  for (uint64_t i = 0; i < n; ++i) col.chunks.push_back(Ciphertext::adopt(h[i]));
  return col;
}

// decode_column without the wait: `out` (col.n_valid doubles) holds the slots once wait() returns.
inline Pending decode_column_async(const EvalContext& ctx, const EncryptedColumn& col, std::span<double> out) {
  if (out.size() < col.n_valid) throw length_mismatch("decode_column: out shorter than n_valid");
  const EncryptedColumn::CView v = col.to_c();
  hs_pending* p = nullptr;
  gpu::check(hs_decode_column_async(ctx.raw(), &v.c, out.data(), &p));
  return Pending(p, col.name);
}

}  // namespace hestat
