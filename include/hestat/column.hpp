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

}  // namespace hestat
