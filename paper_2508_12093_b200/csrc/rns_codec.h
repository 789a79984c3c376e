// rns_codec.h — CKKS encode/decode (canonical embedding) for Tier R; see rns_codec.cpp.
#pragma once

#include <cstddef>
#include <cstdint>

namespace hsg {
namespace rns {

// n <= N/2 real slot values -> N integer coefficients round(scale * m_k)
void encode(uint32_t logN, const double* z, size_t n, double scale, int64_t* coeffs);
// N centred integer coefficients at `scale` -> first n slot values (real parts)
void decode(uint32_t logN, const int64_t* coeffs, double scale, double* z, size_t n);

// the same with integer-valued double coefficients (magnitudes beyond int64)
void encode_real(uint32_t logN, const double* z, size_t n, double scale, double* coeffs);
void decode_real(uint32_t logN, const double* coeffs, double scale, double* z, size_t n);

}  // namespace rns
}  // namespace hsg
