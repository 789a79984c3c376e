// hestat/errors.hpp — drop-in exception taxonomy (reference: errors.hpp:11-38),
// plus the mapping from libhestat_gpu status codes (include/hestat_gpu.h) back
// onto these types.
#pragma once

#include <stdexcept>
#include <string>

#include "hestat_gpu.h"

namespace hestat {

class error : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};

#define HESTAT_DROPIN_ERROR(name) \
  struct name : error {           \
    using error::error;           \
  }
// emulator
HESTAT_DROPIN_ERROR(too_many_values);
HESTAT_DROPIN_ERROR(level_exhausted);
HESTAT_DROPIN_ERROR(length_mismatch);
HESTAT_DROPIN_ERROR(dirty_padding);
// approximation / primitives
HESTAT_DROPIN_ERROR(non_finite_target);
HESTAT_DROPIN_ERROR(domain_violation);
HESTAT_DROPIN_ERROR(divergence);
// statistics
HESTAT_DROPIN_ERROR(empty_column);
HESTAT_DROPIN_ERROR(degenerate_variance);
HESTAT_DROPIN_ERROR(near_zero_mean);
// data pipeline
HESTAT_DROPIN_ERROR(io_error);
HESTAT_DROPIN_ERROR(missing_column);
HESTAT_DROPIN_ERROR(unparsable_cell);
HESTAT_DROPIN_ERROR(non_finite_value);
HESTAT_DROPIN_ERROR(zero_reference);
#undef HESTAT_DROPIN_ERROR

namespace gpu {
// Rethrow a libhestat_gpu status as the reference's exception type.
[[noreturn]] inline void raise(int rc) {
  const std::string m = hs_last_error();
  switch (rc) {
    case HS_E_TOO_MANY_VALUES: throw too_many_values(m);
    case HS_E_LEVEL_EXHAUSTED: throw level_exhausted(m);
    case HS_E_LENGTH_MISMATCH: throw length_mismatch(m);
    case HS_E_DIRTY_PADDING: throw dirty_padding(m);
    case HS_E_NON_FINITE_TARGET: throw non_finite_target(m);
    case HS_E_DOMAIN_VIOLATION: throw domain_violation(m);
    case HS_E_DIVERGENCE: throw divergence(m);
    case HS_E_EMPTY_COLUMN: throw empty_column(m);
    case HS_E_DEGENERATE_VARIANCE: throw degenerate_variance(m);
    case HS_E_NEAR_ZERO_MEAN: throw near_zero_mean(m);
    case HS_E_IO_ERROR: throw io_error(m);
    case HS_E_MISSING_COLUMN: throw missing_column(m);
    case HS_E_UNPARSABLE_CELL: throw unparsable_cell(m);
    case HS_E_NON_FINITE_VALUE: throw non_finite_value(m);
    case HS_E_ZERO_REFERENCE: throw zero_reference(m);
    default: throw error(m);
  }
}
inline void check(int rc) {
  if (rc != HS_OK) raise(rc);
}
}  // namespace gpu

}  // namespace hestat
