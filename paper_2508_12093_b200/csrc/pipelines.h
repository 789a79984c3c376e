// pipelines.h — the hot-path entry points behind the ABI.
//
// Each entry point either
//   (fused)  runs the reference control flow on SymB (levels, meter, errors —
//            before any device work), then evaluates all slot values with the
//            fused kernels of fused.cu (1-3 launches per call), or
//   (op-by-op) runs the same control flow on DevB, one kernel per op.
// The fused path is taken when debug_checks is off, fusion is enabled
// (hs_set_fused), every input ciphertext is known to lie on the 2^-scale_bits
// grid (or quantize is off), and the shape is within the fused kernels' limits.
// Both paths are bit-identical to the reference (tests/test_parity_*.py).
#pragma once

#include "core.h"
#include "flow.h"
#include "series.h"

namespace hsg {
namespace pipe {

using ColC = flow::Col<Ct>;

Ct eval_encrypted(hs_ctx* ctx, const Series& s, const Ct& ct);
Ct newton_loop(hs_ctx* ctx, const Ct& x_op, const Ct& y, int n, int iters, size_t n_valid);
Ct newton_refine(hs_ctx* ctx, const Ct& x, const Ct& y0, int n, int iters, size_t n_valid);
Ct crypto_invsqrt(hs_ctx* ctx, const Ct& ct, double S, const flow::InvCfg& cfg, size_t n_valid);
Ct baseline_invsqrt(hs_ctx* ctx, const Ct& ct, double S, int iters, size_t n_valid);
Ct crypto_inv(hs_ctx* ctx, const Ct& ct, double S, const flow::InvCfg& cfg, size_t n_valid);
Ct crypto_sqrt(hs_ctx* ctx, const Ct& ct, double S, int degree, size_t n_valid);
Ct crypto_sign(hs_ctx* ctx, const Ct& ct, const flow::SignCfg& cfg);

Ct mean_scaled(hs_ctx* ctx, const ColC& col, double B);
Ct variance_to_scale(hs_ctx* ctx, const ColC& col, double S);
Ct variance_scaled(hs_ctx* ctx, const ColC& col, double B);
flow::Moments<Ct> moments(hs_ctx* ctx, const ColC& col, double B);
ColC znorm(hs_ctx* ctx, const ColC& col, double B, const flow::InvCfg& cfg);
Ct kurtosis(hs_ctx* ctx, const ColC& col, double B, const flow::InvCfg& cfg);
Ct skewness(hs_ctx* ctx, const ColC& col, double B, const flow::InvCfg& cfg);
Ct coeff_variation(hs_ctx* ctx, const ColC& col, double B, const flow::SignCfg& sc, const flow::InvCfg& cfg);
Ct pearson(hs_ctx* ctx, const ColC& x, const ColC& y, double B, const flow::InvCfg& cfg);
// znorm(cols[k]) for every k, in order; one launch per 64 single-chunk columns where possible
std::vector<ColC> znorm_batch(hs_ctx* ctx, const std::vector<ColC>& cols, double B, const flow::InvCfg& cfg);
// pearson(cols[i], cols[j]) for every pair i < j in order, one launch where possible
std::vector<Ct> pearson_table(hs_ctx* ctx, const std::vector<ColC>& cols, double B, const flow::InvCfg& cfg);

}  // namespace pipe
}  // namespace hsg
