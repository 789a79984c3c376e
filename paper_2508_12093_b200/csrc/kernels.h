// kernels.h — host-callable launchers for every CUDA kernel of libhestat_gpu.
//
//   ops.cu    E1-E5: slot-wise ops, rotation, requantisation, sum_all_slots
//             (the log-step rotate-and-add reduction, in shared memory across a
//             thread-block cluster via DSMEM).
//   fused.cu  E6-E7: the per-slot program kernel (prog.cuh: Chebyshev BSGS,
//             Newton, inverse roots, sign, sqrt).
//   stat.cu   E8: one cooperative kernel per statistic (moments -> grid barrier
//             -> centred moments -> grid barrier -> per-slot program).
#pragma once

#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>

namespace hsg {

// Arithmetic policy selector (quant.cuh)
enum class QMode : int { None = 0, Exact = 1, Grid = 2 };
struct QSpec {
  QMode mode = QMode::None;
  int bits = 40;
};

namespace k {

// ---- ops.cu ------------------------------------------------------------------------
enum BinOp : int { B_ADD = 0, B_SUB = 1, B_MUL = 2 };
void binary(QSpec q, BinOp op, const double* a, const double* b, double* out, size_t n, cudaStream_t s);
enum ScalOp : int { S_ADD = 0, S_MUL = 1 };
void scalar(QSpec q, ScalOp op, const double* a, double c, double* out, size_t n, cudaStream_t s);
void requant(QSpec q, const double* a, double* out, size_t n, cudaStream_t s);
// encrypt (ckks.hpp:97-104): out[i] = q(src[i]) for i < n, 0 for n <= i < S; src may
// be host-mapped pinned memory (zero-copy).  Sets *bad (device- or host-mapped)
// when any src value is non-finite (column.hpp:28-30 check, done on device).
void encrypt(QSpec q, const double* src, size_t n, double* out, size_t S, int* bad, cudaStream_t s);
void rotate(const double* a, double* out, size_t n, size_t shift, cudaStream_t s);
// batched forms (C5 workloads): `count` independent ciphertexts, one launch per 64
void binary_batch(QSpec q, BinOp op, const double* const* a, const double* const* b, double* const* o,
                  size_t count, size_t n, cudaStream_t s);
void scalar_batch(QSpec q, ScalOp op, const double* const* a, double c, double* const* o, size_t count, size_t n,
                  cudaStream_t s);
void rotate_batch(const double* const* a, double* const* o, size_t count, size_t n, size_t shift, cudaStream_t s);
// sum_all_slots over `batch` ciphertexts of S slots each (a[b], out[b]).
void slot_sum(QSpec q, const double* const* a, double* const* out, int batch, size_t S, cudaStream_t s);
// largest S the single-launch cluster kernel handles with `arrays` concurrent sums
size_t slot_sum_max(int arrays);

// ---- fused.cu: per-slot programs ------------------------------------------------------
enum MOp : int {
  M_LD = 0,   // r[dst] = in(arr[i0][slot])
  M_ST,       // arr_out[i0][slot] = out(r[a])
  M_CONST,    // r[dst] = c (already in the policy's units)
  M_ADD,      // r[dst] = add(r[a], r[b])
  M_SUB,      // r[dst] = sub(r[a], r[b])
  M_MUL,      // r[dst] = mul(r[a], r[b])
  M_ADDC,     // r[dst] = addc(r[a], c)
  M_MULC,     // r[dst] = mulc(r[a], c)
  M_CHEB,     // r[dst] = ChebEncryptedEval(table @ i0, degree i1) on r[a]
  M_NEWTON,   // r[dst] = newton_loop(x_op = r[a], y = r[b], n = i0, iters = i1, (n+1)/n = c)
  M_ZAPPLY,   // for every chunk: zout[c][slot] = out(mul(sub(in(zin[c][slot]), r[a]), r[b]))
  M_LDR,      // r[dst] = per-slot statistic value i0 (stat.cu: 0 mu_x, 1 var_x, 2 mu_y, 3 var_y, 4 num)
  M_CHK       // debug_checks value check of r[a] (real units) on slots < i1, kind i0, constants c, c2:
              // a failing slot sets *Prog::flags (the host then replays the call op by op)
};
// M_CHK kinds: the reference's debug predicates, evaluated with the same fp64 operations
enum ChkKind : int {
  CK_OPEN = 0,       // fail if !(v > c) || !(v <= c2)          check_open_domain, primitives.hpp:134-144
  CK_RANGE = 1,      // fail if v < c || v > c2                  eval_encrypted / sqrt / sign domains
  CK_LT = 2,         // fail if v < c                            moments: negative variance, stats.hpp:144
  CK_SCALED_LT = 3,  // fail if (v * c) * c < c2                 variance below 1e-9 (B^2-scaled), stats.hpp:156
  CK_ABS_LT = 4      // fail if |v| < c                          coeff_variation near-zero mean, stats.hpp:221
};
struct MInst {
  int op, dst, a, b, i0, i1;
  double c;
  int i2 = 0;      // M_NEWTON: divergence check on slots < i2 after every iteration (0 = none)
  double c2 = 0.0;
};
constexpr int kMaxInst = 40;
constexpr int kMaxArr = 6;
#ifndef HS_MAXCH
#define HS_MAXCH 48
#endif
constexpr int kMaxChunks = HS_MAXCH;
constexpr int kRegs = 24;
constexpr int kMaxFusedDegree = 1023;
constexpr int kMaxFusedNewtonN = 6;

struct Prog {
  int n = 0;
  int nchunks = 0;
  unsigned S = 0;
  int ntab = 0;                  // doubles of coefficient tables, staged into shared memory
  const double* tabs = nullptr;  // coefficient tables (device); M_CHEB i0 = offset, b = lane-split
  unsigned* flags = nullptr;     // debug_checks: set nonzero by any failing M_CHK / Newton guard
  MInst ins[kMaxInst];
  const double* in[kMaxArr];
  double* out[kMaxArr];
  const double* zin[kMaxChunks];
  double* zout[kMaxChunks];
};

// Launch one per-slot program over S slots.  lanes = 1, 2, 4 or 8 threads per slot.
void run_prog(QSpec q, const Prog& p, int lanes, cudaStream_t s);
// copies a degree-511 coefficient table (512 doubles, device) into stat.cu's constant-bank copy
void upload_const_table(const double* dev_table, cudaStream_t s);

// moment modes of the statistics kernel (stats.hpp:97-126): mean_scaled terms,
// variance_to_scale terms (squares + mean part), or both
enum MomMode : int { MOM_MEAN = 1, MOM_VAR = 2, MOM_BOTH = 3 };

// ---- stat.cu: one cooperative kernel per statistic ------------------------------------
// Phase A  moment terms of 1-2 columns (MomArgs semantics) -> grid-wide sums
// Phase B  (power > 0) centred power sums (CentArgs semantics) -> grid-wide sum
// Phase C  the per-slot program, with M_LDR reading the per-slot values
//          {mu_x, var_x, mu_y, var_y, num}.
// Each reduction is exact-sum when provable (see slotsum.cuh), else the literal
// log2(S)-step rotate-and-add butterfly runs through global scratch with a grid
// barrier per step.
struct StatArgs {
  int ncols = 1;          // 1 or 2 columns in phase A
  int mom_mode = MOM_BOTH;
  int nchunks = 0;
  const double* x[kMaxChunks];
  const double* y[kMaxChunks];
  uint64_t valid[kMaxChunks];
  double cm[2] = {0, 0}, ca[2] = {0, 0}, cmp[2] = {0, 0};
  int power = 0;          // 0: no phase B; 3, 4: centred power of x; 2: x-y product (pearson)
  double inv_n = 0;
  double* partial = nullptr;  // stat_partial_doubles(), zero between launches: grid-wide totals + counters
  double* scratch = nullptr;  // >= 2 * 6 * S doubles (butterfly fallback)
};
void run_stat(QSpec q, const StatArgs& a, const Prog& p, int lanes, cudaStream_t s);

// ---- stat.cu: the C4 Pearson table in one cooperative kernel -----------------------------
// All ncols (<= 8) single-chunk columns' moments (phase A), every pair's centred product sum
// (phase B: pair p = (pi[p], pj[p]), the x side masked past n_valid as centered_chunks does),
// one inverse square root per COLUMN (phase C: the program `p`, M_LDR 0/1 = mu/var of the
// item's column, its M_ST writes inv + col * S), and per pair out[p] = (cov_p inv_i) inv_j
// (phase D, block-local).  Requires exact grid sums (QGrid): when a sum is not provably exact the
// kernel sets *inexact and writes nothing (the host replays the pairs one by one).
constexpr int kMaxTableCols = 8, kMaxTablePairs = kMaxTableCols * (kMaxTableCols - 1) / 2;
struct PTableArgs {
  int ncols = 0, npairs = 0;
  const double* x[kMaxTableCols];
  uint64_t valid = 0;            // n_valid (< S: the x side of every product is masked)
  double cm = 0, ca = 0, cmp = 0;  // mean_scaled(B = 1), variance_to_scale(B^2) constants
  double inv_n = 0;
  uint8_t pi[kMaxTablePairs], pj[kMaxTablePairs];
  double* out[kMaxTablePairs];
  double* partial = nullptr;     // ptable_partial_doubles(), zero between launches
  unsigned* inexact = nullptr;
};
size_t ptable_partial_doubles();
void run_ptable(QSpec q, const PTableArgs& a, const Prog& p, int lanes, cudaStream_t s);

// ---- stat.cu: many independent single-chunk Z-scores in one cooperative kernel -----------
// Column k: moments (phase A: mean_scaled(B = 1) and variance_scaled(B) terms), the program `p`
// (M_LDR 0/1 = the column's mu/var; its M_ST writes inv + k S: crypto_invsqrt(var, B^2)), then
// z_k = (x_k - mu_k) inv_k (block-local).  A column whose sums are not provably exact takes the
// literal rotate-and-add butterfly in the same launch (scratch: 2 x 3 ncols x S doubles).
constexpr int kMaxZBatch = 64;
struct ZBatchArgs {
  int ncols = 0;
  const double* x[kMaxZBatch];
  double* z[kMaxZBatch];
  double cm[kMaxZBatch], ca[kMaxZBatch], cmp[kMaxZBatch];
  double* partial = nullptr;  // zbatch_partial_doubles(), zero between launches
  double* scratch = nullptr;  // butterfly fallback
};
size_t zbatch_partial_doubles();
void run_zbatch(QSpec q, const ZBatchArgs& a, const Prog& p, int lanes, cudaStream_t s);
size_t stat_partial_doubles();  // scratch sizing for StatArgs::partial

}  // namespace k
}  // namespace hsg
