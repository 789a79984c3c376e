/* hestat_oracle.h — TEST INFRASTRUCTURE ONLY.
 *
 * CPU restatement (plain C11, fp64, -ffp-contract=off) of the reference
 * emulator path: /root/reference/proj/include/hestat/{ckks,chebyshev,
 * primitives,column,stats,plain,data}.hpp.  Exposed with the same C ABI as
 * oracle/ref_shim.cpp (prefix ora_ here, ref_ there) so tests can pin this
 * restatement bit-for-bit against the compiled reference and then use it as
 * the checker for the CUDA product path.  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline leg may load liboracle.so.
 *
 * Parity status: PINNED — tests/test_oracle.py compares every entry point
 * bitwise against the tests/golden fixtures produced by the compiled reference
 * (tests/golden/make_golden.py) and against the reference's own KATs.
 */
#ifndef HESTAT_ORACLE_H
#define HESTAT_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
  uint64_t slot_count;
  int32_t max_level;
  int32_t scale_bits;
  int32_t quantize;
  int32_t auto_bootstrap;
  int32_t debug_checks;
  int32_t _pad;
} orc_params;

typedef struct {
  uint64_t mul_ct, mul_pt, add, rotate, bootstrap;
} orc_meter;

typedef struct {
  int32_t n, cheb_degree, newton_iters, baseline_mode, baseline_iters, _pad;
} orc_invroot;

enum {
  ORC_OP_ADD = 0, ORC_OP_SUB, ORC_OP_ADD_PT, ORC_OP_MUL_CT, ORC_OP_MUL_PT,
  ORC_OP_MUL_PT_VEC, ORC_OP_ROTATE, ORC_OP_BOOTSTRAP, ORC_OP_SUM_ALL
};

const char* ora_last_error(void);
int ora_encrypt(const orc_params* p, const double* v, uint64_t n, double* out, int32_t* lvl);
int ora_op(const orc_params* p, int op, const double* a, uint64_t na, int32_t la,
           const double* b, uint64_t nb, int32_t lb, double c, const double* vec,
           uint64_t nvec, int64_t k, uint64_t n_valid, double* out, int32_t* lout,
           orc_meter* meter);
int ora_fit(int kind, double S, int32_t degree, double lo, double hi, double* coeffs);
double ora_eval_plain(const double* coeffs, uint64_t ncoef, double lo, double hi, double x,
                      int32_t* extrapolated);
int ora_eval_encrypted(const orc_params* p, const double* coeffs, uint64_t ncoef, double lo,
                       double hi, const double* x, int32_t lx, double* out, int32_t* lout,
                       orc_meter* meter);
int ora_newton_refine(const orc_params* p, const double* x, int32_t lx, const double* y0,
                      int32_t ly, int32_t n, int32_t iters, uint64_t n_valid, double* out,
                      int32_t* lout, orc_meter* meter);
int ora_invroot(const orc_params* p, int which, const double* x, int32_t lx, double S,
                const orc_invroot* cfg, uint64_t n_valid, double* out, int32_t* lout,
                orc_meter* meter);
int ora_crypto_sign(const orc_params* p, const double* x, int32_t lx, int32_t mode,
                    int32_t folds, const double* polys, const uint64_t* poly_len,
                    uint64_t npolys, double* out, int32_t* lout, orc_meter* meter);
int ora_stat(const orc_params* p, int which, const double* x, uint64_t n, const double* y,
             uint64_t ny, double B, const orc_invroot* cfg, double* out, int32_t* lout,
             orc_meter* meter);
int ora_synthetic_uniform(uint64_t seed, uint64_t n, double lo, double hi, double* out);
int ora_synthetic_grid(uint64_t n, double lo, double hi, double* out);
int ora_two_subrange_grid(uint64_t n, double lo, double hi, double* out);
int ora_plain(int which, const double* x, uint64_t n, const double* y, double* out);
int ora_znorm_reps(const orc_params* p, const double* x, uint64_t n, double B, int32_t reps,
                   double* out, orc_meter* meter);

#ifdef __cplusplus
}
#endif
#endif
