/* hestat_gpu.h — C ABI of libhestat_gpu.so, the B200 (sm_100a) backend of the
 * hestat CKKS-statistics operator surface.
 *
 * The reference (/root/reference/proj/include/hestat/ headers) is a header-only C++
 * library with no FFI; its "plugin API" is the hestat:: namespace.  This ABI is
 * the narrow waist underneath our drop-in C++ headers (include/hestat/) and
 * the Python mirror (paper_2508_12093_b200/hestat.py).  Every entry point below
 * names the reference declaration it replaces.
 *
 * Conventions
 *   - Every function returning int returns HS_OK (0) or an HS_E_* code; the
 *     message is in hs_last_error() (thread-local).  Codes 1..16 map 1:1 onto
 *     the reference's exception taxonomy (errors.hpp:11-38); on error, output
 *     handles are untouched and the context meter holds exactly the counts the
 *     reference's meter holds when it throws at the same point.
 *   - Ciphertexts (hs_ct) are immutable, reference-counted handles to a device
 *     slot vector plus a host-side level (ckks.hpp:62-78).  Every op returns a
 *     fresh handle that the caller releases with hs_ct_release.  Handles may be
 *     shared across threads and contexts.
 *   - Levels, meters and auto-bootstrap decisions live on the host; slot values
 *     live in HBM.  Ops are asynchronous on the library's CUDA stream; only
 *     hs_ct_read / hs_decrypt / hs_decode_column (and debug-mode value checks)
 *     synchronise.
 *   - Plain pointers and sizes only; no CUDA or torch types cross the ABI.
 */
#ifndef HESTAT_GPU_H
#define HESTAT_GPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes (errors.hpp:11-38) ---------------------------------- */
enum {
  HS_OK = 0,
  HS_E_ERROR = 1,              /* hestat::error                       */
  HS_E_TOO_MANY_VALUES = 2,    /* errors.hpp:18                        */
  HS_E_LEVEL_EXHAUSTED = 3,    /* errors.hpp:19                        */
  HS_E_LENGTH_MISMATCH = 4,    /* errors.hpp:20                        */
  HS_E_DIRTY_PADDING = 5,      /* errors.hpp:21                        */
  HS_E_NON_FINITE_TARGET = 6,  /* errors.hpp:24                        */
  HS_E_DOMAIN_VIOLATION = 7,   /* errors.hpp:25                        */
  HS_E_DIVERGENCE = 8,         /* errors.hpp:26                        */
  HS_E_EMPTY_COLUMN = 9,       /* errors.hpp:29                        */
  HS_E_DEGENERATE_VARIANCE = 10, /* errors.hpp:30                      */
  HS_E_NEAR_ZERO_MEAN = 11,    /* errors.hpp:31                        */
  HS_E_IO_ERROR = 12,          /* errors.hpp:34                        */
  HS_E_MISSING_COLUMN = 13,    /* errors.hpp:35                        */
  HS_E_UNPARSABLE_CELL = 14,   /* errors.hpp:36                        */
  HS_E_NON_FINITE_VALUE = 15,  /* errors.hpp:37                        */
  HS_E_ZERO_REFERENCE = 16,    /* errors.hpp:38                        */
  HS_E_CUDA = 100,             /* device/runtime failure (no reference counterpart) */
  HS_E_INVALID_ARG = 101       /* null handle / bad enum (no reference counterpart) */
};

/* ---- POD mirrors of the reference structs ------------------------------ */
typedef struct {            /* CkksParams, ckks.hpp:19-42 */
  uint64_t slot_count;      /* power of two (default 32768) */
  int32_t max_level;        /* >= 1 (default 11) */
  int32_t scale_bits;       /* >= 1 (default 40) */
  int32_t quantize;         /* bool (default 1) */
  int32_t auto_bootstrap;   /* bool (default 1) */
  int32_t debug_checks;     /* bool (default 0) */
  int32_t _pad;
} hs_params;

typedef struct {            /* CostMeter, ckks.hpp:46-60 */
  uint64_t mul_ct, mul_pt, add, rotate, bootstrap;
} hs_meter;

typedef struct {            /* InvRootConfig, primitives.hpp:23-40 */
  int32_t n;                /* 1 or 2 (default 2) */
  int32_t cheb_degree;      /* default 511 */
  int32_t newton_iters;     /* default 6 */
  int32_t baseline_mode;    /* bool (default 0) */
  int32_t baseline_iters;   /* 0 = default (21 for n=2, 25 for n=1) */
  int32_t _pad;
} hs_invroot_cfg;

typedef struct {            /* SignConfig, primitives.hpp:59-70 */
  int32_t mode;             /* 0 = G3Composition, 1 = CustomComposite */
  int32_t folds;            /* default 7 */
  const double* polys;      /* CustomComposite: concatenated power-basis polys */
  const uint64_t* poly_len; /* length of each */
  uint64_t npolys;
} hs_sign_cfg;

typedef struct {            /* EncryptedColumn, column.hpp:19-23 (name kept host-side) */
  struct hs_ct* const* chunks;
  uint64_t n_chunks;
  uint64_t n_valid;
} hs_column;

typedef struct hs_ctx hs_ctx; /* EvalContext, ckks.hpp:83-257 */
typedef struct hs_ct hs_ct;   /* Ciphertext,  ckks.hpp:64-78  */

enum { HS_TARGET_INVSQRT_SHIFTED = 0, HS_TARGET_SQRT_SHIFTED = 1 }; /* ScaledTargetKind, chebyshev.hpp:37 */

/* ---- runtime ----------------------------------------------------------- */
const char* hs_last_error(void);
const char* hs_version(void);
int hs_init(int device);                 /* optional: pick the CUDA device (default: current) */
int hs_sync(void);                       /* drain the library stream */
void* hs_stream(void);                   /* the library's cudaStream_t (for event timing) */
int hs_set_fused(int enabled);           /* 1 (default): fused pipelines; 0: op-by-op kernels */
uint64_t hs_kernel_launches(void);       /* kernels launched by this process so far */
/* CUDA-graph capture of library calls (launch-bound loops): every fused entry
 * point is capture-safe once warm (its series tables, scratch and ledger memo
 * exist).  Handles created inside the capture and released inside it become
 * graph allocation nodes; replaying re-executes every captured kernel. */
typedef struct hs_graph hs_graph;
int hs_graph_begin(void);
int hs_graph_end(hs_graph** out);
int hs_graph_launch(hs_graph* g);
void hs_graph_destroy(hs_graph* g);
/* diagnostics: FP64-pipe throughput on this GPU (kind 0 DMUL, 1 DADD, 2 DMUL+FRND, 3 DFMA),
 * instructions per second; the roofline denominator of the fused per-slot kernel */
int hs_diag_fp64_rate(int kind, double* ops_per_s);

/* ---- EvalContext (ckks.hpp:83-93) --------------------------------------- */
int hs_params_validate(const hs_params* p);                          /* CkksParams::validate */
int hs_ctx_create(const hs_params* p, uint64_t rng_seed, hs_ctx** out);
int hs_ctx_clone(const hs_ctx* ctx, hs_ctx** out);                   /* EvalContext copy (same backend) */
void hs_ctx_destroy(hs_ctx* ctx);
int hs_ctx_params(const hs_ctx* ctx, hs_params* out);
int hs_ctx_meter(const hs_ctx* ctx, hs_meter* out);
int hs_ctx_set_meter(hs_ctx* ctx, const hs_meter* m);                /* meter() is a mutable ref */
uint64_t hs_ctx_rng_seed(const hs_ctx* ctx);

/* ---- Ciphertext (ckks.hpp:64-78) ----------------------------------------- */
int hs_ct_new(const double* slots, uint64_t n, int32_t level, hs_ct** out); /* Ciphertext(vector, level) */
hs_ct* hs_ct_retain(hs_ct* ct);
void hs_ct_release(hs_ct* ct);
int32_t hs_ct_level(const hs_ct* ct);
uint64_t hs_ct_size(const hs_ct* ct);
int hs_ct_read(const hs_ct* ct, double* out, uint64_t n);             /* slots() (first n) */

/* ---- EvalContext ops (ckks.hpp:97-230) ------------------------------------ */
int hs_encrypt(const hs_ctx* ctx, const double* v, uint64_t n, hs_ct** out);          /* :97  */
int hs_decrypt(const hs_ctx* ctx, const hs_ct* ct, uint64_t n, double* out);          /* :107 */
int hs_add_ct(hs_ctx* ctx, const hs_ct* a, const hs_ct* b, hs_ct** out);             /* :113 */
int hs_sub_ct(hs_ctx* ctx, const hs_ct* a, const hs_ct* b, hs_ct** out);             /* :124 */
int hs_add_pt(hs_ctx* ctx, const hs_ct* a, double c, hs_ct** out);                   /* :137 */
int hs_mul_ct(hs_ctx* ctx, const hs_ct* a, const hs_ct* b, hs_ct** out);             /* :149 */
int hs_mul_pt(hs_ctx* ctx, const hs_ct* a, double c, hs_ct** out);                   /* :168 */
int hs_mul_pt_vec(hs_ctx* ctx, const hs_ct* a, const double* p, uint64_t n, hs_ct** out); /* :179 */
int hs_rotate(hs_ctx* ctx, const hs_ct* a, int64_t k, hs_ct** out);                  /* :193 */
int hs_bootstrap(hs_ctx* ctx, const hs_ct* a, hs_ct** out);                          /* :207 */
int hs_sum_all_slots(hs_ctx* ctx, const hs_ct* a, uint64_t n_valid, hs_ct** out);    /* :218 */
/* batched forms (C5 workloads, no reference counterpart: the reference issues n separate
 * calls): out[i] = op(a[i](, b[i])) with exactly the single op's semantics per element
 * (levels, auto-bootstrap, meter, errors in element order); one kernel per 64 ciphertexts */
int hs_add_ct_batch(hs_ctx* ctx, const hs_ct* const* a, const hs_ct* const* b, uint64_t n, hs_ct** out);
int hs_sub_ct_batch(hs_ctx* ctx, const hs_ct* const* a, const hs_ct* const* b, uint64_t n, hs_ct** out);
int hs_mul_ct_batch(hs_ctx* ctx, const hs_ct* const* a, const hs_ct* const* b, uint64_t n, hs_ct** out);
int hs_add_pt_batch(hs_ctx* ctx, const hs_ct* const* a, double c, uint64_t n, hs_ct** out);
int hs_mul_pt_batch(hs_ctx* ctx, const hs_ct* const* a, double c, uint64_t n, hs_ct** out);
int hs_rotate_batch(hs_ctx* ctx, const hs_ct* const* a, int64_t k, uint64_t n, hs_ct** out);

/* ---- Chebyshev (chebyshev.hpp) --------------------------------------------- */
double hs_scaled_target(int kind, double S, double t);                               /* :39  */
int32_t hs_cheb_eval_depth(int32_t degree);                                           /* :51  */
typedef double (*hs_target_fn)(double x, void* user);
int hs_fit(hs_target_fn f, void* user, int32_t degree, double lo, double hi, double* coeffs); /* :59 */
int hs_fit_target(int kind, double S, int32_t degree, double lo, double hi, double* coeffs);
double hs_eval_plain(const double* coeffs, uint64_t n, double lo, double hi, double x,
                     int32_t* extrapolated);                                          /* :90  */
int hs_eval_encrypted(hs_ctx* ctx, const double* coeffs, uint64_t n, double lo, double hi,
                      const hs_ct* ct, hs_ct** out);                                  /* :171 */

/* ---- inverse-root primitives (primitives.hpp) --------------------------------- */
#define HS_ALL_SLOTS ((uint64_t)-1)                                                   /* :20  */
int hs_newton_loop(hs_ctx* ctx, const hs_ct* x_op, const hs_ct* y, int32_t n, int32_t iters,
                   uint64_t n_valid, hs_ct** out);                                    /* :105 */
int hs_newton_refine(hs_ctx* ctx, const hs_ct* x, const hs_ct* y0, int32_t n, int32_t iters,
                     uint64_t n_valid, hs_ct** out);                                  /* :152 */
int hs_crypto_invsqrt(hs_ctx* ctx, const hs_ct* ct, double S, const hs_invroot_cfg* cfg,
                      uint64_t n_valid, hs_ct** out);                                 /* :186 */
int hs_baseline_invsqrt(hs_ctx* ctx, const hs_ct* ct, double S, int32_t iters, uint64_t n_valid,
                        hs_ct** out);                                                 /* :173 */
int hs_crypto_inv(hs_ctx* ctx, const hs_ct* ct, double S, const hs_invroot_cfg* cfg,
                  uint64_t n_valid, hs_ct** out);                                     /* :211 */
int hs_crypto_sqrt(hs_ctx* ctx, const hs_ct* ct, double S, int32_t degree, uint64_t n_valid,
                   hs_ct** out);                                                      /* :222 */
int hs_crypto_sign(hs_ctx* ctx, const hs_ct* ct, const hs_sign_cfg* cfg, hs_ct** out); /* :279 */

/* ---- columns (column.hpp) ------------------------------------------------------ */
/* chunks_out must hold ceil(n / slot_count) handles; *n_chunks receives the count. */
int hs_encode_column(hs_ctx* ctx, const double* v, uint64_t n, hs_ct** chunks_out,
                     uint64_t* n_chunks);                                             /* :25 */
int hs_decode_column(const hs_ctx* ctx, const hs_column* col, double* out);           /* :41 */

/* Asynchronous forms (extension: the reference's calls are synchronous).  They enqueue the
 * transfer and return; hs_pending_wait blocks until it has completed and returns the deferred
 * status (HS_E_NON_FINITE_VALUE for an encode whose input held a NaN or infinity: discard its
 * chunks).  Until then the caller must not touch `v` / `out`.  Chunks of a pending encode can be
 * passed to any op at once: the library orders its streams behind the upload.  A host loop
 * "encode k+1, compute k, decode k, wait k-1" keeps the copy engines and the SMs busy together.
 * The library keeps the buffers a pending transfer uses alive until it has settled, so the
 * chunk handles may be released earlier.  One thread owns a pending transfer: wait and release are not
 * synchronised against each other.  Every hs_pending is released with hs_pending_release (which
 * waits first if needed). */
typedef struct hs_pending hs_pending;
int hs_encode_column_async(hs_ctx* ctx, const double* v, uint64_t n, hs_ct** chunks_out,
                           uint64_t* n_chunks, hs_pending** pending);
int hs_decode_column_async(const hs_ctx* ctx, const hs_column* col, double* out,
                           hs_pending** pending);
int hs_pending_wait(hs_pending* pending);
void hs_pending_release(hs_pending* pending);

/* ---- statistics (stats.hpp) ------------------------------------------------------ */
int hs_mean_scaled(hs_ctx* ctx, const hs_column* col, double B, hs_ct** out);         /* :97  */
int hs_variance_to_scale(hs_ctx* ctx, const hs_column* col, double S, hs_ct** out);   /* :110 */
int hs_variance_scaled(hs_ctx* ctx, const hs_column* col, double B, hs_ct** out);     /* :130 */
int hs_moments(hs_ctx* ctx, const hs_column* col, double B, hs_ct** mu, hs_ct** var); /* :138 */
/* out_chunks must hold col->n_chunks handles */
int hs_znorm(hs_ctx* ctx, const hs_column* col, double B, const hs_invroot_cfg* cfg,
             hs_ct** out_chunks);                                                     /* :153 */
int hs_kurtosis(hs_ctx* ctx, const hs_column* col, double B, const hs_invroot_cfg* cfg,
                hs_ct** out);                                                         /* :170 */
int hs_skewness(hs_ctx* ctx, const hs_column* col, double B, const hs_invroot_cfg* cfg,
                hs_ct** out);                                                         /* :192 */
int hs_coeff_variation(hs_ctx* ctx, const hs_column* col, double B, const hs_sign_cfg* sign_cfg,
                       const hs_invroot_cfg* cfg, hs_ct** out);                       /* :216 */
int hs_pearson(hs_ctx* ctx, const hs_column* x, const hs_column* y, double B,
               const hs_invroot_cfg* cfg, hs_ct** out);                               /* :239 */
/* Extension: znorm(cols[k]) for k < ncols, in that order, into out_chunks (the result columns'
 * chunks concatenated: sum of the inputs' chunk counts): the same slots, levels and meter as the
 * calls; one launch per 64 single-chunk columns, the calls one by one otherwise. */
int hs_znorm_batch(hs_ctx* ctx, const hs_column* const* cols, uint32_t ncols, double B,
                   const hs_invroot_cfg* cfg, hs_ct** out_chunks);
/* Extension (SURVEY 8(d) C4's "deduplicated batched variant"): pearson(cols[i], cols[j]) for
 * every pair i < j of ncols columns, in that order, into out[ncols (ncols - 1) / 2]: the same
 * slots, levels and meter as the sequential calls; one launch for up to 8 single-chunk columns
 * of equal length (one inverse square root per column), the sequential calls otherwise.  An
 * error leaves no output (the meter is the sequential calls' at the error). */
int hs_pearson_table(hs_ctx* ctx, const hs_column* const* cols, uint32_t ncols, double B,
                     const hs_invroot_cfg* cfg, hs_ct** out);

/* ---- host-side data helpers (data.hpp / plain.hpp; CPU, not the hot path) ------ */
int hs_synthetic_uniform(uint64_t seed, uint64_t n, double lo, double hi, double* out); /* data.hpp:148 */
int hs_synthetic_grid(uint64_t n, double lo, double hi, double* out);                   /* data.hpp:163 */
int hs_two_subrange_grid(uint64_t n, double lo, double hi, double* out);                /* data.hpp:178 */
int hs_mre(const double* approx, const double* exact, uint64_t n, double* out);         /* data.hpp:190 */
int hs_relative_error(double approx, double exact, double* out);                       /* data.hpp:205 */
/* plain.hpp:18-92: which 0 mean 1 variance 2 skewness 3 kurtosis_ratio 4 coeff_variation
 * 5 pearson 6 znorm (n outputs) 7 stddev */
int hs_plain(int which, const double* x, uint64_t n, const double* y, double* out);

#ifdef __cplusplus
}
#endif
#endif /* HESTAT_GPU_H */
