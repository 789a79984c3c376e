// stat.cu — one cooperative kernel per encrypted statistic (stats.hpp:97-265).
//
// A statistic is slot-wise work separated by rotate-and-sum reductions.  Every
// kernel launch costs ~3 us of device time back to back on B200, and a
// cluster-local reduction keeps 140 of 148 SMs idle, so each statistic runs as
// ONE grid-wide cooperative kernel over all SMs:
//
//   phase A  per slot, the moment terms of 1-2 columns (mean, squared, mean
//            part: stats.hpp:41-51, 110-126), summed grid-wide;   grid.sync
//   phase B  (kurtosis / skewness / pearson) per slot, the centred power or
//            product terms using phase A's mean (stats.hpp:56-87), summed
//            grid-wide;                                           grid.sync
//   phase C  per slot, the fused program (prog.cuh): inverse square root of
//            the variance and the statistic's epilogue, written straight to the
//            output ciphertext(s).
//
// Reductions: in grid units every term is an integer; when the grid-wide sum
// of |terms| is provably < 2^53 every addition of the reference's log2(S)-step
// rotate-and-add is exact, so every slot's result is the exact total (see
// slotsum.cuh) and one deterministic reduction suffices.  Otherwise (huge
// magnitudes, or quantize off) the literal butterfly runs through global
// scratch, one grid barrier per step — bit-identical either way.
#include <cooperative_groups.h>

#include <cstdlib>
#include <mutex>
#include <unordered_map>

#include "core.h"
#include "kernels.h"
#include "prog.cuh"
#include "quant.cuh"

namespace hsg {
namespace k {
namespace {
namespace cg = cooperative_groups;

constexpr int kMaxWarps = 32;
constexpr int kNK = 6;  // reduction arrays: up to 3 per column, 2 columns

struct Reduced {
  bool uniform;         // exact-sum: every slot holds tot[k]
  double tot[kNK];
  const double* res;    // otherwise: butterfly result, array k at res + k * S
};

#ifdef HS_STAT_TIMING
__device__ unsigned long long g_stat_t[8];
__device__ __forceinline__ void stamp(int k) {
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    g_stat_t[k] = t;
  }
}
#else
__device__ __forceinline__ void stamp(int) {}
#endif

// Grid barrier over a plain launch (the grid is sized to be co-resident: one block per
// SM, checked against the occupancy calculator on the host).  One word per barrier
// sequence: block 0 adds 2^31 - (blocks - 1), every other block adds 1, so the top bit
// flips exactly when all blocks have arrived and the word's low bits are unchanged
// afterwards (ready for the next barrier and the next launch).  Release on arrival,
// acquire while polling.  A plain launch lets encode_column's kernels (upload stream)
// share the SMs with a running statistic.
__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
struct GridBar {
  unsigned* bar;
  __device__ void sync() const {
    __syncthreads();
    if (threadIdx.x == 0) {
      const unsigned nb = blockIdx.x == 0 ? 0x80000000u - (gridDim.x - 1) : 1u;
      unsigned old;
      asm volatile("atom.add.release.gpu.global.u32 %0, [%1], %2;" : "=r"(old) : "l"(bar), "r"(nb) : "memory");
      while (((old ^ ld_acquire_u32(bar)) & 0x80000000u) == 0) {
      }
    }
    __syncthreads();
  }
};

// Grid-wide rotate-and-sum of NK per-slot term arrays produced by terms(i, t).
// `idle` runs between publishing this block's partials and the grid barrier (work
// that overlaps the wait for the slowest block, e.g. staging the Chebyshev table).
template <class Q, class TermFn, class IdleFn>
__device__ Reduced grid_sum(const Q& q, const GridBar& grid, TermFn terms, int NK, unsigned S,
                            double* accum, unsigned* count, double* scratch, IdleFn idle) {
  __shared__ double red[kMaxWarps][2 * kNK];
  __shared__ double tot[2 * kNK];
  const Range BR = block_range(S);
  Reduced R{};
  R.res = nullptr;
  if constexpr (Q::kExactSum) {
    double acc[2 * kNK];
#pragma unroll
    for (int k = 0; k < 2 * kNK; ++k) acc[k] = 0.0;
    for (unsigned i = BR.lo + threadIdx.x; i < BR.hi; i += blockDim.x) {
      double t[kNK];
      terms(i, t);
#pragma unroll
      for (int k = 0; k < kNK; ++k)
        if (k < NK) {
          acc[2 * k] += t[k];
          acc[2 * k + 1] += fabs(t[k]);
        }
    }
#pragma unroll
    for (int k = 0; k < 2 * kNK; ++k)
      for (int o = 16; o > 0; o >>= 1) acc[k] += __shfl_xor_sync(0xffffffffu, acc[k], o);
    if ((threadIdx.x & 31) == 0)
#pragma unroll
      for (int k = 0; k < 2 * kNK; ++k) red[threadIdx.x >> 5][k] = acc[k];
    __syncthreads();
    // this block's sums go straight into the grid-wide totals: every term is an integer
    // and the checked bound keeps every partial sum below 2^53, so the atomic additions
    // are exact in any order (and a failed bound is never under-reported: rounding is
    // monotone and 2^52 is representable)
    if (threadIdx.x < 2 * NK) {
      double s = 0.0;
      for (unsigned w = 0; w < blockDim.x / 32; ++w) s += red[w][threadIdx.x];
      atomicAdd(accum + threadIdx.x, s);
    }
    stamp(5);
    idle();
    grid.sync();
    stamp(6);
    if (threadIdx.x < 2 * NK) tot[threadIdx.x] = __ldcg(accum + threadIdx.x);
    __syncthreads();
    if (threadIdx.x == 0 && atomicAdd(count, 1u) == gridDim.x - 1) {
      // the last block to read the totals zeroes them for the next launch
      for (int k = 0; k < 2 * NK; ++k) accum[k] = 0.0;
      *count = 0u;
    }
    stamp(7);
    bool exact = true;
    for (int k = 0; k < NK; ++k) {
      R.tot[k] = tot[2 * k];
      exact = exact && tot[2 * k + 1] < 4503599627370496.0;  // 2^52: true sum < 2^53
    }
    __syncthreads();
    if (exact) {
      R.uniform = true;
      return R;
    }
  }
  // literal butterfly (ckks.hpp:218-230) through global memory
  if constexpr (!Q::kExactSum) idle();
  double* cur = scratch;
  double* nxt = scratch + static_cast<size_t>(kNK) * S;
  for (unsigned i = BR.lo + threadIdx.x; i < BR.hi; i += blockDim.x) {
    double t[kNK];
    terms(i, t);
    for (int k = 0; k < NK; ++k) cur[static_cast<size_t>(k) * S + i] = t[k];
  }
  grid.sync();
  for (unsigned d = 1; d < S; d <<= 1) {
    for (unsigned i = BR.lo + threadIdx.x; i < BR.hi; i += blockDim.x) {
      const unsigned j = (i + d) & (S - 1);
      for (int k = 0; k < NK; ++k)
        nxt[static_cast<size_t>(k) * S + i] =
            q.add(__ldcg(cur + static_cast<size_t>(k) * S + i), __ldcg(cur + static_cast<size_t>(k) * S + j));
    }
    grid.sync();
    double* t = cur;
    cur = nxt;
    nxt = t;
  }
  R.uniform = false;
  R.res = cur;
  return R;
}

__device__ __forceinline__ double pick(const Reduced& R, int k, unsigned S, unsigned i) {
  return R.uniform ? R.tot[k] : __ldcg(R.res + static_cast<size_t>(k) * S + i);
}


template <class Q, int P>
__global__ void __launch_bounds__(prog_max_threads<P>(), 1) k_stat(Q q, const __grid_constant__ StatArgs a,
                                                       const __grid_constant__ Prog pg) {
  extern __shared__ double stab[];
  stamp(0);
  const GridBar grid{reinterpret_cast<unsigned*>(a.partial + 4 * kNK + 1)};
  // the table is first needed in phase B/C: stage it while waiting at phase A's barrier
  auto stage = [&] {
    for (int i = threadIdx.x; i < pg.ntab; i += blockDim.x) stab[i] = __ldg(pg.tabs + i);
  };
  const unsigned S = pg.S;
  const int per_col = (a.mom_mode & MOM_MEAN ? 1 : 0) + (a.mom_mode & MOM_VAR ? 2 : 0);
  const int NA = per_col * a.ncols;

  // ---- phase A: moment terms (MomArgs semantics) ----
  auto termsA = [&](unsigned i, double* t) {
    for (int col = 0; col < a.ncols; ++col) {
      double* tc = t + col * per_col;
      for (int c = 0; c < a.nchunks; ++c) {
        const double X = q.in(__ldg((col == 0 ? a.x[c] : a.y[c]) + i));
        double v[3];
        int k = 0;
        if (a.mom_mode & MOM_MEAN) v[k++] = q.mulc(X, a.cm[col]);  // mul_pt(chunk, 1/(B n))
        if (a.mom_mode & MOM_VAR) {
          const double s = q.mulc(X, a.ca[col]);                   // mul_pt(chunk, 1/sqrt(S n))
          v[k++] = q.mul(s, s);                                    // mul_ct(a, a)
          v[k++] = q.mulc(X, a.cmp[col]);                          // mul_pt(chunk, 1/(n sqrt(S)))
        }
        for (int j = 0; j < per_col; ++j) tc[j] = c == 0 ? v[j] : q.add(tc[j], v[j]);
      }
    }
  };
  stamp(1);
  unsigned* counts = reinterpret_cast<unsigned*>(a.partial + 4 * kNK);
  const Reduced RA = grid_sum(q, grid, termsA, NA, S, a.partial, counts, a.scratch, stage);
  stamp(2);

  // per-slot statistic values {mu_x, var_x, mu_y, var_y}
  auto mom = [&](unsigned i, double* sv) {
    for (int col = 0; col < a.ncols; ++col) {
      const int b0 = col * per_col;
      int k = 0;
      if (a.mom_mode & MOM_MEAN) sv[2 * col] = pick(RA, b0 + k++, S, i);
      if (a.mom_mode & MOM_VAR) {
        const double sq = pick(RA, b0 + k, S, i), mp = pick(RA, b0 + k + 1, S, i);
        sv[2 * col + 1] = q.sub(sq, q.mul(mp, mp));  // sub_ct(sq_sum, mul_ct(mp, mp))
      }
    }
  };

  // ---- phase B: centred power / product terms (CentArgs semantics) ----
  Reduced RB{};
  RB.uniform = true;
  RB.tot[0] = 0.0;
  if (a.power > 0) {
    auto termsB = [&](unsigned i, double* t) {
      double sv[4];
      mom(i, sv);
      const double mux = sv[0], muy = sv[2];
      for (int c = 0; c < a.nchunks; ++c) {
        const double mm = a.valid[c] < S ? q.mulc(mux, i < a.valid[c] ? 1.0 : 0.0) : mux;  // mul_pt(mu, mask)
        const double cx = q.sub(q.in(__ldg(a.x[c] + i)), mm);
        double p;
        if (a.power == 4) {
          const double sq = q.mul(cx, cx);
          p = q.mul(sq, sq);
        } else if (a.power == 3) {
          const double sq = q.mul(cx, cx);
          p = q.mul(sq, cx);
        } else {
          p = q.mul(cx, q.sub(q.in(__ldg(a.y[c] + i)), muy));
        }
        const double term = q.mulc(p, a.inv_n);  // mean_of_chunks: mul_pt(chunk, 1/n)
        t[0] = c == 0 ? term : q.add(t[0], term);
      }
    };
    RB = grid_sum(q, grid, termsB, 1, S, a.partial + 2 * kNK, counts + 1,
                  a.scratch + 2 * static_cast<size_t>(kNK) * S, [] {});
  }

  // ---- phase C: the per-slot program over this block's slot range ----
  stamp(3);
  const Range R = block_range(S);
  if (R.lo >= R.hi) return;
  const unsigned iters = (R.spb * P + blockDim.x - 1) / blockDim.x;
  for (unsigned it = 0; it < iters; ++it) {
    const unsigned g = threadIdx.x + it * blockDim.x;
    const unsigned slot = R.lo + g / P;
    const bool live = slot < R.hi;
    const unsigned s = live ? slot : R.hi - 1;
    double sv[5];
    mom(s, sv);
    sv[4] = a.power > 0 ? pick(RB, 0, S, s) : 0.0;
    exec<Q, P>(q, pg, stab, s, static_cast<int>(g % P), live, sv);
  }
  stamp(4);
}

// ---- the C4 Pearson table (kernels.h PTableArgs) ----------------------------------------------
constexpr int kTA = 3 * kMaxTableCols, kTB = kMaxTablePairs;  // phase A / B arrays

// The same totals with one warp per array: warp w sums arrays w, w + warps, ... over the block's
// slots (coalesced loads, shuffles, one pair of atomics per array and block; no block barrier per
// array group).  Used when many arrays are summed (the batched statistics).
template <class TermFn>
__device__ void warp_accumulate(TermFn term, int n, const Range& BR, double* accum) {
  const int warp = static_cast<int>(threadIdx.x >> 5), lane = static_cast<int>(threadIdx.x & 31);
  const int nw = static_cast<int>(blockDim.x >> 5);
  for (int k = warp; k < n; k += nw) {
    double sm = 0.0, ab = 0.0;
    for (unsigned i0 = BR.lo + lane; i0 < BR.hi; i0 += 8 * 32) {
      double t[8];  // eight slots' loads in flight per lane
#pragma unroll
      for (int u = 0; u < 8; ++u) t[u] = i0 + 32 * u < BR.hi ? term(k, i0 + 32 * u) : 0.0;
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        sm += t[u];
        ab += fabs(t[u]);
      }
    }
    for (int o = 16; o > 0; o >>= 1) {
      sm += __shfl_xor_sync(0xffffffffu, sm, o);
      ab += __shfl_xor_sync(0xffffffffu, ab, o);
    }
    if (lane == 0) {  // integer terms, checked bound: exact in any order
      atomicAdd(accum + 2 * k, sm);
      atomicAdd(accum + 2 * k + 1, ab);
    }
  }
}

// The same with NT arrays per group computed together (group g = arrays NT g .. NT g + NT - 1,
// term(g, i, t[NT])): one load serves the group's terms, NT sums in flight per warp.
template <int NT, class TermFn>
__device__ void warp_accumulate_groups(TermFn term, int ngroups, const Range& BR, double* accum) {
  const int warp = static_cast<int>(threadIdx.x >> 5), lane = static_cast<int>(threadIdx.x & 31);
  const int nw = static_cast<int>(blockDim.x >> 5);
  for (int g = warp; g < ngroups; g += nw) {
    double sm[NT], ab[NT];
#pragma unroll
    for (int k = 0; k < NT; ++k) sm[k] = ab[k] = 0.0;
    for (unsigned i0 = BR.lo + lane; i0 < BR.hi; i0 += 4 * 32) {
      double t[4][NT];  // four slots' loads in flight per lane
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        if (i0 + 32 * u < BR.hi) {
          term(g, i0 + 32 * u, t[u]);
        } else {
#pragma unroll
          for (int k = 0; k < NT; ++k) t[u][k] = 0.0;
        }
      }
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int k = 0; k < NT; ++k) {
          sm[k] += t[u][k];
          ab[k] += fabs(t[u][k]);
        }
    }
#pragma unroll
    for (int k = 0; k < NT; ++k)
      for (int o = 16; o > 0; o >>= 1) {
        sm[k] += __shfl_xor_sync(0xffffffffu, sm[k], o);
        ab[k] += __shfl_xor_sync(0xffffffffu, ab[k], o);
      }
    if (lane == 0)
#pragma unroll
      for (int k = 0; k < NT; ++k) {
        atomicAdd(accum + 2 * (NT * g + k), sm[k]);
        atomicAdd(accum + 2 * (NT * g + k) + 1, ab[k]);
      }
  }
}

// Grid barrier, then the totals of arrays [0, n) into tot[] (shared); false when a sum is not
// provably exact.  The last block to read zeroes the totals and its counter for the next launch.
__device__ bool table_totals(const GridBar& grid, double* accum, unsigned* count, int n, double* tot) {
  grid.sync();
  for (int k = threadIdx.x; k < 2 * n; k += blockDim.x) tot[k] = __ldcg(accum + k);
  __syncthreads();
  if (threadIdx.x == 0 && atomicAdd(count, 1u) == gridDim.x - 1) {
    for (int k = 0; k < 2 * n; ++k) accum[k] = 0.0;
    *count = 0u;
  }
  bool exact = true;
  for (int k = 0; k < n; ++k) exact = exact && tot[2 * k + 1] < 4503599627370496.0;  // 2^52
  return exact;
}

// The batched kernels (Pearson table, Z-score batch) have hundreds to thousands of (column, slot)
// items per block whatever P is: every lane count may run the largest block (64 registers per thread).
#ifndef HS_ZB_THREADS
#define HS_ZB_THREADS 1024
#endif
constexpr int kZbThreads = HS_ZB_THREADS;

template <class Q, int P>
__global__ void __launch_bounds__(kZbThreads, 1) k_ptable(Q q, const __grid_constant__ PTableArgs a,
                                                         const __grid_constant__ Prog pg) {
  extern __shared__ double stab[];
  __shared__ double totA[2 * kTA], totB[2 * kTB];
  double* accA = a.partial;
  double* accB = a.partial + 2 * kTA;
  unsigned* counts = reinterpret_cast<unsigned*>(a.partial + 2 * (kTA + kTB));
  const GridBar grid{counts + 2};
  const unsigned S = pg.S;
  const Range BR = block_range(S);
  for (int i = threadIdx.x; i < pg.ntab; i += blockDim.x) stab[i] = __ldg(pg.tabs + i);
  // ---- phase A: per column mean_scaled(B = 1) and variance_to_scale(B^2) terms ----
  const int NA = 3 * a.ncols;
  auto termA = [&](int k, unsigned i) -> double {
    const int c = k / 3, t = k - 3 * c;
    const double X = q.in(__ldg(a.x[c] + i));
    if (t == 0) return q.mulc(X, a.cm);                       // mul_pt(chunk, 1/(B n))
    if (t == 1) {
      const double sx = q.mulc(X, a.ca);                      // mul_pt(chunk, 1/sqrt(S n))
      return q.mul(sx, sx);                                   // mul_ct(a, a)
    }
    return q.mulc(X, a.cmp);                                  // mul_pt(chunk, 1/(n sqrt(S)))
  };
  warp_accumulate(termA, NA, BR, accA);
  if (!table_totals(grid, accA, counts, NA, totA)) {
    if (blockIdx.x == 0 && threadIdx.x == 0) *a.inexact = 1u;
    return;
  }
  // per-column mu, var (every slot holds the exact totals)
  auto mu = [&](int c) { return totA[2 * (3 * c)]; };
  auto var = [&](int c) {
    const double sq = totA[2 * (3 * c + 1)], mp = totA[2 * (3 * c + 2)];
    return q.sub(sq, q.mul(mp, mp));                          // sub_ct(sq_sum, mul_ct(mp, mp))
  };
  // ---- phase B: every pair's centred product, mean_of_chunks(1/n) ----
  auto termB = [&](int p, unsigned i) -> double {
    const int ci = a.pi[p], cj = a.pj[p];
    const double mi = mu(ci);
    const double mm = a.valid < S ? q.mulc(mi, i < a.valid ? 1.0 : 0.0) : mi;  // mul_pt(mu, mask)
    const double cx = q.sub(q.in(__ldg(a.x[ci] + i)), mm);
    const double cy = q.sub(q.in(__ldg(a.x[cj] + i)), mu(cj));
    return q.mulc(q.mul(cx, cy), a.inv_n);
  };
  warp_accumulate(termB, a.npairs, BR, accB);
  if (!table_totals(grid, accB, counts + 1, a.npairs, totB)) {
    if (blockIdx.x == 0 && threadIdx.x == 0) *a.inexact = 1u;
    return;
  }
  if (BR.lo >= BR.hi) return;
  // ---- phase C: the inverse square root of every column's variance, this block's slots ----
  const unsigned items = (BR.hi - BR.lo) * static_cast<unsigned>(a.ncols);
  const unsigned iters = (items * P + blockDim.x - 1) / blockDim.x;
  for (unsigned it = 0; it < iters; ++it) {
    const unsigned g = threadIdx.x + it * blockDim.x, item = g / P;
    const bool live = item < items;
    const unsigned it2 = live ? item : items - 1;
    const unsigned c = it2 / (BR.hi - BR.lo), s = BR.lo + it2 % (BR.hi - BR.lo);
    double sv[5] = {mu(static_cast<int>(c)), var(static_cast<int>(c)), 0.0, 0.0, 0.0};
    exec<Q, P, P == 1>(q, pg, stab, c * S + s, static_cast<int>(g % P), live, sv);
  }
  __syncthreads();  // the block's inverse roots (global, this block's slots) are visible to it
  // ---- phase D: pearson's epilogue per pair, mul_ct(mul_ct(cov, inv_x), inv_y) ----
  const double* inv = pg.out[0];
  const unsigned pitems = (BR.hi - BR.lo) * static_cast<unsigned>(a.npairs);
  for (unsigned g = threadIdx.x; g < pitems; g += blockDim.x) {
    const unsigned p = g / (BR.hi - BR.lo), s = BR.lo + g % (BR.hi - BR.lo);
    const double ix = q.in(__ldcg(inv + a.pi[p] * S + s)), iy = q.in(__ldcg(inv + a.pj[p] * S + s));
    a.out[p][s] = q.out(q.mul(q.mul(totB[2 * p], ix), iy));
  }
}

// ---- many independent Z-scores (kernels.h ZBatchArgs) ----------------------------------------
constexpr int kZA = 3 * kMaxZBatch;

template <class Q, int P>
__global__ void __launch_bounds__(kZbThreads, 1) k_zbatch(Q q, const __grid_constant__ ZBatchArgs a,
                                                         const __grid_constant__ Prog pg) {
  extern __shared__ double stab[];
  __shared__ double tot[2 * kZA];
  __shared__ unsigned char exact[kMaxZBatch];
  __shared__ int any_inexact;
  unsigned* counts = reinterpret_cast<unsigned*>(a.partial + 2 * kZA);
  const GridBar grid{counts + 1};
  const unsigned S = pg.S;
  const Range BR = block_range(S);
  stamp(0);
  for (int i = threadIdx.x; i < pg.ntab; i += blockDim.x) stab[i] = __ldg(pg.tabs + i);
  // ---- phase A: every column's moment terms (stats.hpp:41-51, 110-126) ----
  const int NA = 3 * a.ncols;
  auto termA = [&](int k, unsigned i) -> double {
    const int c = k / 3, t = k - 3 * c;
    const double X = q.in(__ldg(a.x[c] + i));
    if (t == 0) return q.mulc(X, a.cm[c]);                    // mul_pt(chunk, 1/(B n)), B = 1
    if (t == 1) {
      const double sx = q.mulc(X, a.ca[c]);                   // mul_pt(chunk, 1/sqrt(B^2 n))
      return q.mul(sx, sx);                                   // mul_ct(a, a)
    }
    return q.mulc(X, a.cmp[c]);                               // mul_pt(chunk, 1/(n sqrt(B^2)))
  };
  // the column's three terms from one load of each slot
  auto termCol = [&](int c, unsigned i, double (&t)[3]) {
    const double X = q.in(__ldg(a.x[c] + i));
    t[0] = q.mulc(X, a.cm[c]);
    const double sx = q.mulc(X, a.ca[c]);
    t[1] = q.mul(sx, sx);
    t[2] = q.mulc(X, a.cmp[c]);
  };
  warp_accumulate_groups<3>(termCol, a.ncols, BR, a.partial);
  stamp(1);
  table_totals(grid, a.partial, counts, NA, tot);
  // exact-sum per column (uniform across blocks: every block reads the same totals)
  if (threadIdx.x == 0) any_inexact = 0;
  __syncthreads();
  for (int c = threadIdx.x; c < a.ncols; c += blockDim.x) {
    bool e = true;
    for (int t = 0; t < 3; ++t) e = e && tot[2 * (3 * c + t) + 1] < 4503599627370496.0;  // 2^52
    exact[c] = e ? 1 : 0;
    if (!e) any_inexact = 1;
  }
  __syncthreads();
  // ---- a column with a sum beyond the exact bound: the literal butterfly (ckks.hpp:218-230) ----
  double* cur = a.scratch;
  if (any_inexact) {  // uniform
    double* nxt = a.scratch + size_t(NA) * S;
    for (int k = 0; k < NA; ++k)
      if (!exact[k / 3])
        for (unsigned i = BR.lo + threadIdx.x; i < BR.hi; i += blockDim.x) cur[size_t(k) * S + i] = termA(k, i);
    grid.sync();
    for (unsigned d = 1; d < S; d <<= 1) {
      for (int k = 0; k < NA; ++k)
        if (!exact[k / 3])
          for (unsigned i = BR.lo + threadIdx.x; i < BR.hi; i += blockDim.x)
            nxt[size_t(k) * S + i] = q.add(__ldcg(cur + size_t(k) * S + i), __ldcg(cur + size_t(k) * S + ((i + d) & (S - 1))));
      grid.sync();
      double* t = cur;
      cur = nxt;
      nxt = t;
    }
  }
  stamp(2);
  if (BR.lo >= BR.hi) return;
  // per (column, slot): the reduced array values (uniform totals, or the butterfly's slots)
  auto val = [&](int c, int t, unsigned s) {
    return exact[c] ? tot[2 * (3 * c + t)] : __ldcg(cur + size_t(3 * c + t) * S + s);
  };
  auto mu = [&](int c, unsigned s) { return val(c, 0, s); };
  auto var = [&](int c, unsigned s) {
    const double mp = val(c, 2, s);
    return q.sub(val(c, 1, s), q.mul(mp, mp));                // sub_ct(sq_sum, mul_ct(mp, mp))
  };
  // ---- phase C: crypto_invsqrt(var_k, B^2) for every column on this block's slots ----
  const unsigned w = BR.hi - BR.lo, items = w * static_cast<unsigned>(a.ncols);
  const unsigned iters = (items * P + blockDim.x - 1) / blockDim.x;
  for (unsigned it = 0; it < iters; ++it) {
    const unsigned g = threadIdx.x + it * blockDim.x, item = g / P;
    const bool live = item < items;
    const unsigned it2 = live ? item : items - 1;
    const unsigned c = it2 / w, s = BR.lo + it2 % w;
    double sv[5] = {mu(static_cast<int>(c), s), var(static_cast<int>(c), s), 0.0, 0.0, 0.0};
    exec<Q, P, P == 1>(q, pg, stab, c * S + s, static_cast<int>(g % P), live, sv);
  }
  __syncthreads();
  stamp(3);
  // ---- z = mul_ct(sub_ct(x, mu), inv) (stats.hpp:160-165) ----
  const double* inv = pg.out[0];
  for (unsigned g0 = threadIdx.x; g0 < items; g0 += 4 * blockDim.x) {  // four items' loads in flight
    double xv[4], iv[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const unsigned g = g0 + u * blockDim.x;
      if (g < items) {
        const unsigned c = g / w, s = BR.lo + g % w;
        iv[u] = __ldcg(inv + c * S + s);
        xv[u] = __ldg(a.x[c] + s);
      }
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const unsigned g = g0 + u * blockDim.x;
      if (g < items) {
        const unsigned c = g / w, s = BR.lo + g % w;
        a.z[c][s] = q.out(q.mul(q.sub(q.in(xv[u]), mu(static_cast<int>(c), s)), q.in(iv[u])));
      }
    }
  }
  stamp(4);
}

template <class F>
void with_q(QSpec qs, F&& f) {
  const double s = ldexp(1.0, qs.bits), inv = ldexp(1.0, -qs.bits);
  switch (qs.mode) {
    case QMode::None: f(QNone{}); break;
    case QMode::Grid: f(QGrid{s, inv}); break;
    default: fail(HS_E_ERROR, "stat kernels take QNone or QGrid only");
  }
}

// HS_COOP (default 1): launch through cudaLaunchCooperativeKernel, which guarantees the grid is
// co-resident even when other streams' kernels hold SMs; 0 = a plain launch (the occupancy
// check above still sizes the grid to fit).  The barrier is the same either way, and the two
// measured alike (device time and host enqueue).
bool coop_launch() {
  static const bool on = [] {
    const char* e = std::getenv("HS_COOP");
    return !e || std::atoi(e) != 0;
  }();
  return on;
}

std::mutex g_occ_mu;
std::unordered_map<const void*, std::unordered_map<size_t, int>> g_occ;

template <class K>
int max_blocks(K kern, size_t smem, int threads) {
  std::lock_guard<std::mutex> g(g_occ_mu);
  auto& m = g_occ[reinterpret_cast<const void*>(kern)];
  const size_t key = smem * 2048 + static_cast<size_t>(threads);
  auto it = m.find(key);
  if (it != m.end()) return it->second;
  if (smem > 48 * 1024)
    cuda_ok(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)),
            "stat smem attr");
  // same L1/shared carveout as k_encrypt, so an SM can host both at once
  cuda_ok(cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, carveout_pct()), "stat carveout");
  int per_sm = 0;
  cuda_ok(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, threads, smem), "stat occupancy");
  const int n = per_sm * Runtime::get().sm_count();
  m.emplace(key, n);
  return n;
}

}  // namespace

// two sets of 2 kNK totals, two block counters, the grid barrier's two words
size_t stat_partial_doubles() { return 4 * kNK + 2; }
// the table's 2 (kTA + kTB) totals, two block counters and its grid barrier word
size_t ptable_partial_doubles() { return 2 * (kTA + kTB) + 2; }

size_t zbatch_partial_doubles() { return 2 * kZA + 2; }

// The degree-511 table of the next k_zbatch launch into the constant bank (prog.cuh c_cheb511),
// stream-ordered (and captured as a copy node inside a graph capture).
void upload_const_table(const double* dev_table, cudaStream_t s) {
  cuda_ok(cudaMemcpyToSymbolAsync(c_cheb511, dev_table, 512 * sizeof(double), 0, cudaMemcpyDeviceToDevice, s),
          "constant table upload");
}

void run_zbatch(QSpec qs, const ZBatchArgs& a, const Prog& p, int lanes, cudaStream_t s) {
  if (p.S == 0 || a.ncols == 0) return;
  if (qs.mode != QMode::Grid) fail(HS_E_ERROR, "znorm batch: exact grid sums need quantize = true");
  const QGrid Q{ldexp(1.0, qs.bits), ldexp(1.0, -qs.bits)};
  const size_t smem = static_cast<size_t>(p.ntab) * sizeof(double);
  auto go = [&](auto kern, int P) {
    const int maxt = kZbThreads;
    Geo geo = prog_geometry(p.S, P, Runtime::get().sm_count(), maxt);
    {  // a block's items are its slots of EVERY column: size the block for them, not for one column
      const size_t spb = (p.S + geo.blocks - 1) / geo.blocks;
      const size_t want = ((spb * static_cast<size_t>(a.ncols) * P + 31) / 32) * 32;
      geo.threads = static_cast<unsigned>(std::min<size_t>(want, static_cast<size_t>(maxt)));
    }
    const int cap = max_blocks(kern, smem, static_cast<int>(geo.threads));
    if (cap < static_cast<int>(geo.blocks)) fail(HS_E_CUDA, "znorm batch kernel: grid not co-resident");
    QGrid qv = Q;
    ZBatchArgs av = a;
    Prog pv = p;
    void* args[] = {&qv, &av, &pv};
    cuda_ok(cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(kern), dim3(geo.blocks), dim3(geo.threads), args,
                                        smem, s),
            "znorm batch launch");
  };
  if (lanes == 4) go(k_zbatch<QGrid, 4>, 4);
  else if (lanes == 2) go(k_zbatch<QGrid, 2>, 2);
  else go(k_zbatch<QGrid, 1>, 1);
  Runtime::get().note_launch();
}

void run_ptable(QSpec qs, const PTableArgs& a, const Prog& p, int lanes, cudaStream_t s) {
  if (p.S == 0) return;
  if (qs.mode != QMode::Grid) fail(HS_E_ERROR, "pearson table: exact grid sums need quantize = true");
  const QGrid Q{ldexp(1.0, qs.bits), ldexp(1.0, -qs.bits)};
  const size_t smem = static_cast<size_t>(p.ntab) * sizeof(double);
  auto go = [&](auto kern, int P) {
    Geo geo = prog_geometry(p.S, P, Runtime::get().sm_count(), kZbThreads);
    {  // a block's program items are its slots of every column
      const size_t spb = (p.S + geo.blocks - 1) / geo.blocks;
      const size_t want = ((spb * static_cast<size_t>(a.ncols) * P + 31) / 32) * 32;
      geo.threads = static_cast<unsigned>(std::min<size_t>(want, static_cast<size_t>(kZbThreads)));
    }
    const int cap = max_blocks(kern, smem, static_cast<int>(geo.threads));
    if (cap < static_cast<int>(geo.blocks)) fail(HS_E_CUDA, "pearson table kernel: grid not co-resident");
    QGrid qv = Q;
    PTableArgs av = a;
    Prog pv = p;
    void* args[] = {&qv, &av, &pv};
    cuda_ok(cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(kern), dim3(geo.blocks), dim3(geo.threads), args,
                                        smem, s),
            "pearson table launch");
  };
  if (lanes == 4) go(k_ptable<QGrid, 4>, 4);
  else if (lanes == 2) go(k_ptable<QGrid, 2>, 2);
  else go(k_ptable<QGrid, 1>, 1);
  Runtime::get().note_launch();
}

void run_stat(QSpec qs, const StatArgs& a, const Prog& p, int lanes, cudaStream_t s) {
  if (p.S == 0) return;
  with_q(qs, [&](auto Q) {
    using QT = decltype(Q);
    const size_t smem = static_cast<size_t>(p.ntab) * sizeof(double);
    auto go = [&](auto kern, int P) {
      const int maxt = P == 1 ? prog_max_threads<1>() : (P == 2 ? prog_max_threads<2>() : prog_max_threads<4>());
      const Geo geo = prog_geometry(p.S, P, Runtime::get().sm_count(), maxt);
      const int cap = max_blocks(kern, smem, static_cast<int>(geo.threads));
      if (cap < static_cast<int>(geo.blocks)) fail(HS_E_CUDA, "stat kernel: grid not co-resident");
      const int grid = static_cast<int>(geo.blocks);
      QT qv = Q;
      StatArgs av = a;
      Prog pv = p;
      if (coop_launch()) {
        void* args[] = {&qv, &av, &pv};
        cuda_ok(cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(kern), dim3(grid), dim3(geo.threads), args,
                                            smem, s),
                "stat launch");
      } else {
        kern<<<grid, geo.threads, smem, s>>>(qv, av, pv);
        cuda_ok(cudaGetLastError(), "stat launch");
      }
    };
    if (lanes == 8) go(k_stat<QT, 8>, 8);
    else if (lanes == 4) go(k_stat<QT, 4>, 4);
    else if (lanes == 2) go(k_stat<QT, 2>, 2);
    else go(k_stat<QT, 1>, 1);
  });
  Runtime::get().note_launch();
}

}  // namespace k
}  // namespace hsg

#ifdef HS_STAT_TIMING
extern "C" void hs_debug_stat_times(unsigned long long* out) {
  cudaMemcpyFromSymbol(out, hsg::k::g_stat_t, sizeof(unsigned long long) * 8);
}
#endif
