// ntt_cluster.cuh — single-pass NTT: one thread-block cluster of 8 CTAs owns a limb.
//
// The limb is viewed as an R1 x C matrix (element r*C + c).  The two-pass kernels
// (rns.cu k_ntt_pass) read and write the whole limb in HBM twice; here the limb
// goes HBM -> shared memory once:
//
//   forward  phase 1: CTA k transforms columns [k C/8, (k+1) C/8) (the first
//                     log2 R1 stages, twiddle index m + i, loaded straight from HBM);
//            exchange: after a cluster barrier CTA k gathers rows [k R1/8, ...) of
//                     every CTA's column slab through distributed shared memory into
//                     registers, and after a second barrier rewrites its own slab
//                     (one slab per CTA: 64 KiB at N = 2^16, two CTAs per SM);
//            phase 2: the remaining log2 C stages on its rows (twiddle index
//                     m (R1 + row) + i) and stores the rows to HBM.
//   inverse  the mirror image (rows first, columns last, times N^-1).
//
// Both arithmetic paths of rns.cu are supported through a small trait (IntA: 64-bit
// Shoup, lazy [0, 4q); FpA: exact integers in fp64 registers for q < 2^45).  Radix-8
// register groups as in the two-pass kernels; row slabs use the same XOR swizzle.
#pragma once

#include <cooperative_groups.h>

namespace hsg {
namespace rns {
namespace {

namespace cg = cooperative_groups;

constexpr int kCl = 8;  // CTAs per cluster (portable maximum)

template <int LOGN>
struct CGeom {
  static constexpr uint32_t logR1 = LOGN / 2, logC = LOGN - logR1;
  static constexpr uint32_t logCPC = logC - 3;  // columns per CTA
  static constexpr uint32_t logRPC = logR1 - 3; // rows per CTA
  static constexpr uint32_t logSlab = LOGN - 3; // elements per CTA
  static constexpr int threads = (1 << (logSlab - 3)) < 512 ? (1 << (logSlab - 3)) : 512;
  static constexpr int per = (1 << logSlab) / threads;  // exchange elements per thread
};

struct IntA {
  using T = uint64_t;
  using TwT = uint64_t;
  struct Tw {
    uint64_t w, wp;
  };
  uint64_t q, q2, ninv, ninv_sh;
  __device__ explicit IntA(const PrimeC& P) : q(P.q), q2(2 * P.q), ninv(P.ninv), ninv_sh(P.ninv_sh) {}
  __device__ T from(uint64_t v) const { return v; }
  __device__ static Tw tw(const TwT* b, uint32_t N, uint32_t i) { return {__ldg(b + i), __ldg(b + N + i)}; }
  __device__ void fwd(T& x, T& y, Tw t) const {
    const uint64_t X = x >= q2 ? x - q2 : x;
    const uint64_t Tt = mul_shoup_lazy(y, t.w, t.wp, q);
    x = X + Tt;
    y = X - Tt + q2;
  }
  __device__ void inv(T& x, T& y, Tw t) const {
    const uint64_t X = x, Y = y, s = X + Y;
    x = s >= q2 ? s - q2 : s;
    y = mul_shoup_lazy(X - Y + q2, t.w, t.wp, q);
  }
  __device__ void fold(T&) const {}
  __device__ uint64_t out_fwd(T v) const {
    v = v >= q2 ? v - q2 : v;
    return v >= q ? v - q : v;
  }
  __device__ uint64_t out_inv(T v) const { return mul_shoup(v, ninv, ninv_sh, q); }
};

struct FpA {
  using T = double;
  using TwT = double;
  struct Tw {
    double w;
  };
  double q, qinv, ninv;
  __device__ explicit FpA(const PrimeC& P) : q(P.qd), qinv(P.qinvd), ninv(static_cast<double>(P.ninv)) {}
  __device__ T from(uint64_t v) const { return u2d(v); }
  __device__ static Tw tw(const TwT* b, uint32_t, uint32_t i) { return {__ldg(b + i)}; }
  __device__ void fwd(T& x, T& y, Tw t) const {
    const double Tt = fp_mulmod(y, t.w, q, qinv), X = x;
    x = __dadd_rn(X, Tt);
    y = __dadd_rn(X, -Tt);
  }
  __device__ void inv(T& x, T& y, Tw t) const {
    const double X = x, Y = y;
    x = __dadd_rn(X, Y);
    y = fp_mulmod(__dadd_rn(X, -Y), t.w, q, qinv);
  }
  __device__ void fold(T& v) const { v = fp_fold(v, q, qinv); }
  __device__ uint64_t out_fwd(T v) const { return fp_canon(v, q, qinv); }
  __device__ uint64_t out_inv(T v) const { return fp_canon(fp_mulmod(v, ninv, q, qinv), q, qinv); }
};

// One radix-2^RB step over the CTA's slab.  ROWS: transforms are rows (slab [T][C],
// swizzled, twiddle multiplier R1 + row); else columns (slab [R1][T], multiplier 1).
// SRCG: the step reads HBM (global limb `g`); DSTG: it writes HBM.
template <class A, bool INV, bool ROWS, int LOGN, int RB, int DONE, bool SRCG, bool DSTG>
__device__ __forceinline__ void cstep(const A& ar, typename A::T* __restrict__ sm, const uint64_t* __restrict__ gin,
                                      uint64_t* __restrict__ gout, const typename A::TwT* __restrict__ tw,
                                      uint32_t t0) {
  using G = CGeom<LOGN>;
  constexpr uint32_t N = 1u << LOGN, R1 = 1u << G::logR1, logC = G::logC;
  constexpr uint32_t logR = ROWS ? G::logC : G::logR1;       // transform length
  constexpr uint32_t logT = ROWS ? G::logRPC : G::logCPC;    // transforms per CTA
  constexpr uint32_t logG = logR - RB;
  constexpr uint32_t total = 1u << (logG + logT);
  constexpr int NT = G::threads;
  constexpr uint32_t logs = INV ? DONE : logR - 1 - DONE - (RB - 1);
  using T = typename A::T;
#pragma unroll
  for (uint32_t it = 0; it < (total + NT - 1) / NT; ++it) {
    const uint32_t idx = threadIdx.x + it * NT;
    if (total % NT != 0 && idx >= total) break;
    uint32_t tr, g;
    if (ROWS) {
      g = idx & ((1u << logG) - 1);
      tr = idx >> logG;
    } else {
      tr = idx & ((1u << logT) - 1);
      g = idx >> logT;
    }
    const uint32_t blk0 = g >> logs;
    const uint32_t j0 = (blk0 << (logs + RB)) | (g & ((1u << logs) - 1));
    const uint32_t S = ROWS ? R1 + t0 + tr : 1u;
    T x[1 << RB];
#pragma unroll
    for (int k = 0; k < (1 << RB); ++k) {
      const uint32_t e = j0 + (uint32_t(k) << logs);
      if (SRCG)
        x[k] = ar.from(ROWS ? gin[(size_t(t0 + tr) << logC) + e] : gin[(size_t(e) << logC) + t0 + tr]);
      else
        x[k] = ROWS ? sm[swz((tr << logR) + e)] : sm[(e << logT) + tr];
    }
    if (!INV) {
#pragma unroll
      for (int st = 0; st < RB; ++st) {
        const int d = 1 << (RB - 1 - st);
#pragma unroll
        for (int b = 0; b < (1 << st); ++b) {
          const typename A::Tw w = A::tw(tw, N, ((1u << (DONE + st)) * S) + (blk0 << st) + b);
#pragma unroll
          for (int o = 0; o < d; ++o) ar.fwd(x[b * 2 * d + o], x[b * 2 * d + o + d], w);
        }
      }
    } else {
      constexpr uint32_t logh0 = logR - 1 - DONE;
#pragma unroll
      for (int st = 0; st < RB; ++st) {
        const int d = 1 << st;
#pragma unroll
        for (int b = 0; b < (1 << (RB - 1 - st)); ++b) {
          const typename A::Tw w = A::tw(tw, N, ((1u << (logh0 - st)) * S) + (blk0 << (RB - 1 - st)) + b);
#pragma unroll
          for (int o = 0; o < d; ++o) ar.inv(x[b * 2 * d + o], x[b * 2 * d + o + d], w);
        }
      }
#pragma unroll
      for (int k = 0; k < (1 << RB); ++k) ar.fold(x[k]);
    }
#pragma unroll
    for (int k = 0; k < (1 << RB); ++k) {
      const uint32_t e = j0 + (uint32_t(k) << logs);
      if (DSTG) {
        const uint64_t v = INV ? ar.out_inv(x[k]) : ar.out_fwd(x[k]);
        if (ROWS)
          gout[(size_t(t0 + tr) << logC) + e] = v;
        else
          gout[(size_t(e) << logC) + t0 + tr] = v;
      } else {
        if (ROWS)
          sm[swz((tr << logR) + e)] = x[k];
        else
          sm[(e << logT) + tr] = x[k];
      }
    }
  }
}

template <class A, bool INV, bool ROWS, int LOGN, int DONE, bool SRCG, bool DSTG>
__device__ __forceinline__ void csteps(const A& ar, typename A::T* sm, const uint64_t* gin, uint64_t* gout,
                                       const typename A::TwT* tw, uint32_t t0) {
  constexpr int logR = ROWS ? CGeom<LOGN>::logC : CGeom<LOGN>::logR1;
  if constexpr (DONE < logR) {
    constexpr int rem = logR - DONE;
    constexpr int RB = rem == 4 ? 2 : (rem < 3 ? rem : 3);
    if constexpr (DONE > 0) __syncthreads();
    cstep<A, INV, ROWS, LOGN, RB, DONE, SRCG && DONE == 0, DSTG && DONE + RB == logR>(ar, sm, gin, gout, tw, t0);
    csteps<A, INV, ROWS, LOGN, DONE + RB, SRCG, DSTG>(ar, sm, gin, gout, tw, t0);
  }
}

template <class A, bool INV, int LOGN>
__device__ __forceinline__ void ntt_cluster_body(const A& ar, const uint64_t* gin, uint64_t* gout,
                                                 const typename A::TwT* tw, unsigned char* smraw) {
  using G = CGeom<LOGN>;
  using T = typename A::T;
  constexpr uint32_t C = 1u << G::logC, CPC = 1u << G::logCPC, RPC = 1u << G::logRPC;
  constexpr int NT = G::threads, PER = G::per;
  T* sm = reinterpret_cast<T*>(smraw);  // one slab: column layout [R1][CPC] or row layout [RPC][C]
  cg::cluster_group cl = cg::this_cluster();
  const uint32_t k = cl.block_rank();
  T v[PER];
  if (!INV) {
    csteps<A, false, false, LOGN, 0, true, false>(ar, sm, gin, gout, tw, k * CPC);
    cl.sync();  // every column slab complete and visible
#pragma unroll
    for (int i = 0; i < PER; ++i) {  // rows k*RPC.. of every CTA's column slab, into registers
      const uint32_t idx = threadIdx.x + i * NT, t = idx >> G::logC, c = idx & (C - 1);
      const T* rem = cl.map_shared_rank(sm, c >> G::logCPC);
      v[i] = rem[((k * RPC + t) << G::logCPC) + (c & (CPC - 1))];
    }
    cl.sync();  // every remote read done: slabs may be overwritten
#pragma unroll
    for (int i = 0; i < PER; ++i) sm[swz(threadIdx.x + i * NT)] = v[i];
    __syncthreads();
    csteps<A, false, true, LOGN, 0, false, true>(ar, sm, gin, gout, tw, k * RPC);
  } else {
    csteps<A, true, true, LOGN, 0, true, false>(ar, sm, gin, gout, tw, k * RPC);
    cl.sync();
#pragma unroll
    for (int i = 0; i < PER; ++i) {  // columns k*CPC.. of every CTA's row slab
      const uint32_t idx = threadIdx.x + i * NT, r = idx >> G::logCPC, c = idx & (CPC - 1);
      const T* rem = cl.map_shared_rank(sm, r >> G::logRPC);
      v[i] = rem[swz(((r & (RPC - 1)) << G::logC) + k * CPC + c)];
    }
    cl.sync();
#pragma unroll
    for (int i = 0; i < PER; ++i) sm[threadIdx.x + i * NT] = v[i];
    __syncthreads();
    csteps<A, true, false, LOGN, 0, false, true>(ar, sm, gin, gout, tw, k * CPC);
  }
}

// grid (8, rows, batch), cluster (8, 1, 1): one cluster per (row, batch item)
template <bool INV, int LOGN>
__global__ void __launch_bounds__(CGeom<LOGN>::threads, 2)
    k_ntt_cluster(const uint64_t* in, size_t in_stride, uint64_t* out, size_t out_stride,
                  const __grid_constant__ RowMap rm, const PrimeC* pcs, const uint64_t* tw, const double* twd) {
  extern __shared__ __align__(16) unsigned char smraw[];
  constexpr uint32_t N = 1u << LOGN;
  const uint32_t pi = rm.prime[blockIdx.y];
  const PrimeC& P = pcs[pi];
  const uint64_t* gi = in + blockIdx.z * in_stride + (size_t(rm.irow[blockIdx.y]) << LOGN);
  uint64_t* go = out + blockIdx.z * out_stride + (size_t(rm.orow[blockIdx.y]) << LOGN);
  if (P.fp) {
    const double* t = twd + size_t(pi) * 2 * N + (INV ? N : 0);
    ntt_cluster_body<FpA, INV, LOGN>(FpA(P), gi, go, t, smraw);
  } else {
    const uint64_t* t = tw + size_t(pi) * 4 * N + (INV ? 2 * N : 0);
    ntt_cluster_body<IntA, INV, LOGN>(IntA(P), gi, go, t, smraw);
  }
}

template <int LOGN>
void launch_ntt_cluster(const uint64_t* in, size_t in_stride, uint64_t* out, size_t out_stride, const RowMap& rm,
                        uint32_t n, uint32_t batch, bool inverse, const PrimeC* pcs, const uint64_t* tw,
                        const double* twd, cudaStream_t s) {
  using G = CGeom<LOGN>;
  const size_t smem = size_t(1) << (G::logSlab + 3);  // one slab of 8-byte words
  auto kern = inverse ? k_ntt_cluster<true, LOGN> : k_ntt_cluster<false, LOGN>;
  static bool attr_set[2] = {false, false};
  if (!attr_set[inverse]) {
    cuda_ok(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)),
            "cluster ntt smem");
    attr_set[inverse] = true;
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(kCl, n, batch);
  cfg.blockDim = dim3(G::threads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = kCl;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cuda_ok(cudaLaunchKernelEx(&cfg, kern, in, in_stride, out, out_stride, rm, pcs, tw, twd), "cluster ntt launch");
}

}  // namespace
}  // namespace rns
}  // namespace hsg
