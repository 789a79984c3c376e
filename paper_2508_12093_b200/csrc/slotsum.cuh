// slotsum.cuh — sum_all_slots as one kernel per ciphertext.
//
// Reference semantics (ckks.hpp:218-230): log2(S) steps of
//     acc <- q(acc + rotate(acc, 2^j))         (left rotation: acc[(i + 2^j) mod S])
// so slot i of the result is a balanced tree over the cyclic window starting at
// i.  We replay exactly those S*log2(S) additions (bit-exact in every quantize
// mode, no reassociation), but keep the whole ciphertext on chip: the S slots
// are split across a thread-block cluster of C CTAs (S/C slots each, double-
// buffered in shared memory), partners at distance >= S/C are read from the
// owning CTA's shared memory through DSMEM, and one cluster barrier separates
// steps.  HBM traffic is one read of the inputs and one write of the outputs.
//
// A prologue functor produces NA independent arrays per slot (e.g. the three
// moment terms of stats.hpp) and an epilogue consumes the NA replicated sums,
// so the statistics pipelines fuse their slot-wise producers/consumers into the
// reduction kernel.
#pragma once

#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include "core.h"

namespace hsg {
namespace cg = cooperative_groups;

constexpr int kSumThreads = 1024;
constexpr unsigned kSlotsPerCta = 4096;  // 32 KB per array per buffer
constexpr unsigned kMaxCluster = 16;     // 16 is non-portable on sm_100

template <class Q, int NA, class Pro, class Epi>
__global__ void __launch_bounds__(kSumThreads, 1)
    k_slotsum(Q q, Pro pro, Epi epi, unsigned S, unsigned L) {
  extern __shared__ double sm[];  // [2][NA][L]
  cg::cluster_group cl = cg::this_cluster();
  const unsigned rank = cl.block_rank();
  const unsigned b = blockIdx.y;
  const unsigned base = rank * L;
  double* buf0 = sm;
  double* buf1 = sm + NA * L;

  double part[2 * NA];  // per-thread sum and |sum| of each array (exact-sum test)
#pragma unroll
  for (int a = 0; a < 2 * NA; ++a) part[a] = 0.0;
  for (unsigned j = threadIdx.x; j < L; j += blockDim.x) {
    double v[NA];
    pro(b, base + j, v);
#pragma unroll
    for (int a = 0; a < NA; ++a) {
      buf0[a * L + j] = v[a];
      if constexpr (Q::kExactSum) {
        part[2 * a] += v[a];
        part[2 * a + 1] += fabs(v[a]);
      }
    }
  }

  if constexpr (Q::kExactSum) {
    // Grid units: every term is an integer.  If sum|A| < 2^52 (computed bound;
    // the true sum is then < 2^53), every partial sum of every rotate-and-add
    // window is an exactly representable integer, so all log2(S) additions are
    // exact and every slot of the reference's result equals the exact total,
    // whatever the order: reduce once and broadcast.  Otherwise fall through
    // to the literal butterfly below.
    __shared__ double red[32][2 * NA];
    __shared__ double tot[2 * NA];
#pragma unroll
    for (int a = 0; a < 2 * NA; ++a)
      for (int o = 16; o > 0; o >>= 1) part[a] += __shfl_xor_sync(0xffffffffu, part[a], o);
    if ((threadIdx.x & 31) == 0)
#pragma unroll
      for (int a = 0; a < 2 * NA; ++a) red[threadIdx.x >> 5][a] = part[a];
    __syncthreads();
    if (threadIdx.x < 2 * NA) {
      double acc = 0.0;
      for (unsigned w = 0; w < (blockDim.x + 31) / 32; ++w) acc += red[w][threadIdx.x];
      tot[threadIdx.x] = acc;
    }
    cl.sync();
    double all[2 * NA];
#pragma unroll
    for (int a = 0; a < 2 * NA; ++a) all[a] = 0.0;
    for (unsigned r = 0; r < cl.num_blocks(); ++r) {
      const double* t = cl.map_shared_rank(tot, r);
#pragma unroll
      for (int a = 0; a < 2 * NA; ++a) all[a] += t[a];
    }
    bool exact = true;
#pragma unroll
    for (int a = 0; a < NA; ++a) exact = exact && all[2 * a + 1] < 4503599627370496.0;  // 2^52
    if (exact) {
      double v[NA];
#pragma unroll
      for (int a = 0; a < NA; ++a) v[a] = all[2 * a];
      for (unsigned j = threadIdx.x; j < L; j += blockDim.x) epi(b, base + j, v);
      cl.sync();  // keep `tot` alive until every CTA has read it
      return;
    }
  }
  cl.sync();

  double* cur = buf0;
  double* nxt = buf1;
  for (unsigned d = 1; d < S; d <<= 1) {
    for (unsigned j = threadIdx.x; j < L; j += blockDim.x) {
      const unsigned p = (base + j + d) & (S - 1);
      const unsigned pr = p / L;
      const unsigned pj = p - pr * L;
      const double* src = pr == rank ? cur : cl.map_shared_rank(cur, pr);
#pragma unroll
      for (int a = 0; a < NA; ++a) nxt[a * L + j] = q.add(cur[a * L + j], src[a * L + pj]);
    }
    cl.sync();
    double* t = cur;
    cur = nxt;
    nxt = t;
  }

  for (unsigned j = threadIdx.x; j < L; j += blockDim.x) {
    double v[NA];
#pragma unroll
    for (int a = 0; a < NA; ++a) v[a] = cur[a * L + j];
    epi(b, base + j, v);
  }
}

// Cluster geometry for S slots and NA arrays; returns false when S is too large
// for one cluster (the caller then uses the multi-launch fallback).
inline bool slotsum_geometry(size_t S, int NA, unsigned* C, unsigned* L) {
  unsigned c = 1;
  size_t l = S;
  while (l > kSlotsPerCta && c < kMaxCluster) {
    c *= 2;
    l /= 2;
  }
  const size_t smem = 2ull * NA * l * sizeof(double);
  if (smem > 227ull * 1024) return false;
  *C = c;
  *L = static_cast<unsigned>(l);
  return true;
}

template <class Q, int NA, class Pro, class Epi>
void launch_slotsum(Q q, Pro pro, Epi epi, size_t S, int batch, cudaStream_t s) {
  unsigned C = 1, L = 1;
  if (!slotsum_geometry(S, NA, &C, &L)) fail(HS_E_CUDA, "slot_sum: slot count too large for one cluster");
  auto kern = k_slotsum<Q, NA, Pro, Epi>;
  const size_t smem = 2ull * NA * L * sizeof(double);
  cuda_ok(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)),
          "slotsum smem attr");
  if (C > 8)
    cuda_ok(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1),
            "slotsum cluster attr");
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(C, static_cast<unsigned>(batch), 1);
  cfg.blockDim = dim3(L < kSumThreads ? ((L + 31) / 32) * 32 : kSumThreads, 1, 1);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = C;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cuda_ok(cudaLaunchKernelEx(&cfg, kern, q, pro, epi, static_cast<unsigned>(S), L), "slotsum launch");
  Runtime::get().note_launch();
}

}  // namespace hsg
