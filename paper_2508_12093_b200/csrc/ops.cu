// ops.cu — E1-E5: the EvalContext slot-wise ops as HBM-streaming kernels.
//
//   binary   add_ct / sub_ct / mul_ct               ckks.hpp:113-164   24 B/slot
//   scalar   add_pt / mul_pt(scalar)                ckks.hpp:137-176   16 B/slot
//   binary   mul_pt(vector) == B_MUL with p         ckks.hpp:179-189   24 B/slot
//   rotate   left cyclic shift (no quantisation)    ckks.hpp:193-202   16 B/slot
//   requant  bootstrap / encrypt quantisation       ckks.hpp:207-213   16 B/slot
//   slot_sum sum_all_slots (slotsum.cuh)            ckks.hpp:218-230   16 B/slot
//
// Streaming kernels use 16-byte vector accesses and a grid of a few CTAs per
// SM with a grid-stride loop; each is bandwidth-bound (<= 0.17 flop/B).
#include <algorithm>
#include <vector>

#include "core.h"
#include "kernels.h"
#include "quant.cuh"
#include "slotsum.cuh"

namespace hsg {
namespace k {
namespace {

constexpr int kThreads = 256;
constexpr int kBatch = 64;  // ciphertexts per batched launch (pointer table passed by value)

inline unsigned grid_for(size_t n_items) {
  const size_t want = (n_items + kThreads - 1) / kThreads;
  const size_t cap = static_cast<size_t>(Runtime::get().sm_count()) * 8;
  return static_cast<unsigned>(want < 1 ? 1 : (want > cap ? cap : want));
}

template <class Q, int OP>
__device__ __forceinline__ double bin(const Q& q, double x, double y) {
  if constexpr (OP == B_ADD) return q.add(x, y);
  else if constexpr (OP == B_SUB) return q.sub(x, y);
  else return q.mul(x, y);
}

template <class Q, int OP>
__global__ void __launch_bounds__(kThreads) k_binary(Q q, const double* __restrict__ a,
                                                      const double* __restrict__ b,
                                                      double* __restrict__ o, size_t n) {
  const size_t n2 = n / 2;
  const size_t stride = static_cast<size_t>(gridDim.x) * blockDim.x;
  const double2* a2 = reinterpret_cast<const double2*>(a);
  const double2* b2 = reinterpret_cast<const double2*>(b);
  double2* o2 = reinterpret_cast<double2*>(o);
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n2; i += stride) {
    const double2 x = __ldg(a2 + i), y = __ldg(b2 + i);
    o2[i] = make_double2(bin<Q, OP>(q, x.x, y.x), bin<Q, OP>(q, x.y, y.y));
  }
  if ((n & 1) && blockIdx.x == 0 && threadIdx.x == 0) o[n - 1] = bin<Q, OP>(q, a[n - 1], b[n - 1]);
}

template <class Q, int OP>
__global__ void __launch_bounds__(kThreads) k_scalar(Q q, const double* __restrict__ a, double c,
                                                      double* __restrict__ o, size_t n) {
  const size_t n2 = n / 2;
  const size_t stride = static_cast<size_t>(gridDim.x) * blockDim.x;
  const double2* a2 = reinterpret_cast<const double2*>(a);
  double2* o2 = reinterpret_cast<double2*>(o);
  auto f = [&](double x) { return OP == S_ADD ? q.addc(x, c) : q.mulc(x, c); };
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n2; i += stride) {
    const double2 x = __ldg(a2 + i);
    o2[i] = make_double2(f(x.x), f(x.y));
  }
  if ((n & 1) && blockIdx.x == 0 && threadIdx.x == 0) o[n - 1] = f(a[n - 1]);
}

template <class Q>
__global__ void __launch_bounds__(kThreads) k_requant(Q q, const double* __restrict__ a,
                                                       double* __restrict__ o, size_t n) {
  const size_t stride = static_cast<size_t>(gridDim.x) * blockDim.x;
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n; i += stride)
    o[i] = q.req(a[i]);
}

// encrypt (ckks.hpp:97-104): zero-pad to S, quantise, flag non-finite inputs.  `src`
// may be host memory mapped into the device (zero-copy over PCIe): two slots per
// thread with 16-byte reads when `src` is 16-byte aligned, so each PCIe read carries
// more payload.
// Small blocks (64 threads, <= 32 registers): they fit in the register file a running
// statistics kernel leaves free on every SM sub-partition (k_stat: 448 threads x 120
// registers), so encode_column on the upload stream overlaps the compute stream instead
// of queueing behind it.
constexpr int kEncThreads = 64;
template <class Q, bool VEC>
__global__ void __launch_bounds__(kEncThreads, 32) k_encrypt(Q q, const double* __restrict__ src, size_t n,
                                                       double* __restrict__ o, size_t S, int* bad) {
  const size_t stride = static_cast<size_t>(gridDim.x) * blockDim.x;
  bool nf = false;
  if (VEC) {
    double2* o2 = reinterpret_cast<double2*>(o);
    for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < S / 2; i += stride) {
      double2 v = make_double2(0.0, 0.0);
      if (2 * i + 1 < n) {
        v = *reinterpret_cast<const double2*>(src + 2 * i);
      } else if (2 * i < n) {
        v.x = src[2 * i];
      }
      nf = nf || !isfinite(v.x) || !isfinite(v.y);
      o2[i] = make_double2(q.req(v.x), q.req(v.y));
    }
    if ((S & 1) && blockIdx.x == 0 && threadIdx.x == 0) {
      const double v = S - 1 < n ? src[S - 1] : 0.0;
      nf = nf || !isfinite(v);
      o[S - 1] = q.req(v);
    }
  } else {
    for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < S; i += stride) {
      double v = 0.0;
      if (i < n) {
        v = src[i];
        nf = nf || !isfinite(v);
      }
      o[i] = q.req(v);
    }
  }
  if (bad && __any_sync(0xffffffffu, nf) && (threadIdx.x & 31) == 0) atomicOr(bad, 1);
}

__global__ void __launch_bounds__(kThreads) k_rotate(const double* __restrict__ a, double* __restrict__ o,
                                                      size_t n, size_t shift) {
  const size_t mask = n - 1;  // n is a power of two
  const size_t stride = static_cast<size_t>(gridDim.x) * blockDim.x;
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n; i += stride)
    o[i] = __ldg(a + ((i + shift) & mask));
}

// one step of the multi-launch fallback of sum_all_slots (S beyond one cluster)
template <class Q>
__global__ void __launch_bounds__(kThreads) k_sum_step(Q q, const double* __restrict__ a,
                                                        double* __restrict__ o, size_t n, size_t d) {
  const size_t mask = n - 1;
  const size_t stride = static_cast<size_t>(gridDim.x) * blockDim.x;
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n; i += stride)
    o[i] = q.add(a[i], a[(i + d) & mask]);
}

// ---- batched forms (C5): blockIdx.y = ciphertext of the batch, pointers by value ----
struct BatchPtrs {
  const double* a[kBatch];
  const double* b[kBatch];
  double* o[kBatch];
};

template <class Q, int OP>
__global__ void __launch_bounds__(kThreads) k_binary_batch(Q q, const __grid_constant__ BatchPtrs p, size_t n) {
  const unsigned e = blockIdx.y;
  const size_t n2 = n / 2, stride = static_cast<size_t>(gridDim.x) * blockDim.x;
  const double2* a2 = reinterpret_cast<const double2*>(p.a[e]);
  const double2* b2 = reinterpret_cast<const double2*>(p.b[e]);
  double2* o2 = reinterpret_cast<double2*>(p.o[e]);
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n2; i += stride) {
    const double2 x = __ldg(a2 + i), y = __ldg(b2 + i);
    o2[i] = make_double2(bin<Q, OP>(q, x.x, y.x), bin<Q, OP>(q, x.y, y.y));
  }
  if ((n & 1) && blockIdx.x == 0 && threadIdx.x == 0) p.o[e][n - 1] = bin<Q, OP>(q, p.a[e][n - 1], p.b[e][n - 1]);
}

template <class Q, int OP>
__global__ void __launch_bounds__(kThreads) k_scalar_batch(Q q, const __grid_constant__ BatchPtrs p, double c,
                                                            size_t n) {
  const unsigned e = blockIdx.y;
  const size_t n2 = n / 2, stride = static_cast<size_t>(gridDim.x) * blockDim.x;
  const double2* a2 = reinterpret_cast<const double2*>(p.a[e]);
  double2* o2 = reinterpret_cast<double2*>(p.o[e]);
  auto f = [&](double x) { return OP == S_ADD ? q.addc(x, c) : q.mulc(x, c); };
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n2; i += stride) {
    const double2 x = __ldg(a2 + i);
    o2[i] = make_double2(f(x.x), f(x.y));
  }
  if ((n & 1) && blockIdx.x == 0 && threadIdx.x == 0) p.o[e][n - 1] = f(p.a[e][n - 1]);
}

// out[i] = a[(i + shift) mod n], two slots per thread with 16-byte loads: an even shift
// is an aligned double2 read; an odd one reads the aligned pair ending at i+shift and
// takes the next slot from the neighbouring lane (shuffle); lane 31 and the last live
// lane read it from memory.
__global__ void __launch_bounds__(kThreads) k_rotate_batch(const __grid_constant__ BatchPtrs p, size_t n,
                                                            size_t shift) {
  const unsigned e = blockIdx.y;
  const size_t mask = n - 1, n2 = n / 2, stride = static_cast<size_t>(gridDim.x) * blockDim.x;
  const double* a = p.a[e];
  double2* o2 = reinterpret_cast<double2*>(p.o[e]);
  const bool odd = shift & 1;
  const unsigned lane = threadIdx.x & 31;
  // grid-stride loop with a warp-uniform trip count so the shuffle sees full warps
  for (size_t base = blockIdx.x * static_cast<size_t>(blockDim.x); base < n2; base += stride) {
    const size_t i = base + threadIdx.x;
    const bool live = i < n2;
    const size_t j = (2 * i + shift - (odd ? 1 : 0)) & mask;  // even index
    double2 v = live ? __ldg(reinterpret_cast<const double2*>(a + j)) : make_double2(0.0, 0.0);
    if (!odd) {
      if (live) o2[i] = v;
      continue;
    }
    double nx = __shfl_down_sync(0xffffffffu, v.x, 1);
    if ((lane == 31 || i + 1 >= n2) && live) nx = __ldg(a + ((j + 2) & mask));
    if (live) o2[i] = make_double2(v.y, nx);
  }
}

// x-blocks per ciphertext: ~8 grid-stride iterations per thread, at least one wave over the batch
inline unsigned batch_gx(size_t items, size_t count) {
  const size_t per = (items + kThreads * 8 - 1) / (kThreads * 8);
  const size_t wave = (static_cast<size_t>(Runtime::get().sm_count()) * 8 + count - 1) / count;
  return static_cast<unsigned>(std::max<size_t>(1, std::max(per, std::min(wave, (items + kThreads - 1) / kThreads))));
}

template <class F>
void with_q(QSpec qs, F&& f) {
  const double s = ldexp(1.0, qs.bits), inv = ldexp(1.0, -qs.bits);
  switch (qs.mode) {
    case QMode::None: f(QNone{}); break;
    case QMode::Exact: f(QExact{s, inv}); break;
    case QMode::Grid: f(QGrid{s, inv}); break;
  }
}

constexpr int kSumBatch = 8;
struct PtrPro {
  const double* a[kSumBatch];
  template <int NA>
  __device__ void operator()(unsigned b, unsigned i, double (&v)[NA]) const { v[0] = a[b][i]; }
};
struct PtrEpi {
  double* o[kSumBatch];
  template <int NA>
  __device__ void operator()(unsigned b, unsigned i, const double (&v)[NA]) const { o[b][i] = v[0]; }
};

}  // namespace

void binary(QSpec q, BinOp op, const double* a, const double* b, double* out, size_t n, cudaStream_t s) {
  if (n == 0) return;
  with_q(q, [&](auto Q) {
    using QT = decltype(Q);
    const unsigned g = grid_for((n + 1) / 2);
    if (op == B_ADD) k_binary<QT, B_ADD><<<g, kThreads, 0, s>>>(Q, a, b, out, n);
    else if (op == B_SUB) k_binary<QT, B_SUB><<<g, kThreads, 0, s>>>(Q, a, b, out, n);
    else k_binary<QT, B_MUL><<<g, kThreads, 0, s>>>(Q, a, b, out, n);
  });
  cuda_ok(cudaGetLastError(), "binary launch");
  Runtime::get().note_launch();
}

void scalar(QSpec q, ScalOp op, const double* a, double c, double* out, size_t n, cudaStream_t s) {
  if (n == 0) return;
  with_q(q, [&](auto Q) {
    using QT = decltype(Q);
    const unsigned g = grid_for((n + 1) / 2);
    if (op == S_ADD) k_scalar<QT, S_ADD><<<g, kThreads, 0, s>>>(Q, a, c, out, n);
    else k_scalar<QT, S_MUL><<<g, kThreads, 0, s>>>(Q, a, c, out, n);
  });
  cuda_ok(cudaGetLastError(), "scalar launch");
  Runtime::get().note_launch();
}

void requant(QSpec q, const double* a, double* out, size_t n, cudaStream_t s) {
  if (n == 0) return;
  with_q(q, [&](auto Q) { k_requant<<<grid_for(n), kThreads, 0, s>>>(Q, a, out, n); });
  cuda_ok(cudaGetLastError(), "requant launch");
  Runtime::get().note_launch();
}

inline unsigned enc_grid(size_t n_items) {
  const size_t want = (n_items + kEncThreads - 1) / kEncThreads;
  const size_t cap = static_cast<size_t>(Runtime::get().sm_count()) * 16;
  return static_cast<unsigned>(want < 1 ? 1 : (want > cap ? cap : want));
}

void encrypt(QSpec q, const double* src, size_t n, double* out, size_t S, int* bad, cudaStream_t s) {
  if (S == 0) return;
  const bool vec = (reinterpret_cast<uintptr_t>(src) & 15) == 0;
  static const bool attr = [] {  // same carveout as the statistics kernels (stat.cu): SMs are shared
    for (const void* f : {reinterpret_cast<const void*>(k_encrypt<QGrid, true>),
                          reinterpret_cast<const void*>(k_encrypt<QGrid, false>),
                          reinterpret_cast<const void*>(k_encrypt<QExact, true>),
                          reinterpret_cast<const void*>(k_encrypt<QExact, false>),
                          reinterpret_cast<const void*>(k_encrypt<QNone, true>),
                          reinterpret_cast<const void*>(k_encrypt<QNone, false>)})
      cuda_ok(cudaFuncSetAttribute(f, cudaFuncAttributePreferredSharedMemoryCarveout, carveout_pct()), "encrypt carveout");
    return true;
  }();
  (void)attr;
  with_q(q, [&](auto Q) {
    if (vec)
      k_encrypt<decltype(Q), true><<<enc_grid((S + 1) / 2), kEncThreads, 0, s>>>(Q, src, n, out, S, bad);
    else
      k_encrypt<decltype(Q), false><<<enc_grid(S), kEncThreads, 0, s>>>(Q, src, n, out, S, bad);
  });
  cuda_ok(cudaGetLastError(), "encrypt launch");
  Runtime::get().note_launch();
}

void rotate(const double* a, double* out, size_t n, size_t shift, cudaStream_t s) {
  if (n == 0) return;
  k_rotate<<<grid_for(n), kThreads, 0, s>>>(a, out, n, shift);
  cuda_ok(cudaGetLastError(), "rotate launch");
  Runtime::get().note_launch();
}

size_t slot_sum_max(int arrays) {
  size_t S = 1;
  unsigned C, L;
  while (slotsum_geometry(S * 2, arrays, &C, &L) && S < (size_t(1) << 30)) S *= 2;
  return S;
}

void slot_sum(QSpec q, const double* const* a, double* const* out, int batch, size_t S, cudaStream_t s) {
  if (S == 0 || batch == 0) return;
  Runtime& rt = Runtime::get();
  unsigned C, L;
  if (slotsum_geometry(S, 1, &C, &L)) {
    for (int b0 = 0; b0 < batch; b0 += kSumBatch) {
      const int nb = std::min(kSumBatch, batch - b0);
      PtrPro pro{};
      PtrEpi epi{};
      for (int i = 0; i < nb; ++i) {
        pro.a[i] = a[b0 + i];
        epi.o[i] = out[b0 + i];
      }
      with_q(q, [&](auto Q) { launch_slotsum<decltype(Q), 1>(Q, pro, epi, S, nb, s); });
    }
    return;
  }
  // multi-launch fallback: log2(S) global-memory steps (ping-pong)
  DevBuf tmp = rt.alloc(S);
  for (int i = 0; i < batch; ++i) {
    const double* src = a[i];
    int steps = 0;
    for (size_t d = 1; d < S; d <<= 1) ++steps;
    // arrange the ping-pong so the last step lands in out[i]
    double* bufs[2] = {(steps % 2) ? out[i] : tmp.get(), (steps % 2) ? tmp.get() : out[i]};
    int w = 0;
    if (steps == 0) {
      cuda_ok(cudaMemcpyAsync(out[i], src, S * sizeof(double), cudaMemcpyDeviceToDevice, s), "copy");
      continue;
    }
    for (size_t d = 1; d < S; d <<= 1) {
      with_q(q, [&](auto Q) { k_sum_step<<<grid_for(S), kThreads, 0, s>>>(Q, src, bufs[w], S, d); });
      cuda_ok(cudaGetLastError(), "sum step launch");
      rt.note_launch();
      src = bufs[w];
      w ^= 1;
    }
  }
}

void binary_batch(QSpec q, BinOp op, const double* const* a, const double* const* b, double* const* o,
                  size_t count, size_t n, cudaStream_t s) {
  for (size_t base = 0; base < count; base += kBatch) {
    const size_t m = std::min<size_t>(kBatch, count - base);
    BatchPtrs p{};
    for (size_t i = 0; i < m; ++i) {
      p.a[i] = a[base + i];
      p.b[i] = b[base + i];
      p.o[i] = o[base + i];
    }
    const dim3 g(batch_gx((n + 1) / 2, m), static_cast<unsigned>(m));
    with_q(q, [&](auto Q) {
      using QT = decltype(Q);
      if (op == B_ADD) k_binary_batch<QT, B_ADD><<<g, kThreads, 0, s>>>(Q, p, n);
      else if (op == B_SUB) k_binary_batch<QT, B_SUB><<<g, kThreads, 0, s>>>(Q, p, n);
      else k_binary_batch<QT, B_MUL><<<g, kThreads, 0, s>>>(Q, p, n);
    });
    cuda_ok(cudaGetLastError(), "binary batch launch");
    Runtime::get().note_launch();
  }
}

void scalar_batch(QSpec q, ScalOp op, const double* const* a, double c, double* const* o, size_t count, size_t n,
                  cudaStream_t s) {
  for (size_t base = 0; base < count; base += kBatch) {
    const size_t m = std::min<size_t>(kBatch, count - base);
    BatchPtrs p{};
    for (size_t i = 0; i < m; ++i) {
      p.a[i] = a[base + i];
      p.o[i] = o[base + i];
    }
    const dim3 g(batch_gx((n + 1) / 2, m), static_cast<unsigned>(m));
    with_q(q, [&](auto Q) {
      using QT = decltype(Q);
      if (op == S_ADD) k_scalar_batch<QT, S_ADD><<<g, kThreads, 0, s>>>(Q, p, c, n);
      else k_scalar_batch<QT, S_MUL><<<g, kThreads, 0, s>>>(Q, p, c, n);
    });
    cuda_ok(cudaGetLastError(), "scalar batch launch");
    Runtime::get().note_launch();
  }
}

void rotate_batch(const double* const* a, double* const* o, size_t count, size_t n, size_t shift, cudaStream_t s) {
  if (n < 2) {  // one slot: every rotation is the identity
    for (size_t i = 0; i < count; ++i)
      cuda_ok(cudaMemcpyAsync(o[i], a[i], n * sizeof(double), cudaMemcpyDeviceToDevice, s), "rotate copy");
    return;
  }
  for (size_t base = 0; base < count; base += kBatch) {
    const size_t m = std::min<size_t>(kBatch, count - base);
    BatchPtrs p{};
    for (size_t i = 0; i < m; ++i) {
      p.a[i] = a[base + i];
      p.o[i] = o[base + i];
    }
    const dim3 g(batch_gx(n / 2, m), static_cast<unsigned>(m));
    k_rotate_batch<<<g, kThreads, 0, s>>>(p, n, shift);
    cuda_ok(cudaGetLastError(), "rotate batch launch");
    Runtime::get().note_launch();
  }
}

}  // namespace k
}  // namespace hsg
