// rns.cu — Tier R kernels and host orchestration (see rns.h).
//
//   NTT / iNTT   two shared-memory passes per limb: the first log2(R1) stages
//                act on columns (stride C = N/R1, coalesced 2048-element tiles),
//                the remaining stages on contiguous blocks of C; Shoup twiddles,
//                lazy Harvey butterflies in [0, 4q), canonical output.
//   tensor       d0 = a0 b0, d1 = a0 b1 + a1 b0, d2 = a1 b1 (Barrett).
//   ModUp        fast base conversion of each digit (coefficient form) to the
//                extended basis Q_l u P, then NTT of the new limbs.
//   inner        sum_j ModUp(d_j) * key_j over all digits (streams the key).
//   ModDown      iNTT of the P limbs, base conversion P -> Q_l, NTT, then
//                (acc - conv) * P^-1 (+ the tensor's d0/d1 for HMult).
//   rescale      iNTT of the last limb, reduce into q_i, NTT, (c_i - t_i) q_l^-1.
//   automorph    NTT-domain Galois permutation for 5^k.
// Every kernel takes a batch index in blockIdx.z (ciphertexts of one call).
#include "rns.h"

#include <algorithm>
#include <cstring>
#include <stdexcept>
#include <string>

namespace hsg {
namespace rns {
namespace {

constexpr int kT = 256;        // threads per block
constexpr uint32_t kTile = 2048;  // NTT elements per CTA (16 KB of shared memory)

enum : uint64_t { D_SECRET = 1, D_KEY_A = 2, D_KEY_E = 3, D_CT = 4 };

__host__ __device__ inline uint64_t hash64(uint64_t seed, uint64_t domain, uint64_t a, uint64_t b) {
  uint64_t z = seed ^ (domain * 0x9E3779B97F4A7C15ULL) ^ (a * 0xC2B2AE3D27D4EB4FULL) ^ (b * 0x165667B19E3779F9ULL);
  z += 0x9E3779B97F4A7C15ULL;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}
__host__ __device__ inline uint64_t uniform_mod(uint64_t h, uint64_t q) {
  return static_cast<uint64_t>((static_cast<u128>(h) * q) >> 64);
}
__device__ inline uint64_t lift(int64_t v, uint64_t q) {
  return v >= 0 ? static_cast<uint64_t>(v) % q : q - (static_cast<uint64_t>(-v) % q);
}
__device__ inline uint32_t bitrev(uint32_t x, uint32_t bits) { return __brev(x) >> (32 - bits); }

struct PrimeMap {
  uint8_t p[64];
};

// ---------------------------------------------------------------- NTT kernels
// forward, phase 1: the first log2(R1) stages on columns r*C + c
__global__ void __launch_bounds__(kT) k_ntt_fwd_cols(uint64_t* data, const __grid_constant__ PrimeMap pm, size_t gstride, const PrimeC* pcs,
                                                     const uint64_t* tw, uint32_t N, uint32_t R1, uint32_t CPB) {
  __shared__ uint64_t sm[kTile];
  const uint32_t pi = pm.p[blockIdx.y];
  const uint64_t q = pcs[pi].q, q2 = 2 * q;
  const uint64_t* psi = tw + size_t(pi) * 4 * N;
  const uint64_t* psip = psi + N;
  uint64_t* a = data + blockIdx.z * gstride + size_t(blockIdx.y) * N;
  const uint32_t C = N / R1, c0 = blockIdx.x * CPB;
  for (uint32_t e = threadIdx.x; e < R1 * CPB; e += blockDim.x) sm[e] = a[c0 + (e % CPB) + (e / CPB) * C];
  __syncthreads();
  for (uint32_t m = 1, tr = R1 / 2; m < R1; m <<= 1, tr >>= 1) {
    for (uint32_t b = threadIdx.x; b < (R1 / 2) * CPB; b += blockDim.x) {
      const uint32_t cc = b % CPB, bi = b / CPB, g = bi / tr, r0 = g * 2 * tr + bi % tr;
      const uint64_t w = __ldg(psi + m + g), wp = __ldg(psip + m + g);
      uint64_t X = sm[r0 * CPB + cc];
      const uint64_t Y = sm[(r0 + tr) * CPB + cc];
      X = X >= q2 ? X - q2 : X;
      const uint64_t T = mul_shoup_lazy(Y, w, wp, q);
      sm[r0 * CPB + cc] = X + T;
      sm[(r0 + tr) * CPB + cc] = X - T + q2;
    }
    __syncthreads();
  }
  for (uint32_t e = threadIdx.x; e < R1 * CPB; e += blockDim.x) a[c0 + (e % CPB) + (e / CPB) * C] = sm[e];
}

// forward, phase 2: the remaining stages on contiguous blocks of C; canonical output
__global__ void __launch_bounds__(kT) k_ntt_fwd_rows(uint64_t* data, const __grid_constant__ PrimeMap pm, size_t gstride, const PrimeC* pcs,
                                                     const uint64_t* tw, uint32_t N, uint32_t R1, uint32_t BPB) {
  __shared__ uint64_t sm[kTile];
  const uint32_t pi = pm.p[blockIdx.y];
  const uint64_t q = pcs[pi].q, q2 = 2 * q;
  const uint64_t* psi = tw + size_t(pi) * 4 * N;
  const uint64_t* psip = psi + N;
  const uint32_t C = N / R1;
  uint64_t* a = data + blockIdx.z * gstride + size_t(blockIdx.y) * N + size_t(blockIdx.x) * BPB * C;
  for (uint32_t e = threadIdx.x; e < BPB * C; e += blockDim.x) sm[e] = a[e];
  __syncthreads();
  for (uint32_t m = R1, t = C / 2; m < N; m <<= 1, t >>= 1) {
    for (uint32_t b = threadIdx.x; b < BPB * C / 2; b += blockDim.x) {
      const uint32_t k = b / (C / 2), bi = b % (C / 2), g = bi / t, u0 = g * 2 * t + bi % t;
      const uint32_t gb = blockIdx.x * BPB + k;
      const uint32_t wi = m + gb * (m / R1) + g;
      const uint64_t w = __ldg(psi + wi), wp = __ldg(psip + wi);
      uint64_t X = sm[k * C + u0];
      const uint64_t Y = sm[k * C + u0 + t];
      X = X >= q2 ? X - q2 : X;
      const uint64_t T = mul_shoup_lazy(Y, w, wp, q);
      sm[k * C + u0] = X + T;
      sm[k * C + u0 + t] = X - T + q2;
    }
    __syncthreads();
  }
  for (uint32_t e = threadIdx.x; e < BPB * C; e += blockDim.x) {
    uint64_t v = sm[e];
    v = v >= q2 ? v - q2 : v;
    a[e] = v >= q ? v - q : v;
  }
}

// inverse, phase 1: the first stages (t = 1 .. C/2) on contiguous blocks of C
__global__ void __launch_bounds__(kT) k_ntt_inv_rows(uint64_t* data, const __grid_constant__ PrimeMap pm, size_t gstride, const PrimeC* pcs,
                                                     const uint64_t* tw, uint32_t N, uint32_t R1, uint32_t BPB) {
  __shared__ uint64_t sm[kTile];
  const uint32_t pi = pm.p[blockIdx.y];
  const uint64_t q = pcs[pi].q, q2 = 2 * q;
  const uint64_t* ipsi = tw + size_t(pi) * 4 * N + 2 * N;
  const uint64_t* ipsip = ipsi + N;
  const uint32_t C = N / R1;
  uint64_t* a = data + blockIdx.z * gstride + size_t(blockIdx.y) * N + size_t(blockIdx.x) * BPB * C;
  for (uint32_t e = threadIdx.x; e < BPB * C; e += blockDim.x) sm[e] = a[e];
  __syncthreads();
  for (uint32_t t = 1, h = N / 2; t < C; t <<= 1, h >>= 1) {
    for (uint32_t b = threadIdx.x; b < BPB * C / 2; b += blockDim.x) {
      const uint32_t k = b / (C / 2), bi = b % (C / 2), g = bi / t, u0 = g * 2 * t + bi % t;
      const uint32_t gb = blockIdx.x * BPB + k;
      const uint32_t wi = h + gb * (C / (2 * t)) + g;
      const uint64_t w = __ldg(ipsi + wi), wp = __ldg(ipsip + wi);
      const uint64_t X = sm[k * C + u0], Y = sm[k * C + u0 + t];
      uint64_t s = X + Y;
      s = s >= q2 ? s - q2 : s;
      sm[k * C + u0] = s;
      sm[k * C + u0 + t] = mul_shoup_lazy(X - Y + q2, w, wp, q);
    }
    __syncthreads();
  }
  for (uint32_t e = threadIdx.x; e < BPB * C; e += blockDim.x) a[e] = sm[e];
}

// inverse, phase 2: the last log2(R1) stages on columns, then * N^-1; canonical output
__global__ void __launch_bounds__(kT) k_ntt_inv_cols(uint64_t* data, const __grid_constant__ PrimeMap pm, size_t gstride, const PrimeC* pcs,
                                                     const uint64_t* tw, uint32_t N, uint32_t R1, uint32_t CPB) {
  __shared__ uint64_t sm[kTile];
  const uint32_t pi = pm.p[blockIdx.y];
  const PrimeC P = pcs[pi];
  const uint64_t q = P.q, q2 = 2 * q;
  const uint64_t* ipsi = tw + size_t(pi) * 4 * N + 2 * N;
  const uint64_t* ipsip = ipsi + N;
  uint64_t* a = data + blockIdx.z * gstride + size_t(blockIdx.y) * N;
  const uint32_t C = N / R1, c0 = blockIdx.x * CPB;
  for (uint32_t e = threadIdx.x; e < R1 * CPB; e += blockDim.x) sm[e] = a[c0 + (e % CPB) + (e / CPB) * C];
  __syncthreads();
  for (uint32_t tr = 1, h = R1 / 2; tr < R1; tr <<= 1, h >>= 1) {
    for (uint32_t b = threadIdx.x; b < (R1 / 2) * CPB; b += blockDim.x) {
      const uint32_t cc = b % CPB, bi = b / CPB, g = bi / tr, r0 = g * 2 * tr + bi % tr;
      const uint64_t w = __ldg(ipsi + h + g), wp = __ldg(ipsip + h + g);
      const uint64_t X = sm[r0 * CPB + cc], Y = sm[(r0 + tr) * CPB + cc];
      uint64_t s = X + Y;
      s = s >= q2 ? s - q2 : s;
      sm[r0 * CPB + cc] = s;
      sm[(r0 + tr) * CPB + cc] = mul_shoup_lazy(X - Y + q2, w, wp, q);
    }
    __syncthreads();
  }
  for (uint32_t e = threadIdx.x; e < R1 * CPB; e += blockDim.x)
    a[c0 + (e % CPB) + (e / CPB) * C] = mul_shoup(sm[e], P.ninv, P.ninv_sh, q);
}

// ---------------------------------------------------------------- elementwise
__global__ void k_random_ct(uint64_t* out, const PrimeC* pcs, uint64_t seed, uint64_t tag, uint32_t nl, uint32_t N) {
  const size_t total = size_t(2) * nl * N;
  for (size_t x = blockIdx.x * size_t(blockDim.x) + threadIdx.x; x < total; x += size_t(gridDim.x) * blockDim.x) {
    const uint32_t n = x % N, i = (x / N) % nl, p = x / (size_t(N) * nl);
    out[x] = uniform_mod(hash64(seed, D_CT, tag * 1024 + p * 64 + i, n), pcs[i].q);
  }
}

__global__ void k_secret(uint64_t* sk, const PrimeC* pcs, uint64_t seed, uint32_t np, uint32_t N) {
  for (size_t x = blockIdx.x * size_t(blockDim.x) + threadIdx.x; x < size_t(np) * N; x += size_t(gridDim.x) * blockDim.x) {
    const uint32_t n = x % N, i = x / N;
    sk[x] = lift(static_cast<int64_t>(hash64(seed, D_SECRET, 0, n) % 3) - 1, pcs[i].q);
  }
}

__device__ inline int64_t cbd(uint64_t h) {
  return static_cast<int64_t>(__popcll(h & 0x1FFFFFULL)) - static_cast<int64_t>(__popcll((h >> 21) & 0x1FFFFFULL));
}

// key digit j: a uniform (NTT form), e small (coefficient form, NTT'd by the host after)
__global__ void k_key_ae(uint64_t* a, uint64_t* e, const PrimeC* pcs, uint64_t seed, uint64_t keyid, uint32_t j,
                         uint32_t np, uint32_t N) {
  for (size_t x = blockIdx.x * size_t(blockDim.x) + threadIdx.x; x < size_t(np) * N; x += size_t(gridDim.x) * blockDim.x) {
    const uint32_t n = x % N, i = x / N;
    const uint64_t q = pcs[i].q;
    a[x] = uniform_mod(hash64(seed, D_KEY_A, keyid * 4096 + j * 64 + i, n), q);
    e[x] = lift(cbd(hash64(seed, D_KEY_E, keyid * 4096 + j, n)), q);
  }
}

// b = e - a s + [i in digit j] P_i s'
__global__ void k_key_b(uint64_t* b, const uint64_t* a, const uint64_t* e, const uint64_t* s, const uint64_t* sp,
                        const PrimeC* pcs, const uint64_t* Pmod, uint32_t j, uint32_t alpha, uint32_t nq,
                        uint32_t np, uint32_t N) {
  for (size_t x = blockIdx.x * size_t(blockDim.x) + threadIdx.x; x < size_t(np) * N; x += size_t(gridDim.x) * blockDim.x) {
    const uint32_t i = x / N;
    const PrimeC& P = pcs[i];
    uint64_t v = sub_mod(e[x], mul_mod(a[x], s[x], P), P.q);
    if (i < nq && i / alpha == j) v = add_mod(v, mul_mod(Pmod[i], sp[x], P), P.q);
    b[x] = v;
  }
}

__global__ void k_square(uint64_t* out, const uint64_t* in, const PrimeC* pcs, uint32_t np, uint32_t N) {
  for (size_t x = blockIdx.x * size_t(blockDim.x) + threadIdx.x; x < size_t(np) * N; x += size_t(gridDim.x) * blockDim.x)
    out[x] = mul_mod(in[x], in[x], pcs[x / N]);
}

__device__ inline uint32_t galois_src(uint32_t j, uint64_t g, uint32_t logN) {
  const uint64_t mask = (2ULL << logN) - 1;
  const uint64_t e = ((2ULL * bitrev(j, logN) + 1) * g) & mask;
  return bitrev(static_cast<uint32_t>((e - 1) >> 1), logN);
}

// out[p][i][n] = in[p][i][src(n)] for `npoly` polys of nl limbs
__global__ void k_automorph(uint64_t* out, const uint64_t* in, uint64_t g, uint32_t logN, uint32_t rows,
                            size_t gstride) {
  const uint32_t N = 1u << logN;
  const uint64_t* src = in + blockIdx.z * gstride;
  uint64_t* dst = out + blockIdx.z * gstride;
  for (size_t x = blockIdx.x * size_t(blockDim.x) + threadIdx.x; x < size_t(rows) * N; x += size_t(gridDim.x) * blockDim.x) {
    const uint32_t n = x % N;
    dst[x] = src[(x - n) + galois_src(n, g, logN)];
  }
}

// tensor: d0 = a0 b0, d1 = a0 b1 + a1 b0, d2 = a1 b1 (all NTT form, nl limbs)
__global__ void k_tensor(const uint64_t* a, const uint64_t* b, uint64_t* d0, uint64_t* d1, uint64_t* d2,
                         const PrimeC* pcs, uint32_t nl, uint32_t N, size_t ct_stride, size_t d_stride) {
  const uint64_t* A = a + blockIdx.z * ct_stride;
  const uint64_t* Bb = b + blockIdx.z * ct_stride;
  const size_t off = blockIdx.z * d_stride, half = size_t(nl) * N;
  for (size_t x = blockIdx.x * size_t(blockDim.x) + threadIdx.x; x < half; x += size_t(gridDim.x) * blockDim.x) {
    const PrimeC& P = pcs[x / N];
    const uint64_t a0 = A[x], a1 = A[half + x], b0 = Bb[x], b1 = Bb[half + x];
    d0[off + x] = mul_mod(a0, b0, P);
    d1[off + x] = add_mod(mul_mod(a0, b1, P), mul_mod(a1, b0, P), P.q);
    d2[off + x] = mul_mod(a1, b1, P);
  }
}

// ---------------------------------------------------------------- key switching
// Base-conversion constants of one (source set -> target set) conversion:
//   y_i = [x_i * hinv_i]_{src_i};  out_t = sum_i y_i * h[t][i] mod t  (Shoup constants)
struct Conv {
  uint32_t nsrc, ntgt;
  uint8_t src[32];      // source prime indices
  uint8_t tgt[64];      // target prime indices
  uint8_t tgt_row[64];  // destination row (limb) of each target in the output array
  uint64_t hinv[32], hinv_sh[32];
};

__global__ void k_conv(const uint64_t* in, uint32_t in_row0, uint64_t* out, const Conv* cv, const PrimeC* pcs,
                       const uint64_t* h, const uint64_t* h_sh, uint32_t N, size_t in_stride, size_t out_stride) {
  const Conv& C = *cv;
  const uint64_t* I = in + blockIdx.z * in_stride;
  uint64_t* O = out + blockIdx.z * out_stride;
  for (uint32_t n = blockIdx.x * blockDim.x + threadIdx.x; n < N; n += gridDim.x * blockDim.x) {
    uint64_t y[32];
    for (uint32_t i = 0; i < C.nsrc; ++i)
      y[i] = mul_shoup(I[size_t(in_row0 + i) * N + n], C.hinv[i], C.hinv_sh[i], pcs[C.src[i]].q);
    for (uint32_t t = blockIdx.y; t < C.ntgt; t += gridDim.y) {
      const uint64_t qt = pcs[C.tgt[t]].q, q2 = 2 * qt;
      const uint64_t* ht = h + size_t(t) * 32;
      const uint64_t* hs = h_sh + size_t(t) * 32;
      uint64_t acc = 0;
      for (uint32_t i = 0; i < C.nsrc; ++i) {
        acc += mul_shoup_lazy(y[i], ht[i], hs[i], qt);
        acc = acc >= q2 ? acc - q2 : acc;
      }
      O[size_t(C.tgt_row[t]) * N + n] = acc >= qt ? acc - qt : acc;
    }
  }
}

// acc_w[x] = sum_j ext_j[x] * key_w[j][gi(x)]  (w = 0: b, 1: a), nx rows
__global__ void k_ks_inner(const uint64_t* ext, uint64_t* acc, const uint64_t* kb, const uint64_t* ka, const __grid_constant__ PrimeMap pm,
                           const PrimeC* pcs, uint32_t nd, uint32_t nx, uint32_t np, uint32_t N, size_t ext_stride,
                           size_t acc_stride) {
  const uint64_t* E = ext + blockIdx.z * ext_stride;
  uint64_t* A = acc + blockIdx.z * acc_stride;
  const size_t rowN = size_t(nx) * N;
  for (size_t x = blockIdx.x * size_t(blockDim.x) + threadIdx.x; x < rowN; x += size_t(gridDim.x) * blockDim.x) {
    const uint32_t row = x / N, n = x % N, gi = pm.p[row];
    const PrimeC& P = pcs[gi];
    uint64_t s0 = 0, s1 = 0;
    for (uint32_t j = 0; j < nd; ++j) {
      const uint64_t e = E[size_t(j) * rowN + x];
      const size_t kx = (size_t(j) * np + gi) * N + n;
      s0 = add_mod(s0, mul_mod(e, __ldg(kb + kx), P), P.q);
      s1 = add_mod(s1, mul_mod(e, __ldg(ka + kx), P), P.q);
    }
    A[x] = s0;
    A[rowN + x] = s1;
  }
}

// out_w[i] = (acc_w[i] - conv_w[i]) * pinv_i (+ add_w[i] when given)
__global__ void k_moddown(const uint64_t* acc, const uint64_t* conv, const uint64_t* add0, const uint64_t* add1,
                          uint64_t* out, const PrimeC* pcs, const uint64_t* pinv, const uint64_t* pinv_sh, uint32_t nl,
                          uint32_t nx, uint32_t N, size_t acc_stride, size_t conv_stride, size_t add_stride,
                          size_t out_stride) {
  const uint64_t* A = acc + blockIdx.z * acc_stride;
  const uint64_t* Cv = conv + blockIdx.z * conv_stride;
  uint64_t* O = out + blockIdx.z * out_stride;
  const size_t half = size_t(nl) * N;
  for (size_t x = blockIdx.x * size_t(blockDim.x) + threadIdx.x; x < 2 * half; x += size_t(gridDim.x) * blockDim.x) {
    const uint32_t w = x / half;
    const size_t r = x - w * half;
    const uint32_t i = r / N;
    const uint64_t q = pcs[i].q;
    uint64_t v = mul_shoup(sub_mod(A[size_t(w) * nx * N + r], Cv[x], q), pinv[i], pinv_sh[i], q);
    const uint64_t* ad = w == 0 ? add0 : add1;
    if (ad) v = add_mod(v, ad[blockIdx.z * add_stride + r], q);
    O[x] = v;
  }
}

__global__ void k_rescale_sub(const uint64_t* in, const uint64_t* t, uint64_t* out, const PrimeC* pcs,
                              const uint64_t* qinv, const uint64_t* qinv_sh, uint32_t level, uint32_t N,
                              size_t in_stride, size_t t_stride, size_t out_stride) {
  const size_t per = size_t(level) * N;
  for (size_t x = blockIdx.x * size_t(blockDim.x) + threadIdx.x; x < 2 * per; x += size_t(gridDim.x) * blockDim.x) {
    const uint32_t p = x / per;
    const size_t r = x - p * per;
    const uint32_t i = r / N;
    const uint64_t q = pcs[i].q;
    const uint64_t c = in[blockIdx.z * in_stride + size_t(p) * (level + 1) * N + r];
    out[blockIdx.z * out_stride + x] = mul_shoup(sub_mod(c, t[blockIdx.z * t_stride + x], q), qinv[i], qinv_sh[i], q);
  }
}

// t[p][i][n] = last[p][n] mod q_i (the last limb, coefficient form, replicated into every q_i)
__global__ void k_rescale_spread(const uint64_t* last, uint64_t* t, const PrimeC* pcs, uint32_t level, uint32_t N,
                                 size_t last_stride, size_t t_stride) {
  const size_t per = size_t(level) * N;
  for (size_t x = blockIdx.x * size_t(blockDim.x) + threadIdx.x; x < 2 * per; x += size_t(gridDim.x) * blockDim.x) {
    const uint32_t p = x / per;
    const size_t r = x - p * per;
    const uint32_t i = r / N, n = r % N;
    t[blockIdx.z * t_stride + x] = reduce64(last[blockIdx.z * last_stride + size_t(p) * N + n], pcs[i]);
  }
}

__global__ void k_copy_rows(const uint64_t* in, uint64_t* out, uint32_t rows, uint32_t N, size_t in_stride,
                            size_t out_stride) {
  for (size_t x = blockIdx.x * size_t(blockDim.x) + threadIdx.x; x < size_t(rows) * N; x += size_t(gridDim.x) * blockDim.x)
    out[blockIdx.z * out_stride + x] = in[blockIdx.z * in_stride + x];
}

// host helpers -----------------------------------------------------------------------
uint64_t h_mulmod(uint64_t a, uint64_t b, uint64_t q) { return static_cast<uint64_t>(static_cast<u128>(a) * b % q); }
uint64_t h_pow(uint64_t a, uint64_t e, uint64_t q) {
  uint64_t r = 1 % q;
  a %= q;
  while (e) {
    if (e & 1) r = h_mulmod(r, a, q);
    a = h_mulmod(a, a, q);
    e >>= 1;
  }
  return r;
}
uint64_t h_inv(uint64_t a, uint64_t q) { return h_pow(a, q - 2, q); }
bool h_prime(uint64_t n) {
  static const uint64_t bases[] = {2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37};
  if (n < 2) return false;
  for (uint64_t b : bases)
    if (n % b == 0) return n == b;
  uint64_t d = n - 1;
  int r = 0;
  while ((d & 1) == 0) {
    d >>= 1;
    ++r;
  }
  for (uint64_t b : bases) {
    uint64_t x = h_pow(b, d, n);
    if (x == 1 || x == n - 1) continue;
    bool comp = true;
    for (int j = 1; j < r; ++j) {
      x = h_mulmod(x, x, n);
      if (x == n - 1) {
        comp = false;
        break;
      }
    }
    if (comp) return false;
  }
  return true;
}
uint32_t h_bitrev(uint32_t x, uint32_t bits) {
  uint32_t r = 0;
  for (uint32_t i = 0; i < bits; ++i) r |= ((x >> i) & 1u) << (bits - 1 - i);
  return r;
}

unsigned grid_of(size_t n) {
  const size_t g = (n + kT - 1) / kT;
  return static_cast<unsigned>(std::min<size_t>(std::max<size_t>(g, 1), size_t(Runtime::get().sm_count()) * 16));
}

template <class T>
DevBuf upload(const std::vector<T>& v) {
  Runtime& rt = Runtime::get();
  const size_t words = (v.size() * sizeof(T) + 7) / 8;
  DevBuf d = rt.alloc(std::max<size_t>(words, 1));
  cuda_ok(cudaMemcpyAsync(d.get(), v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice, rt.stream()), "upload");
  rt.sync();
  return d;
}

PrimeMap map_of(const std::vector<uint32_t>& p) {
  PrimeMap m{};
  for (size_t i = 0; i < p.size() && i < 64; ++i) m.p[i] = static_cast<uint8_t>(p[i]);
  return m;
}

}  // namespace

// ================================================================== context
uint64_t Ctx::galois_elt(int64_t k, uint32_t logN) {
  const uint64_t twoN = 2ULL << logN, half = 1ULL << (logN - 1);
  int64_t kk = k % static_cast<int64_t>(half);
  if (kk < 0) kk += static_cast<int64_t>(half);
  uint64_t g = 1;
  for (int64_t i = 0; i < kk; ++i) g = g * 5 % twoN;
  return g;
}

Ctx::Ctx(const Spec& s) : spec(s) {
  if (s.logN < 9 || s.logN > 17) fail(HS_E_INVALID_ARG, "rns: logN must be in [9, 17]");
  if (s.dnum < 1 || s.K < 1 || s.L + 1 + s.K > 64) fail(HS_E_INVALID_ARG, "rns: bad prime counts");
  if (s.logq0 > 61 || s.logq > 61 || s.logp > 61 || s.logq < 20) fail(HS_E_INVALID_ARG, "rns: primes must be 20..61 bits");
  N = 1u << s.logN;
  nq = s.L + 1;
  np = nq + s.K;
  alpha = (nq + s.dnum - 1) / s.dnum;
  if (alpha > 32) fail(HS_E_INVALID_ARG, "rns: digits wider than 32 primes");
  // primes (rns_oracle.c rnso_primes)
  const uint64_t twoN = 2ULL << s.logN;
  const uint32_t bits[3] = {s.logq0, s.logq, s.logp}, cnt[3] = {1, s.L, s.K};
  for (int g = 0; g < 3; ++g) {
    uint64_t c = ((1ULL << bits[g]) / twoN) * twoN + 1;
    if (c >= (1ULL << bits[g])) c -= twoN;
    for (uint32_t taken = 0; taken < cnt[g];) {
      if (c < twoN) fail(HS_E_INVALID_ARG, "rns: ran out of NTT primes");
      if (std::find(primes.begin(), primes.end(), c) == primes.end() && h_prime(c)) {
        primes.push_back(c);
        ++taken;
      }
      c -= twoN;
    }
  }
  // per-prime constants and twiddle tables
  std::vector<uint64_t> tw(size_t(np) * 4 * N);
  for (uint32_t i = 0; i < np; ++i) {
    const uint64_t q = primes[i];
    PrimeC p{};
    p.q = q;
    p.k = 64 - __builtin_clzll(q);
    p.mu = static_cast<uint64_t>((static_cast<u128>(1) << (2 * p.k)) / q);
    p.m64 = static_cast<uint64_t>((static_cast<u128>(1) << 64) / q);
    p.ninv = h_inv(N % q, q);
    p.ninv_sh = shoup_of(p.ninv, q);
    pc.push_back(p);
    uint64_t psi = 0;
    for (uint64_t x = 2;; ++x) {
      psi = h_pow(x, (q - 1) / twoN, q);
      if (h_pow(psi, N, q) == q - 1) break;
    }
    const uint64_t ipsi = h_inv(psi, q);
    uint64_t* t = tw.data() + size_t(i) * 4 * N;
    for (uint32_t k = 0; k < N; ++k) {
      const uint32_t r = h_bitrev(k, s.logN);
      t[k] = h_pow(psi, r, q);
      t[N + k] = shoup_of(t[k], q);
      t[2 * N + k] = h_pow(ipsi, r, q);
      t[3 * N + k] = shoup_of(t[2 * N + k], q);
    }
  }
  d_pc = upload(pc);
  d_tw = upload(tw);
  // secret key (NTT form over every prime)
  Runtime& rt = Runtime::get();
  d_sk = rt.alloc(size_t(np) * N);
  k_secret<<<grid_of(size_t(np) * N), kT, 0, rt.stream()>>>(reinterpret_cast<uint64_t*>(d_sk.get()), dpc(), s.seed, np, N);
  cuda_ok(cudaGetLastError(), "secret");
  std::vector<uint32_t> all(np);
  for (uint32_t i = 0; i < np; ++i) all[i] = i;
  ntt(*this, reinterpret_cast<uint64_t*>(d_sk.get()), all, 1, 0, false);
  rt.sync();
}

void Ctx::make_key(uint64_t keyid, const uint64_t* sprime, Key* out) {
  Runtime& rt = Runtime::get();
  const size_t kw = size_t(spec.dnum) * np * N;
  out->b = rt.alloc(kw);
  out->a = rt.alloc(kw);
  DevBuf e = rt.alloc(size_t(np) * N);
  std::vector<uint64_t> Pm(np);
  for (uint32_t i = 0; i < np; ++i) {
    uint64_t v = 1;
    for (uint32_t k = 0; k < spec.K; ++k) v = h_mulmod(v, primes[nq + k] % primes[i], primes[i]);
    Pm[i] = v;
  }
  DevBuf dP = upload(Pm);
  std::vector<uint32_t> all(np);
  for (uint32_t i = 0; i < np; ++i) all[i] = i;
  uint64_t* B = reinterpret_cast<uint64_t*>(out->b.get());
  uint64_t* A = reinterpret_cast<uint64_t*>(out->a.get());
  uint64_t* E = reinterpret_cast<uint64_t*>(e.get());
  for (uint32_t j = 0; j < spec.dnum; ++j) {
    uint64_t* aj = A + size_t(j) * np * N;
    uint64_t* bj = B + size_t(j) * np * N;
    k_key_ae<<<grid_of(size_t(np) * N), kT, 0, rt.stream()>>>(aj, E, dpc(), spec.seed, keyid, j, np, N);
    ntt(*this, E, all, 1, 0, false);
    k_key_b<<<grid_of(size_t(np) * N), kT, 0, rt.stream()>>>(bj, aj, E, reinterpret_cast<const uint64_t*>(d_sk.get()),
                                                             sprime, dpc(), reinterpret_cast<const uint64_t*>(dP.get()),
                                                             j, alpha, nq, np, N);
    cuda_ok(cudaGetLastError(), "keygen");
  }
  rt.sync();
}

const Ctx::Key& Ctx::relin_key() {
  std::lock_guard<std::mutex> g(key_mu);
  if (!relin_) {
    Runtime& rt = Runtime::get();
    DevBuf s2 = rt.alloc(size_t(np) * N);
    k_square<<<grid_of(size_t(np) * N), kT, 0, rt.stream()>>>(reinterpret_cast<uint64_t*>(s2.get()),
                                                              reinterpret_cast<const uint64_t*>(d_sk.get()), dpc(), np, N);
    relin_ = std::make_unique<Key>();
    make_key(0, reinterpret_cast<const uint64_t*>(s2.get()), relin_.get());
  }
  return *relin_;
}

const Ctx::Key& Ctx::galois_key(uint64_t g) {
  std::lock_guard<std::mutex> lk(key_mu);
  auto it = gal_.find(g);
  if (it != gal_.end()) return *it->second;
  Runtime& rt = Runtime::get();
  DevBuf sg = rt.alloc(size_t(np) * N);
  k_automorph<<<dim3(grid_of(size_t(np) * N), 1, 1), kT, 0, rt.stream()>>>(
      reinterpret_cast<uint64_t*>(sg.get()), reinterpret_cast<const uint64_t*>(d_sk.get()), g, spec.logN, np, 0);
  auto k = std::make_unique<Key>();
  make_key(1 + g, reinterpret_cast<const uint64_t*>(sg.get()), k.get());
  return *gal_.emplace(g, std::move(k)).first->second;
}

// ================================================================== device ops
void ntt(const Ctx& c, uint64_t* data, const std::vector<uint32_t>& prime_of, uint32_t batch, size_t gstride,
         bool inverse) {
  if (prime_of.empty() || batch == 0) return;
  Runtime& rt = Runtime::get();
  const uint32_t N = c.N, s1 = c.spec.logN / 2, R1 = 1u << s1, C = N / R1;
  const uint32_t CPB = std::min<uint32_t>(kTile / R1, C), BPB = std::min<uint32_t>(kTile / C, R1);
  const PrimeMap pm = map_of(prime_of);
  const uint32_t nl = static_cast<uint32_t>(prime_of.size());
  const dim3 g1(C / CPB, nl, batch), g2(N / (BPB * C), nl, batch);
  const uint64_t* tw = reinterpret_cast<const uint64_t*>(c.d_tw.get());
  if (!inverse) {
    k_ntt_fwd_cols<<<g1, kT, 0, rt.stream()>>>(data, pm, gstride, c.dpc(), tw, N, R1, CPB);
    k_ntt_fwd_rows<<<g2, kT, 0, rt.stream()>>>(data, pm, gstride, c.dpc(), tw, N, R1, BPB);
  } else {
    k_ntt_inv_rows<<<g2, kT, 0, rt.stream()>>>(data, pm, gstride, c.dpc(), tw, N, R1, BPB);
    k_ntt_inv_cols<<<g1, kT, 0, rt.stream()>>>(data, pm, gstride, c.dpc(), tw, N, R1, CPB);
  }
  cuda_ok(cudaGetLastError(), "ntt launch");
  rt.note_launch(2);
}

void random_ct(const Ctx& c, uint32_t level, uint64_t tag, uint64_t* out) {
  Runtime& rt = Runtime::get();
  k_random_ct<<<grid_of(size_t(2) * (level + 1) * c.N), kT, 0, rt.stream()>>>(out, c.dpc(), c.spec.seed, tag, level + 1,
                                                                             c.N);
  cuda_ok(cudaGetLastError(), "random_ct");
  rt.note_launch();
}

namespace {

// Base-conversion plan (host-built, device-resident, cached per (level, digit)).
struct ConvPlan {
  DevBuf cv, h, h_sh;
};

ConvPlan build_conv(const Ctx& c, const std::vector<uint32_t>& src, const std::vector<uint32_t>& tgt,
                    const std::vector<uint32_t>& tgt_row) {
  Conv cv{};
  cv.nsrc = static_cast<uint32_t>(src.size());
  cv.ntgt = static_cast<uint32_t>(tgt.size());
  std::vector<uint64_t> h(tgt.size() * 32, 0), hs(tgt.size() * 32, 0);
  for (size_t i = 0; i < src.size(); ++i) {
    const uint64_t qi = c.primes[src[i]];
    uint64_t v = 1;
    for (size_t m = 0; m < src.size(); ++m)
      if (m != i) v = h_mulmod(v, c.primes[src[m]] % qi, qi);
    cv.src[i] = static_cast<uint8_t>(src[i]);
    cv.hinv[i] = h_inv(v, qi);
    cv.hinv_sh[i] = shoup_of(cv.hinv[i], qi);
  }
  for (size_t t = 0; t < tgt.size(); ++t) {
    const uint64_t qt = c.primes[tgt[t]];
    cv.tgt[t] = static_cast<uint8_t>(tgt[t]);
    cv.tgt_row[t] = static_cast<uint8_t>(tgt_row[t]);
    for (size_t i = 0; i < src.size(); ++i) {
      uint64_t v = 1;
      for (size_t m = 0; m < src.size(); ++m)
        if (m != i) v = h_mulmod(v, c.primes[src[m]] % qt, qt);
      h[t * 32 + i] = v;
      hs[t * 32 + i] = shoup_of(v, qt);
    }
  }
  ConvPlan p;
  p.cv = upload(std::vector<Conv>{cv});
  p.h = upload(h);
  p.h_sh = upload(hs);
  return p;
}

struct KsPlan {
  uint32_t nl, nx, nd;
  std::vector<uint32_t> ext_primes;  // extended basis row -> prime
  std::vector<ConvPlan> up;          // per digit
  ConvPlan down;                     // P -> Q_l
  DevBuf pinv, pinv_sh;              // [nl] P^-1 mod q_i
  DevBuf qinv, qinv_sh;              // [level] q_level^-1 mod q_i (rescale)
};

std::mutex g_plan_mu;
std::map<std::pair<const Ctx*, uint32_t>, std::unique_ptr<KsPlan>> g_plans;

std::unique_ptr<KsPlan> build_plan(const Ctx& c, uint32_t level) {
  auto p = std::make_unique<KsPlan>();
  p->nl = level + 1;
  p->nx = p->nl + c.spec.K;
  p->nd = (p->nl + c.alpha - 1) / c.alpha;
  for (uint32_t i = 0; i < p->nl; ++i) p->ext_primes.push_back(i);
  for (uint32_t k = 0; k < c.spec.K; ++k) p->ext_primes.push_back(c.nq + k);
  for (uint32_t j = 0; j < p->nd; ++j) {
    const uint32_t lo = j * c.alpha, hi = std::min(lo + c.alpha, p->nl);
    std::vector<uint32_t> src, tgt, row;
    for (uint32_t i = lo; i < hi; ++i) src.push_back(i);
    for (uint32_t x = 0; x < p->nx; ++x)
      if (x < lo || x >= hi) {
        tgt.push_back(p->ext_primes[x]);
        row.push_back(x);
      }
    p->up.push_back(build_conv(c, src, tgt, row));
  }
  std::vector<uint32_t> src, tgt, row;
  for (uint32_t k = 0; k < c.spec.K; ++k) src.push_back(c.nq + k);
  for (uint32_t i = 0; i < p->nl; ++i) {
    tgt.push_back(i);
    row.push_back(i);
  }
  p->down = build_conv(c, src, tgt, row);
  std::vector<uint64_t> pinv(p->nl), pinv_sh(p->nl);
  for (uint32_t i = 0; i < p->nl; ++i) {
    const uint64_t q = c.primes[i];
    uint64_t v = 1;
    for (uint32_t k = 0; k < c.spec.K; ++k) v = h_mulmod(v, c.primes[c.nq + k] % q, q);
    pinv[i] = h_inv(v, q);
    pinv_sh[i] = shoup_of(pinv[i], q);
  }
  p->pinv = upload(pinv);
  p->pinv_sh = upload(pinv_sh);
  std::vector<uint64_t> qinv(std::max<uint32_t>(level, 1)), qinv_sh(std::max<uint32_t>(level, 1));
  for (uint32_t i = 0; i < level; ++i) {
    qinv[i] = h_inv(c.primes[level] % c.primes[i], c.primes[i]);
    qinv_sh[i] = shoup_of(qinv[i], c.primes[i]);
  }
  p->qinv = upload(qinv);
  p->qinv_sh = upload(qinv_sh);
  return p;
}

const KsPlan& ks_plan(const Ctx& c, uint32_t level) {
  std::lock_guard<std::mutex> g(g_plan_mu);
  auto key = std::make_pair(&c, level);
  auto it = g_plans.find(key);
  if (it != g_plans.end()) return *it->second;
  return *g_plans.emplace(key, build_plan(c, level)).first->second;
}

// Key-switch `batch` polynomials d ([nl][N] each, NTT form, stride d_stride) with key
// kk; out_w = ModDown(acc_w) + add_w  ([2][nl][N] per batch item, stride out_stride).
void key_switch(Ctx& c, uint32_t level, const uint64_t* d, size_t d_stride, const Ctx::Key& kk, const uint64_t* add0,
                const uint64_t* add1, size_t add_stride, uint64_t* out, size_t out_stride, uint32_t batch) {
  Runtime& rt = Runtime::get();
  cudaStream_t s = rt.stream();
  const KsPlan& P = ks_plan(c, level);
  const uint32_t N = c.N, nl = P.nl, nx = P.nx, nd = P.nd, K = c.spec.K;
  const size_t ext_stride = size_t(nd) * nx * N, acc_stride = size_t(2) * nx * N;
  DevBuf dc = rt.alloc(size_t(batch) * nl * N);
  DevBuf ext = rt.alloc(size_t(batch) * ext_stride);
  DevBuf acc = rt.alloc(size_t(batch) * acc_stride);
  uint64_t* DC = reinterpret_cast<uint64_t*>(dc.get());
  uint64_t* EXT = reinterpret_cast<uint64_t*>(ext.get());
  uint64_t* ACC = reinterpret_cast<uint64_t*>(acc.get());
  std::vector<uint32_t> qmap(nl);
  for (uint32_t i = 0; i < nl; ++i) qmap[i] = i;
  // d -> coefficient form
  k_copy_rows<<<dim3(grid_of(size_t(nl) * N), 1, batch), kT, 0, s>>>(d, DC, nl, N, d_stride, size_t(nl) * N);
  ntt(c, DC, qmap, batch, size_t(nl) * N, true);
  // ModUp per digit: own rows copied (NTT form), new rows base-converted then NTT'd
  for (uint32_t j = 0; j < nd; ++j) {
    const uint32_t lo = j * c.alpha, hi = std::min(lo + c.alpha, nl);
    uint64_t* Ej = EXT + size_t(j) * nx * N;
    k_copy_rows<<<dim3(grid_of(size_t(hi - lo) * N), 1, batch), kT, 0, s>>>(d + size_t(lo) * N, Ej + size_t(lo) * N,
                                                                          hi - lo, N, d_stride, ext_stride);
    const ConvPlan& cp = P.up[j];
    const uint32_t ntgt = nx - (hi - lo);
    k_conv<<<dim3((N + kT - 1) / kT, std::min<uint32_t>(ntgt, 8), batch), kT, 0, s>>>(
        DC, lo, Ej, reinterpret_cast<const Conv*>(cp.cv.get()), c.dpc(), reinterpret_cast<const uint64_t*>(cp.h.get()),
        reinterpret_cast<const uint64_t*>(cp.h_sh.get()), N, size_t(nl) * N, ext_stride);
    // NTT the converted rows: [0, lo) and [hi, nx) as two contiguous runs
    if (lo > 0) {
      std::vector<uint32_t> pm(P.ext_primes.begin(), P.ext_primes.begin() + lo);
      ntt(c, Ej, pm, batch, ext_stride, false);
    }
    std::vector<uint32_t> pm2(P.ext_primes.begin() + hi, P.ext_primes.end());
    ntt(c, Ej + size_t(hi) * N, pm2, batch, ext_stride, false);
  }
  // inner product with the key
  k_ks_inner<<<dim3(grid_of(size_t(nx) * N), 1, batch), kT, 0, s>>>(
      EXT, ACC, reinterpret_cast<const uint64_t*>(kk.b.get()), reinterpret_cast<const uint64_t*>(kk.a.get()),
      map_of(P.ext_primes), c.dpc(), nd, nx, c.np, N, ext_stride, acc_stride);
  // ModDown: P rows -> coefficient form -> base-convert into Q_l -> NTT -> combine
  DevBuf pc = rt.alloc(size_t(batch) * 2 * K * N);
  DevBuf conv = rt.alloc(size_t(batch) * 2 * nl * N);
  uint64_t* PC = reinterpret_cast<uint64_t*>(pc.get());
  uint64_t* CV = reinterpret_cast<uint64_t*>(conv.get());
  std::vector<uint32_t> pmap(K);
  for (uint32_t k = 0; k < K; ++k) pmap[k] = c.nq + k;
  for (uint32_t w = 0; w < 2; ++w) {
    k_copy_rows<<<dim3(grid_of(size_t(K) * N), 1, batch), kT, 0, s>>>(ACC + size_t(w) * nx * N + size_t(nl) * N,
                                                                     PC + size_t(w) * K * N, K, N, acc_stride,
                                                                     size_t(2) * K * N);
    ntt(c, PC + size_t(w) * K * N, pmap, batch, size_t(2) * K * N, true);
    k_conv<<<dim3((N + kT - 1) / kT, std::min<uint32_t>(nl, 8), batch), kT, 0, s>>>(
        PC + size_t(w) * K * N, 0, CV + size_t(w) * nl * N, reinterpret_cast<const Conv*>(P.down.cv.get()), c.dpc(),
        reinterpret_cast<const uint64_t*>(P.down.h.get()), reinterpret_cast<const uint64_t*>(P.down.h_sh.get()), N,
        size_t(2) * K * N, size_t(2) * nl * N);
  }
  ntt(c, CV, qmap, 2 * batch, size_t(nl) * N, false);  // both halves: 2*batch groups of nl rows
  k_moddown<<<dim3(grid_of(size_t(2) * nl * N), 1, batch), kT, 0, s>>>(
      ACC, CV, add0, add1, out, c.dpc(), reinterpret_cast<const uint64_t*>(P.pinv.get()),
      reinterpret_cast<const uint64_t*>(P.pinv_sh.get()), nl, nx, N, acc_stride, size_t(2) * nl * N, add_stride,
      out_stride);
  cuda_ok(cudaGetLastError(), "key switch");
  rt.note_launch(6 + 4 * nd);
}

}  // namespace

void mul_relin(Ctx& c, uint32_t level, const uint64_t* a, const uint64_t* b, uint64_t* out, uint32_t batch) {
  if (level > c.spec.L) fail(HS_E_INVALID_ARG, "rns mul_relin: level > L");
  Runtime& rt = Runtime::get();
  const uint32_t N = c.N, nl = level + 1;
  const size_t ct = size_t(2) * nl * N, half = size_t(nl) * N;
  const Ctx::Key& key = c.relin_key();
  DevBuf d = rt.alloc(size_t(batch) * 3 * half);
  uint64_t* D = reinterpret_cast<uint64_t*>(d.get());
  // layout per batch item: [d0 | d1 | d2], stride 3*half
  k_tensor<<<dim3(grid_of(half), 1, batch), kT, 0, rt.stream()>>>(a, b, D, D + half, D + 2 * half, c.dpc(), nl, N, ct,
                                                                 3 * half);
  rt.note_launch();
  key_switch(c, level, D + 2 * half, 3 * half, key, D, D + half, 3 * half, out, ct, batch);
}

void rescale(Ctx& c, uint32_t level, const uint64_t* in, uint64_t* out, uint32_t batch) {
  if (level < 1 || level > c.spec.L) fail(HS_E_INVALID_ARG, "rns rescale: level must be in [1, L]");
  Runtime& rt = Runtime::get();
  cudaStream_t s = rt.stream();
  const uint32_t N = c.N, nl = level + 1;
  const size_t in_stride = size_t(2) * nl * N, out_stride = size_t(2) * level * N;
  DevBuf last = rt.alloc(size_t(batch) * 2 * N);
  DevBuf t = rt.alloc(size_t(batch) * out_stride);
  uint64_t* LAST = reinterpret_cast<uint64_t*>(last.get());
  uint64_t* T = reinterpret_cast<uint64_t*>(t.get());
  for (uint32_t p = 0; p < 2; ++p)
    k_copy_rows<<<dim3(grid_of(N), 1, batch), kT, 0, s>>>(in + (size_t(p) * nl + level) * N, LAST + size_t(p) * N, 1, N,
                                                        in_stride, size_t(2) * N);
  ntt(c, LAST, {level}, 2 * batch, N, true);
  k_rescale_spread<<<dim3(grid_of(out_stride), 1, batch), kT, 0, s>>>(LAST, T, c.dpc(), level, N, size_t(2) * N,
                                                                     out_stride);
  std::vector<uint32_t> qmap(level);
  for (uint32_t i = 0; i < level; ++i) qmap[i] = i;
  ntt(c, T, qmap, 2 * batch, size_t(level) * N, false);
  const KsPlan& P = ks_plan(c, level);
  const uint64_t* QI = reinterpret_cast<const uint64_t*>(P.qinv.get());
  const uint64_t* QS = reinterpret_cast<const uint64_t*>(P.qinv_sh.get());
  k_rescale_sub<<<dim3(grid_of(out_stride), 1, batch), kT, 0, s>>>(in, T, out, c.dpc(), QI, QS, level, N, in_stride,
                                                                  out_stride, out_stride);
  cuda_ok(cudaGetLastError(), "rescale");
  rt.note_launch(5);
}

void rotate(Ctx& c, uint32_t level, int64_t k, const uint64_t* in, uint64_t* out, uint32_t batch) {
  if (level > c.spec.L) fail(HS_E_INVALID_ARG, "rns rotate: level > L");
  Runtime& rt = Runtime::get();
  const uint32_t N = c.N, nl = level + 1;
  const size_t ct = size_t(2) * nl * N;
  const uint64_t g = Ctx::galois_elt(k, c.spec.logN);
  const Ctx::Key& key = c.galois_key(g);
  DevBuf perm = rt.alloc(size_t(batch) * ct);
  uint64_t* PM = reinterpret_cast<uint64_t*>(perm.get());
  k_automorph<<<dim3(grid_of(ct), 1, batch), kT, 0, rt.stream()>>>(PM, in, g, c.spec.logN, 2 * nl, ct);
  rt.note_launch();
  // out0 = sigma(c0) + ks0, out1 = ks1
  key_switch(c, level, PM + size_t(nl) * N, ct, key, PM, nullptr, ct, out, ct, batch);
}

void prepare_level(Ctx& c, uint32_t level) {
  if (level > c.spec.L) fail(HS_E_INVALID_ARG, "rns: level > L");
  ks_plan(c, level);
}

void forget(const Ctx& c) {
  std::lock_guard<std::mutex> g(g_plan_mu);
  for (auto it = g_plans.begin(); it != g_plans.end();) it = it->first.first == &c ? g_plans.erase(it) : std::next(it);
}

}  // namespace rns
}  // namespace hsg
