// codec_gpu.cu — CKKS canonical-embedding encode / decode on the device (Tier R).
//
// The same transform as the host codec (rns_codec.cpp): slot j of m(X) is m(zeta^{t_j}),
// t_j = 5^j mod 2N, computed with one 2N-point complex FFT — bit-reversed input, radix-2
// Cooley-Tukey stages, the host plan's twiddle table, and per butterfly the same fp64
// operations in the same order (vr = v.re wr - v.im wi, vi = v.re wi + v.im wr, u +- v; every
// op an explicit _rn intrinsic, no contraction), so each butterfly rounds exactly as the host
// loop does and the device output is bit-identical to rns_codec.cpp's.
//
//   stages of length <= 2048: one kernel, 2048-point sub-transforms in shared memory;
//   longer stages (2N = 2^17 at N = 2^16: 6 of them): one grid-wide launch each.
// A batch of independent transforms (a column's chunks) rides on blockIdx.y.  The 2N complex
// workspace per item (2 MiB at N = 2^16) comes from the stream-ordered pool.
#include <cmath>
#include <mutex>
#include <unordered_map>
#include <vector>

#include "rns.h"

namespace hsg {
namespace rns {
namespace {

constexpr int kCT = 256;        // threads per codec block
constexpr int kLogLocal = 11;   // 2048-point shared-memory sub-transforms

struct DevPlan {
  uint32_t logn = 0, n = 0;
  DevBuf w;    // double2[n/2]: exp(2 pi i k / n), exactly the host plan's values
  DevBuf rev;  // uint32[n]: bit reversal
  DevBuf t;    // uint32[N/2]: 5^j mod n
};

unsigned blocks_for(size_t n) { return static_cast<unsigned>(std::min<size_t>((n + kCT - 1) / kCT, 148 * 16)); }

const DevPlan& dev_plan(uint32_t logN) {
  static std::mutex mu;
  static std::unordered_map<uint32_t, DevPlan> plans;
  std::lock_guard<std::mutex> g(mu);
  auto it = plans.find(logN);
  if (it != plans.end()) return it->second;
  DevPlan p;
  p.logn = logN + 1;
  p.n = 1u << p.logn;
  std::vector<double> w(p.n);  // interleaved re, im; same expressions as rns_codec.cpp plan()
  for (uint32_t k = 0; k < p.n / 2; ++k) {
    const double a = 2.0 * M_PI * static_cast<double>(k) / static_cast<double>(p.n);
    w[2 * k] = std::cos(a);
    w[2 * k + 1] = std::sin(a);
  }
  std::vector<uint32_t> rev(p.n);
  for (uint32_t k = 0; k < p.n; ++k) {
    uint32_t r = 0;
    for (uint32_t b = 0; b < p.logn; ++b) r |= ((k >> b) & 1u) << (p.logn - 1 - b);
    rev[k] = r;
  }
  const uint32_t S = 1u << (logN - 1);
  std::vector<uint32_t> t(S);
  uint64_t v = 1;
  for (uint32_t j = 0; j < S; ++j) {
    t[j] = static_cast<uint32_t>(v);
    v = (v * 5) % p.n;
  }
  Runtime& rt = Runtime::get();
  // uploaded on the upload stream and waited for: legal while the compute stream is captured
  cudaStream_t up = rt.upload_stream();
  p.w = rt.alloc_on(w.size(), up);
  p.rev = rt.alloc_on((rev.size() + 1) / 2, up);
  p.t = rt.alloc_on((t.size() + 1) / 2, up);
  cuda_ok(cudaMemcpyAsync(p.w.get(), w.data(), w.size() * 8, cudaMemcpyHostToDevice, up), "codec plan");
  cuda_ok(cudaMemcpyAsync(p.rev.get(), rev.data(), rev.size() * 4, cudaMemcpyHostToDevice, up), "codec plan");
  cuda_ok(cudaMemcpyAsync(p.t.get(), t.data(), t.size() * 4, cudaMemcpyHostToDevice, up), "codec plan");
  cuda_ok(cudaStreamSynchronize(up), "codec plan");
  return plans.emplace(logN, std::move(p)).first->second;
}

__device__ __forceinline__ void butterfly(double2& u, double2& v, double wr, double wi) {
  const double vr = __dsub_rn(__dmul_rn(v.x, wr), __dmul_rn(v.y, wi));
  const double vi = __dadd_rn(__dmul_rn(v.x, wi), __dmul_rn(v.y, wr));
  const double ur = u.x, ui = u.y;
  u = make_double2(__dadd_rn(ur, vr), __dadd_rn(ui, vi));
  v = make_double2(__dsub_rn(ur, vr), __dsub_rn(ui, vi));
}

// stages len = 2 .. 2^kLogLocal on 2^kLogLocal-point sub-transforms, in shared memory
__global__ void __launch_bounds__(kCT) k_fft_local(double2* b, const double2* __restrict__ w, uint32_t logn,
                                                   double sg) {
  constexpr uint32_t L = 1u << kLogLocal;
  __shared__ double2 s[L];
  double2* B = b + (size_t(blockIdx.y) << logn) + (size_t(blockIdx.x) << kLogLocal);
  for (uint32_t i = threadIdx.x; i < L; i += kCT) s[i] = B[i];
  for (uint32_t lh = 0; lh < kLogLocal; ++lh) {  // half = 2^lh, len = 2^(lh+1)
    __syncthreads();
    const uint32_t sh = logn - lh - 1;  // step = n / len
    for (uint32_t id = threadIdx.x; id < L / 2; id += kCT) {
      const uint32_t k = id & ((1u << lh) - 1), i = (id >> lh) << (lh + 1);
      const double2 tw = __ldg(w + (size_t(k) << sh));
      butterfly(s[i + k], s[i + k + (1u << lh)], tw.x, __dmul_rn(sg, tw.y));
    }
  }
  __syncthreads();
  for (uint32_t i = threadIdx.x; i < L; i += kCT) B[i] = s[i];
}

// one stage of length 2^(lh+1) > 2^kLogLocal over the whole transform
__global__ void __launch_bounds__(kCT) k_fft_stage(double2* b, const double2* __restrict__ w, uint32_t logn,
                                                   uint32_t lh, double sg) {
  double2* B = b + (size_t(blockIdx.y) << logn);
  const uint32_t sh = logn - lh - 1;
  for (uint32_t id = blockIdx.x * kCT + threadIdx.x; id < (1u << (logn - 1)); id += gridDim.x * kCT) {
    const uint32_t k = id & ((1u << lh) - 1), i = (id >> lh) << (lh + 1);
    const double2 tw = __ldg(w + (size_t(k) << sh));
    double2 u = B[i + k], v = B[i + k + (1u << lh)];
    butterfly(u, v, tw.x, __dmul_rn(sg, tw.y));
    B[i + k] = u;
    B[i + k + (1u << lh)] = v;
  }
}

void fft(double2* b, const DevPlan& p, uint32_t batch, double sg, cudaStream_t s) {
  const uint32_t local = p.logn < kLogLocal ? p.logn : kLogLocal;
  const double2* w = reinterpret_cast<const double2*>(p.w.get());
  if (local == kLogLocal) {
    k_fft_local<<<dim3(p.n >> kLogLocal, batch), kCT, 0, s>>>(b, w, p.logn, sg);
  } else {
    for (uint32_t lh = 0; lh < p.logn; ++lh)
      k_fft_stage<<<dim3(blocks_for(p.n / 2), batch), kCT, 0, s>>>(b, w, p.logn, lh, sg);
  }
  if (local == kLogLocal)
    for (uint32_t lh = kLogLocal; lh < p.logn; ++lh)
      k_fft_stage<<<dim3(blocks_for(p.n / 2), batch), kCT, 0, s>>>(b, w, p.logn, lh, sg);
  cuda_ok(cudaGetLastError(), "codec fft");
  Runtime::get().note_launch(local == kLogLocal ? 1 + p.logn - local : p.logn);
}

// encode input: item k holds z[k S .. k S + n_k), n_k = min(S, n - k S), placed at rev[t_j]
__global__ void k_enc_scatter(double2* b, const double* z, size_t n, uint32_t S, const uint32_t* rev,
                              const uint32_t* t, uint32_t logn) {
  const size_t off = size_t(blockIdx.y) * S;
  const size_t nk = n > off ? (n - off < S ? n - off : S) : 0;
  double2* B = b + (size_t(blockIdx.y) << logn);
  for (uint32_t j = blockIdx.x * kCT + threadIdx.x; j < nk; j += gridDim.x * kCT)
    B[rev[t[j]]] = make_double2(z[off + j], 0.0);
}

// coefficients: co[k] = rint((Re a_k * (2/N)) * scale), k < N
__global__ void k_enc_finish(const double2* b, double* co, uint32_t logn, double f, double scale) {
  const uint32_t N = 1u << (logn - 1);
  const double2* B = b + (size_t(blockIdx.y) << logn);
  double* C = co + (size_t(blockIdx.y) << (logn - 1));
  for (uint32_t k = blockIdx.x * kCT + threadIdx.x; k < N; k += gridDim.x * kCT)
    C[k] = rint(__dmul_rn(__dmul_rn(B[k].x, f), scale));
}

// decode input: a[rev[k]] = co[k] / scale (k < N; the upper half stays zero)
__global__ void k_dec_scatter(double2* b, const double* co, const uint32_t* rev, uint32_t logn, double scale) {
  const uint32_t N = 1u << (logn - 1);
  double2* B = b + (size_t(blockIdx.y) << logn);
  const double* C = co + (size_t(blockIdx.y) << (logn - 1));
  for (uint32_t k = blockIdx.x * kCT + threadIdx.x; k < N; k += gridDim.x * kCT)
    B[rev[k]] = make_double2(__ddiv_rn(C[k], scale), 0.0);
}

__global__ void k_dec_gather(const double2* b, const uint32_t* t, double* z, size_t n, size_t z_stride,
                             uint32_t logn) {
  const double2* B = b + (size_t(blockIdx.y) << logn);
  double* Z = z + size_t(blockIdx.y) * z_stride;
  for (uint32_t j = blockIdx.x * kCT + threadIdx.x; j < n; j += gridDim.x * kCT) Z[j] = B[t[j]].x;
}

}  // namespace

void encode_dev(uint32_t logN, const double* z, size_t n, double scale, double* co, uint32_t batch) {
  if (batch == 0) return;
  const DevPlan& p = dev_plan(logN);
  const uint32_t S = 1u << (logN - 1);
  if (n > size_t(S) * batch) fail(HS_E_INVALID_ARG, "encode: more values than slots");
  Runtime& rt = Runtime::get();
  cudaStream_t s = rt.stream();
  DevBuf ws = rt.alloc(size_t(batch) * 2 * p.n);
  double2* b = reinterpret_cast<double2*>(ws.get());
  cuda_ok(cudaMemsetAsync(b, 0, size_t(batch) * p.n * sizeof(double2), s), "codec zero");
  k_enc_scatter<<<dim3(blocks_for(S), batch), kCT, 0, s>>>(b, z, n, S, reinterpret_cast<const uint32_t*>(p.rev.get()),
                                                           reinterpret_cast<const uint32_t*>(p.t.get()), p.logn);
  fft(b, p, batch, -1.0, s);
  k_enc_finish<<<dim3(blocks_for(p.n / 2), batch), kCT, 0, s>>>(b, co, p.logn, 2.0 / static_cast<double>(p.n / 2),
                                                                scale);
  cuda_ok(cudaGetLastError(), "codec encode");
  rt.note_launch(2);
}

void decode_dev(uint32_t logN, const double* co, double scale, double* z, size_t n, size_t z_stride, uint32_t batch) {
  if (batch == 0) return;
  const DevPlan& p = dev_plan(logN);
  if (n > (p.n >> 2)) fail(HS_E_INVALID_ARG, "decode: more values than slots");
  Runtime& rt = Runtime::get();
  cudaStream_t s = rt.stream();
  DevBuf ws = rt.alloc(size_t(batch) * 2 * p.n);
  double2* b = reinterpret_cast<double2*>(ws.get());
  cuda_ok(cudaMemsetAsync(b, 0, size_t(batch) * p.n * sizeof(double2), s), "codec zero");
  k_dec_scatter<<<dim3(blocks_for(p.n / 2), batch), kCT, 0, s>>>(b, co, reinterpret_cast<const uint32_t*>(p.rev.get()),
                                                                 p.logn, scale);
  fft(b, p, batch, 1.0, s);
  k_dec_gather<<<dim3(blocks_for(n), batch), kCT, 0, s>>>(b, reinterpret_cast<const uint32_t*>(p.t.get()), z, n,
                                                          z_stride, p.logn);
  cuda_ok(cudaGetLastError(), "codec decode");
  rt.note_launch(2);
}

}  // namespace rns
}  // namespace hsg
