// diag.cu — FP64-pipe throughput probe used as the roofline denominator of the
// fused per-slot kernel (bench.py).  MEASURED_PEAKS.json only carries HBM and
// bf16 tensor peaks; the fused inverse-root kernel is bound by the FP64 pipe
// (DMUL / DADD / FRND.F64), so bench.py measures that pipe on the same GPU with
// this kernel: 8 independent dependency chains per thread, full grid.
#include "core.h"

namespace hsg {
namespace {

template <int KIND>
__global__ void __launch_bounds__(256) k_fp64_rate(double* sink, double c, int iters) {
  double x[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) x[j] = 1.0 + 1e-3 * (threadIdx.x + j);
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      if constexpr (KIND == 0) x[j] = __dmul_rn(x[j], c);
      else if constexpr (KIND == 1) x[j] = __dadd_rn(x[j], c);
      else if constexpr (KIND == 2) x[j] = rint(__dmul_rn(x[j], c));
      else x[j] = __fma_rn(x[j], c, c);
    }
  }
  double s = 0.0;
#pragma unroll
  for (int j = 0; j < 8; ++j) s += x[j];
  if (s == 12345.678) sink[threadIdx.x] = s;  // keep the chains alive
}

}  // namespace
}  // namespace hsg

extern "C" int hs_diag_fp64_rate(int kind, double* ops_per_s) {
  using namespace hsg;
  try {
    Runtime& rt = Runtime::get();
    DevBuf sink = rt.alloc(256);
    const int blocks = rt.sm_count() * 8, threads = 256, iters = 4096;
    cudaEvent_t e0, e1;
    cuda_ok(cudaEventCreate(&e0), "event");
    cuda_ok(cudaEventCreate(&e1), "event");
    float best = 1e30f;
    for (int rep = 0; rep < 4; ++rep) {
      cuda_ok(cudaEventRecord(e0, rt.stream()), "record");
      switch (kind) {
        case 0: k_fp64_rate<0><<<blocks, threads, 0, rt.stream()>>>(sink.get(), 1.0000001, iters); break;
        case 1: k_fp64_rate<1><<<blocks, threads, 0, rt.stream()>>>(sink.get(), 1e-9, iters); break;
        case 2: k_fp64_rate<2><<<blocks, threads, 0, rt.stream()>>>(sink.get(), 1.0000001, iters); break;
        default: k_fp64_rate<3><<<blocks, threads, 0, rt.stream()>>>(sink.get(), 1e-9, iters); break;
      }
      cuda_ok(cudaEventRecord(e1, rt.stream()), "record");
      cuda_ok(cudaEventSynchronize(e1), "sync");
      float ms = 0.f;
      cuda_ok(cudaEventElapsedTime(&ms, e0, e1), "elapsed");
      if (rep > 0 && ms < best) best = ms;
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    const double insts = static_cast<double>(blocks) * threads * iters * 8 * (kind == 2 ? 2 : 1);
    *ops_per_s = insts / (best * 1e-3);
    return HS_OK;
  } catch (const Error& e) {
    return e.code;
  }
}
