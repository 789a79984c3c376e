// Zero-copy (pinned host) read bandwidth for a 256 KiB column: kernel device time and
// launch+sync wall time for several launch shapes, against a DMA copy.
#include <chrono>
#include <cstdio>
#include <cuda_runtime.h>

__global__ void rd(const double2* __restrict__ src, double2* __restrict__ dst, size_t n2, int per) {
  size_t i = (blockIdx.x * size_t(blockDim.x) + threadIdx.x) * per;
  double2 v[8];
#pragma unroll
  for (int k = 0; k < 8; ++k)
    if (k < per && i + k < n2) v[k] = src[i + k];
#pragma unroll
  for (int k = 0; k < 8; ++k)
    if (k < per && i + k < n2) dst[i + k] = v[k];
}

__global__ void rd_strided(const double2* __restrict__ src, double2* __restrict__ dst, size_t n2) {
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n2; i += size_t(gridDim.x) * blockDim.x)
    dst[i] = src[i];
}

int main() {
  const size_t S = 32768, bytes = S * 8, n2 = S / 2;
  double *h, *d;
  cudaHostAlloc(&h, bytes, cudaHostAllocDefault);
  cudaMalloc(&d, bytes);
  for (size_t i = 0; i < S; ++i) h[i] = i * 0.5;
  cudaStream_t s;
  cudaStreamCreate(&s);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto wall = [](auto f) {
    auto t0 = std::chrono::steady_clock::now();
    for (int r = 0; r < 200; ++r) f();
    return std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count() / 200;
  };
  for (int per : {1, 2, 4, 8}) {
    for (int thr : {128, 256, 512}) {
      const unsigned blocks = unsigned((n2 / per + thr - 1) / thr);
      auto f = [&] { rd<<<blocks, thr, 0, s>>>(reinterpret_cast<const double2*>(h), reinterpret_cast<double2*>(d), n2, per); };
      for (int r = 0; r < 20; ++r) f();
      cudaStreamSynchronize(s);
      cudaEventRecord(e0, s);
      for (int r = 0; r < 100; ++r) f();
      cudaEventRecord(e1, s);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      const double w = wall([&] { f(); cudaStreamSynchronize(s); });
      printf("zero-copy per=%d thr=%d blocks=%u: device %.2f us/launch (%.1f GB/s), launch+sync %.2f us\n", per, thr,
             blocks, ms * 10, bytes / (ms * 10) / 1e3, w);
    }
  }
  for (unsigned blocks : {148u, 296u, 592u}) {
    auto f = [&] { rd_strided<<<blocks, 256, 0, s>>>(reinterpret_cast<const double2*>(h), reinterpret_cast<double2*>(d), n2); };
    for (int r = 0; r < 20; ++r) f();
    cudaStreamSynchronize(s);
    cudaEventRecord(e0, s);
    for (int r = 0; r < 100; ++r) f();
    cudaEventRecord(e1, s);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("zero-copy grid-stride blocks=%u: device %.2f us/launch\n", blocks, ms * 10);
  }
  {
    auto f = [&] { cudaMemcpyAsync(d, h, bytes, cudaMemcpyHostToDevice, s); };
    for (int r = 0; r < 20; ++r) f();
    cudaStreamSynchronize(s);
    cudaEventRecord(e0, s);
    for (int r = 0; r < 100; ++r) f();
    cudaEventRecord(e1, s);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double w = wall([&] { f(); cudaStreamSynchronize(s); });
    printf("DMA H2D: device %.2f us/copy, copy+sync %.2f us\n", ms * 10, w);
    auto g = [&] { cudaMemcpyAsync(h, d, bytes, cudaMemcpyDeviceToHost, s); };
    for (int r = 0; r < 20; ++r) g();
    cudaStreamSynchronize(s);
    cudaEventRecord(e0, s);
    for (int r = 0; r < 100; ++r) g();
    cudaEventRecord(e1, s);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    const double w2 = wall([&] { g(); cudaStreamSynchronize(s); });
    printf("DMA D2H: device %.2f us/copy, copy+sync %.2f us\n", ms * 10, w2);
    const double w3 = wall([&] { cudaStreamSynchronize(s); });
    printf("bare sync %.2f us\n", w3);
  }
  return 0;
}
