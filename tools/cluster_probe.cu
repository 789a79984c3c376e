// cluster_probe.cu — microbenchmark: fixed cost of cluster launches vs smem size.
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

__global__ void k_empty(double* o, int n) {
  extern __shared__ double sm[];
  cg::cluster_group cl = cg::this_cluster();
  for (int i = threadIdx.x; i < n; i += blockDim.x) sm[i] = i;
  cl.sync();
  if (threadIdx.x == 0 && o && n > 5) o[blockIdx.x] = sm[5];
}

__global__ void k_plain(double* o) {
  if (threadIdx.x == 0 && o) o[blockIdx.x] = 1.0;
}

int main() {
  double* o;
  cudaMalloc(&o, 1 << 20);
  cudaStream_t s;
  cudaStreamCreate(&s);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int C : {1, 2, 4, 8, 16}) {
    for (int smemkb : {0, 32, 96, 196}) {
      size_t smem = smemkb * 1024;
      cudaFuncSetAttribute(k_empty, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      cudaFuncSetAttribute(k_empty, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
      cudaLaunchConfig_t cfg{};
      cfg.gridDim = dim3(C, 1, 1);
      cfg.blockDim = dim3(1024, 1, 1);
      cfg.dynamicSmemBytes = smem;
      cfg.stream = s;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = C;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      int n = smem / 8;
      for (int w = 0; w < 20; ++w) cudaLaunchKernelEx(&cfg, k_empty, o, n);
      cudaEventRecord(a, s);
      for (int w = 0; w < 200; ++w) cudaLaunchKernelEx(&cfg, k_empty, o, n);
      cudaEventRecord(b, s);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      printf("cluster %2d smem %3d KB: %7.2f us/launch (%s)\n", C, smemkb, ms * 1e3 / 200,
             cudaGetErrorString(cudaGetLastError()));
    }
  }
  for (int w = 0; w < 20; ++w) k_plain<<<148, 256, 0, s>>>(o);
  cudaEventRecord(a, s);
  for (int w = 0; w < 200; ++w) k_plain<<<148, 256, 0, s>>>(o);
  cudaEventRecord(b, s);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  printf("plain 148x256: %7.2f us/launch\n", ms * 1e3 / 200);
  return 0;
}
