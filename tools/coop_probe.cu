// coop_probe.cu — fixed cost of cooperative launches and grid.sync on B200.
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

__global__ void k_coop(double* o, int syncs) {
  cg::grid_group g = cg::this_grid();
  for (int i = 0; i < syncs; ++i) g.sync();
  if (threadIdx.x == 0 && o) o[blockIdx.x] = 1.0;
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
  float ms;
  for (int threads : {256, 512, 1024}) {
    for (int syncs : {0, 1, 2, 8}) {
      void* args[] = {&o, &syncs};
      for (int w = 0; w < 20; ++w) cudaLaunchCooperativeKernel((void*)k_coop, 148, threads, args, 0, s);
      cudaEventRecord(a, s);
      for (int w = 0; w < 200; ++w) cudaLaunchCooperativeKernel((void*)k_coop, 148, threads, args, 0, s);
      cudaEventRecord(b, s);
      cudaEventSynchronize(b);
      cudaEventElapsedTime(&ms, a, b);
      printf("coop 148x%4d syncs %d: %6.2f us/launch (%s)\n", threads, syncs, ms * 1e3 / 200,
             cudaGetErrorString(cudaGetLastError()));
    }
  }
  // graph of 50 cooperative launches with 1 sync
  int syncs = 1;
  void* args[] = {&o, &syncs};
  cudaGraph_t gr;
  cudaGraphExec_t ge;
  cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
  for (int w = 0; w < 50; ++w) cudaLaunchCooperativeKernel((void*)k_coop, 148, 512, args, 0, s);
  cudaStreamEndCapture(s, &gr);
  cudaGraphInstantiate(&ge, gr, 0);
  cudaGraphLaunch(ge, s);
  cudaStreamSynchronize(s);
  cudaEventRecord(a, s);
  cudaGraphLaunch(ge, s);
  cudaEventRecord(b, s);
  cudaEventSynchronize(b);
  cudaEventElapsedTime(&ms, a, b);
  printf("graph coop 148x512 1 sync: %6.2f us/node (%s)\n", ms * 1e3 / 50, cudaGetErrorString(cudaGetLastError()));
  cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
  for (int w = 0; w < 50; ++w) k_plain<<<148, 512, 0, s>>>(o);
  cudaStreamEndCapture(s, &gr);
  cudaGraphInstantiate(&ge, gr, 0);
  cudaGraphLaunch(ge, s);
  cudaStreamSynchronize(s);
  cudaEventRecord(a, s);
  cudaGraphLaunch(ge, s);
  cudaEventRecord(b, s);
  cudaEventSynchronize(b);
  cudaEventElapsedTime(&ms, a, b);
  printf("graph plain 148x512: %6.2f us/node\n", ms * 1e3 / 50);
  return 0;
}
