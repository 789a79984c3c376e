// Host-side cost of the e2e API calls (encode_column / znorm / decode_column) in C++,
// without Python in the loop.  Build: see tools/README or the command in the commit.
#include <chrono>
#include <cmath>
#include <cstdio>
#include <vector>

#include <cuda_runtime.h>

#include "hestat_gpu.h"

int main() {
  const uint64_t S = 32768;
  hs_params p{S, 11, 40, 1, 1, 0, 0};
  hs_ctx* ctx = nullptr;
  hs_ctx_create(&p, 0, &ctx);
  double *x = nullptr, *z = nullptr;
  cudaHostAlloc(reinterpret_cast<void**>(&x), S * 8, cudaHostAllocDefault);
  cudaHostAlloc(reinterpret_cast<void**>(&z), S * 8, cudaHostAllocDefault);
  std::vector<double> u(S);
  hs_synthetic_uniform(21, S, 0.0, 1.0, u.data());
  for (uint64_t i = 0; i < S; ++i) x[i] = 50.0 + 10.0 * std::sqrt(-2 * std::log(u[i] + 1e-12)) * std::cos(6.283185307179586 * u[(i + 1) % S]);
  hs_invroot_cfg cfg{2, 511, 6, 0, 0, 0};
  auto now = [] { return std::chrono::steady_clock::now(); };
  auto us = [](auto a, auto b) { return std::chrono::duration<double, std::micro>(b - a).count(); };
  double t_enc = 0, t_z = 0, t_dec = 0;
  const int N = 300;
  for (int it = 0; it < N + 20; ++it) {
    hs_ct* chunk = nullptr;
    uint64_t nch = 0;
    auto t0 = now();
    hs_encode_column(ctx, x, S, &chunk, &nch);
    auto t1 = now();
    hs_column col{&chunk, 1, S};
    hs_ct* out = nullptr;
    hs_znorm(ctx, &col, 100.0, &cfg, &out);
    auto t2 = now();
    hs_column zc{&out, 1, S};
    hs_decode_column(ctx, &zc, z);
    auto t3 = now();
    hs_ct_release(chunk);
    hs_ct_release(out);
    if (it >= 20) {
      t_enc += us(t0, t1);
      t_z += us(t1, t2);
      t_dec += us(t2, t3);
    }
  }
  std::printf("C++ e2e: encode %.1f us, znorm enqueue %.1f us, decode (incl. wait) %.1f us, total %.1f us\n",
              t_enc / N, t_z / N, t_dec / N, (t_enc + t_z + t_dec) / N);
  {  // pipelined: encode step k+1 while step k computes
    hs_ct* cur = nullptr;
    uint64_t nch = 0;
    auto t0 = now();
    hs_encode_column(ctx, x, S, &cur, &nch);
    double pz = 0, pe = 0, pd = 0;
    for (int it = 0; it < N; ++it) {
      hs_column col{&cur, 1, S};
      hs_ct* out = nullptr;
      auto a = now();
      hs_znorm(ctx, &col, 100.0, &cfg, &out);
      auto b = now();
      hs_ct* next = nullptr;
      if (it + 1 < N) hs_encode_column(ctx, x, S, &next, &nch);
      auto c = now();
      hs_column zc{&out, 1, S};
      hs_decode_column(ctx, &zc, z);
      auto d = now();
      pz += us(a, b), pe += us(b, c), pd += us(c, d);
      hs_ct_release(cur);
      hs_ct_release(out);
      cur = next;
    }
    auto t1 = now();
    std::printf("C++ e2e pipelined: %.1f us/step (znorm enqueue %.1f, encode next %.1f, decode %.1f)\n",
                us(t0, t1) / N, pz / N, pe / N, pd / N);
  }
  // znorm enqueue alone, device kept busy
  hs_ct* chunk = nullptr;
  uint64_t nch = 0;
  hs_encode_column(ctx, x, S, &chunk, &nch);
  hs_column col{&chunk, 1, S};
  hs_sync();
  auto t0 = now();
  for (int it = 0; it < N; ++it) {
    hs_ct* out = nullptr;
    hs_znorm(ctx, &col, 100.0, &cfg, &out);
    hs_ct_release(out);
  }
  auto t1 = now();
  hs_sync();
  auto t2 = now();
  std::printf("znorm: %.1f us/call host enqueue, %.1f us/call incl. drain\n", us(t0, t1) / N, us(t0, t2) / N);
  return 0;
}
