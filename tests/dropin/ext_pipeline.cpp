// tests/dropin/ext_pipeline.cpp — the C++ extension surface over the drop-in headers (our own
// source, not the reference's): znorm_batch and the asynchronous column transfers give the bits
// of the reference-shaped calls, a deferred non_finite_value is raised by wait(), and the
// three-stage host pipeline (encode k+1 | znorm_batch k | decode k) runs from pinned memory.
// Prints one line "ext_pipeline ok ... us/ciphertext"; any mismatch exits 1.
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <deque>
#include <vector>

#include <cuda_runtime_api.h>

#include "hestat/hestat.hpp"

using namespace hestat;

static bool same_bits(const double* a, const double* b, size_t n) { return std::memcmp(a, b, n * sizeof(double)) == 0; }

int main(int argc, char** argv) {
  const size_t S = argc > 1 ? std::stoul(argv[1]) : 32768;
  const size_t KB = argc > 2 ? std::stoul(argv[2]) : 64;
  const int steps = argc > 3 ? std::stoi(argv[3]) : 30;
  const double B = 100.0;
  CkksParams p;
  p.slot_count = S;
  EvalContext ctx(p);
  // KB columns of S values ~ N(50, 10^2) from the reference's seeded uniforms (data.hpp:148-160)
  std::vector<double> u = synthetic_uniform(21, 2 * S, 0.0, 1.0);
  std::vector<double> x(S);
  for (size_t i = 0; i < S; ++i)
    x[i] = 50.0 + 10.0 * std::sqrt(-2.0 * std::log(u[2 * i] + 1e-300)) * std::cos(6.283185307179586 * u[2 * i + 1]);
  constexpr int NBUF = 4;
  double *hx[NBUF], *hz[NBUF];
  for (int b = 0; b < NBUF; ++b) {
    if (cudaHostAlloc(reinterpret_cast<void**>(&hx[b]), KB * S * 8, cudaHostAllocDefault) != cudaSuccess ||
        cudaHostAlloc(reinterpret_cast<void**>(&hz[b]), KB * S * 8, cudaHostAllocDefault) != cudaSuccess) {
      std::fprintf(stderr, "pinned allocation failed\n");
      return 1;
    }
    for (size_t j = 0; j < KB; ++j)
      for (size_t i = 0; i < S; ++i) hx[b][j * S + i] = x[(i + 97 * j) % S];
    std::memset(hz[b], 0, KB * S * 8);
  }
  // reference-shaped calls: the expected bits
  std::vector<std::vector<double>> want;
  for (size_t j = 0; j < KB; ++j) {  // every column of the step
    const EncryptedColumn c = encode_column(ctx, std::span<const double>(hx[0] + j * S, S));
    want.push_back(decode_column(ctx, znorm(ctx, c, B)));
  }
  auto split = [&](const EncryptedColumn& big) {
    std::vector<EncryptedColumn> cols;
    for (const Ciphertext& c : big.chunks) {
      EncryptedColumn one;
      one.chunks.push_back(c);
      one.n_valid = S;
      cols.push_back(std::move(one));
    }
    return cols;
  };
  auto join = [&](const std::vector<EncryptedColumn>& zs) {
    EncryptedColumn all;
    for (const EncryptedColumn& z : zs) all.chunks.push_back(z.chunks.at(0));
    all.n_valid = zs.size() * S;
    return all;
  };
  // deferred error
  {
    std::vector<double> bad(hx[0], hx[0] + 2 * S);
    bad[S + 5] = std::nan("");
    Pending pe;
    const EncryptedColumn c = encode_column_async(ctx, bad, pe, "bad");
    bool threw = false;
    try {
      pe.wait();
    } catch (const non_finite_value&) {
      threw = true;
    }
    if (!threw) {
      std::fprintf(stderr, "non-finite input not reported by wait()\n");
      return 1;
    }
  }
  // handles dropped before their transfer has settled: the library keeps the buffers alive
  {
    Pending pe;
    { const EncryptedColumn gone = encode_column_async(ctx, std::span<const double>(hx[0], 2 * S), pe); }
    pe.wait();
    const EncryptedColumn c = encode_column(ctx, std::span<const double>(hx[0], S));
    std::vector<double> got(S, 0.0);
    Pending pd;
    {
      const EncryptedColumn z = znorm(ctx, c, B);
      pd = decode_column_async(ctx, z, got);
    }
    for (int i = 0; i < 4; ++i) (void)znorm(ctx, c, B);  // pool churn while the copy may be in flight
    pd.wait();
    if (!same_bits(got.data(), want[0].data(), S)) {
      std::fprintf(stderr, "decode_column_async of a released column differs\n");
      return 1;
    }
  }
  // the pipeline
  auto run = [&](int n) {
    Pending pe;
    std::vector<EncryptedColumn> cols = split(encode_column_async(ctx, std::span<const double>(hx[0], KB * S), pe));
    std::deque<Pending> dq;
    for (int k = 0; k < n; ++k) {
      const std::vector<EncryptedColumn> zs = znorm_batch(ctx, cols, B);
      Pending pk = std::move(pe);
      if (k + 1 < n)
        cols = split(encode_column_async(ctx, std::span<const double>(hx[(k + 1) % NBUF], KB * S), pe));
      dq.push_back(decode_column_async(ctx, join(zs), std::span<double>(hz[k % NBUF], KB * S)));
      pk.wait();
      while (dq.size() > 2) {
        dq.front().wait();
        dq.pop_front();
      }
    }
    while (!dq.empty()) {
      dq.front().wait();
      dq.pop_front();
    }
  };
  run(6);
  for (int b = 0; b < NBUF; ++b) std::memset(hz[b], 0, KB * S * 8);
  const auto t0 = std::chrono::steady_clock::now();
  run(steps);
  const double us = std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count();
  for (int b = 0; b < std::min(NBUF, steps); ++b)
    for (size_t j = 0; j < want.size(); ++j)
      if (!same_bits(hz[b] + j * S, want[j].data(), S)) {
        std::fprintf(stderr, "pipeline output differs from znorm(encode_column) at buffer %d column %zu\n", b, j);
        return 1;
      }
  std::printf("ext_pipeline ok: %zu x %zu slots per step, %d steps, %.2f us/ciphertext end to end (C++ host, pinned "
              "buffers, H2D + znorm_batch + D2H per step)\n", KB, S, steps, us / (double(steps) * double(KB)));
  return 0;
}
