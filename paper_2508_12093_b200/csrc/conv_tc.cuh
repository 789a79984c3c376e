// conv_tc.cuh — fast base conversion on the 5th-generation tensor cores
// (tcgen05.mma kind::i8, accumulators in TMEM), included by rns.cu.
//
// out_t[n] = sum_i y_i[n] h[t][i] mod q_t,  y_i = [x_i hinv_i]_{q_i}, is an exact
// integer GEMM over bytes (the same identity as k_conv_mma, rns.cu):
//   A[n][8i + a]     = byte a of y_i[n]                      M = 128 coefficients
//   B[8t + b][8i + a] = byte b of (h[t][i] 2^(8a) mod q_t)   N = 8 x targets (host-built)
//   D[n][8t + b]     = sum_k A[n][k] B[8t + b][k] < 8 nsrc 255^2 < 2^23   (exact s32)
//   out_t[n]         = sum_b D[n][8t + b] 2^(8b) mod q_t
// A tile is 128 coefficients of one job, converted to every target at once.  CTAs are
// persistent (one per SM, 16 warps) and walk a contiguous run of one job's tiles:
//   * B (the job's constant matrix, <= 32 KB) lands in shared memory once, by one
//     bulk copy (cp.async.bulk, the TMA engine) completing on an mbarrier;
//   * A: the threads load a tile's source residues (coalesced), multiply by hinv_i and
//     store each coefficient's residues as its K-major A row (16-byte core-matrix
//     rows, SWIZZLE_NONE canonical layout); two A buffers;
//   * one elected thread issues KS x ceil(N / 256) tcgen05.mma (K = 32 bytes each)
//     into one of two TMEM accumulators and commits them to that buffer's mbarrier;
//   * every warp reads its 32 TMEM lanes (= 32 coefficients) with tcgen05.ld: each
//     thread owns one coefficient and gets a target's 8 byte-column sums in 8
//     consecutive registers, so the recombination and the modular reduction run in
//     registers and the store is a coalesced row segment.
// Warp roles: 16 compute warps and one MMA warp.  Compute warps, iteration j: store
// A(j+1) from the registers loaded during iteration j-1, issue the global loads of
// tile j+2, arrive on ready[(j+1) & 1]; wait full[j & 1]; epilogue(j).  The MMA warp:
// wait ready[j & 1] (A(j) stored, and every epilogue of tile j-2 done with that
// accumulator), issue MMA(j), commit to full[j & 1].  No CTA-wide barrier per tile.
// The output is canonical, so it equals k_conv's / k_conv_mma's word for word.
#pragma once

namespace tc {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_fence_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ bool mbar_test(uint32_t bar, uint32_t phase) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(bar), "r"(phase)
      : "memory");
  return ok != 0;
}
// polling with a back-off: a spinning warp would take issue slots from the compute warps
__device__ __forceinline__ void mbar_wait_sleep(uint32_t bar, uint32_t phase, uint32_t ns) {
  while (!mbar_test(bar, phase)) __nanosleep(ns);
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t phase) {
  uint32_t ok = 0;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(bar), "r"(phase)
        : "memory");
  } while (!ok);
}
// global -> shared bulk copy (TMA engine), completion counted in bytes on `bar`
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
               "l"(src), "r"(bytes), "r"(bar)
               : "memory");
}
// generic-proxy shared-memory writes -> visible to the tensor core (async proxy)
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

__device__ __forceinline__ void tmem_alloc(uint32_t slot, uint32_t ncols) {  // one full warp
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(slot), "r"(ncols) : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t ncols) {  // the allocating warp
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols) : "memory");
}

// Shared-memory matrix descriptor, SWIZZLE_NONE K-major canonical layout: core
// matrices of 8 rows x 16 bytes (128 contiguous bytes); LBO = byte distance between
// the two K-adjacent core matrices of one MMA (K = 32 bytes), SBO = byte distance
// between 8-row groups.  Version 1 (sm_100).
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return uint64_t((saddr >> 4) & 0x3FFFu) | (uint64_t((lbo >> 4) & 0x3FFFu) << 16) |
         (uint64_t((sbo >> 4) & 0x3FFFu) << 32) | (uint64_t(1) << 46);
}
// Instruction descriptor of tcgen05.mma kind::i8: D s32, A and B unsigned 8-bit,
// both K-major, M = 128, N (multiple of 16, <= 256).
__host__ __device__ constexpr uint32_t idesc_u8(uint32_t n) {
  return (2u << 4) | (0u << 7) | (0u << 10) | ((n >> 3) << 17) | ((128u >> 4) << 24);
}
__device__ __forceinline__ void mma_u8(uint32_t dtmem, uint64_t ad, uint64_t bd, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(dtmem),
      "l"(ad), "l"(bd), "r"(idesc), "r"(acc)
      : "memory");
}
__device__ __forceinline__ void mma_commit(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar) : "memory");
}
// 32 lanes x 8 consecutive 32-bit columns: thread i of the warp gets lane (base lane + i)
__device__ __forceinline__ void tmem_ld8(uint32_t taddr, uint32_t (&v)[8]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
               : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
               : "r"(taddr));
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

}  // namespace tc

constexpr int kTcRows = 128;      // coefficients per tile (MMA M)
constexpr int kTcCompute = 512;  // 16 compute warps: 4 per TMEM lane quarter, 4 threads per A row
constexpr int kTcThreads = kTcCompute + 32;  // + the MMA-issuing warp
constexpr int kTcParts = kTcCompute / kTcRows;

struct TcTgt {
  double qd, qinvd, c32d;  // fp targets: q, 1/q, 2^32 mod q
  uint64_t off;            // output row offset (words) inside a batch item
  uint32_t fp;
};

__host__ __device__ constexpr uint32_t tc_rows(uint32_t ntgt) { return (8 * ntgt + 15) / 16 * 16; }
// two accumulators when they fit in TMEM's 512 columns (targets <= 32), else one (the next
// tile's MMAs then wait for the current epilogue)
__host__ __device__ constexpr bool tc_dbuf(uint32_t rows) { return 2 * rows <= 512; }
__host__ __device__ constexpr uint32_t tc_cols(uint32_t rows) {
  return 2 * rows <= 32 ? 32 : 2 * rows <= 64 ? 64 : 2 * rows <= 128 ? 128 : 2 * rows <= 256 ? 256 : 512;
}
template <int KS>
constexpr uint32_t tc_smem_a() {
  return uint32_t(2 * KS) * kTcRows * 16;  // one A buffer
}

// KS = k-steps of 32 bytes (nsrc <= 4 KS); blockIdx.y = job, blockIdx.x = run of tiles
// over (batch item, coefficient tile), `per` tiles per CTA.
template <int KS>
__global__ void __launch_bounds__(kTcThreads, 1) k_conv_tc(const uint64_t* in, size_t in_stride, uint64_t* out,
                                                          size_t out_stride, const ConvJob* jobs, const uint8_t* img,
                                                          const PrimeC* pcs, uint32_t logN, uint32_t ntiles,
                                                          uint32_t per) {
  constexpr uint32_t KC = 2 * KS;                   // 16-byte K chunks (two sources each)
  constexpr uint32_t CPT = (KC + kTcParts - 1) / kTcParts;  // chunks per thread
  extern __shared__ __align__(128) uint8_t tc_smem[];
  uint8_t* As = tc_smem;                            // [2][KC][128 rows][16 B]
  uint8_t* Bs = tc_smem + 2 * tc_smem_a<KS>();      // [KC][NR rows][16 B]
  __shared__ __align__(8) uint64_t bars[5];  // 0: B landed; 1, 2: full (MMAs done); 3, 4: ready (A stored)
  __shared__ uint32_t tslot;
  __shared__ TcTgt tgs[kMaxTgt];
  __shared__ PrimeC tq[kMaxTgt];
  __shared__ uint64_t hinv_s[4 * KS], hinvsh_s[4 * KS], qs_s[4 * KS];
  const ConvJob& J = jobs[blockIdx.y];
  const uint32_t nsrc = J.nsrc, ntgt = J.ntgt, NR = tc_rows(ntgt), ncols = tc_cols(NR);
  const bool dbuf = tc_dbuf(NR);
  const uint32_t t0 = blockIdx.x * per, t1 = min(t0 + per, ntiles);
  if (t0 >= t1) return;
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t bar_b = tc::smem_u32(&bars[0]);
  auto full = [&](uint32_t b) { return tc::smem_u32(&bars[1 + b]); };
  auto ready = [&](uint32_t b) { return tc::smem_u32(&bars[3 + b]); };
  if (threadIdx.x == 0) {
    tc::mbar_init(bar_b, 1);
    tc::mbar_init(full(0), 1);
    tc::mbar_init(full(1), 1);
    tc::mbar_init(ready(0), kTcCompute / 32);
    tc::mbar_init(ready(1), kTcCompute / 32);
    tc::mbar_fence_init();
  }
  if (warp == 0) tc::tmem_alloc(tc::smem_u32(&tslot), ncols);
  for (uint32_t k = threadIdx.x; k < ntgt; k += kTcThreads) {
    const PrimeC P = pcs[J.tgt[k]];
    tq[k] = P;
    const uint64_t c32 = (uint64_t(1) << 32) % P.q;
    tgs[k] = TcTgt{P.qd, P.qinvd, static_cast<double>(c32), uint64_t(J.out_row + J.tgt_row[k]) << logN, P.fp};
  }
  if (threadIdx.x < nsrc) {
    hinv_s[threadIdx.x] = J.hinv[threadIdx.x];
    hinvsh_s[threadIdx.x] = J.hinv_sh[threadIdx.x];
    qs_s[threadIdx.x] = pcs[J.src[threadIdx.x]].q;
  }
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = tslot;
  const uint32_t tiles_per_item = 1u << (logN - 7);
  auto issue = [&](uint32_t buf) {  // one thread: the tile's MMAs into accumulator `buf`
    const uint32_t a0 = tc::smem_u32(As + buf * tc_smem_a<KS>()), b0 = tc::smem_u32(Bs);
    for (uint32_t nb = 0; nb < NR; nb += 256) {
      const uint32_t n = NR - nb < 256 ? NR - nb : 256;
      const uint32_t id = tc::idesc_u8(n);
#pragma unroll
      for (int ks = 0; ks < KS; ++ks) {
        const uint64_t ad = tc::sdesc(a0 + 2 * ks * kTcRows * 16, kTcRows * 16, 128);
        const uint64_t bd = tc::sdesc(b0 + 2 * ks * NR * 16 + nb * 16, NR * 16, 128);
        tc::mma_u8(tmem + (dbuf ? buf * NR : 0) + nb, ad, bd, id, ks > 0 ? 1u : 0u);
      }
    }
    tc::mma_commit(full(buf));
  };
  if (warp == kTcCompute / 32) {  // ---- the MMA warp ----
    if (lane == 0) {
      const uint32_t bytes = KC * NR * 16;  // the job's B image: one bulk copy
      tc::mbar_expect_tx(bar_b, bytes);
      tc::bulk_g2s(tc::smem_u32(Bs), img + J.img_off, bytes, bar_b);
      tc::mbar_wait(bar_b, 0);
      for (uint32_t j = 0; j < t1 - t0; ++j) {
        tc::mbar_wait_sleep(ready(j & 1), (j >> 1) & 1, 32);
        tc::fence_after();
        issue(j & 1);
      }
    }
    __syncwarp();
  } else {  // ---- compute warps ----
  // A rows: thread (row m, part p) owns chunks p, p + 4, ... of row m
  const uint32_t m = threadIdx.x & (kTcRows - 1), part = threadIdx.x / kTcRows;
  uint64_t x[CPT][2];
  auto load = [&](uint32_t tile) {
    const uint32_t item = tile / tiles_per_item, n0 = (tile % tiles_per_item) * kTcRows;
    const uint64_t* I = in + item * in_stride + (size_t(J.in_row) << logN) + n0 + m;
#pragma unroll
    for (uint32_t c = 0; c < CPT; ++c) {
      const uint32_t kc = part + kTcParts * c, i0 = 2 * kc, i1 = i0 + 1;
      x[c][0] = kc < KC && i0 < nsrc ? __ldcs(I + (size_t(i0) << logN)) : 0;
      x[c][1] = kc < KC && i1 < nsrc ? __ldcs(I + (size_t(i1) << logN)) : 0;
    }
  };
  auto store_a = [&](uint32_t buf) {  // then this warp's arrival on ready[buf]
    uint8_t* A = As + buf * tc_smem_a<KS>();
#pragma unroll
    for (uint32_t c = 0; c < CPT; ++c) {
      const uint32_t kc = part + kTcParts * c, i0 = 2 * kc, i1 = i0 + 1;
      if (kc >= KC) break;
      const uint64_t y0 = i0 < nsrc ? mul_shoup(x[c][0], hinv_s[i0], hinvsh_s[i0], qs_s[i0]) : 0;
      const uint64_t y1 = i1 < nsrc ? mul_shoup(x[c][1], hinv_s[i1], hinvsh_s[i1], qs_s[i1]) : 0;
      *reinterpret_cast<uint4*>(A + (kc * kTcRows + m) * 16) =
          make_uint4(uint32_t(y0), uint32_t(y0 >> 32), uint32_t(y1), uint32_t(y1 >> 32));
    }
    tc::fence_async_smem();
    tc::fence_before();
    __syncwarp();
    if (lane == 0) tc::mbar_arrive(ready(buf));
  };
  // epilogue mapping: warp w reads TMEM lanes 32 (w & 3) .. + 31; the four warps of a lane
  // quarter take targets g, g + 4, ... (g = w >> 2)
  const uint32_t q4 = warp & 3, grp = warp >> 2;
  // lo = sum_{b<4} v_b 2^(8b), hi = sum_{b>=4} v_b 2^(8(b-4)), each < 2^47 (v_b < 2^23)
  auto lohi = [](const uint32_t (&v)[8], uint64_t& lo, uint64_t& hi) {
    lo = (uint64_t(v[2] + (v[3] << 8)) << 16) + (v[0] + (v[1] << 8));
    hi = (uint64_t(v[6] + (v[7] << 8)) << 16) + (v[4] + (v[5] << 8));
  };
  auto fin_int = [&](uint64_t* O, uint32_t t, const uint32_t (&v)[8]) {
    uint64_t lo, hi;
    lohi(v, lo, hi);
    __stcs(O + tgs[t].off, reduce128((static_cast<u128>(hi) << 32) + lo, tq[t]));
  };
  // targets < 2^45: lo + hi (2^32 mod q) on the FP64 pipe, every step exact
  auto fin_fp = [&](uint64_t* O, uint32_t t, const uint32_t (&v)[8]) {
    uint64_t lo, hi;
    lohi(v, lo, hi);
    const TcTgt T = tgs[t];
    const double hh = fp_mulmod(u2d(hi), T.c32d, T.qd, T.qinvd);
    __stcs(O + T.off, fp_canon(__dadd_rn(hh, u2d(lo)), T.qd, T.qinvd));
  };
  const uint32_t nint = J.nint;
  // prologue: A(t0) stored (ready[0]), loads of t0 + 1 in flight
  load(t0);
  store_a(0);
  if (t0 + 1 < t1) load(t0 + 1);
#pragma unroll 1
  for (uint32_t tile = t0, j = 0; tile < t1; ++tile, ++j) {
    const uint32_t buf = j & 1;
    if (tile + 1 < t1 && dbuf) {
      store_a(buf ^ 1);                  // the loads issued one iteration ago
      if (tile + 2 < t1) load(tile + 2);  // in flight during this epilogue
    }
    tc::mbar_wait_sleep(full(buf), (j >> 1) & 1, 64);
    tc::fence_after();
    const uint32_t item = tile / tiles_per_item, n0 = (tile % tiles_per_item) * kTcRows;
    uint64_t* O = out + item * out_stride + n0 + 32 * q4 + lane;
    const uint32_t taddr = tmem + ((32 * q4) << 16) + (dbuf ? buf * NR : 0);
    // integer targets first (at most a few), then the FP64 ones four at a time, branch-free
    uint32_t t = grp;
#pragma unroll 1
    for (; t < nint; t += 4) {
      uint32_t v0[8];
      tc::tmem_ld8(taddr + 8 * t, v0);
      tc::tmem_wait_ld();
      fin_int(O, t, v0);
    }
    t = nint + grp;
#pragma unroll 1
    for (; t + 12 < ntgt; t += 16) {
      uint32_t v0[8], v1[8], v2[8], v3[8];
      tc::tmem_ld8(taddr + 8 * t, v0);
      tc::tmem_ld8(taddr + 8 * (t + 4), v1);
      tc::tmem_ld8(taddr + 8 * (t + 8), v2);
      tc::tmem_ld8(taddr + 8 * (t + 12), v3);
      tc::tmem_wait_ld();
      fin_fp(O, t, v0);
      fin_fp(O, t + 4, v1);
      fin_fp(O, t + 8, v2);
      fin_fp(O, t + 12, v3);
    }
#pragma unroll 1
    for (; t < ntgt; t += 4) {
      uint32_t v0[8];
      tc::tmem_ld8(taddr + 8 * t, v0);
      tc::tmem_wait_ld();
      fin_fp(O, t, v0);
    }
    if (tile + 1 < t1 && !dbuf) {  // one accumulator: A(j+1) and its MMAs after this epilogue
      store_a(buf ^ 1);
      if (tile + 2 < t1) load(tile + 2);
    }
  }
  }  // compute warps
  tc::fence_before();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc(tmem, ncols);
}
