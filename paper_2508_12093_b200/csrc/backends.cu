// backends.cu — DevB: one CUDA kernel per EvalContext op (ckks.hpp:97-230).
#include "backends.h"

#include <cstring>
#include <mutex>
#include <vector>
#include <string>

namespace hsg {

DevB::DevB(const Params& p, Meter& m) : LedgerBase(p, m) {
  qs_.mode = p.quantize ? QMode::Exact : QMode::None;
  qs_.bits = p.scale_bits;
}

namespace {
// Where the device can read the caller's buffer directly (pinned, host-mapped
// under UVA) the encrypt kernel reads it zero-copy; otherwise stage it through
// a device buffer.  Returns the device-visible source pointer.
// Large pinned inputs (>= kDmaBytes) go through the copy engine instead (encrypt_column's own
// branch, or the staged copy below for a single ciphertext): the DMA runs at PCIe rate beside a
// statistics kernel that fills every SM (a zero-copy k_encrypt would queue behind it, and reads
// host memory at less than half that rate), and the encrypt kernel then reads HBM.
constexpr size_t kDmaBytes = size_t(2) << 20;
const double* device_source(const double* v, size_t n, DevBuf* stage, bool* pinned, cudaStream_t s) {
  Runtime& rt = Runtime::get();
  cudaPointerAttributes at{};
  *pinned = cudaPointerGetAttributes(&at, v) == cudaSuccess && at.type == cudaMemoryTypeHost;
  cudaGetLastError();
  if (*pinned && at.devicePointer && n * sizeof(double) < kDmaBytes)
    return static_cast<const double*>(at.devicePointer);
  if (at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged) return v;
  *stage = s == rt.stream() ? rt.alloc(n) : rt.alloc_on(n, s);
  cuda_ok(cudaMemcpyAsync(stage->get(), v, n * sizeof(double), cudaMemcpyHostToDevice, s), "encrypt upload");
  return stage->get();
}

int* bad_flag() {  // host-mapped pinned flag word, one per thread
  thread_local int* f = nullptr;
  if (!f) cuda_ok(cudaHostAlloc(reinterpret_cast<void**>(&f), sizeof(int), cudaHostAllocMapped), "flag alloc");
  return f;
}

// flag words of asynchronous encodes (one per call in flight), recycled
std::mutex g_flag_mu;
std::vector<int*> g_flags;
int* take_flag() {
  {
    std::lock_guard<std::mutex> g(g_flag_mu);
    if (!g_flags.empty()) {
      int* f = g_flags.back();
      g_flags.pop_back();
      return f;
    }
  }
  int* f = nullptr;
  cuda_ok(cudaHostAlloc(reinterpret_cast<void**>(&f), sizeof(int), cudaHostAllocMapped), "flag alloc");
  return f;
}
void give_flag(int* f) {
  std::lock_guard<std::mutex> g(g_flag_mu);
  g_flags.push_back(f);
}
}  // namespace

void EncodePending::finish() {
  const bool nf = bad && *bad;
  if (bad) give_flag(bad);
  bad = nullptr;
  stage.reset();
  block.reset();
  if (nf) fail(HS_E_NON_FINITE_VALUE, "encode_column: non-finite value in column");
}
EncodePending::~EncodePending() {
  if (bad) give_flag(bad);
}

Ct DevB::encrypt(const double* v, size_t n) const {
  if (n > p_.S) fail(HS_E_TOO_MANY_VALUES, "encrypt: more values than slots");
  Runtime& rt = Runtime::get();
  DevBuf d = rt.alloc(p_.S);
  DevBuf stage;
  bool pinned = false;
  const double* src = n ? device_source(v, n, &stage, &pinned, rt.stream()) : nullptr;
  if (pinned && rt.capturing())  // a captured graph would keep reading the caller's buffer later
    fail(HS_E_INVALID_ARG, "encrypt of a pinned host buffer cannot be captured into a graph");
  k::encrypt(qs_, src, n, d.get(), p_.S, nullptr, rt.stream());
  if (pinned) rt.sync();  // the caller may reuse its pinned buffer on return
  return ct_device(d, p_.S, p_.max_level, p_.quantize ? p_.scale_bits : 0);
}

std::vector<Ct> DevB::encrypt_column(const double* v, size_t n, EncodePending* pend) const {
  Runtime& rt = Runtime::get();
  std::vector<Ct> out;
  if (n == 0) return out;
  // The column is read from host memory and its finiteness verdict is needed before
  // returning (a stream synchronisation), neither of which a CUDA graph can capture.
  if (rt.capturing())
    fail(HS_E_INVALID_ARG, "encode_column cannot run inside hs_graph_begin/hs_graph_end: encode the "
                           "columns first and capture the computation on them");
  // On an upload stream: the host input is read and encrypted beside whatever the compute
  // stream is running, and only this work is waited for below.
  const unsigned ui = rt.next_upload();
  cudaStream_t s = rt.upload_stream_at(ui);
  const size_t nch = (n + p_.S - 1) / p_.S;
  int* bad = pend ? take_flag() : bad_flag();
  *bad = 0;
  DevBuf stage, block;
  bool pinned = false;
  cudaPointerAttributes at{};
  const bool host_pinned = cudaPointerGetAttributes(&at, v) == cudaSuccess && at.type == cudaMemoryTypeHost;
  cudaGetLastError();
  const double* src;
  if (host_pinned && n * sizeof(double) >= kDmaBytes) {
    // Large pinned column: copy-engine DMA into the stream's persistent staging buffer, output
    // block from the compute stream's pool (whose freed blocks are reusable at once; an
    // upload-stream allocation would have to map new memory whenever the pool's free blocks still
    // wait on compute-stream work), the encrypt kernel ordered behind the allocation point.
    double* st = rt.upload_stage(ui, n);
    cuda_ok(cudaMemcpyAsync(st, v, n * sizeof(double), cudaMemcpyHostToDevice, s), "encrypt upload");
    block = rt.alloc(nch * p_.S);
    const auto here = rt.mark_on(rt.stream());
    cuda_ok(cudaStreamWaitEvent(s, here->e, 0), "encode_column order");
    src = st;
    pinned = true;
  } else {
    src = device_source(v, n, &stage, &pinned, s);
    block = rt.alloc_on(nch * p_.S, s);
  }
  // One allocation and one launch for the whole column: chunk c is the slice [c S, (c + 1) S) of
  // the block (zero padding behind the last value included), so the kernel is the single-chunk
  // one over n values and nch * S slots.
  k::encrypt(qs_, src, n, block.get(), nch * p_.S, bad, s);
  for (size_t c = 0; c < nch; ++c)
    out.push_back(ct_device(DevBuf(block, block.get() + c * p_.S), p_.S, p_.max_level,
                            p_.quantize ? p_.scale_bits : 0));
  // the finiteness verdict (and the caller's buffer) must be settled before returning; the
  // outputs are then complete for any later compute-stream work
  if (pend) {  // asynchronous: consumers order themselves behind `done` (CtData::device)
    pend->done = rt.mark_on(s);
    pend->bad = bad;
    pend->stage = std::move(stage);
    pend->block = block;
    for (const Ct& c : out) c->filling = pend->done;
    return out;
  }
  rt.wait(s);  // releases the API lock while this thread sleeps (api.cu wait_unlocked)
  if (*bad) fail(HS_E_NON_FINITE_VALUE, "encode_column: non-finite value in column");
  return out;
}

Ct DevB::encrypt_const(double c) const {
  std::vector<double> v(p_.S, c);
  return encrypt(v.data(), v.size());
}

Ct DevB::addsub(const C& a, const C& b, k::BinOp op) {  // ckks.hpp:113-133
  check_shape(sz(a));
  check_shape(sz(b));
  DevBuf o = Runtime::get().alloc(p_.S);
  k::binary(qs_, op, a->device(), b->device(), o.get(), p_.S, Runtime::get().stream());
  ++m_.add;
  return ct_device(o, p_.S, std::min(a->level, b->level), p_.quantize ? p_.scale_bits : 0);
}

Ct DevB::add_pt(const C& a, double c) {  // ckks.hpp:137-144
  check_shape(sz(a));
  DevBuf o = Runtime::get().alloc(p_.S);
  k::scalar(qs_, k::S_ADD, a->device(), c, o.get(), p_.S, Runtime::get().stream());
  ++m_.add;
  return ct_device(o, p_.S, a->level, p_.quantize ? p_.scale_bits : 0);
}

Ct DevB::bootstrap(const C& a) {  // ckks.hpp:207-213
  check_shape(sz(a));
  DevBuf o = Runtime::get().alloc(p_.S);
  k::requant(qs_, a->device(), o.get(), p_.S, Runtime::get().stream());
  ++m_.bootstrap;
  return ct_device(o, p_.S, p_.max_level, p_.quantize ? p_.scale_bits : a->grid);
}

Ct DevB::mul_ct(C a, C b) {  // ckks.hpp:149-164
  check_shape(sz(a));
  check_shape(sz(b));
  if (std::min(a->level, b->level) < 1) {
    if (!p_.auto_bootstrap) fail(HS_E_LEVEL_EXHAUSTED, "mul_ct: no multiplicative level left");
    if (a->level < 1) a = bootstrap(a);
    if (b->level < 1) b = bootstrap(b);
  }
  DevBuf o = Runtime::get().alloc(p_.S);
  k::binary(qs_, k::B_MUL, a->device(), b->device(), o.get(), p_.S, Runtime::get().stream());
  ++m_.mul_ct;
  return ct_device(o, p_.S, std::min(a->level, b->level) - 1, p_.quantize ? p_.scale_bits : 0);
}

Ct DevB::prepare_mul_pt(C a) {  // ckks.hpp:233-240
  if (a->level < 1) {
    if (!p_.auto_bootstrap) fail(HS_E_LEVEL_EXHAUSTED, "mul_pt: no multiplicative level left");
    a = bootstrap(a);
  }
  return a;
}

Ct DevB::mul_pt(C a, double c) {  // ckks.hpp:168-176
  check_shape(sz(a));
  a = prepare_mul_pt(a);
  DevBuf o = Runtime::get().alloc(p_.S);
  k::scalar(qs_, k::S_MUL, a->device(), c, o.get(), p_.S, Runtime::get().stream());
  ++m_.mul_pt;
  return ct_device(o, p_.S, a->level - 1, p_.quantize ? p_.scale_bits : 0);
}

Ct DevB::mul_pt_vec(C a, const std::vector<double>& v) {  // ckks.hpp:179-189
  check_shape(sz(a));
  if (v.size() != p_.S) fail(HS_E_LENGTH_MISMATCH, "mul_pt: plaintext vector length != slot count");
  a = prepare_mul_pt(a);
  Runtime& rt = Runtime::get();
  DevBuf pv = rt.alloc(p_.S);
  cuda_ok(cudaMemcpyAsync(pv.get(), v.data(), p_.S * sizeof(double), cudaMemcpyHostToDevice, rt.stream()),
          "mul_pt plaintext upload");
  DevBuf o = rt.alloc(p_.S);
  k::binary(qs_, k::B_MUL, a->device(), pv.get(), o.get(), p_.S, rt.stream());
  ++m_.mul_pt;
  return ct_device(o, p_.S, a->level - 1, p_.quantize ? p_.scale_bits : 0);
}

Ct DevB::rotate(const C& a, long kk) {  // ckks.hpp:193-202
  check_shape(sz(a));
  const long n = static_cast<long>(p_.S);
  const long shift = ((kk % n) + n) % n;
  DevBuf o = Runtime::get().alloc(p_.S);
  k::rotate(a->device(), o.get(), p_.S, static_cast<size_t>(shift), Runtime::get().stream());
  ++m_.rotate;
  return ct_device(o, p_.S, a->level, a->grid);
}

Ct DevB::sum_all_slots(const C& a, size_t n_valid) {  // ckks.hpp:218-230
  check_shape(sz(a));
  if (p_.debug && n_valid < p_.S) {
    const double eps = std::ldexp(1.0, -(p_.scale_bits - 1));
    const std::vector<double>& h = a->host_slots();
    for (size_t i = n_valid; i < p_.S; ++i)
      if (std::abs(h[i]) > eps) fail(HS_E_DIRTY_PADDING, "sum_all_slots: nonzero padding slot");
  }
  DevBuf o = Runtime::get().alloc(p_.S);
  const double* src = a->device();
  double* dst = o.get();
  k::slot_sum(qs_, &src, &dst, 1, p_.S, Runtime::get().stream());
  int steps = 0;
  for (size_t s = 1; s < p_.S; s <<= 1) ++steps;
  m_.rotate += steps;
  m_.add += steps;
  int grid = p_.quantize ? p_.scale_bits : 0;
  if (steps == 0) grid = a->grid;  // S == 1: no add, value passes through untouched
  return ct_device(o, p_.S, a->level, grid);
}

// ---- batched ops (C5) -------------------------------------------------------------------------
std::vector<Ct> DevB::binary_batch(const std::vector<Ct>& a, const std::vector<Ct>& b, k::BinOp op) {
  if (a.size() != b.size()) fail(HS_E_LENGTH_MISMATCH, "batch: operand counts differ");
  const size_t n = a.size();
  std::vector<Ct> x(a), y(b);
  std::vector<int> lvl(n);
  for (size_t i = 0; i < n; ++i) {  // ckks.hpp:113-164, element by element
    check_shape(sz(x[i]));
    check_shape(sz(y[i]));
    if (op == k::B_MUL) {
      if (std::min(x[i]->level, y[i]->level) < 1) {
        if (!p_.auto_bootstrap) fail(HS_E_LEVEL_EXHAUSTED, "mul_ct: no multiplicative level left");
        if (x[i]->level < 1) x[i] = bootstrap(x[i]);
        if (y[i]->level < 1) y[i] = bootstrap(y[i]);
      }
      ++m_.mul_ct;
      lvl[i] = std::min(x[i]->level, y[i]->level) - 1;
    } else {
      ++m_.add;
      lvl[i] = std::min(x[i]->level, y[i]->level);
    }
  }
  std::vector<Ct> out;
  if (n == 0) return out;
  Runtime& rt = Runtime::get();
  DevBuf block = rt.alloc(n * p_.S);
  std::vector<const double*> pa(n), pb(n);
  std::vector<double*> po(n);
  for (size_t i = 0; i < n; ++i) {
    pa[i] = x[i]->device();
    pb[i] = y[i]->device();
    po[i] = block.get() + i * p_.S;
  }
  k::binary_batch(qs_, op, pa.data(), pb.data(), po.data(), n, p_.S, rt.stream());
  for (size_t i = 0; i < n; ++i)
    out.push_back(ct_device(DevBuf(block, po[i]), p_.S, lvl[i], p_.quantize ? p_.scale_bits : 0));
  return out;
}

std::vector<Ct> DevB::scalar_batch(const std::vector<Ct>& a, double c, k::ScalOp op) {
  const size_t n = a.size();
  std::vector<Ct> x(a);
  std::vector<int> lvl(n);
  for (size_t i = 0; i < n; ++i) {  // ckks.hpp:137-176
    check_shape(sz(x[i]));
    if (op == k::S_MUL) {
      x[i] = prepare_mul_pt(x[i]);
      ++m_.mul_pt;
      lvl[i] = x[i]->level - 1;
    } else {
      ++m_.add;
      lvl[i] = x[i]->level;
    }
  }
  std::vector<Ct> out;
  if (n == 0) return out;
  Runtime& rt = Runtime::get();
  DevBuf block = rt.alloc(n * p_.S);
  std::vector<const double*> pa(n);
  std::vector<double*> po(n);
  for (size_t i = 0; i < n; ++i) {
    pa[i] = x[i]->device();
    po[i] = block.get() + i * p_.S;
  }
  k::scalar_batch(qs_, op, pa.data(), c, po.data(), n, p_.S, rt.stream());
  for (size_t i = 0; i < n; ++i)
    out.push_back(ct_device(DevBuf(block, po[i]), p_.S, lvl[i], p_.quantize ? p_.scale_bits : 0));
  return out;
}

std::vector<Ct> DevB::rotate_batch(const std::vector<Ct>& a, long kk) {  // ckks.hpp:193-202
  const size_t n = a.size();
  for (size_t i = 0; i < n; ++i) {
    check_shape(sz(a[i]));
    ++m_.rotate;
  }
  std::vector<Ct> out;
  if (n == 0) return out;
  const long S = static_cast<long>(p_.S);
  const size_t shift = static_cast<size_t>(((kk % S) + S) % S);
  Runtime& rt = Runtime::get();
  DevBuf block = rt.alloc(n * p_.S);
  std::vector<const double*> pa(n);
  std::vector<double*> po(n);
  for (size_t i = 0; i < n; ++i) {
    pa[i] = a[i]->device();
    po[i] = block.get() + i * p_.S;
  }
  k::rotate_batch(pa.data(), po.data(), n, p_.S, shift, rt.stream());
  for (size_t i = 0; i < n; ++i) out.push_back(ct_device(DevBuf(block, po[i]), p_.S, a[i]->level, a[i]->grid));
  return out;
}

// ---- debug-mode value checks (host reads; debug is the diagnostics path) ----
double DevB::first_slot(const C& c) {  // stats.hpp:89-91 (decrypt(ct, 1)[0])
  double v = 0.0;
  c->read(&v, 1);
  return v;
}

void DevB::check_open_domain(const C& c, size_t n_valid, double lo, double hi, const char* who) {
  const size_t n = std::min(n_valid, c->n);  // primitives.hpp:134-144
  const std::vector<double>& h = c->host_slots();
  for (size_t i = 0; i < n; ++i) {
    const double t = h[i];
    if (!(t > lo) || !(t <= hi)) fail(HS_E_DOMAIN_VIOLATION, std::string(who) + ": scaled slot outside domain");
  }
}

void DevB::check_eval_domain(const C& c, double lo, double hi) {  // chebyshev.hpp:174-179
  const double eps = 1e-9;
  for (double v : c->host_slots())
    if (v < lo - eps || v > hi + eps) fail(HS_E_DOMAIN_VIOLATION, "eval_encrypted: slot outside series domain");
}

void DevB::check_divergence(const C& c, size_t n_valid) {  // primitives.hpp:89-96
  const size_t n = std::min(n_valid, c->n);
  const std::vector<double>& h = c->host_slots();
  for (size_t i = 0; i < n; ++i)
    if (!(std::abs(h[i]) <= 1e6)) fail(HS_E_DIVERGENCE, "newton iterate exceeded the divergence guard");
}

void DevB::check_sqrt_domain(const C& c, size_t n_valid) {  // primitives.hpp:225-232
  const size_t n = std::min(n_valid, c->n);
  const std::vector<double>& h = c->host_slots();
  for (size_t i = 0; i < n; ++i)
    if (h[i] < -1e-9 || h[i] > 2.0 + 1e-9) fail(HS_E_DOMAIN_VIOLATION, "crypto_sqrt: scaled slot outside [0, 2]");
}

void DevB::check_sign_domain(const C& c) {  // primitives.hpp:282-286
  for (double v : c->host_slots())
    if (v < -1.0 - 1e-9 || v > 1.0 + 1e-9) fail(HS_E_DOMAIN_VIOLATION, "crypto_sign: slot outside [-1, 1]");
}

}  // namespace hsg
