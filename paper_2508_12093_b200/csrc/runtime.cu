// runtime.cu — device runtime and ciphertext storage (see core.h).
#include <cstdlib>
#include <cstring>
#include <string>

#include "core.h"
#include "kernels.h"

namespace hsg {

void cuda_ok(cudaError_t e, const char* what) {
  if (e != cudaSuccess) fail(HS_E_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

Params Params::from(const hs_params& p) {
  Params r;
  r.S = static_cast<size_t>(p.slot_count);
  r.max_level = p.max_level;
  r.scale_bits = p.scale_bits;
  r.quantize = p.quantize != 0;
  r.auto_bootstrap = p.auto_bootstrap != 0;
  r.debug = p.debug_checks != 0;
  return r;
}

hs_params Params::to() const {
  hs_params p{};
  p.slot_count = S;
  p.max_level = max_level;
  p.scale_bits = scale_bits;
  p.quantize = quantize;
  p.auto_bootstrap = auto_bootstrap;
  p.debug_checks = debug;
  return p;
}

// CkksParams::validate, ckks.hpp:34-39
void Params::validate() const {
  if (S == 0 || (S & (S - 1)) != 0) fail(HS_E_ERROR, "CkksParams: slot_count must be a power of two");
  if (max_level < 1) fail(HS_E_ERROR, "CkksParams: max_level must be >= 1");
  if (scale_bits < 1) fail(HS_E_ERROR, "CkksParams: scale_bits must be >= 1");
}

// ---- Runtime -------------------------------------------------------------------
namespace {
std::mutex g_init_mu;
Runtime* g_rt = nullptr;
int g_req_device = -1;
}  // namespace

Runtime::Runtime(int device) {
  int count = 0;
  cuda_ok(cudaGetDeviceCount(&count), "cudaGetDeviceCount");
  if (count == 0) fail(HS_E_CUDA, "no CUDA device visible");
  if (device < 0) cuda_ok(cudaGetDevice(&device), "cudaGetDevice");
  device_ = device;
  cuda_ok(cudaSetDevice(device_), "cudaSetDevice");
  cudaDeviceProp prop{};
  cuda_ok(cudaGetDeviceProperties(&prop, device_), "cudaGetDeviceProperties");
  if (prop.major < 10)
    fail(HS_E_CUDA, std::string("libhestat_gpu targets sm_100a (B200); found ") + prop.name);
  sms_ = prop.multiProcessorCount;
  if (const char* e = std::getenv("HESTAT_LANES")) {
    const int l = std::atoi(e);
    if (l == 1 || l == 2 || l == 4 || l == 8) prog_lanes = l;
  }
  if (const char* e = std::getenv("HESTAT_BATCH_LANES")) {  // batched kernels: default by batch size (core.h)
    const int l = std::atoi(e);
    if (l == 1 || l == 2 || l == 4) batch_lanes = l;
  }
  cuda_ok(cudaStreamCreateWithFlags(&stream_, cudaStreamNonBlocking), "cudaStreamCreate");
  // The side streams carry short work that a caller is blocked on (encode_column's encrypt kernel,
  // decode_column's copies): highest priority, so their blocks are placed before the next queued
  // statistics launch when SMs free up.
  int prio_lo = 0, prio_hi = 0;
  cuda_ok(cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi), "cudaDeviceGetStreamPriorityRange");
  for (cudaStream_t& u : upload_)
    cuda_ok(cudaStreamCreateWithPriority(&u, cudaStreamNonBlocking, prio_hi), "cudaStreamCreate (upload)");
  cuda_ok(cudaStreamCreateWithPriority(&download_, cudaStreamNonBlocking, prio_hi), "cudaStreamCreate (download)");
  // Keep freed blocks in the stream-ordered pool: ciphertexts are churned per op.
  cudaMemPool_t pool;
  cuda_ok(cudaDeviceGetDefaultMemPool(&pool, device_), "cudaDeviceGetDefaultMemPool");
  uint64_t thr = UINT64_MAX;
  cuda_ok(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr), "pool threshold");
  // An upload-stream allocation must never wait on compute-stream work behind a pending
  // free (that would serialise encode_column behind the running statistic): reuse a block
  // freed on the other stream only once its free has completed.
#ifndef HS_POOL_XDEP
  int no = 0;
  cuda_ok(cudaMemPoolSetAttribute(pool, cudaMemPoolReuseAllowInternalDependencies, &no), "pool reuse attr");
#endif
}

Runtime& Runtime::get() {
  std::lock_guard<std::mutex> g(g_init_mu);
  if (!g_rt) g_rt = new Runtime(g_req_device);  // intentionally leaked (outlives handles)
  return *g_rt;
}

void Runtime::init(int device) {
  std::lock_guard<std::mutex> g(g_init_mu);
  if (g_rt) {
    if (g_rt->device_ != device)
      fail(HS_E_CUDA, "hs_init: runtime already initialised on another device");
    return;
  }
  g_req_device = device;
}

DevBuf Runtime::alloc(size_t n) {
  double* p = nullptr;
  const size_t bytes = (n ? n : 1) * sizeof(double);
  cuda_ok(cudaSetDevice(device_), "cudaSetDevice");
  cuda_ok(cudaMallocAsync(reinterpret_cast<void**>(&p), bytes, stream_), "cudaMallocAsync");
  cudaStream_t s = stream_;
  return DevBuf(p, [s](double* q) { cudaFreeAsync(q, s); });  // errors at teardown ignored
}

DevBuf Runtime::alloc_on(size_t n, cudaStream_t on) {
  double* p = nullptr;
  const size_t bytes = (n ? n : 1) * sizeof(double);
  cuda_ok(cudaSetDevice(device_), "cudaSetDevice");
  cuda_ok(cudaMallocAsync(reinterpret_cast<void**>(&p), bytes, on), "cudaMallocAsync");
  cudaStream_t s = stream_;
  return DevBuf(p, [s](double* q) { cudaFreeAsync(q, s); });
}

bool Runtime::capturing() const {
  cudaStreamCaptureStatus st = cudaStreamCaptureStatusNone;
  cuda_ok(cudaStreamIsCapturing(stream_, &st), "cudaStreamIsCapturing");
  return st != cudaStreamCaptureStatusNone;
}

void Runtime::sync() { cuda_ok(cudaStreamSynchronize(stream_), "cudaStreamSynchronize"); }

namespace {
void (*g_wait_hook)(cudaStream_t) = nullptr;
}
void Runtime::set_wait_hook(void (*hook)(cudaStream_t)) { g_wait_hook = hook; }
void Runtime::wait(cudaStream_t s) const {
  if (g_wait_hook)
    g_wait_hook(s);
  else
    cuda_ok(cudaStreamSynchronize(s), "cudaStreamSynchronize");
}

double* Runtime::upload_stage(unsigned i, size_t n) {
  std::lock_guard<std::mutex> g(stage_mu_);
  if (stage_n_[i] < n) {
    cuda_ok(cudaStreamSynchronize(upload_[i]), "upload stage sync");
    if (stage_[i]) cuda_ok(cudaFree(stage_[i]), "upload stage free");
    stage_[i] = nullptr;
    stage_n_[i] = 0;
    cuda_ok(cudaMalloc(reinterpret_cast<void**>(&stage_[i]), n * sizeof(double)), "upload stage alloc");
    stage_n_[i] = n;
  }
  return stage_[i];
}

cudaEvent_t Runtime::take_event() {
  {
    std::lock_guard<std::mutex> g(ev_mu_);
    if (!ev_free_.empty()) {
      cudaEvent_t e = ev_free_.back();
      ev_free_.pop_back();
      return e;
    }
  }
  cudaEvent_t e = nullptr;
  cuda_ok(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "cudaEventCreate");
  return e;
}
void Runtime::give_event(cudaEvent_t e) {
  std::lock_guard<std::mutex> g(ev_mu_);
  ev_free_.push_back(e);
}
ReadyEv::~ReadyEv() {
  if (e) Runtime::get().give_event(e);
}
std::shared_ptr<ReadyEv> Runtime::mark_ready() {
  if (capturing()) return nullptr;
  return mark_on(stream_);
}
std::shared_ptr<ReadyEv> Runtime::mark_on(cudaStream_t s) {
  auto r = std::make_shared<ReadyEv>();
  r->e = take_event();
  r->serial = ++ev_serial_;
  cuda_ok(cudaEventRecord(r->e, s), "cudaEventRecord (ready)");
  return r;
}
void Runtime::compute_waits(const std::shared_ptr<ReadyEv>& ev) {
  if (!ev) return;
  std::lock_guard<std::mutex> g(ev_mu_);
  if (last_waited_ == ev->serial) return;  // the chunks of one column share one event
  cuda_ok(cudaStreamWaitEvent(stream_, ev->e, 0), "cudaStreamWaitEvent (upload)");
  last_waited_ = ev->serial;
}

double* Runtime::scratch(int slot, size_t n, bool zero) {
  std::lock_guard<std::mutex> g(scratch_mu_);
  if (scratch_n_[slot] < n) {
    scratch_[slot] = alloc(n);  // the old buffer is freed stream-ordered
    scratch_n_[slot] = n;
    if (zero) cuda_ok(cudaMemsetAsync(scratch_[slot].get(), 0, n * sizeof(double), stream_), "scratch zero");
  }
  return scratch_[slot].get();
}

// ---- ciphertext storage -----------------------------------------------------------
// An asynchronous encode_column may still be writing `dev` on an upload stream: order the compute
// stream behind it.  While the compute stream is being captured into a graph an outside event
// cannot become a dependency of the capture, so the host waits for the upload instead.
void CtData::settle_locked() const {
  if (!filling) return;
  Runtime& rt = Runtime::get();
  if (rt.capturing())
    cuda_ok(cudaEventSynchronize(filling->e), "cudaEventSynchronize (upload)");
  else
    rt.compute_waits(filling);
  filling.reset();
}

const double* CtData::device() const {
  std::lock_guard<std::mutex> g(mu);
  settle_locked();
  if (!dev) {
    Runtime& rt = Runtime::get();
    DevBuf d = rt.alloc(n);
    if (n)
      cuda_ok(cudaMemcpyAsync(d.get(), host.data(), n * sizeof(double), cudaMemcpyHostToDevice,
                              rt.stream()),
              "ciphertext upload");
    const_cast<CtData*>(this)->dev = d;
  }
  return dev.get();
}

const std::vector<double>& CtData::host_slots() const {
  std::lock_guard<std::mutex> g(mu);
  settle_locked();
  if (!host_ok) {
    host.resize(n);
    if (n) {
      Runtime& rt = Runtime::get();
      cuda_ok(cudaMemcpyAsync(host.data(), dev.get(), n * sizeof(double), cudaMemcpyDeviceToHost,
                              rt.stream()),
              "ciphertext download");
      rt.sync();
    }
    host_ok = true;
  }
  return host;
}

void CtData::read(double* out, size_t count) const {
  if (count == 0) return;
  read_async(out, count, 0);
  Runtime::get().sync();
}

// Enqueue a D2H copy of slots [0, count) straight into the caller's buffer
// (pinned buffers DMA directly; no intermediate host cache).  The caller syncs.
void CtData::read_async(double* out, size_t count, size_t) const {
  {
    std::lock_guard<std::mutex> g(mu);
    if (host_ok) {
      std::memcpy(out, host.data(), count * sizeof(double));
      return;
    }
    settle_locked();
  }
  Runtime& rt = Runtime::get();
  // copy-engine DMA straight into the caller's buffer (measured faster than SM stores
  // into host-mapped memory for 256 KiB on this box: 23.5 vs 29 us per decode call)
  cuda_ok(cudaMemcpyAsync(out, dev.get(), count * sizeof(double), cudaMemcpyDeviceToHost, rt.stream()),
          "ciphertext read");
}

Ct ct_device(DevBuf buf, size_t n, int level, int grid, std::shared_ptr<ReadyEv> ready) {
  auto c = std::make_shared<CtData>();
  c->ready = std::move(ready);
  c->n = n;
  c->level = level;
  c->grid = grid;
  c->dev = std::move(buf);
  return c;
}

Ct ct_host(std::vector<double> v, int level) {
  auto c = std::make_shared<CtData>();
  c->n = v.size();
  c->level = level;
  c->grid = 0;
  c->host = std::move(v);
  c->host_ok = true;
  return c;
}

Ct ct_empty() { return ct_host({}, 0); }

}  // namespace hsg
