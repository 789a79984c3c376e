// core.h — host-side core of libhestat_gpu.so: errors, parameters, meter,
// device runtime (stream + stream-ordered memory pool) and ciphertext storage.
//
// Reference counterparts: CkksParams / CostMeter / Ciphertext / EvalContext
// (/root/reference/proj/include/hestat/ckks.hpp:19-93).  The reference keeps a
// std::vector<double> per ciphertext; here a ciphertext is an immutable device
// buffer in HBM plus a host-side level, with a lazily filled host mirror for
// slots() reads.
#pragma once

#include <cstdlib>
#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <unordered_map>
#include <vector>

#include "hestat_gpu.h"

namespace hsg {

// ---- errors: one C++ type carrying the ABI status code (errors.hpp:11-38) ----
struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};
[[noreturn]] inline void fail(int code, const std::string& msg) { throw Error(code, msg); }
void cuda_ok(cudaError_t e, const char* what);

// ---- CkksParams (ckks.hpp:19-42) ----
struct Params {
  size_t S = 32768;
  int max_level = 11;
  int scale_bits = 40;
  bool quantize = true;
  bool auto_bootstrap = true;
  bool debug = false;

  static Params from(const hs_params& p);
  hs_params to() const;
  void validate() const;  // ckks.hpp:34-39
};

// ---- CostMeter (ckks.hpp:46-60) ----
struct Meter {
  uint64_t mul_ct = 0, mul_pt = 0, add = 0, rotate = 0, bootstrap = 0;
};

// ---- device runtime --------------------------------------------------------
using DevBuf = std::shared_ptr<double>;

class Runtime {
 public:
  static Runtime& get();        // lazily initialised, never destroyed
  static void init(int device); // optional explicit device choice (before first use)

  cudaStream_t stream() const { return stream_; }
  // Host-input stream of encode_column: its copy/encrypt kernels run beside the compute
  // stream's kernels (a caller can encode the next column while the current one computes).
  // encode_column synchronises it before returning, so its outputs are complete for any
  // later work on the compute stream without an event.
  // One of kUploadStreams, round-robin per call: consecutive encode_column calls (host threads
  // encoding ahead) do not order one column's copy behind the previous column's encrypt kernel,
  // which may be waiting for SMs.  A caller keeps the stream it got for its whole operation.
  cudaStream_t upload_stream() { return upload_[next_upload()]; }
  unsigned next_upload() { return up_next_.fetch_add(1) % kUploadStreams; }
  cudaStream_t upload_stream_at(unsigned i) const { return upload_[i]; }
  // Upload stream i's persistent staging buffer of at least n doubles (grown on demand, which
  // synchronises that stream; steady state allocates nothing).  Work that uses it is ordered by
  // the stream, so consecutive encodes on one stream reuse it safely.
  double* upload_stage(unsigned i, size_t n);
  // Result stream of decode_column: the D2H copies of ciphertexts that carry a `ready` event
  // (outputs of the fused statistics) run here, beside the compute stream's next kernels.
  cudaStream_t download_stream() const { return download_; }
  // Block the calling thread until `s` has drained.  api.cu installs a hook that releases the
  // API lock for the duration (hs_encode_column / hs_decode_column of one thread then overlap
  // another thread's calls: PCIe is full duplex and the copy engines are independent).
  void wait(cudaStream_t s) const;
  static void set_wait_hook(void (*hook)(cudaStream_t));
  // An event recorded on the compute stream now (null while the stream is being captured):
  // the completion marker a fused statistic attaches to its outputs.
  std::shared_ptr<struct ReadyEv> mark_ready();
  std::shared_ptr<struct ReadyEv> mark_on(cudaStream_t s);  // the same on any stream
  void compute_waits(const std::shared_ptr<struct ReadyEv>& ev);  // compute stream waits (deduplicated)
  cudaEvent_t take_event();
  void give_event(cudaEvent_t e);
  bool capturing() const;                   // the compute stream is being captured into a graph
  int device() const { return device_; }
  int sm_count() const { return sms_; }
  DevBuf alloc(size_t n_doubles);           // stream-ordered; freed stream-ordered
  // allocated in `on`'s order, freed in the compute stream's order (where its consumers run)
  DevBuf alloc_on(size_t n_doubles, cudaStream_t on);
  void sync();
  void note_launch(uint64_t n = 1) { launches_ += n; }
  uint64_t launches() const { return launches_.load(); }
  bool fused = true;
  int prog_lanes = 2;  // threads per slot of the fused program kernel (HESTAT_LANES: 1, 2, 4, 8)
  // the same for the batched kernels (HESTAT_BATCH_LANES: 1, 2, 4); 0 = by batch size: one thread
  // per slot once a block has a full round of items (no work repeated across lanes, and the
  // degree-511 tree then runs from the constant bank)
  int batch_lanes = 0;

  // Persistent device scratch buffer `slot` of at least n doubles (grown on
  // demand; zero-filled when (re)allocated if `zero`).  All device work is ordered
  // on one stream, so reuse is race-free.
  double* scratch(int slot, size_t n, bool zero = false);

 private:
  Runtime(int device);
  int device_ = 0;
  int sms_ = 148;
  cudaStream_t stream_ = nullptr;
  static constexpr unsigned kUploadStreams = 3;
  cudaStream_t upload_[kUploadStreams] = {nullptr, nullptr, nullptr};
  std::atomic<unsigned> up_next_{0};
  std::mutex stage_mu_;
  double* stage_[kUploadStreams] = {nullptr, nullptr, nullptr};
  size_t stage_n_[kUploadStreams] = {0, 0, 0};
  cudaStream_t download_ = nullptr;
  std::mutex ev_mu_;
  std::atomic<uint64_t> ev_serial_{0};
  uint64_t last_waited_ = 0;
  std::vector<cudaEvent_t> ev_free_;
  std::atomic<uint64_t> launches_{0};
  std::mutex scratch_mu_;
  DevBuf scratch_[6];
  size_t scratch_n_[6] = {0, 0, 0, 0, 0, 0};
};

// L1/shared carveout (percent of the unified 228 KB) shared by the statistics kernels and
// encode_column's k_encrypt: SMs only host kernels of one carveout at a time, so both use
// the same small one (k_stat needs <= ~15 KB of shared memory).  HS_CARVEOUT overrides.
inline int carveout_pct() {
  static const int v = [] {
    const char* e = std::getenv("HS_CARVEOUT");
    return e ? std::atoi(e) : 10;
  }();
  return v;
}

// ---- Ciphertext storage ------------------------------------------------------
// grid > 0 records that every slot is a multiple of 2^-grid (the output of a
// quantising op under scale_bits == grid); fused kernels rely on it to carry
// values in exact integer grid units.
struct ReadyEv {  // pooled event, returned to the runtime when the last holder drops it
  cudaEvent_t e = nullptr;
  uint64_t serial = 0;  // unique per recording (events are recycled)
  ~ReadyEv();
};

struct CtData {
  size_t n = 0;
  int level = 0;
  int grid = 0;
  DevBuf dev;  // null for host-constructed ciphertexts until first device use
  std::shared_ptr<ReadyEv> ready;  // set by the fused statistics: `dev` is complete once it has fired
  // set by an asynchronous encode_column: `dev` is being written on an upload stream; the first
  // device() use makes the compute stream wait for it
  mutable std::shared_ptr<ReadyEv> filling;
  mutable std::mutex mu;
  mutable std::vector<double> host;
  mutable bool host_ok = false;

  const double* device() const;                 // uploads a host-only ciphertext once
  void read(double* out, size_t count) const;   // synchronous D2H into the caller's buffer
  void read_async(double* out, size_t count, size_t) const;  // enqueue only
  const std::vector<double>& host_slots() const;

 private:
  void settle_locked() const;  // caller holds mu
};
using Ct = std::shared_ptr<const CtData>;

Ct ct_device(DevBuf buf, size_t n, int level, int grid, std::shared_ptr<ReadyEv> ready = nullptr);
Ct ct_host(std::vector<double> v, int level);  // Ciphertext(std::vector<double>, int)
Ct ct_empty();                                 // Ciphertext()

// ---- EncryptedColumn (column.hpp:19-23) ----
struct Column {
  std::vector<Ct> chunks;
  size_t n_valid = 0;
};

}  // namespace hsg

namespace hsg {
namespace rns {
struct RCtData;
struct Home;
}  // namespace rns
}  // namespace hsg

// ABI handle types.  A context is Tier E (slot vectors with the reference's emulator
// semantics) unless `rns` is set, in which case every op runs on RNS-CKKS ciphertexts
// (Tier R, rns_eval.h); a handle then carries `r` and the context's RNS home (keys, scales),
// which decrypts it for hs_ct_read (Ciphertext::slots()).
struct hs_ct {
  hsg::Ct p;
  std::shared_ptr<const hsg::rns::RCtData> r;
  std::shared_ptr<hsg::rns::Home> home;
};
struct hs_ctx {
  hsg::Params p;
  hsg::Meter m;
  uint64_t seed = 0;
  std::shared_ptr<hsg::rns::Home> rns;
};
