// runtime.h -- process-wide device context and small HBM helpers.
#pragma once
#include <cuda_runtime.h>

#include <cstddef>
#include <cstring>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include "servesim_b200.hpp"
#include "ssg_device.h"

namespace ssg {

// CUDA failures map to status 3 at the C ABI (never a silent fallback).
class CudaError : public std::runtime_error {
 public:
  explicit CudaError(const std::string& m) : std::runtime_error(m) {}
};

inline void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw CudaError(std::string(what) + ": " + cudaGetErrorString(e));
}

struct Context {
  int device = -1;
  cudaStream_t stream = nullptr;
  int math_fma = -1;  // SSG_MATH_FMA / SSG_MATH_PLAIN, probed from the host libm
  int num_sms = 0;
};

// Initializes on first use (device 0) unless ssg_init chose another device.
Context& context();
void init_context(int device);
void shutdown_context();

// HBM for DeviceBuffer: stream-ordered allocations on the context stream from the
// device's memory pool, which keeps freed blocks (release threshold = max), so a
// new search session or simulation reuses the previous one's HBM instead of paying
// cudaMalloc/cudaFree (a device-wide sync) per buffer.  SSG_POOL=0 falls back to
// plain cudaMalloc/cudaFree (A/B only).  Every library kernel and copy runs on the
// context stream; callers that pass their own stream only read buffers whose
// upload was synchronised.
// Buffers are ordered on the stream current for the allocating thread
// (StreamScope), or the context stream; a buffer is freed on the stream it was
// allocated on, which is the only stream that uses it.
void* device_alloc(std::size_t bytes, cudaStream_t s);
void device_free(void* p, cudaStream_t s);
cudaStream_t current_stream();  // StreamScope's stream, else the context stream

struct StreamScope {
  explicit StreamScope(cudaStream_t s);
  ~StreamScope();
  StreamScope(const StreamScope&) = delete;
  StreamScope& operator=(const StreamScope&) = delete;
  cudaStream_t prev;
};

// Which glibc contraction this host's libm runs (host_math.cpp).
int probe_host_math_variant();
// mathcheck.cu: fn 0 = log1p, 1 = exp of x_k = base + k * step, k in [k0, k0 + n)
void launch_math_eval(int fn, int fma_variant, double base, double step, int64_t k0, int64_t n,
                      double* d_out, cudaStream_t s);

// Counters over the library's own kernels (reset/read through the C ABI; the
// bench reports them next to its timings).
struct RunStats {
  int64_t launches_simulate = 0, launches_select = 0, launches_predict = 0, launches_batch = 0;
  int64_t launches_setup = 0;
  int64_t units = 0, iterations = 0, entries = 0, events = 0;
  int64_t predictor_bytes = 0, entry_bytes = 0;
  double simulate_ms = 0.0;  // k_simulate device time, CUDA events on the launching stream
  int64_t queries = 0;       // k_predict queries
  double predict_ms = 0.0;
  int64_t h2d_bytes = 0, d2h_bytes = 0;
  double simulate_busy_ms = 0.0;  // union of k_simulate intervals (launches overlap across streams)
  // sweep work the sequential reference search would do (probes its replay asks + SLO runs)
  int64_t useful_iterations = 0, useful_entries = 0, useful_bytes = 0;
  int64_t cancelled_probes = 0;  // speculative probes stopped once a lower rate of their group failed
  int64_t spec_slo_runs = 0, spec_slo_used = 0;  // speculative SLO runs taken / used by the replay
  void add(const RunStats& o);
};
// The calling thread's counters: the process-wide ones, or a StatsScope's
// private accumulator, merged into the process-wide ones when the scope ends.
RunStats& stats();
struct StatsScope {
  StatsScope();
  ~StatsScope();
  StatsScope(const StatsScope&) = delete;
  StatsScope& operator=(const StatsScope&) = delete;
  RunStats local;
  RunStats* prev;
};

// Pinned host staging for one stream's copies: a bump allocator over pinned
// chunks, reset after the stream is synchronised.  Copies from pageable memory
// can hold the issuing thread behind other streams' kernels; the sweep lanes
// stage through pinned memory so their launches overlap.
class HostStaging {
 public:
  HostStaging() = default;
  ~HostStaging();
  HostStaging(const HostStaging&) = delete;
  HostStaging& operator=(const HostStaging&) = delete;
  void* take(std::size_t bytes);  // valid until reset()
  void reset();                   // only after the stream's copies completed

 private:
  struct Chunk {
    char* p;
    std::size_t cap;
  };
  std::vector<Chunk> chunks_;
  std::size_t used_ = 0;  // in the last chunk
  std::size_t total_ = 0;
};

// Host phase timing to stderr when SSG_TIMING is set (diagnostics only).
class PhaseTimer {
 public:
  explicit PhaseTimer(const char* what);
  ~PhaseTimer();
  PhaseTimer(const PhaseTimer&) = delete;
  PhaseTimer& operator=(const PhaseTimer&) = delete;

 private:
  const char* what_;
  double t0_;
};

// Owning HBM buffer.
template <typename T>
struct DeviceBuffer {
  T* ptr = nullptr;
  std::size_t count = 0;
  cudaStream_t stream = nullptr;  // allocation stream
  DeviceBuffer() = default;
  explicit DeviceBuffer(std::size_t n) { resize(n); }
  ~DeviceBuffer() { release(); }
  DeviceBuffer(const DeviceBuffer&) = delete;
  DeviceBuffer& operator=(const DeviceBuffer&) = delete;
  DeviceBuffer(DeviceBuffer&& o) noexcept : ptr(o.ptr), count(o.count), stream(o.stream) {
    o.ptr = nullptr;
    o.count = 0;
  }
  DeviceBuffer& operator=(DeviceBuffer&& o) noexcept {
    if (this != &o) {
      release();
      ptr = o.ptr;
      count = o.count;
      stream = o.stream;
      o.ptr = nullptr;
      o.count = 0;
    }
    return *this;
  }
  void resize(std::size_t n) {
    if (n <= count && ptr) return;
    release();
    if (n == 0) return;
    stream = current_stream();
    ptr = static_cast<T*>(device_alloc(n * sizeof(T), stream));
    count = n;
  }
  void release() {
    if (ptr) device_free(ptr, stream);
    ptr = nullptr;
    count = 0;
  }
  void upload(const T* src, std::size_t n, cudaStream_t s) {
    resize(n);
    if (n) cuda_check(cudaMemcpyAsync(ptr, src, n * sizeof(T), cudaMemcpyHostToDevice, s), "H2D");
    stats().h2d_bytes += static_cast<int64_t>(n * sizeof(T));
  }
  void upload(const std::vector<T>& v, cudaStream_t s) { upload(v.data(), v.size(), s); }
  void upload(const std::vector<T>& v, cudaStream_t s, HostStaging& st) {
    resize(v.size());
    if (v.empty()) return;
    void* p = st.take(v.size() * sizeof(T));
    std::memcpy(p, v.data(), v.size() * sizeof(T));
    cuda_check(cudaMemcpyAsync(ptr, p, v.size() * sizeof(T), cudaMemcpyHostToDevice, s), "H2D");
    stats().h2d_bytes += static_cast<int64_t>(v.size() * sizeof(T));
  }
  // D2H into staging; the caller copies out of the returned pointer after syncing s
  const T* download_staged(std::size_t n, cudaStream_t s, HostStaging& st) const {
    T* p = static_cast<T*>(st.take(n * sizeof(T)));
    if (n) cuda_check(cudaMemcpyAsync(p, ptr, n * sizeof(T), cudaMemcpyDeviceToHost, s), "D2H");
    stats().d2h_bytes += static_cast<int64_t>(n * sizeof(T));
    return p;
  }
  void download(T* dst, std::size_t n, cudaStream_t s) const {
    if (n) cuda_check(cudaMemcpyAsync(dst, ptr, n * sizeof(T), cudaMemcpyDeviceToHost, s), "D2H");
    stats().d2h_bytes += static_cast<int64_t>(n * sizeof(T));
  }
};

}  // namespace ssg

namespace servesim {

// HBM-resident flattened estimator (built by predictor.cu from EstimatorModel).
struct DeviceEstimator {
  ssg::DeviceBuffer<SsgModelDesc> models;
  ssg::DeviceBuffer<double> dpool;
  ssg::DeviceBuffer<SsgNode> nodes;
  ssg::DeviceBuffer<int32_t> roots;
  // single-query path (EstimatorModel::predict): kept buffers, one caller at a time
  std::mutex one_mu;
  ssg::DeviceBuffer<double> one_dev;
  double* one_host = nullptr;  // pinned
  ~DeviceEstimator();
  ssg::DeviceBuffer<double> node_a;  // SoA mirror (SSG_FOREST_SOA A/B builds)
  ssg::DeviceBuffer<int2> node_fr;
  std::vector<SsgModelDesc> host_models;
  std::map<OpModelKey, int32_t> index;  // (op, tp) -> model slot
  std::vector<int64_t> qbytes;          // algorithmic bytes of one query per slot
  SsgEstView view{};
  std::size_t bytes = 0;  // HBM footprint
  bool has_forest = false;

  int32_t slot(OpName op, std::int64_t tp) const {
    auto it = index.find({op, tp});
    return it == index.end() ? -1 : it->second;
  }
};

// Formats the reference's extrapolation-margin message for one query
// (estimator.hpp:115-119).
std::string bbox_error_message(const EstimatorModel::PerOpModel& m, const OpModelKey& key,
                               int feature, double value);

}  // namespace servesim
