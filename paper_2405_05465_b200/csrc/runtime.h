// runtime.h -- process-wide device context and small HBM helpers.
#pragma once
#include <cuda_runtime.h>

#include <cstddef>
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
void* device_alloc(std::size_t bytes);
void device_free(void* p);

// Which glibc contraction this host's libm runs (host_math.cpp).
int probe_host_math_variant();

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
};
RunStats& stats();

// Owning HBM buffer.
template <typename T>
struct DeviceBuffer {
  T* ptr = nullptr;
  std::size_t count = 0;
  DeviceBuffer() = default;
  explicit DeviceBuffer(std::size_t n) { resize(n); }
  ~DeviceBuffer() { release(); }
  DeviceBuffer(const DeviceBuffer&) = delete;
  DeviceBuffer& operator=(const DeviceBuffer&) = delete;
  DeviceBuffer(DeviceBuffer&& o) noexcept : ptr(o.ptr), count(o.count) {
    o.ptr = nullptr;
    o.count = 0;
  }
  DeviceBuffer& operator=(DeviceBuffer&& o) noexcept {
    if (this != &o) {
      release();
      ptr = o.ptr;
      count = o.count;
      o.ptr = nullptr;
      o.count = 0;
    }
    return *this;
  }
  void resize(std::size_t n) {
    if (n <= count && ptr) return;
    release();
    if (n == 0) return;
    ptr = static_cast<T*>(device_alloc(n * sizeof(T)));
    count = n;
  }
  void release() {
    if (ptr) device_free(ptr);
    ptr = nullptr;
    count = 0;
  }
  void upload(const T* src, std::size_t n, cudaStream_t s) {
    resize(n);
    if (n) cuda_check(cudaMemcpyAsync(ptr, src, n * sizeof(T), cudaMemcpyHostToDevice, s), "H2D");
    stats().h2d_bytes += static_cast<int64_t>(n * sizeof(T));
  }
  void upload(const std::vector<T>& v, cudaStream_t s) { upload(v.data(), v.size(), s); }
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
