// runtime.cpp -- device context and the host-libm variant probe.
#include "runtime.h"

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <mutex>

#include "glibc_math.h"

namespace ssg {

namespace {
Context g_ctx;
RunStats g_stats;
std::mutex g_mu;
bool g_pool = true;
std::mutex g_stats_mu;
thread_local RunStats* t_stats = nullptr;
thread_local cudaStream_t t_stream = nullptr;
}  // namespace

void RunStats::add(const RunStats& o) {
  launches_simulate += o.launches_simulate;
  launches_select += o.launches_select;
  launches_predict += o.launches_predict;
  launches_batch += o.launches_batch;
  launches_setup += o.launches_setup;
  units += o.units;
  iterations += o.iterations;
  entries += o.entries;
  events += o.events;
  predictor_bytes += o.predictor_bytes;
  entry_bytes += o.entry_bytes;
  simulate_ms += o.simulate_ms;
  queries += o.queries;
  predict_ms += o.predict_ms;
  h2d_bytes += o.h2d_bytes;
  d2h_bytes += o.d2h_bytes;
  simulate_busy_ms += o.simulate_busy_ms;
  useful_iterations += o.useful_iterations;
  useful_entries += o.useful_entries;
  useful_bytes += o.useful_bytes;
  cancelled_probes += o.cancelled_probes;
  spec_slo_runs += o.spec_slo_runs;
  spec_slo_used += o.spec_slo_used;
}

StatsScope::StatsScope() : prev(t_stats) { t_stats = &local; }
StatsScope::~StatsScope() {
  t_stats = prev;
  std::lock_guard<std::mutex> lk(g_stats_mu);
  stats().add(local);
}

StreamScope::StreamScope(cudaStream_t s) : prev(t_stream) { t_stream = s; }
StreamScope::~StreamScope() { t_stream = prev; }
cudaStream_t current_stream() { return t_stream ? t_stream : context().stream; }

int probe_host_math_variant() {
  // Walk inputs until both routines have separated the two contractions at
  // least a few times; the host libm must agree with exactly one of them on
  // every sample, or device parity with this host is impossible.
  std::uint64_t s = 0x9e3779b97f4a7c15ULL;
  auto next = [&] {
    s ^= s << 13;
    s ^= s >> 7;
    s ^= s << 17;
    return s;
  };
  int agree[2] = {0, 0}, seen = 0;
  for (int i = 0; i < 400000 && seen < 64; ++i) {
    const double xe = -25.0 + 35.0 * (static_cast<double>(next() >> 11) * 0x1p-53);
    const double xl = static_cast<double>(next() % 4000000) * static_cast<double>(1u << (next() % 12));
    const double he = std::exp(xe), hl = std::log1p(xl);
    double v[2][2];
    for (int k = 0; k < 2; ++k) {
      v[k][0] = ssg_exp(xe, k);
      v[k][1] = ssg_log1p(xl, k);
    }
    const bool differ_e = std::memcmp(&v[0][0], &v[1][0], 8) != 0;
    const bool differ_l = std::memcmp(&v[0][1], &v[1][1], 8) != 0;
    for (int k = 0; k < 2; ++k) {
      if (std::memcmp(&he, &v[k][0], 8) != 0 || std::memcmp(&hl, &v[k][1], 8) != 0)
        agree[k] = -1;
      else if (agree[k] >= 0 && (differ_e || differ_l))
        ++agree[k];
    }
    if (differ_e || differ_l) ++seen;
  }
  if (agree[SSG_MATH_FMA] > 0 && agree[SSG_MATH_PLAIN] < 0) return SSG_MATH_FMA;
  if (agree[SSG_MATH_PLAIN] > 0 && agree[SSG_MATH_FMA] < 0) return SSG_MATH_PLAIN;
  throw servesim::InternalError(
      "host libm exp/log1p match neither glibc contraction variant; device predictions "
      "cannot be made bit-identical to this host");
}

RunStats& stats() { return t_stats ? *t_stats : g_stats; }

void init_context(int device) {
  std::lock_guard<std::mutex> lk(g_mu);
  if (g_ctx.device == device && g_ctx.stream) return;
  if (g_ctx.stream) {
    cudaStreamDestroy(g_ctx.stream);
    g_ctx.stream = nullptr;
  }
  int n = 0;
  cuda_check(cudaGetDeviceCount(&n), "cudaGetDeviceCount");
  if (device < 0 || device >= n)
    throw CudaError("ssg_init: device " + std::to_string(device) + " not present (" +
                    std::to_string(n) + " visible)");
  cuda_check(cudaSetDevice(device), "cudaSetDevice");
  cudaDeviceProp prop{};
  cuda_check(cudaGetDeviceProperties(&prop, device), "cudaGetDeviceProperties");
  if (prop.major != 10)
    throw CudaError(std::string("ssg: built for sm_100a, found ") + prop.name);
  cuda_check(cudaStreamCreateWithFlags(&g_ctx.stream, cudaStreamNonBlocking), "stream");
  g_ctx.device = device;
  g_ctx.num_sms = prop.multiProcessorCount;
  const char* pool_env = std::getenv("SSG_POOL");
  g_pool = !(pool_env && pool_env[0] == '0');
  if (g_pool) {
    cudaMemPool_t pool;
    cuda_check(cudaDeviceGetDefaultMemPool(&pool, device), "cudaDeviceGetDefaultMemPool");
    std::uint64_t keep = UINT64_MAX;
    cuda_check(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep),
               "cudaMemPoolSetAttribute");
    // no allocator-inserted waits: a block freed on one sweep lane's stream
    // behind a running kernel must not make another lane's allocation wait
    // for that kernel (lanes exist to overlap); opportunistic reuse of frees
    // that already completed stays on
    int no = 0;
    cuda_check(cudaMemPoolSetAttribute(pool, cudaMemPoolReuseAllowInternalDependencies, &no),
               "cudaMemPoolSetAttribute");
  }
  if (g_ctx.math_fma < 0) g_ctx.math_fma = probe_host_math_variant();
}

Context& context() {
  if (!g_ctx.stream) init_context(0);
  cuda_check(cudaSetDevice(g_ctx.device), "cudaSetDevice");
  return g_ctx;
}

void* device_alloc(std::size_t bytes, cudaStream_t s) {
  context();
  void* p = nullptr;
  if (g_pool)
    cuda_check(cudaMallocAsync(&p, bytes, s), "cudaMallocAsync");
  else
    cuda_check(cudaMalloc(&p, bytes), "cudaMalloc");
  return p;
}

void device_free(void* p, cudaStream_t s) {
  if (g_pool && g_ctx.stream && s)
    cudaFreeAsync(p, s);
  else
    cudaFree(p);
}

namespace {
double now_s() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}
bool timing_on() {
  static const bool on = std::getenv("SSG_TIMING") != nullptr;
  return on;
}
}  // namespace

PhaseTimer::PhaseTimer(const char* what) : what_(what), t0_(timing_on() ? now_s() : 0.0) {}
PhaseTimer::~PhaseTimer() {
  if (timing_on()) std::fprintf(stderr, "[ssg timing] %-28s %9.3f ms\n", what_, 1e3 * (now_s() - t0_));
}

HostStaging::~HostStaging() {
  for (auto& c : chunks_) cudaFreeHost(c.p);
}

void* HostStaging::take(std::size_t bytes) {
  bytes = (bytes + 255) & ~static_cast<std::size_t>(255);
  if (chunks_.empty() || used_ + bytes > chunks_.back().cap) {
    const std::size_t cap = std::max<std::size_t>(bytes, std::max<std::size_t>(1 << 20, total_));
    char* p = nullptr;
    cuda_check(cudaHostAlloc(reinterpret_cast<void**>(&p), cap, cudaHostAllocPortable),
               "cudaHostAlloc");
    chunks_.push_back({p, cap});
    total_ += cap;
    used_ = 0;
  }
  void* p = chunks_.back().p + used_;
  used_ += bytes;
  return p;
}

void HostStaging::reset() {
  if (chunks_.size() > 1) {  // consolidate into one chunk of the high-water size
    for (auto& c : chunks_) cudaFreeHost(c.p);
    chunks_.clear();
    const std::size_t cap = total_;
    total_ = 0;
    char* p = nullptr;
    cuda_check(cudaHostAlloc(reinterpret_cast<void**>(&p), cap, cudaHostAllocPortable),
               "cudaHostAlloc");
    chunks_.push_back({p, cap});
    total_ = cap;
  }
  used_ = 0;
}

void shutdown_context() {
  std::lock_guard<std::mutex> lk(g_mu);
  if (g_ctx.stream) cudaStreamDestroy(g_ctx.stream);
  g_ctx = Context{};
}

}  // namespace ssg
