// select.cu -- K5: exact nearest-rank percentiles by segmented radix select.
//
// reference: stats.hpp:15-24 (percentile: sort, then sorted[ceil(q n) - 1]),
//            metrics.hpp:58-67 (summaries), search.hpp:333,351-356 (p99 / p90)
//
// One block per (segment, rank): eight 8-bit digit passes over the segment's
// order-preserving 64-bit keys narrow the candidate prefix until the rank-th
// smallest key is fixed -- an exact selection, so the returned double is the
// very element std::sort would have put at that index.  Histograms live in
// shared memory; the segment is streamed from HBM/L2 once per pass with
// coalesced loads; the digit's bin is found by a warp scan.
#include <cmath>
#include <vector>

#include "runtime.h"
#include "select.h"

namespace ssgk {

__device__ __forceinline__ unsigned long long order_key(double d) {
  unsigned long long u = (unsigned long long)__double_as_longlong(d);
  return (u >> 63) ? ~u : (u | (1ull << 63));
}
__device__ __forceinline__ double key_value(unsigned long long k) {
  const unsigned long long u = (k >> 63) ? (k & ~(1ull << 63)) : ~k;
  return __longlong_as_double((long long)u);
}

constexpr int kSelectThreads = 512;
constexpr int kSelectWarps = kSelectThreads / 32;

// tasks[t] = {segment, rank (0-based)}; seg_off[s]..seg_off[s+1] spans the samples
__global__ void __launch_bounds__(kSelectThreads)
    k_select(const double* __restrict__ samples, const int64_t* __restrict__ seg_off,
             const SelectTask* __restrict__ tasks, int64_t ntasks, double* __restrict__ out) {
  // per-warp histograms (atomics contend within a warp only), summed per pass
  __shared__ unsigned int whist[kSelectWarps][256];
  __shared__ unsigned int hist[256];
  __shared__ unsigned long long s_prefix;
  __shared__ long long s_rank;
  const int64_t t = blockIdx.x;
  if (t >= ntasks) return;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const SelectTask task = tasks[t];
  const int64_t lo = seg_off[task.segment], hi = seg_off[task.segment + 1];
  if (threadIdx.x == 0) {
    s_prefix = 0;
    s_rank = task.rank;
  }
  for (int pass = 0; pass < 8; ++pass) {
    const int shift = 56 - 8 * pass;
    for (int b = lane; b < 256; b += 32) whist[warp][b] = 0;
    __syncthreads();
    const unsigned long long prefix = s_prefix;
    const unsigned long long pmask = pass == 0 ? 0ull : (~0ull << (shift + 8));
    for (int64_t i = lo + threadIdx.x; i < hi; i += blockDim.x) {
      const unsigned long long k = order_key(__ldg(samples + i));
      if ((k & pmask) == prefix) atomicAdd(&whist[warp][(k >> shift) & 0xff], 1u);
    }
    __syncthreads();
    if (threadIdx.x < 256) {
      unsigned int c = 0;
#pragma unroll
      for (int w = 0; w < kSelectWarps; ++w) c += whist[w][threadIdx.x];
      hist[threadIdx.x] = c;
    }
    __syncthreads();
    if (warp == 0) {
      // the digit: first bin whose inclusive count exceeds the rank -- lane l
      // owns bins 8l..8l+7, a warp scan gives each lane the count before them
      unsigned int own[8], sum = 0;
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        own[q] = hist[8 * lane + q];
        sum += own[q];
      }
      unsigned long long incl = sum;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const unsigned long long v = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += v;
      }
      const long long r = s_rank;
      const unsigned long long before = incl - sum;
      const unsigned hit = __ballot_sync(0xffffffffu, (long long)incl > r);
      const int L = __ffs(hit) - 1;  // the rank lies in the segment, so some lane hits
      if (lane == L) {
        long long rr = r - (long long)before;
        int b = 0;
        for (; b < 7; ++b) {
          if (rr < (long long)own[b]) break;
          rr -= own[b];
        }
        s_rank = rr;
        s_prefix = prefix | ((unsigned long long)(8 * L + b) << shift);
      }
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) out[t] = key_value(s_prefix);
}

}  // namespace ssgk

namespace ssg {

int64_t nearest_rank_index(int64_t n, double q) {
  // stats.hpp:20-23: rank = ceil(q * n) (as size_t), at least 1; index = rank - 1
  auto rank = static_cast<int64_t>(std::ceil(q * static_cast<double>(n)));
  if (rank < 1) rank = 1;
  return rank - 1;
}

void launch_select(const double* d_samples, const int64_t* d_seg_off, const SelectTask* d_tasks,
                   int64_t ntasks, double* d_out, cudaStream_t s) {
  if (ntasks <= 0) return;
  ssgk::k_select<<<(unsigned)ntasks, ssgk::kSelectThreads, 0, s>>>(d_samples, d_seg_off, d_tasks,
                                                                   ntasks, d_out);
  cuda_check(cudaGetLastError(), "k_select launch");
  stats().launches_select += 1;
}

std::vector<double> device_percentiles(const std::vector<double>& samples,
                                       const std::vector<double>& qs) {
  auto& ctx = context();
  cudaStream_t s = ctx.stream;
  const int64_t n = static_cast<int64_t>(samples.size());
  DeviceBuffer<double> d_samples, d_out;
  DeviceBuffer<int64_t> d_off;
  DeviceBuffer<SelectTask> d_tasks;
  std::vector<int64_t> off = {0, n};
  std::vector<SelectTask> tasks;
  for (double q : qs) tasks.push_back(SelectTask{0, nearest_rank_index(n, q)});
  d_samples.upload(samples, s);
  d_off.upload(off, s);
  d_tasks.upload(tasks, s);
  d_out.resize(tasks.size());
  launch_select(d_samples.ptr, d_off.ptr, d_tasks.ptr, static_cast<int64_t>(tasks.size()), d_out.ptr, s);
  std::vector<double> out(tasks.size());
  d_out.download(out.data(), out.size(), s);
  cuda_check(cudaStreamSynchronize(s), "percentile select");
  return out;
}

}  // namespace ssg
