// sweep.cu -- device-side setup and measurement for the capacity sweep.
//
// k_probe_setup   one warp per probe rebuilds the probe's Poisson arrivals
//                 t_i = t_{i-1} + max(E_i / qps, 1e-12) from the resident unit
//                 exponentials (workload.hpp:96-103) and scatters the request
//                 stream into the probe's simulation units (RR replica r owns
//                 trace positions r, r+R, ...), so a round uploads only the unit
//                 descriptors, never request data.
// k_slo_samples   per SLO-run request: scheduling delay and TTFT; per emission:
//                 the time-between-tokens gap (first emission of a request -> +inf,
//                 which sorts past every rank the select asks for)
//                 (metrics.hpp:38-52).
#include "runtime.h"
#include "sim_engine.h"
#include "sweep.h"

namespace ssgk {

// One warp per probe: lanes take 32 trace positions at a time (gaps, request
// records, emission bases in parallel); the arrival times are the exact
// left-to-right fp64 running sum, a chain of one add per request that reads
// the gaps through shuffles issued ahead of it.
__global__ void k_probe_setup(const ProbeDesc* __restrict__ probes, int32_t nprobes,
                              const SimUnit* __restrict__ units, const int32_t* __restrict__ pre,
                              const int32_t* __restrict__ dec, const double* __restrict__ unit_exp,
                              const int64_t* __restrict__ dec_prefix, int32_t n, ReqHot* hot,
                              ReqTimes* tm, int64_t* ids, int64_t* emit_base) {
  const int32_t p = (int32_t)((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5);
  const int lane = threadIdx.x & 31;
  if (p >= nprobes) return;  // warp-uniform
  const ProbeDesc P = probes[p];
  double t = 0.0;
  for (int32_t base = 0; base < n; base += 32) {
    const int32_t i = base + lane;
    const bool on = i < n;
    double gap = 0.0;
    if (on && !P.static_run) {
      gap = __ddiv_rn(unit_exp[i], P.qps);
      gap = gap < 1e-12 ? 1e-12 : gap;  // std::max(gap, 1e-12)
    }
    double arrival = 0.0;
    const int32_t kmax = n - base < 32 ? n - base : 32;
#pragma unroll
    for (int k = 0; k < 32; ++k) {
      const double gk = __shfl_sync(0xffffffffu, gap, k);
      if (k < kmax) t = P.static_run ? 0.0 : __dadd_rn(t, gk);
      if (k == lane) arrival = t;
    }
    if (!on) continue;
    const int32_t u = P.first_unit + (P.decoupled ? i % P.R : 0);
    const int32_t local = P.decoupled ? i / P.R : i;
    const int64_t g = units[u].req_off + local;
    ReqHot h;
    h.target = 0;
    h.done = 0;
    h.emitted = 0;
    h.kv = 0;
    h.held = 0;
    h.planned = 0;
    h.decode = dec[i];
    h.prefill = pre[i];
    hot[g] = h;
    ReqTimes r;
    r.arrival = arrival;
    r.first_sched = -1.0;
    r.first_tok = -1.0;
    r.completion = -1.0;
    tm[g] = r;
    ids[g] = i;
    if (emit_base) emit_base[g] = P.emis_base >= 0 ? P.emis_base + dec_prefix[i] : -1;
  }
}

// grid: (ceil(n / 256), nprobes); requests in trace order per probe
__global__ void k_slo_request_samples(const ProbeDesc* __restrict__ probes,
                                      const SimUnit* __restrict__ units,
                                      const ReqTimes* __restrict__ tm, int32_t n,
                                      double* __restrict__ delay, double* __restrict__ ttft) {
  const int32_t p = blockIdx.y;
  const int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const ProbeDesc P = probes[p];
  const int32_t u = P.first_unit + (P.decoupled ? i % P.R : 0);
  const int32_t local = P.decoupled ? i / P.R : i;
  const ReqTimes t = tm[units[u].req_off + local];
  delay[(int64_t)p * n + i] = t.first_sched - t.arrival;
  ttft[(int64_t)p * n + i] = t.first_tok - t.arrival;
}

// emissions of one probe are laid out in trace order (emis_base + dec_prefix[i]);
// first[k] marks the first emission slot of a request within that layout
__global__ void k_slo_gaps(const double* __restrict__ emis, const uint8_t* __restrict__ first,
                           int64_t per_probe, int64_t total, double* __restrict__ gaps) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= total) return;
  const int64_t w = k % per_probe;
  gaps[k] = first[w] ? INFINITY : __dsub_rn(emis[k], emis[k - 1]);
}

}  // namespace ssgk

namespace ssg {

void launch_probe_setup(const ProbeDesc* d_probes, int32_t nprobes, const SimUnit* d_units,
                        const ResidentWorkload& w, ReqHot* hot, ReqTimes* tm, int64_t* ids,
                        int64_t* emit_base, cudaStream_t s) {
  if (nprobes <= 0) return;
  const int threads = 128;  // 4 probes (warps) per block
  const int64_t blocks = ((int64_t)nprobes * 32 + threads - 1) / threads;
  ssgk::k_probe_setup<<<(unsigned)blocks, threads, 0, s>>>(
      d_probes, nprobes, d_units, w.pre.ptr, w.dec.ptr, w.unit_exp.ptr, w.dec_prefix.ptr, w.n, hot,
      tm, ids, emit_base);
  cuda_check(cudaGetLastError(), "k_probe_setup launch");
  stats().launches_setup += 1;
}

void launch_slo_samples(const ProbeDesc* d_probes, int32_t nprobes, const SimUnit* d_units,
                        const ReqTimes* tm, const ResidentWorkload& w, const double* emis,
                        double* delay, double* ttft, double* gaps, cudaStream_t s) {
  if (nprobes <= 0) return;
  dim3 g1((w.n + 255) / 256, nprobes);
  ssgk::k_slo_request_samples<<<g1, 256, 0, s>>>(d_probes, d_units, tm, w.n, delay, ttft);
  cuda_check(cudaGetLastError(), "k_slo_request_samples launch");
  const int64_t total = w.emis_per_probe * nprobes;
  ssgk::k_slo_gaps<<<(unsigned)((total + 255) / 256), 256, 0, s>>>(emis, w.first_emis.ptr,
                                                                    w.emis_per_probe, total, gaps);
  cuda_check(cudaGetLastError(), "k_slo_gaps launch");
  stats().launches_setup += 2;
}

}  // namespace ssg
