// sweep.h -- device-resident probe streams for the capacity sweep.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "runtime.h"
#include "sim_device.h"

// One probe / SLO run / static run of one candidate: which units carry it.
struct ProbeDesc {
  double qps;          // arrival rate (ignored for static runs)
  int32_t R;           // replicas of the candidate
  int32_t first_unit;  // its units are [first_unit, first_unit + (decoupled ? R : 1))
  int32_t decoupled;   // 1: one unit per RR replica; 0: one coupled unit
  int32_t static_run;  // all arrivals at t = 0 (makespan objective)
  int64_t emis_base;   // trace-order emission layout base, or -1 (no emissions)
};

namespace ssg {

// The probe trace (first probe_requests workload lengths, ids 0..n-1) and the
// unit exponentials of the probe seed, resident in HBM for a whole sweep.
struct ResidentWorkload {
  int32_t n = 0;
  int64_t emis_per_probe = 0;  // sum of decode tokens
  DeviceBuffer<int32_t> pre, dec;
  DeviceBuffer<double> unit_exp;
  DeviceBuffer<int64_t> dec_prefix;  // exclusive prefix of decode tokens
  DeviceBuffer<uint8_t> first_emis;  // 1 at each request's first emission slot
};

// Drops the pooled sweep lanes (streams, HBM, pinned staging); ssg_shutdown.
void release_sweep_lanes();

void launch_probe_setup(const ProbeDesc* d_probes, int32_t nprobes, const SimUnit* d_units,
                        const ResidentWorkload& w, ReqHot* hot, ReqTimes* tm, int64_t* ids,
                        int64_t* emit_base, cudaStream_t s);
void launch_slo_samples(const ProbeDesc* d_probes, int32_t nprobes, const SimUnit* d_units,
                        const ReqTimes* tm, const ResidentWorkload& w, const double* emis,
                        double* delay, double* ttft, double* gaps, cudaStream_t s);

}  // namespace ssg
