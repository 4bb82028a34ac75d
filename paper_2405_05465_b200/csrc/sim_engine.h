// sim_engine.h -- launch descriptor of the simulation kernel (host <-> device).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "sim_device.h"
#include "ssg_device.h"

#ifndef SSG_SIM_WARPS
#define SSG_SIM_WARPS 2  // warps per block: units differ wildly in length, keep blocks small
#endif

struct SimLaunch {
  const SimConfig* configs;
  const SimUnit* units;
  const int32_t* order;  // unit launch order (longest first), may be null
  int64_t nunits;
  const SsgEstView* ests;
  ReqHot* hot;
  ReqTimes* tm;
  const int64_t* ids;
  int32_t* restarts;
  const int64_t* emit_base;  // may be null
  double* emissions;         // may be null
  const int32_t* arr_order;  // may be null (identity)
  RepState* reps;
  int32_t* ws;
  int64_t* log;              // may be null
  SimUnitOut* out;
  const double* tables;       // token tables pool, may be null
  int32_t fast_forward;       // 1: pure-decode stretches of lone replicas take the fast loop
  int32_t has_forest;         // any estimator of the launch has forest models
  uint32_t* group_fail;       // per speculation group: bits of the probes that failed, may be null
  int32_t all_lone;           // every unit is one replica without the deferred pool (LONE kernels)
};

namespace ssg {
// SSG_NO_FASTFWD=1 disables the pure-decode fast-forward (A/B checks).
int fast_forward_enabled();
// Sweeps compile the fast-forward out (measured faster: the many concurrent
// probe warps are instruction-fetch bound); SSG_SWEEP_FASTFWD=1 turns it on.
int sweep_fast_forward_enabled();
void launch_simulate(const SimLaunch& L, cudaStream_t s);
// Diagnostic builds (-DSSG_PHASE_CYCLES): per-unit phase cycles of the last
// k_simulate launch, SSG_PH_N per unit (engine.cuh SSG_PH_*); false otherwise.
bool phase_cycles(long long* dst, int64_t n);
// True when every unit simulates one replica that does not route through the
// deferred pool and the launch has no batch log and no arrival permutation --
// the launch may take the LONE kernel variant.
template <class Units, class Configs>
inline bool all_lone_units(const SimLaunch& L, const Units& units, const Configs& configs) {
  if (L.log || L.arr_order) return false;
  for (const auto& u : units)
    if (u.R != 1 || configs[u.config].routing == SSG_ROUTE_DEFERRED ||
        (u.flags & (SSG_UF_BATCH_LOG | SSG_UF_OBSERVER)))
      return false;
  return true;
}
// Builds the token tables of `n` configs (cfgs[i].tab_off / tab_stride set by
// the caller); valid[i*stride + t] gets bit0 = token/comm terms valid, bit1 =
// prefill-at-prior-0 valid.
void launch_build_tables(const SimConfig* d_cfgs, int32_t n, int32_t stride,
                         const SsgEstView* d_ests, double* d_pool, uint8_t* d_valid, cudaStream_t s);
}
