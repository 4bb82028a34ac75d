// sim_host.h -- host staging for simulation launches (used by sim.cpp and the
// sweep in search.cpp).
#pragma once
#include <vector>

#include "runtime.h"
#include "servesim_b200.hpp"
#include "sim_engine.h"

namespace ssg {

// Flattens one cluster config for the device (validations and error messages
// as run_simulation's preamble, sim.hpp:139-150).
SimConfig make_sim_config(const servesim::ClusterConfig& cluster,
                          const servesim::EstimatorModel& est, int32_t est_index,
                          servesim::MemoryPlan* plan_out = nullptr);

// The per-stage operator table (derive_operators order) with model slots.
void fill_sim_ops(SimConfig& c, const std::vector<servesim::OperatorDescriptor>& ops,
                  const servesim::DeviceEstimator& de);

// predict_batch + batch_device_flops over compositions (CSR), one warp each,
// through the same device code the engine uses (engine.cu).
void predict_batches(const servesim::EstimatorModel& est, const SimConfig& cfg, int64_t n,
                     const int64_t* p_off, const int64_t* p_len, const int64_t* p_prior,
                     const int64_t* d_off, const int64_t* d_ctx, double* seconds, double* flops);

// Same over compositions of several configs (cfgs[comp_cfg[c]]; cfgs[].est
// indexes ests); per-composition status instead of exceptions.
void predict_batches_multi(const std::vector<SimConfig>& cfgs, const std::vector<SsgEstView>& ests,
                           const std::vector<int32_t>& comp_cfg, int64_t n, const int64_t* p_off,
                           const int64_t* p_len, const int64_t* p_prior, const int64_t* d_off,
                           const int64_t* d_ctx, double* seconds, double* flops,
                           std::vector<SimUnitOut>& status);

// Token tables (SimConfig::tab_*) for `cfgs`: configs with equal operator
// tables (same estimator, tp, pp) share one table.  Fills tab_off / stride /
// tmax / pmax in place and leaves the pool in `pool` (device).
void build_token_tables(std::vector<SimConfig>& cfgs, const std::vector<SsgEstView>& ests,
                        const std::vector<const servesim::DeviceEstimator*>& est_of,
                        DeviceBuffer<double>& pool);

struct UnitSpec {
  int32_t config = 0;
  int32_t R = 1;
  int32_t flags = 0;
  double abort_thr = 0.0;
  int32_t abort_max_late = 0;
  int64_t log_cap = 0;
};

// Everything one k_simulate launch needs, staged on the host.
struct SimJobs {
  std::vector<SimConfig> configs;
  std::vector<SsgEstView> ests;
  std::vector<SimUnit> units;
  std::vector<ReqHot> hot;
  std::vector<ReqTimes> tm;
  std::vector<int64_t> ids;
  std::vector<int64_t> emit_base;
  std::vector<int32_t> arr_order;
  int64_t ws_words = 0, nreps = 0, log_words = 0, emissions = 0;
  bool any_order = false;
  const double* tables = nullptr;  // token tables pool (device), if built
  bool has_forest = false;         // any estimator of the launch uses forests

  // Adds a unit over the given requests, which must already be in (arrival,
  // id) order; `event_order` (may be empty = identity) lists local indices in
  // arrival-event order.  Returns the unit index.
  int32_t add_unit(const UnitSpec& spec, const std::vector<servesim::Request>& reqs,
                   const std::vector<int32_t>& event_order);
};

struct SimResults {
  std::vector<SimUnitOut> out;
  std::vector<RepState> reps;
  std::vector<ReqTimes> tm;
  std::vector<int32_t> restarts;
  std::vector<double> emissions;
  std::vector<int64_t> log;
};

// Uploads, runs and downloads one launch on the library stream.
void run_jobs(const SimJobs& jobs, SimResults& res, bool want_requests);

// Reference-format messages for device error codes.
[[noreturn]] void raise_unit_error(const SimUnitOut& o, const SimConfig& cfg,
                                   const servesim::EstimatorModel& est);

}  // namespace ssg
