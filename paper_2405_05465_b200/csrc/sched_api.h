// sched_api.h -- launch descriptor of the step-wise scheduler kernel
// (sched_api.cu), shared by the host ReplicaScheduler (host/scheduler.cpp).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "sim_device.h"

#define SSG_SCHED_ENQUEUE 0   // enqueue slot `arg` (scheduler.hpp:146-155)
#define SSG_SCHED_SCHEDULE 1  // schedule_iteration at `now` (scheduler.hpp:184-194)
#define SSG_SCHED_COMPLETE 2  // complete_iteration of the np/nd plan in P_*/D_* (scheduler.hpp:197-233)
#define SSG_SCHED_RENUMBER 3  // open slot `arg` among `n` slots (out-of-order enqueue)

struct SchedArgs {
  int32_t op, arg;
  int32_t n;       // slots in use (RENUMBER)
  int32_t serial;  // schedule_iteration counter (the planned_ set's stamp)
  int32_t np, nd;  // COMPLETE: plan sizes
  double now;
  const SimConfig* cfg;
  const SimUnit* unit;
  ReqHot* hot;
  ReqTimes* tm;
  int64_t* ids;
  int32_t* restarts;
  RepState* reps;
  int32_t* ws;
  SimUnitOut* out;
};

namespace ssg {
void launch_sched_op(const SchedArgs& a, cudaStream_t s);
}
