// sched_api.cu -- the reference's step-wise scheduler plugin API
// (ReplicaScheduler, scheduler.hpp:136-233) on the GPU: the replica's queues,
// block accounting and per-request progress live in HBM, and every call
// (enqueue, schedule_iteration, complete_iteration) is one warp running the
// same device scheduler code the simulation kernel runs (engine.cuh), so a
// plan produced here is by construction the plan the engine would form.
//
// Request slots are ordered by (arrival, id) -- the device queues compare slot
// indices, exactly like the engine's unit-local indices.  A request enqueued
// out of that order is inserted by renumbering: slots >= p move up by one and
// every queued index is remapped (k_sched_op, op RENUMBER).
#include "engine.cuh"
#include "runtime.h"
#include "sched_api.h"

namespace ssgk {

// One warp; every op loads the replica, acts, stores it back.
__global__ void __launch_bounds__(32) k_sched_op(SchedArgs A) {
  Unit U;
  U.cfg = A.cfg;
  U.u = A.unit;
  U.E = SsgEstView{};
  U.hot = A.hot;
  U.tm = A.tm;
  U.ids = A.ids;
  U.restarts = A.restarts;
  U.emit_base = nullptr;
  U.emissions = nullptr;
  U.arr_order = nullptr;
  U.reps = A.reps;
  U.ws = A.ws;
  U.log = nullptr;
  U.out = A.out;
  U.smem_stats = nullptr;
  U.tables = nullptr;
  U.smem_part = nullptr;
  U.pcap = SSG_MAX_PP;
  U.group_fail = nullptr;
  U.fast = 0;
  U.lane = threadIdx.x & 31;
  U.MB = A.cfg->max_batch;
  U.WC = A.unit->wait_cap;
  U.rep_stride = 6LL * U.MB + U.WC;
  U.serial = A.serial;
  U.qbytes = 0;
  U.iters = 0;
  U.entries = 0;
  U.clock = A.now;
  U.flops = 0.0;
  U.seq = 0;
  U.ax1_hint = 0;
  U.qb_lane = 0;
  U.plan_tokens = 0;
  U.plan_late = 0;
  if (U.lane == 0) {
    SimUnitOut o;
    memset(&o, 0, sizeof o);
    *U.out = o;
  }
  __syncwarp();
  RepState S = load_rep(U, 0);
  switch (A.op) {
    case SSG_SCHED_ENQUEUE:
      enqueue(U, S, 0, A.arg);
      break;
    case SSG_SCHED_SCHEDULE: {
      S.np = 0;
      S.nd = 0;
      schedule_batch(U, S, 0);
      const int32_t tokens = U.plan_tokens + S.nd;
      // sarathi's closing check (scheduler.hpp:441-442)
      if (!failed(U) && U.cfg->policy == SSG_POL_SARATHI && tokens > U.cfg->chunk)
        set_error(U, SSG_ERR_INTERNAL, 5, tokens, 0, 0.0);
      break;
    }
    case SSG_SCHED_COMPLETE:
      // the plan's entries were written to P_*/D_* by the host
      S.np = A.np;
      S.nd = A.nd;
      complete_batch(U, S, 0);
      S.np = 0;
      S.nd = 0;
      break;
    case SSG_SCHED_RENUMBER: {
      // make room for a request whose (arrival, id) sorts at slot p
      const int32_t p = A.arg, n = A.n;
      for (int32_t c = n; c > p; c -= 32) {
        const int32_t i = c - 1 - U.lane;
        ReqHot h;
        ReqTimes t;
        int64_t id = 0;
        int32_t rs = 0;
        if (i >= p) {
          h = U.hot[i];
          t = U.tm[i];
          id = U.ids[i];
          rs = U.restarts[i];
        }
        __syncwarp();
        if (i >= p) {
          U.hot[i + 1] = h;
          U.tm[i + 1] = t;
          A.ids[i + 1] = id;
          U.restarts[i + 1] = rs;
        }
        __syncwarp();
      }
      int32_t* run = RUN(U, 0);
      for (int32_t k = U.lane; k < S.run_n; k += 32)
        if (run[k] >= p) run[k] += 1;
      int32_t* w = WAIT(U, 0);
      const int32_t mask = U.WC - 1;
      for (int32_t k = U.lane; k < S.wait_n; k += 32) {
        int32_t& v = w[(S.wait_head + k) & mask];
        if (v >= p) v += 1;
      }
      __syncwarp();
      break;
    }
    default:
      set_error(U, SSG_ERR_INTERNAL, 0, 0, 0, 0.0);
  }
  store_rep(U, 0, S);
  if (U.lane == 0) U.out->late = U.plan_tokens;  // tokens of prefill chunks planned (diagnostic)
}

}  // namespace ssgk

namespace ssg {

void launch_sched_op(const SchedArgs& a, cudaStream_t s) {
  ssgk::k_sched_op<<<1, 32, 0, s>>>(a);
  cuda_check(cudaGetLastError(), "k_sched_op launch");
  stats().launches_setup += 1;
}

}  // namespace ssg
