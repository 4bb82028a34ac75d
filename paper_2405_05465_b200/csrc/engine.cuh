// engine.cuh -- K3: one warp simulates one unit (a replica, or a routed group
// of replicas) event by event, exactly as the reference's engine and
// schedulers do.
//
// reference: sim.hpp:135-320 (event loop), scheduler.hpp:136-561 (policies,
//            preemption, routing), memory.hpp:51-104 (block accounting),
//            estimator.hpp:294-380 (batch latency and flops),
//            scheduler.hpp:566-579 (pipeline makespan)
//
// Execution model.  All 32 lanes run the scheduler's control flow together on
// identical (warp-uniform) scalars held in registers.  Every store of shared
// sequential state goes through wput(): a warp barrier (all lanes finished
// reading the old value), one store from lane 0, a second barrier (the value is
// visible to every lane) -- so no lane ever depends on implicit lockstep.
// The data-parallel pieces -- decode admission over the running queue,
// completion of a batch, queue shifts, per-entry reductions and the per-
// operator predictor evaluations -- spread over lanes and end in __syncwarp().
// Sequential semantics that matter for parity (admission order, preemption of
// the latest unplanned runner, operator-order fp64 sums, tree-order forest
// sums) are kept exactly; parallel fast paths are taken only where they are
// provably equivalent (e.g. a decode window whose cumulative block shortfall
// fits in free memory cannot preempt).
#pragma once
#include "predictor.cuh"
#include "sim_device.h"

#define SSG_FULL 0xffffffffu

// Code-placement knobs (the simulation kernel is instruction-fetch bound):
// SSG_COLD marks rarely executed scheduler paths, SSG_WARM the per-policy
// schedulers.  Each expands to __noinline__ or __forceinline__ at build time.
#ifndef SSG_COLD
#define SSG_COLD __forceinline__
#endif
#ifndef SSG_WARM
#define SSG_WARM __forceinline__
#endif

namespace ssgk {

// The attention query's libm calls at the two per-iteration sites (batch
// latency, fast-forward).  SSG_LIBM_CALLS=1 (A/B builds) emits them once as
// out-of-line functions instead of inlining a copy at each site.
#if defined(SSG_LIBM_CALLS) && SSG_LIBM_CALLS
template <int FMA>
__device__ __noinline__ double hot_log1p(double x) { return ssg_log1p(x, FMA); }
template <int FMA>
__device__ __noinline__ double hot_exp(double x) { return ssg_exp(x, FMA); }
#else
template <int FMA>
__device__ __forceinline__ double hot_log1p(double x) { return ssg_log1p(x, FMA); }
template <int FMA>
__device__ __forceinline__ double hot_exp(double x) { return ssg_exp(x, FMA); }
#endif

struct Unit {
  const SimConfig* cfg;
  const SimUnit* u;
  SsgEstView E;
  ReqHot* hot;
  ReqTimes* tm;
  const int64_t* ids;
  int32_t* restarts;
  const int64_t* emit_base;
  double* emissions;
  const int32_t* arr_order;
  RepState* reps;
  int32_t* ws;
  int64_t* log;
  SimUnitOut* out;
  int64_t* smem_stats;  // per-warp scratch [pcap * 6] (shared memory, HBM for deep pipelines)
  const double* tables; // token tables pool (SimConfig::tab_off)
  double* smem_part;    // per-warp scratch [4 * pcap]
  int32_t pcap;         // microbatches the scratch holds (SSG_MAX_PP, or pp above it)
  uint32_t* group_fail;  // this unit's speculation-group failure mask (may be null)
  int fast;         // pure-decode fast-forward enabled
  int lane;
  int64_t rep_stride;  // int32 words per replica in ws
  int32_t MB, WC;
  int32_t serial;      // schedule_iteration counter (planned_ stamp)
  int64_t qbytes;      // predictor bytes (accounting only)
  int64_t iters, entries;
  double clock;
  uint64_t seq;
  int32_t ax1_hint;    // per lane: last axis-1 interp cell of this lane's attention query
  int64_t qb_lane;     // per lane: predictor bytes of the microbatches this lane summed
  // counted while the scheduler forms a batch (reset by batch_start):
  int32_t plan_tokens; // prefill chunk tokens pushed
  int32_t plan_late;   // requests first scheduled now, later than the abort threshold
  double flops;        // total_model_flops so far (written to SimUnitOut at the end)
#ifdef SSG_PHASE_CYCLES
  long long ph[SSG_PH_N];  // diagnostic build: cycles per event-loop phase (SSG_PH_*)
#endif
};

// Diagnostic builds (-DSSG_PHASE_CYCLES) charge clock64 deltas to phases:
// 0 schedule, 1 batch latency, 2 batch complete, 3 fast-forward calls,
// 4 arrivals, 5 fast-forwarded iterations (a count), 6 whole unit,
// 7 fast-forward calls (a count); inside the batch latency (table path):
// 8 per-microbatch sums, 9 query setup and attention queries, 11 operator-order
// sums, 10 makespan; counts: 12 BatchStarts with more than 32 runners, 13 with
// requests waiting and room in the batch, 14 fast-forward calls that ran no
// iteration, 15 batches with a prefill chunk.
#ifdef SSG_PHASE_CYCLES
#define SSG_PH_BEGIN(v) const long long v = clock64()
#define SSG_PH_END(v, k) (U.ph[k] += clock64() - (v))
#else
#define SSG_PH_BEGIN(v)
#define SSG_PH_END(v, k)
#endif

// ---------------------------------------------------------------- workspace
__device__ __forceinline__ int32_t* rep_ws(Unit& U, int r) { return U.ws + r * U.rep_stride; }
__device__ __forceinline__ int32_t* RUN(Unit& U, int r) { return rep_ws(U, r); }
__device__ __forceinline__ int32_t* WAIT(Unit& U, int r) { return rep_ws(U, r) + U.MB; }
__device__ __forceinline__ int32_t* P_IDX(Unit& U, int r) { return rep_ws(U, r) + U.MB + U.WC; }
__device__ __forceinline__ int32_t* P_CHUNK(Unit& U, int r) { return P_IDX(U, r) + U.MB; }
__device__ __forceinline__ int32_t* P_PRIOR(Unit& U, int r) { return P_IDX(U, r) + 2 * U.MB; }
__device__ __forceinline__ int32_t* D_IDX(Unit& U, int r) { return P_IDX(U, r) + 3 * U.MB; }
__device__ __forceinline__ int32_t* D_CTX(Unit& U, int r) { return P_IDX(U, r) + 4 * U.MB; }
__device__ __forceinline__ int32_t* POOL(Unit& U) { return U.ws + U.u->R * U.rep_stride; }
// pool ring state lives after the pool itself
__device__ __forceinline__ int32_t* POOL_HEAD(Unit& U) { return POOL(U) + U.WC; }

__host__ __device__ inline int64_t unit_ws_words(int R, int MB, int WC) {
  return (int64_t)R * (6LL * MB + WC) + WC + 2;
}

// ---------------------------------------------------------------- stores
template <typename T>
__device__ __forceinline__ void wput(const Unit& U, T* p, T v) {
  __syncwarp();
  if (U.lane == 0) *p = v;
  __syncwarp();
}
// Several lane-0 stores under one pair of barriers.
#define WSTORE_BEGIN(U) \
  __syncwarp();         \
  if ((U).lane == 0) {
#define WSTORE_END \
  }                \
  __syncwarp();

// Warp sum of non-negative 64-bit values: one REDUX when every lane's value is
// below 2^26 (the 32-lane total then fits 31 bits), else a shuffle tree.
__device__ __forceinline__ int64_t warp_sum64(int64_t v) {
  if (__all_sync(SSG_FULL, (v >> 26) == 0)) return (int64_t)__reduce_add_sync(SSG_FULL, (unsigned)v);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(SSG_FULL, v, o);
  return v;
}

// ---------------------------------------------------------------- errors
static __device__ SSG_COLD void set_error(Unit& U, int code, int32_t i32, int64_t a, int64_t b,
                                          double f) {
  __syncwarp();
  if (U.lane == 0 && U.out->code == SSG_OK) {
    U.out->code = code;
    U.out->err_i32 = i32;
    U.out->err_i64[0] = a;
    U.out->err_i64[1] = b;
    U.out->err_f64 = f;
    U.out->err_time = U.clock;
  }
  __syncwarp();
}
__device__ __forceinline__ bool failed(Unit& U) { return U.out->code != SSG_OK; }

// ---------------------------------------------------------------- blocks
__device__ __forceinline__ int64_t units_for(const SimConfig& c, int64_t tokens) {
  // ceil(tokens / block_size), tokens >= 0, as one 64-bit multiply-high of
  // tokens + block_size - 1 by bs_magic (block_magic, sim_device.h): exact for
  // every power of two and for numerators below 2^32 otherwise (tokens < 2^31,
  // block_size < 2^31, both checked on the host).  bs_magic == 0: one unit per
  // token (LightLLM, or block_size 1).  A single branch-free form keeps the
  // dozen inlined block-accounting sites small (the kernel is fetch bound).
  return c.bs_magic ? (int64_t)__umul64hi((uint64_t)(tokens + c.block_size - 1), c.bs_magic) : tokens;
}
__device__ __forceinline__ int64_t shortfall_held(const SimConfig& c, int32_t held, int64_t tokens) {
  int64_t s = units_for(c, tokens) - (int64_t)held;
  return s > 0 ? s : 0;
}
__device__ __forceinline__ int64_t shortfall(const SimConfig& c, const ReqHot& h, int64_t tokens) {
  int64_t s = units_for(c, tokens) - (int64_t)h.held;
  return s > 0 ? s : 0;
}
// BlockManager::try_reserve (memory.hpp:82-89)
__device__ __forceinline__ bool try_reserve(Unit& U, RepState& S, int32_t j, int64_t tokens) {
  const SimConfig& c = *U.cfg;
  const int64_t need = shortfall(c, U.hot[j], tokens);
  if (need > c.total_units - S.allocated) return false;
  wput(U, &U.hot[j].held, U.hot[j].held + (int32_t)need);
  S.allocated += need;
  return true;
}
// BlockManager::release (memory.hpp:91-97)
__device__ __forceinline__ void release(Unit& U, RepState& S, int32_t j) {
  S.allocated -= U.hot[j].held;
  wput(U, &U.hot[j].held, 0);
}

// ---------------------------------------------------------------- queues
// Shift a[lo, hi) by `delta` (+1 or -1) positions, warp-cooperatively; the
// ring variant maps logical positions through (base + p) & mask.
__device__ __forceinline__ void ring_shift(Unit& U, int32_t* a, int32_t mask, int32_t base,
                                           int32_t lo, int32_t hi, int delta) {
  const int n = hi - lo;
  if (n <= 0) return;
  if (delta < 0) {
#pragma unroll 1
    for (int c = 0; c < n; c += 32) {
      const int p = lo + c + U.lane;
      int32_t v = 0;
      if (p < hi) v = a[(base + p) & mask];
      __syncwarp();
      if (p < hi) a[(base + p - 1) & mask] = v;
      __syncwarp();
    }
  } else {
#pragma unroll 1
    for (int c = n; c > 0; c -= 32) {
      const int p = lo + c - 1 - U.lane;
      int32_t v = 0;
      if (p >= lo) v = a[(base + p) & mask];
      __syncwarp();
      if (p >= lo) a[(base + p + 1) & mask] = v;
      __syncwarp();
    }
  }
}

// first logical position whose value is > x (upper_bound) in a sorted ring
__device__ __forceinline__ int32_t ring_upper(const int32_t* a, int32_t mask, int32_t base,
                                              int32_t n, int32_t x) {
  int32_t first = 0, count = n;
  while (count > 0) {
    int32_t step = count >> 1;
    if (!(x < a[(base + first + step) & mask])) {
      first += step + 1;
      count -= step + 1;
    } else {
      count = step;
    }
  }
  return first;
}

// insert_sorted(waiting_, r) (scheduler.hpp:243-247)
__device__ __forceinline__ void wait_insert(Unit& U, RepState& S, int r, int32_t j) {
  int32_t* w = WAIT(U, r);
  const int32_t mask = U.WC - 1;
  int32_t pos;
  if (S.wait_n == 0 || w[(S.wait_head + S.wait_n - 1) & mask] < j)
    pos = S.wait_n;
  else
    pos = ring_upper(w, mask, S.wait_head, S.wait_n, j);
  if (pos < S.wait_n - pos) {  // shift the front part left by one
    ring_shift(U, w, mask, S.wait_head, 0, pos, -1);
    S.wait_head = (S.wait_head - 1) & mask;
  } else {
    ring_shift(U, w, mask, S.wait_head, pos, S.wait_n, +1);
  }
  wput(U, &w[(S.wait_head + pos) & mask], j);
  S.wait_n += 1;
}

// erase_from_waiting (scheduler.hpp:474-478); the queue is sorted, so the
// element's position is its lower bound.
__device__ __forceinline__ void wait_erase(Unit& U, RepState& S, int r, int32_t j) {
  int32_t* w = WAIT(U, r);
  const int32_t mask = U.WC - 1;
  if (S.wait_n > 0 && w[S.wait_head & mask] == j) {
    // the admitted head (every admission): no search, no shift
    if (S.wait_n > 1) S.wait_head = (S.wait_head + 1) & mask;
    S.wait_n -= 1;
    __syncwarp();
    return;
  }
  int32_t pos = ring_upper(w, mask, S.wait_head, S.wait_n, j - 1);
  if (pos >= S.wait_n || w[(S.wait_head + pos) & mask] != j) {
    set_error(U, SSG_ERR_INTERNAL, 1, j, 0, 0.0);  // "request not in waiting queue"
    return;
  }
  if (pos < S.wait_n - 1 - pos) {
    ring_shift(U, w, mask, S.wait_head, 0, pos, +1);
    S.wait_head = (S.wait_head + 1) & mask;
  } else {
    ring_shift(U, w, mask, S.wait_head, pos + 1, S.wait_n, -1);
  }
  S.wait_n -= 1;
  __syncwarp();
}

__device__ __forceinline__ int32_t wait_front(Unit& U, const RepState& S, int r) {
  return WAIT(U, r)[S.wait_head & (U.WC - 1)];
}

// insert_sorted_running (scheduler.hpp:249-252)
__device__ __forceinline__ void run_insert(Unit& U, RepState& S, int r, int32_t j) {
  int32_t* a = RUN(U, r);
  int32_t pos;
  if (S.run_n == 0 || a[S.run_n - 1] < j)
    pos = S.run_n;
  else
    pos = ring_upper(a, 0x7fffffff, 0, S.run_n, j);
  ring_shift(U, a, 0x7fffffff, 0, pos, S.run_n, +1);
  wput(U, &a[pos], j);
  S.run_n += 1;
}

__device__ __forceinline__ void run_erase_at(Unit& U, RepState& S, int r, int32_t pos) {
  int32_t* a = RUN(U, r);
  ring_shift(U, a, 0x7fffffff, 0, pos + 1, S.run_n, -1);
  S.run_n -= 1;
  __syncwarp();
}

// ---------------------------------------------------------------- scheduler
__device__ __forceinline__ bool finished(const ReqHot& h) { return h.emitted >= h.decode; }
__device__ __forceinline__ bool prefill_complete(const ReqHot& h) { return h.done >= h.target; }

// mark_scheduled (scheduler.hpp:262-265)
__device__ __forceinline__ void mark_scheduled(Unit& U, int32_t j) {
  const ReqTimes t = U.tm[j];
  const bool first = t.first_sched < 0;
  // the probe abort counts batch entries with first_scheduled == clock that
  // waited past the threshold (sim.hpp:231-239); a request is marked at most
  // once per schedule, is in the batch iff marked, and gets first_scheduled ==
  // clock only here -- so the count can be taken as it happens
  if (first && U.clock - t.arrival > U.u->abort_thr) U.plan_late += 1;
  WSTORE_BEGIN(U)
  if (first) U.tm[j].first_sched = U.clock;
  U.hot[j].planned = U.serial;
  WSTORE_END
}

// preempt_latest (scheduler.hpp:269-285): returns the victim or -1.
static __device__ SSG_COLD int32_t preempt_latest(Unit& U, RepState& S, int r) {
  int32_t* a = RUN(U, r);
  for (int32_t p = S.run_n - 1; p >= 0; --p) {
    const int32_t v = a[p];
    if (U.hot[v].planned == U.serial) continue;
    run_erase_at(U, S, r, p);
    release(U, S, v);
    ReqHot& h = U.hot[v];
    const int32_t target = h.prefill + h.emitted, restarts = U.restarts[v] + 1;
    WSTORE_BEGIN(U)
    h.kv = 0;
    h.done = 0;
    h.target = target;
    U.restarts[v] = restarts;
    WSTORE_END
    S.preemptions += 1;
    wait_insert(U, S, r, v);  // victim was unfinished: outstanding unchanged
    return v;
  }
  return -1;
}

// ensure_decode_memory (scheduler.hpp:290-296)
__device__ __forceinline__ bool ensure_decode_memory(Unit& U, RepState& S, int r, int32_t j) {
  while (!try_reserve(U, S, j, (int64_t)U.hot[j].kv + 1)) {
    const int32_t victim = preempt_latest(U, S, r);
    if (victim < 0 || victim == j) return false;
  }
  return true;
}

// admit_reserve (scheduler.hpp:302-316)
__device__ __forceinline__ bool admit_reserve(Unit& U, RepState& S, int r, int32_t j, int64_t target,
                              bool allow_preempt, bool use_watermark) {
  const SimConfig& c = *U.cfg;
  while (true) {
    const int64_t need = shortfall(c, U.hot[j], target);
    const int64_t floor = (use_watermark && S.run_n > 0) ? c.watermark_units : 0;
    if ((c.total_units - S.allocated) - need >= floor) break;
    if (!allow_preempt) return false;
    const int32_t victim = preempt_latest(U, S, r);
    if (victim < 0 || victim == j) return false;
  }
  return try_reserve(U, S, j, target);
}

__device__ __forceinline__ void push_prefill(Unit& U, RepState& S, int r, int32_t j, int32_t chunk,
                                             int32_t prior) {
  WSTORE_BEGIN(U)
  P_IDX(U, r)[S.np] = j;
  P_CHUNK(U, r)[S.np] = chunk;
  P_PRIOR(U, r)[S.np] = prior;
  WSTORE_END
  S.np += 1;
  U.plan_tokens += chunk;
}

// schedule_decodes (scheduler.hpp:449-472).  Fast path: a 32-entry window of
// the running queue is judged at once -- eligibility, batch cap / token budget
// and the cumulative block shortfall against free units.  Entries up to the
// first one that would not fit are admitted together (no preemption can occur
// for them); that entry, if any, replays the sequential ensure_decode_memory
// path, after which the window scan resumes.
static __device__ void schedule_decodes(Unit& U, RepState& S, int r, int32_t max_entries,
                                 int32_t* budget) {
  const SimConfig& c = *U.cfg;
  int32_t i = 0;
  while (i < S.run_n) {
    const int32_t* a = RUN(U, r);
    const int p = i + U.lane;
    int32_t j = -1;
    bool elig = false;
    int64_t need = 0;
    if (p < S.run_n) {
      j = a[p];
      const ReqHot h = U.hot[j];
      elig = !finished(h) && prefill_complete(h) && h.planned != U.serial;
      if (elig) need = shortfall(c, h, (int64_t)h.kv + 1);
    }
    const unsigned em = __ballot_sync(SSG_FULL, elig);
    if (em == 0) {
      i += 32;
      continue;
    }
    // exclusive count of eligible entries before this lane; inclusive need sum
    // (32-bit scan when every need is small -- the common case: 0 or 1 block)
    const int before = __popc(em & ((1u << U.lane) - 1u));
    int64_t incl = need;
    const unsigned ones = __ballot_sync(SSG_FULL, need == 1);
    if (__all_sync(SSG_FULL, need <= 1)) {
      // the usual case: a decode needs no new block or exactly one
      incl = __popc(ones & ((2u << U.lane) - 1u));
    } else if (__all_sync(SSG_FULL, need < (1 << 25))) {
      int32_t inc32 = (int32_t)need;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int32_t t = __shfl_up_sync(SSG_FULL, inc32, o);
        if (U.lane >= o) inc32 += t;
      }
      incl = inc32;
    } else {
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int64_t t = __shfl_up_sync(SSG_FULL, incl, o);
        if (U.lane >= o) incl += t;
      }
    }
    const int32_t batch0 = S.np + S.nd;
    const int64_t free0 = c.total_units - S.allocated;
    const bool cap_ok = (batch0 + before < max_entries) && (!budget || *budget - before >= 1);
    const bool mem_ok = incl <= free0;
    const unsigned stop = __ballot_sync(SSG_FULL, elig && !(cap_ok && mem_ok));
    const int first_stop = stop ? __ffs(stop) - 1 : 32;
    // admit the eligible entries before first_stop
    const bool take = elig && U.lane < first_stop;
    const unsigned tm = __ballot_sync(SSG_FULL, take);
    const int ntake = __popc(tm);
    bool late_first = false;
    if (take) {
      ReqHot& h = U.hot[j];
      h.held += (int32_t)need;  // distinct requests per lane
      const ReqTimes t = U.tm[j];
      if (t.first_sched < 0) {
        U.tm[j].first_sched = U.clock;
        late_first = U.clock - t.arrival > U.u->abort_thr;
      }
      h.planned = U.serial;
      D_IDX(U, r)[S.nd + before] = j;
      D_CTX(U, r)[S.nd + before] = h.kv + 1;
    }
    U.plan_late += __popc(__ballot_sync(SSG_FULL, late_first));
    __syncwarp();
    int64_t taken_need = __shfl_sync(SSG_FULL, incl, first_stop == 0 ? 0 : first_stop - 1);
    // inclusive prefix at the last taken lane (non-eligible lanes add 0)
    if (ntake == 0) taken_need = 0;
    __syncwarp();
    S.allocated += taken_need;
    S.nd += ntake;
    if (budget) *budget -= ntake;
    if (first_stop == 32) {
      i += 32;
      continue;
    }
    // the stopping entry: cap/budget -> the reference breaks out of the loop
    const int32_t js = __shfl_sync(SSG_FULL, j, first_stop);
    if (S.np + S.nd >= max_entries) return;
    if (budget && *budget < 1) return;
    // memory shortfall: sequential ensure_decode_memory with preemption
    i = i + first_stop;
    if (!ensure_decode_memory(U, S, r, js)) {
      if (i < S.run_n && RUN(U, r)[i] == js) ++i;
      continue;
    }
    mark_scheduled(U, js);
    const int32_t ctx = U.hot[js].kv + 1;
    WSTORE_BEGIN(U)
    D_IDX(U, r)[S.nd] = js;
    D_CTX(U, r)[S.nd] = ctx;
    WSTORE_END
    S.nd += 1;
    if (budget) *budget -= 1;
    int32_t pos = 0;
    const int32_t* a2 = RUN(U, r);
    while (pos < S.run_n && a2[pos] != js) ++pos;
    i = pos + 1;
  }
}

// First position >= i of the running queue whose request matches `pred`
// (warp-parallel 32-entry windows); run_n if none.
#define PRED_PREFILL_LEFT 0
static __device__ SSG_WARM int32_t next_running(Unit& U, const RepState& S, int r, int32_t i, int pred) {
  const int32_t* a = RUN(U, r);
#pragma unroll 1
  for (; i < S.run_n; i += 32) {
    const int32_t p = i + U.lane;
    bool hit = false;
    if (p < S.run_n) {
      const ReqHot h = U.hot[a[p]];
      hit = !finished(h) && !prefill_complete(h);
    }
    const unsigned m = __ballot_sync(SSG_FULL, hit);
    if (m) return i + __ffs(m) - 1;
  }
  return S.run_n;
}

// vLLM, Orca+ / LightLLM and Sarathi-Serve batch formation in one body
// (scheduler.hpp:354-444).  The three differ only in phase order -- vLLM and
// Orca+ admit waiting prompts, then decode; Sarathi decodes, continues in-flight
// chunks, then admits -- and in a few per-phase rules, so each phase has ONE
// call site (the admission's admit_reserve, schedule_decodes and their
// preemption paths are emitted once): the simulation kernel is instruction-
// fetch bound, and co-resident warps of different policies now share this code.
//   vLLM:    budget max_tokens, admission may preempt; decodes only when no
//            prefill was admitted, with no token budget
//   Orca+:   budget max_tokens, no preemption; decodes share the budget left;
//            a prompt longer than the budget runs alone (no decodes)
//   Sarathi: budget chunk_size; decodes first; then in-flight chunks in running
//            order; then admission of chunk = min(budget, prompt)
static __device__ SSG_WARM void schedule_chunked(Unit& U, RepState& S, int r) {
  const SimConfig& c = *U.cfg;
  const bool sar = c.policy == SSG_POL_SARATHI, vl = c.policy == SSG_POL_VLLM;
  int32_t budget = sar ? c.chunk : c.max_tokens;
  bool decodes = true;
#pragma unroll 1
  for (int ph = 0; ph < 2; ++ph) {
    if (ph == (sar ? 0 : 1)) {
      if (decodes) schedule_decodes(U, S, r, c.max_batch, vl ? nullptr : &budget);
      continue;
    }
    // prefills: Sarathi first continues in-flight chunks in running order (a
    // 32-entry window is scanned at once; only requests with prefill left are
    // visited), then every policy admits waiting heads -- one reservation site
    bool inflight = sar;
    int32_t i = 0;
#pragma unroll 1
    while (true) {
      int32_t j, chunk, prior = 0, t = 0;
      bool alone = false;
      if (inflight) {
        int32_t k = S.run_n;
        if (budget >= 1 && S.np + S.nd < c.max_batch) k = next_running(U, S, r, i, PRED_PREFILL_LEFT);
        if (k >= S.run_n) {
          inflight = false;
          continue;
        }
        j = RUN(U, r)[k];
        const ReqHot h = U.hot[j];
        const int32_t rem = h.target - h.done;
        chunk = budget < rem ? budget : rem;
        prior = h.done;
        i = k + 1;
      } else {
        if (!(S.wait_n > 0 && S.run_n < c.max_batch)) break;
        if (sar && !(budget > 0 && S.np + S.nd < c.max_batch)) break;
        j = wait_front(U, S, r);
        t = U.hot[j].target;
        chunk = t;
        if (sar) {
          chunk = budget < t ? budget : t;
        } else {
          alone = t > c.max_tokens;
          if (alone && S.np > 0) break;
          if (!alone && t > budget) break;
        }
      }
      // in-flight chunks: no watermark, no preemption; admissions: watermark,
      // preemption for vLLM only (scheduler.hpp:302-316)
      if (!admit_reserve(U, S, r, j, (int64_t)prior + chunk, !inflight && vl, !inflight)) {
        if (!inflight) break;
        inflight = false;
        continue;
      }
      if (!inflight) {
        wait_erase(U, S, r, j);
        run_insert(U, S, r, j);
      }
      mark_scheduled(U, j);
      push_prefill(U, S, r, j, chunk, prior);
      if (inflight) {
        budget -= chunk;
        continue;
      }
      budget -= sar ? chunk : (t < budget ? t : budget);
      if (alone) {
        decodes = false;
        break;
      }
      if (!sar && budget == 0) break;
    }
    __syncwarp();
    if (vl && S.np > 0) decodes = false;
  }
  __syncwarp();
}

static __device__ SSG_COLD void schedule_ft(Unit& U, RepState& S, int r) {
  const SimConfig& c = *U.cfg;
  if (!S.ft_inflight) {
    while (S.wait_n > 0 && S.run_n < c.max_batch) {
      const int32_t head = wait_front(U, S, r);
      const ReqHot h = U.hot[head];
      const int64_t final_ctx = (int64_t)h.target + (h.decode - h.emitted);
      if (!try_reserve(U, S, head, final_ctx)) break;
      S.wait_head = (S.wait_head + 1) & (U.WC - 1);
      S.wait_n -= 1;
      run_insert(U, S, r, head);
    }
    __syncwarp();
    if (S.run_n == 0) return;
    S.ft_inflight = 1;
  }
  // prompts run one member per iteration ...
  const int32_t k = next_running(U, S, r, 0, PRED_PREFILL_LEFT);
  if (k < S.run_n) {
    const int32_t j = RUN(U, r)[k];
    const ReqHot h = U.hot[j];
    mark_scheduled(U, j);
    push_prefill(U, S, r, j, h.target - h.done, h.done);
    return;
  }
  // ... then every unfinished member decodes in lockstep (order = running order)
  const int32_t* a = RUN(U, r);
#pragma unroll 1
  for (int32_t base = 0; base < S.run_n; base += 32) {
    const int32_t p = base + U.lane;
    bool live = false;
    int32_t j = -1;
    if (p < S.run_n) {
      j = a[p];
      live = !finished(U.hot[j]);
    }
    const unsigned m = __ballot_sync(SSG_FULL, live);
    bool late_first = false;
    if (live) {
      const int32_t slot = S.nd + __popc(m & ((1u << U.lane) - 1u));
      const ReqTimes t = U.tm[j];
      if (t.first_sched < 0) {
        U.tm[j].first_sched = U.clock;
        late_first = U.clock - t.arrival > U.u->abort_thr;
      }
      U.hot[j].planned = U.serial;
      D_IDX(U, r)[slot] = j;
      D_CTX(U, r)[slot] = U.hot[j].kv + 1;
    }
    U.plan_late += __popc(__ballot_sync(SSG_FULL, late_first));
    __syncwarp();
    S.nd += __popc(m);
  }
}

// ReplicaScheduler::schedule_iteration's policy dispatch (scheduler.hpp:184-194)
__device__ __forceinline__ void schedule_batch(Unit& U, RepState& S, int r) {
  if (U.cfg->policy == SSG_POL_FT)
    schedule_ft(U, S, r);
  else
    schedule_chunked(U, S, r);
}

// ---------------------------------------------------------------- replica state
// ---------------------------------------------------------------- helpers
__device__ __forceinline__ RepState load_rep(Unit& U, int r) {
  __syncwarp();
  RepState s = U.reps[r];
  __syncwarp();
  return s;
}
__device__ __forceinline__ void store_rep(Unit& U, int r, const RepState& s) {
  __syncwarp();
  if (U.lane == 0) U.reps[r] = s;
  __syncwarp();
}

// ReplicaScheduler::enqueue (scheduler.hpp:146-155)
__device__ __forceinline__ bool enqueue(Unit& U, RepState& S, int r, int32_t j) {
  const SimConfig& c = *U.cfg;
  const ReqHot h = U.hot[j];
  const int64_t need = units_for(c, (int64_t)h.prefill + h.decode);
  if (need > c.total_units) {
    set_error(U, SSG_ERR_ENQUEUE, r, U.ids[j], need, (double)c.total_units);
    return false;
  }
  wput(U, &U.hot[j].target, h.prefill + h.emitted);
  wait_insert(U, S, r, j);
  S.outstanding += 1;
  return true;
}

// start_if_idle (sim.hpp:191-195): has_work() == outstanding() > 0
__device__ __forceinline__ void start_if_idle(Unit& U, RepState& S) {
  if (S.busy || S.outstanding == 0) return;
  S.ev_kind = 1;
  S.ev_time = U.clock;
  S.ev_seq = U.seq++;
  S.busy = 1;
}

// complete_iteration (scheduler.hpp:197-233), warp-parallel over the batch.
static __device__ void complete_batch(Unit& U, RepState& S, int r) {
  const int32_t np = S.np, nd = S.nd;
  const bool emit_times = (U.u->flags & SSG_UF_EMISSIONS) != 0;
  int newly_finished = 0;
  bool bad = false;
#pragma unroll 1
  for (int32_t k = U.lane; k < np + nd; k += 32) {
    int32_t j;
    bool emit;
    if (k < np) {
      j = P_IDX(U, r)[k];
      ReqHot& h = U.hot[j];
      const int32_t done = h.done + P_CHUNK(U, r)[k];
      h.done = done;
      h.kv = done;
      if (done > h.target) bad = true;  // "prefill progressed past its target"
      emit = done >= h.target;
    } else {
      j = D_IDX(U, r)[k - np];
      U.hot[j].kv = D_CTX(U, r)[k - np];
      emit = true;
    }
    if (emit) {
      ReqHot& h = U.hot[j];
      if (h.emitted >= h.decode) bad = true;  // "emit_token on finished request"
      const int32_t e = h.emitted + 1;
      h.emitted = e;
      if (emit_times) U.emissions[U.emit_base[j] + e - 1] = U.clock;
      ReqTimes& t = U.tm[j];
      if (t.first_tok < 0) t.first_tok = U.clock;
      if (e >= h.decode) {
        t.completion = U.clock;
        ++newly_finished;
      }
    }
  }
  __syncwarp();
  if (__any_sync(SSG_FULL, bad)) {
    set_error(U, SSG_ERR_INTERNAL, 4, 0, 0, 0.0);
    return;
  }
  newly_finished = (int)__reduce_add_sync(SSG_FULL, (unsigned)newly_finished);
  S.outstanding -= newly_finished;
  // only a request that just emitted its last token holds KV and sits in the
  // running queue while finished (earlier finishers were released and dropped,
  // or -- FT -- released with held = 0 and still unfinished members remain):
  // with none, the release/compaction pass below changes nothing
  if (newly_finished == 0) return;
  // release finished runners; drop them from running unless FT froze membership
  int32_t* a = RUN(U, r);
  int32_t write = 0;
  int64_t freed = 0;
  bool any_unfinished = false;
#pragma unroll 1
  for (int32_t base = 0; base < S.run_n; base += 32) {
    const int32_t p = base + U.lane;
    int32_t j = -1;
    bool fin = false;
    if (p < S.run_n) {
      j = a[p];
      ReqHot& h = U.hot[j];
      fin = h.emitted >= h.decode;
      if (fin) {
        freed += h.held;
        h.held = 0;
      } else {
        any_unfinished = true;
      }
    }
    if (!S.ft_inflight) {
      const unsigned keep = __ballot_sync(SSG_FULL, p < S.run_n && !fin);
      const int dst = write + __popc(keep & ((1u << U.lane) - 1u));
      __syncwarp();
      if (p < S.run_n && !fin) a[dst] = j;
      write += __popc(keep);
    }
    __syncwarp();
  }
  freed = warp_sum64(freed);
  S.allocated -= freed;
  if (!S.ft_inflight) {
    S.run_n = write;
  } else if (!__any_sync(SSG_FULL, any_unfinished)) {
    S.run_n = 0;
    S.ft_inflight = 0;
  }
  __syncwarp();
}

// ---------------------------------------------------------------- latency
// predict_batch / batch_device_flops per microbatch (estimator.hpp:294-380),
// split_microbatches (sim.hpp:118-130) and pipeline_makespan
// (scheduler.hpp:566-579).  Per-entry sums are integer (exact in any order);
// the per-operator predictions run one per lane and are then added strictly
// in operator order, microbatch by microbatch, as the reference does.
// The generic per-(microbatch, op) evaluation for batches outside the token
// tables' range (or configs without tables): one lane per task, operator-order
// accumulation.  Out of line -- it is the cold path of batch_latency.
template <int FMA, int FOREST>
static __device__ SSG_COLD void batch_latency_full(Unit& U, const int64_t* st, int& err, int& err_task,
                                                int& err_feat, double& err_val, int64_t& qb) {
  const SimConfig& c = *U.cfg;
  const int pp = c.pp;
  const int nops = c.nops;
  double* secs_part = U.smem_part;
  double* flop_part = U.smem_part + U.pcap;
  const int work = pp * nops;
  double acc_s = 0.0, acc_f = 0.0;
  int cur_m = 0;
  for (int base = 0; base < work; base += 32) {
    const int t = base + U.lane;
    double pred = 0.0, fl = 0.0, v0 = 0.0, v1 = 0.0;
    bool active = false;
    int code = SSG_OK, bad = 0;
    if (t < work) {
      const int m = t / nops;
      const SimOp& o = c.ops[t - m * nops];
      const int64_t* s = st + m * 6;
      const double tokens = (double)s[1];
      if (s[1] > 0) {
        if (o.cls == SSG_CLS_TOKEN) {
          active = true;
          v0 = tokens;
          if (o.flop_kind == 0)
            fl = __dmul_rn(__dmul_rn(__dmul_rn(2.0, tokens), o.fa), o.fb);
          else if (o.flop_kind == 1)
            fl = __dmul_rn(tokens, o.fa);
          else
            fl = __dmul_rn(__dmul_rn(8.0, tokens), o.fa);
        } else if (o.cls == SSG_CLS_SEQ) {
          if (o.flop_kind == 3 && s[0] > 0) {
            active = true;
            const double n_eq = (double)ssg_llround_nonneg(sqrt((double)s[2]));
            v0 = n_eq;
            v1 = __dmul_rn((double)s[3], o.kvb);
            const double ctx_tokens = v1 / o.kvb;
            fl = __dmul_rn(__dmul_rn(__dmul_rn(4.0, n_eq), __dadd_rn(n_eq, ctx_tokens)), o.fa);
          } else if (o.flop_kind == 4 && s[4] > 0) {
            active = true;
            v0 = (double)s[4];
            v1 = __dmul_rn((double)s[5], o.kvb);
            const double ctx_tokens = v1 / o.kvb;
            fl = __dmul_rn(__dmul_rn(4.0, ctx_tokens), o.fa);
          }
        } else {
          active = true;
          v0 = __dmul_rn(tokens, o.payload);
        }
      }
      if (active) {
        qb += o.qbytes;
        code = ssg_predict_t<FMA, FOREST>(U.E, o.slot, v0, v1, &pred, &bad);
        pred = __dmul_rn(o.count, pred);
        fl = (o.cls == SSG_CLS_COMM) ? 0.0 : __dmul_rn(o.count, fl);
      }
    }
    const unsigned em = __ballot_sync(SSG_FULL, code != SSG_OK);
    if (em && err == SSG_OK) {
      const int src = __ffs(em) - 1;
      err = __shfl_sync(SSG_FULL, code, src);
      err_task = base + src;
      err_feat = __shfl_sync(SSG_FULL, bad, src);
      err_val = __shfl_sync(SSG_FULL, bad ? v1 : v0, src);
    }
    const int kmax = (work - base) < 32 ? (work - base) : 32;
    for (int k = 0; k < kmax; ++k) {
      const double pk = __shfl_sync(SSG_FULL, pred, k);
      const double fk = __shfl_sync(SSG_FULL, fl, k);
      const int ak = __shfl_sync(SSG_FULL, (int)active, k);
      const int m = (base + k) / nops;
      if (m != cur_m) {
        if (U.lane == 0) {
          secs_part[cur_m] = acc_s;
          flop_part[cur_m] = acc_f;
        }
        acc_s = 0.0;
        acc_f = 0.0;
        cur_m = m;
      }
      if (ak) {
        acc_s = __dadd_rn(acc_s, pk);
        if (c.ops[(base + k) - m * nops].cls != SSG_CLS_COMM) acc_f = __dadd_rn(acc_f, fk);
      }
    }
  }
  if (U.lane == 0) {
    secs_part[cur_m] = acc_s;
    flop_part[cur_m] = acc_f;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) qb += __shfl_xor_sync(SSG_FULL, qb, o);
  U.qbytes += qb;
  __syncwarp();
}

// Result of one attention query: the prediction, SSG_OK or the error code
// with the failing feature, and the axis-1 cell for the lane's next search.
struct AttnQuery {
  double pred;
  int32_t code;
  int32_t bad;
  int32_t hint;
};

// One out-of-line copy serves the batch latency and the decode fast-forward
// (the kernel is instruction-fetch bound: SSG_ATTN_INLINE=1 inlines both, A/B).
#ifdef SSG_ATTN_INLINE
#define SSG_ATTN_QUERY __forceinline__
#else
#define SSG_ATTN_QUERY __noinline__
#endif

// EstimatorModel::predict of one attention query on a 2-D interpolator whose
// axis-0 cell at the integer v0 comes from the token tables (lo0, f0 =
// ssg_axis_cell(log1p(v0)), computed by k_build_tables with the same code) and
// whose axis-1 search starts from the lane's previous cell: the bracket test
// below holds exactly when std::upper_bound would land in that cell, so the
// cell, the fraction and every later operation are the reference's.
// estimator.hpp:105-123, regressor.hpp:308-341.
template <int FMA>
__device__ SSG_ATTN_QUERY AttnQuery ssg_attn_interp(const double* __restrict__ dpool,
                                                    const SsgModelDesc* __restrict__ m, double v0,
                                                    double v1, int32_t lo0, double f0, int32_t hint) {
  AttnQuery q;
  q.pred = 0.0;
  q.code = SSG_OK;
  q.bad = 0;
  q.hint = hint;
  if (!(v0 >= m->lower[0] && v0 <= m->upper[0])) {
    q.code = SSG_ERR_BBOX;
    return q;
  }
  if (!(v1 >= m->lower[1] && v1 <= m->upper[1])) {
    q.code = SSG_ERR_BBOX;
    q.bad = 1;
    return q;
  }
  const int32_t n1 = m->axis_len[1];
  int32_t lo1;
  double f1;
  ssg_axis_cell_hint(dpool + m->axis_off[1], n1, hot_log1p<FMA>(v1), &q.hint, &lo1, &f1);
  const int32_t n0 = m->axis_len[0];
  const double* vals = dpool + m->values_off;
  const int32_t h0 = n0 == 1 ? 0 : 1;
  const int32_t h1 = n1 == 1 ? 0 : 1;
  const double g0 = __dsub_rn(1.0, f0), g1 = __dsub_rn(1.0, f1);
  const int64_t r0 = (int64_t)lo0 * n1, r1 = (int64_t)(lo0 + h0) * n1;
  const double w1lo = g1, w1hi = h1 ? f1 : g1;
  const double w0lo = g0, w0hi = h0 ? f0 : g0;
  double acc = __dmul_rn(__dmul_rn(w1lo, w0lo), __ldg(vals + r0 + lo1));
  acc = __dadd_rn(acc, __dmul_rn(__dmul_rn(w1lo, w0hi), __ldg(vals + r1 + lo1)));
  acc = __dadd_rn(acc, __dmul_rn(__dmul_rn(w1hi, w0lo), __ldg(vals + r0 + lo1 + h1)));
  acc = __dadd_rn(acc, __dmul_rn(__dmul_rn(w1hi, w0hi), __ldg(vals + r1 + lo1 + h1)));
  if (!ssg_exp_in_range(acc)) {
    q.code = SSG_ERR_EXP_RANGE;
    return q;
  }
  q.pred = hot_exp<FMA>(acc);
  return q;
}

template <int FMA, int FOREST>
__device__ int batch_latency(Unit& U, RepState& S, int r, double* latency, double* flops_out) {
  const SimConfig& c = *U.cfg;
  const int pp = c.pp;
  int64_t* st = U.smem_stats;  // [pp][6]: prefills, tokens, sum p^2, sum prior, decodes, sum ctx
  const int32_t total = S.np + S.nd;
  // per-microbatch sums: prefills, tokens, sum p^2, sum prior, decodes, sum ctx
  SSG_PH_BEGIN(ph_a);
  auto accumulate = [&](int32_t k, int64_t& a0, int64_t& a1, int64_t& a2, int64_t& a3, int64_t& a4,
                        int64_t& a5) {
    if (k < S.np) {
      const int64_t ch = P_CHUNK(U, r)[k];
      a0 += 1;
      a1 += ch;
      a2 += ch * ch;
      a3 += P_PRIOR(U, r)[k];
    } else {
      a1 += 1;
      a4 += 1;
      a5 += D_CTX(U, r)[k - S.np];
    }
  };
  if ((32 % pp) == 0) {
    // entry k belongs to microbatch k mod pp (split_microbatches, sim.hpp:118-130);
    // with pp | 32 lane l only sees entries of microbatch l mod pp, so one pass
    // and a reduction over the lanes sharing l mod pp give every microbatch
    int64_t a0 = 0, a1 = 0, a2 = 0, a3 = 0, a4 = 0, a5 = 0;
#pragma unroll 1
    for (int32_t k = U.lane; k < total; k += 32) accumulate(k, a0, a1, a2, a3, a4, a5);
    // 32-lane sums of values below 2^26 fit in 31 bits: one REDUX each
    const bool small = ((a1 | a2 | a3 | a5) >> 26) == 0;
    if (pp == 1 && __all_sync(SSG_FULL, small)) {
      a0 = __reduce_add_sync(SSG_FULL, (unsigned)a0);
      a1 = __reduce_add_sync(SSG_FULL, (unsigned)a1);
      a2 = __reduce_add_sync(SSG_FULL, (unsigned)a2);
      a3 = __reduce_add_sync(SSG_FULL, (unsigned)a3);
      a4 = __reduce_add_sync(SSG_FULL, (unsigned)a4);
      a5 = __reduce_add_sync(SSG_FULL, (unsigned)a5);
    } else {
      for (int o = 16; o >= pp; o >>= 1) {
        a0 += __shfl_xor_sync(SSG_FULL, a0, o);
        a1 += __shfl_xor_sync(SSG_FULL, a1, o);
        a2 += __shfl_xor_sync(SSG_FULL, a2, o);
        a3 += __shfl_xor_sync(SSG_FULL, a3, o);
        a4 += __shfl_xor_sync(SSG_FULL, a4, o);
        a5 += __shfl_xor_sync(SSG_FULL, a5, o);
      }
    }
    __syncwarp();
    if (U.lane < pp) {
      int64_t* s6 = st + U.lane * 6;
      s6[0] = a0;
      s6[1] = a1;
      s6[2] = a2;
      s6[3] = a3;
      s6[4] = a4;
      s6[5] = a5;
    }
  } else {
    for (int m = 0; m < pp; ++m) {
      int64_t a0 = 0, a1 = 0, a2 = 0, a3 = 0, a4 = 0, a5 = 0;
      for (int32_t k = m + U.lane * pp; k < total; k += 32 * pp) accumulate(k, a0, a1, a2, a3, a4, a5);
      a0 = warp_sum64(a0);
      a1 = warp_sum64(a1);
      a2 = warp_sum64(a2);
      a3 = warp_sum64(a3);
      a4 = warp_sum64(a4);
      a5 = warp_sum64(a5);
      if (U.lane == 0) {
        st[m * 6 + 0] = a0;
        st[m * 6 + 1] = a1;
        st[m * 6 + 2] = a2;
        st[m * 6 + 3] = a3;
        st[m * 6 + 4] = a4;
        st[m * 6 + 5] = a5;
      }
      __syncwarp();
    }
  }
  __syncwarp();
  SSG_PH_END(ph_a, 8);
  SSG_PH_BEGIN(ph_q);
  const int nops = c.nops;
  double* secs_part = U.smem_part;       // [pp]
  double* flop_part = U.smem_part + U.pcap;
  int err = SSG_OK, err_task = 0, err_feat = 0;
  double err_val = 0.0;
  int64_t qb = 0;
  // token-table fast path: every non-empty microbatch within the tables' range
  const bool use_tab =
      c.tab_off >= 0 && pp <= SSG_MAX_PP && !__any_sync(SSG_FULL, U.lane < pp && st[U.lane * 6 + 1] > c.tab_tmax);
  if (use_tab) {
    const int T1 = c.tab_stride;
    const double* tab = U.tables + c.tab_off;
    // per-lane work: lane 2m = prefill attention of microbatch m, 2m+1 = decode attention
    const int m = U.lane >> 1;
    const bool is_dec = U.lane & 1;
    double pred = 0.0, fl = 0.0, v0 = 0.0, v1 = 0.0;
    int code = SSG_OK, bad = 0;
    bool active = false, query = false;
    int64_t t0 = 0;  // integer v0 of the query
    const int op_index = is_dec ? c.idx_dec : c.idx_pre;
    if (m < pp && op_index >= 0) {
      const int64_t* s6 = st + m * 6;
      const SimOp& o = c.ops[op_index];
      if (s6[1] > 0 && !is_dec && s6[0] > 0) {
        active = true;
        const int64_t n_eq = ssg_llround_nonneg(sqrt((double)s6[2]));
        if (s6[3] == 0 && n_eq <= c.tab_pmax) {
          pred = tab[5 * (int64_t)T1 + n_eq];
          fl = tab[6 * (int64_t)T1 + n_eq];
        } else {
          query = true;
          t0 = n_eq;
          v0 = (double)n_eq;
          v1 = __dmul_rn((double)s6[3], o.kvb);
          const double ctx_tokens = v1 / o.kvb;
          fl = __dmul_rn(o.count, __dmul_rn(__dmul_rn(__dmul_rn(4.0, v0), __dadd_rn(v0, ctx_tokens)), o.fa));
        }
      } else if (s6[1] > 0 && is_dec && s6[4] > 0) {
        active = true;
        query = true;
        t0 = s6[4];
        v0 = (double)s6[4];
        v1 = __dmul_rn((double)s6[5], o.kvb);
        const double ctx_tokens = v1 / o.kvb;
        fl = __dmul_rn(o.count, __dmul_rn(__dmul_rn(4.0, ctx_tokens), o.fa));
      }
    }
    // one converged predictor call for every querying lane (prefill and
    // decode attention of every microbatch evaluate side by side)
    if (query) {
      const SimOp& o = c.ops[op_index];
      if (!FOREST && c.tab_cells && t0 <= c.tab_tmax) {
        const int64_t row = is_dec ? 7 : 9;
        const double f0 = tab[row * T1 + t0];
        const int32_t lo0 = (int32_t)tab[(row + 1) * T1 + t0];
        const AttnQuery aq = ssg_attn_interp<FMA>(U.E.dpool, U.E.models + o.slot, v0, v1, lo0, f0, U.ax1_hint);
        code = aq.code;
        bad = aq.bad;
        pred = aq.pred;
        U.ax1_hint = aq.hint;
      } else {
        code = ssg_predict_t<FMA, FOREST>(U.E, o.slot, v0, v1, &pred, &bad);
      }
      pred = __dmul_rn(o.count, pred);
    }
    SSG_PH_END(ph_q, 9);
    SSG_PH_BEGIN(ph_e);
    const unsigned em = __ballot_sync(SSG_FULL, code != SSG_OK);
    if (em) {
      const int src = __ffs(em) - 1;  // lanes are in (microbatch, prefill < decode) order
      err = __shfl_sync(SSG_FULL, code, src);
      err_feat = __shfl_sync(SSG_FULL, bad, src);
      err_val = __shfl_sync(SSG_FULL, bad ? v1 : v0, src);
      err_task = __shfl_sync(SSG_FULL, op_index, src);  // op index within microbatch 0's numbering
    }
    // microbatch mm's operator-order sum on lane mm: token-level ops (table),
    // prefill attention (lane 2mm), decode attention (lane 2mm + 1), comm ops
    const double pp_pred = __shfl_sync(SSG_FULL, pred, (2 * U.lane) & 31);
    const double pp_fl = __shfl_sync(SSG_FULL, fl, (2 * U.lane) & 31);
    const int pp_act = __shfl_sync(SSG_FULL, (int)active, (2 * U.lane) & 31);
    const double dd_pred = __shfl_sync(SSG_FULL, pred, (2 * U.lane + 1) & 31);
    const double dd_fl = __shfl_sync(SSG_FULL, fl, (2 * U.lane + 1) & 31);
    const int dd_act = __shfl_sync(SSG_FULL, (int)active, (2 * U.lane + 1) & 31);
    if (U.lane < pp) {
      const int64_t* s6 = st + U.lane * 6;
      const int64_t t = s6[1];
      double acc_s = 0.0, acc_f = 0.0;
      if (t > 0) {
        // algorithmic bytes: every query the reference makes, however it is served
        U.qb_lane += c.qb_fixed + (s6[0] > 0 ? c.qb_pre : 0) + (s6[4] > 0 ? c.qb_dec : 0);
        acc_s = tab[t];
        acc_f = tab[(int64_t)T1 + t];
        if (pp_act) {
          acc_s = __dadd_rn(acc_s, pp_pred);
          acc_f = __dadd_rn(acc_f, pp_fl);
        }
        if (dd_act) {
          acc_s = __dadd_rn(acc_s, dd_pred);
          acc_f = __dadd_rn(acc_f, dd_fl);
        }
        // comm ops (at most 3), op order
        const double* comm = tab + 2 * (int64_t)T1 + t;
        if (c.ncomm > 0) acc_s = __dadd_rn(acc_s, comm[0]);
        if (c.ncomm > 1) acc_s = __dadd_rn(acc_s, comm[T1]);
        if (c.ncomm > 2) acc_s = __dadd_rn(acc_s, comm[2 * (int64_t)T1]);
      }
      secs_part[U.lane] = acc_s;
      flop_part[U.lane] = acc_f;
    }
    __syncwarp();
    SSG_PH_END(ph_e, 11);
  } else {
    batch_latency_full<FMA, FOREST>(U, st, err, err_task, err_feat, err_val, qb);
  }
  SSG_PH_BEGIN(ph_m);
  if (err != SSG_OK) {  // first failing (microbatch, op) in order -- either path
    const SimOp& o = c.ops[err_task % nops];
    set_error(U, err, o.slot, err_feat, 0, err_val);
    return err;
  }
  double lat = 0.0, flops = 0.0;
  if (pp == 1) {
    lat = secs_part[0];
    if (!(lat > 0.0)) {
      set_error(U, SSG_ERR_INTERNAL, 2, 0, 0, lat);  // predict_batch: non-positive prediction
      return SSG_ERR_INTERNAL;
    }
    flops = __dmul_rn(flop_part[0], (double)c.tp);
  } else if (pp <= 4) {
    // pipeline_makespan (scheduler.hpp:566-579) over the non-empty microbatches
    // in order, in registers: stage after stage, each microbatch starts when it
    // and its predecessor are both done
    double tim[4], fin[4];
    bool ne[4];
#pragma unroll
    for (int m = 0; m < 4; ++m) {
      ne[m] = m < pp && st[m * 6 + 1] != 0;
      tim[m] = ne[m] ? secs_part[m] : 0.0;
      fin[m] = 0.0;
    }
#pragma unroll
    for (int m = 0; m < 4; ++m) {
      if (!ne[m]) continue;
      if (!(tim[m] > 0.0)) {
        set_error(U, SSG_ERR_INTERNAL, 2, 0, 0, tim[m]);
        return SSG_ERR_INTERNAL;
      }
      flops = __dadd_rn(flops, __dmul_rn(flop_part[m], (double)(c.tp * c.pp)));
    }
#pragma unroll 1
    for (int st_i = 0; st_i < pp; ++st_i) {
      double prev = 0.0;
#pragma unroll
      for (int m = 0; m < 4; ++m) {
        if (!ne[m]) continue;
        const double f = fin[m];
        const double start = f < prev ? prev : f;
        prev = __dadd_rn(start, tim[m]);
        fin[m] = prev;
      }
    }
    lat = 0.0;
#pragma unroll
    for (int m = 0; m < 4; ++m)
      if (ne[m]) lat = fin[m];  // the last non-empty microbatch
    __syncwarp();
  } else {
    // compact the non-empty microbatches' times into part[2*MAX..]; makespan
    double* times = U.smem_part + 2 * U.pcap;
    double* finish = U.smem_part + 3 * U.pcap;
    int nt = 0;
    for (int m = 0; m < pp; ++m) {
      if (st[m * 6 + 1] == 0) continue;
      if (!(secs_part[m] > 0.0)) {
        set_error(U, SSG_ERR_INTERNAL, 2, 0, 0, secs_part[m]);
        return SSG_ERR_INTERNAL;
      }
      flops = __dadd_rn(flops, __dmul_rn(flop_part[m], (double)(c.tp * c.pp)));
      if (U.lane == 0) {
        times[nt] = secs_part[m];
        finish[nt] = 0.0;
      }
      ++nt;
    }
    __syncwarp();
    // every lane runs the makespan on its own registers-through-smem copy;
    // lane 0 owns the stores
    for (int s = 0; s < pp; ++s) {
      double prev = 0.0;
      for (int m = 0; m < nt; ++m) {
        const double f = finish[m];
        const double start = f < prev ? prev : f;
        prev = __dadd_rn(start, times[m]);
        __syncwarp();
        if (U.lane == 0) finish[m] = prev;
        __syncwarp();
      }
    }
    lat = nt ? finish[nt - 1] : 0.0;
    __syncwarp();
  }
  lat = __dadd_rn(lat, c.cpu_overhead);
  if (!(lat > 0.0)) {
    set_error(U, SSG_ERR_INTERNAL, 3, 0, 0, lat);  // non-positive iteration latency
    return SSG_ERR_INTERNAL;
  }
  *latency = lat;
  *flops_out = flops;
  SSG_PH_END(ph_m, 10);
  return SSG_OK;
}

}  // namespace ssgk
