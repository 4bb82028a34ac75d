// engine.cu -- K3 kernel: the discrete-event loop over a unit's replicas.
//
// reference: sim.hpp:135-320 (run_simulation), sim.hpp:42-47 (event order),
//            scheduler.hpp:146-233 (enqueue, complete_iteration),
//            scheduler.hpp:492-561 (Router)
//
// Event order.  The reference pushes every arrival first (seq 0..N-1) and then
// BatchStart/BatchComplete events with increasing seq; ties on time break on
// seq.  Each replica has at most one pending BatchStart/BatchComplete, so the
// device queue is "next arrival" plus one slot per replica, and the next event
// is a warp-wide (time, seq) argmin over those slots.  RequestComplete events
// are pure bookkeeping in the reference and are not materialised; seq stays
// monotone in push order, which is all the ordering depends on.
#include <cstdlib>

#include "engine.cuh"
#ifndef SSG_FFWD
#define SSG_FFWD __forceinline__
#endif
#include "runtime.h"
#include "sim_engine.h"
#include "sim_host.h"

namespace ssgk {
#ifdef SSG_FF_STATS
// diagnostics build only: fast-forward calls, committed iterations, histogram
// of stretch lengths (0, 1, 2-3, 4-7, 8-15, 16-31, 32+), event-loop iterations
__device__ unsigned long long g_ff_stats[16];
#define FFSTAT(i) do { if (U.lane == 0) atomicAdd(&g_ff_stats[i], 1ull); } while (0)
#else
#define FFSTAT(i) do { } while (0)
#endif

// Router::drain for the deferred policy (scheduler.hpp:532-551) followed by the
// engine's enqueue + start_if_idle per assignment (sim.hpp:197-202).
__device__ SSG_COLD void drain_pool(Unit& U) {
  const SimConfig& c = *U.cfg;
  if (c.routing != SSG_ROUTE_DEFERRED) return;
  int32_t* pool = POOL(U);
  int32_t* ph = POOL_HEAD(U);  // [0] head, [1] size
  int32_t head = ph[0], size = ph[1];
  if (size == 0) return;
  const int R = U.u->R;
  const int mask = U.WC - 1;
  // The reference snapshots outstanding counts and bumps counts[best] per
  // assignment; each assignment's enqueue bumps the replica's outstanding count
  // too, so the live counts equal the snapshot throughout -- read them live,
  // 32 replicas per pass (any replica count).
  while (size > 0) {
    // best = lowest index among counts < threshold with the smallest count
    int64_t key = INT64_MAX;
#pragma unroll 1
    for (int r0 = 0; r0 < R; r0 += 32) {
      const int r = r0 + U.lane;
      int64_t k2 = INT64_MAX;
      if (r < R) {
        const int64_t cnt = U.reps[r].outstanding;
        if (cnt < c.defer_threshold) k2 = (cnt << 16) | r;
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const int64_t t = __shfl_xor_sync(SSG_FULL, k2, o);
        k2 = t < k2 ? t : k2;
      }
      key = k2 < key ? k2 : key;
    }
    if (key == INT64_MAX) break;
    const int best = (int)(key & 0xffff);
    const int32_t j = pool[head & mask];
    head = (head + 1) & mask;
    size -= 1;
    RepState S = load_rep(U, best);
    const bool ok = enqueue(U, S, best, j);
    if (ok) start_if_idle(U, S);
    store_rep(U, best, S);
    if (!ok) break;
  }
  wput(U, &ph[0], head);
  wput(U, &ph[1], size);
}

// One BatchStart event (sim.hpp:221-283).  Returns false when the unit must
// stop (error or probe abort).
// request slot of the q-th arrival (LONE launches have no permutation)
template <int LONE>
__device__ __forceinline__ int32_t arrival_slot(const Unit& U, int32_t q) {
  return (!LONE && U.arr_order) ? U.arr_order[q] : q;
}

template <int FMA, int FOREST, int LONE>
__device__ bool batch_start(Unit& U, RepState& S, int r) {
  const SimConfig& c = *U.cfg;
  U.serial += 1;
  S.np = 0;
  S.nd = 0;
  U.plan_tokens = 0;
  U.plan_late = 0;
  SSG_PH_BEGIN(ph_s);
  schedule_batch(U, S, r);
  SSG_PH_END(ph_s, 0);
  if (failed(U)) return false;
  if (S.np + S.nd == 0) {
    S.busy = 0;
    S.ev_kind = 0;
    return true;
  }
  const int32_t tokens = U.plan_tokens + S.nd;
#ifdef SSG_PHASE_CYCLES
  U.ph[15] += S.np > 0;
#endif
  if (c.policy == SSG_POL_SARATHI && tokens > c.chunk) {
    set_error(U, SSG_ERR_INTERNAL, 5, tokens, 0, 0.0);  // sarathi: token budget exceeded
    return false;
  }
  // batch log (SimObserver::on_batch payload, before the abort check)
  int64_t log_hdr = -1;
  if (!LONE && (U.u->flags & SSG_UF_BATCH_LOG)) {
    // observer runs append the scheduler state the SimObserver may query:
    // outstanding, preemptions, ft_inflight, FT member count + ids (running order)
    const bool obs = (U.u->flags & SSG_UF_OBSERVER) != 0;
    const int32_t members = obs && S.ft_inflight ? S.run_n : 0;
    const int64_t need = 6 + 3LL * S.np + 2LL * S.nd + (obs ? 4 + members : 0);
    const int64_t used = U.out->log_used;
    if (used >= 0 && used + need <= U.u->log_cap) {
      int64_t* L = U.log + used;
      if (U.lane == 0) {
        L[0] = r;
        L[1] = __double_as_longlong(U.clock);
        L[2] = S.allocated;
        L[3] = S.np;
        L[4] = S.nd;
        L[5] = 0;
      }
#pragma unroll 1
      for (int32_t k = U.lane; k < S.np; k += 32) {
        L[6 + 3 * k] = U.ids[P_IDX(U, r)[k]];
        L[7 + 3 * k] = P_CHUNK(U, r)[k];
        L[8 + 3 * k] = P_PRIOR(U, r)[k];
      }
#pragma unroll 1
      for (int32_t k = U.lane; k < S.nd; k += 32) {
        L[6 + 3 * S.np + 2 * k] = U.ids[D_IDX(U, r)[k]];
        L[7 + 3 * S.np + 2 * k] = D_CTX(U, r)[k];
      }
      if (obs) {
        int64_t* X = L + 6 + 3 * S.np + 2 * S.nd;
        if (U.lane == 0) {
          X[0] = S.outstanding;
          X[1] = S.preemptions;
          X[2] = S.ft_inflight;
          X[3] = members;
        }
#pragma unroll 1
        for (int32_t k = U.lane; k < members; k += 32) X[4 + k] = U.ids[RUN(U, r)[k]];
      }
      log_hdr = used;
      wput(U, &U.out->log_used, used + need);
    } else {
      wput(U, &U.out->log_used, (int64_t)-1);  // overflow: log incomplete
    }
  }
  // capacity-probe abort (sim.hpp:231-240)
  if (U.u->flags & SSG_UF_ABORT) {
    const int late = U.plan_late;
    if (late) {
      const int total = U.out->late + late;
      wput(U, &U.out->late, total);
      if (total > U.u->abort_max_late) {
        wput(U, &U.out->aborted, 1);
        return false;
      }
    }
  }
  double lat = 0.0, flops = 0.0;
  SSG_PH_BEGIN(ph_l);
  const int lat_code = batch_latency<FMA, FOREST>(U, S, r, &lat, &flops);
  SSG_PH_END(ph_l, 1);
  if (lat_code != SSG_OK) return false;
  if (!LONE && log_hdr >= 0) wput(U, &U.log[log_hdr + 5], (int64_t)__double_as_longlong(lat));
  S.busy_time = __dadd_rn(S.busy_time, lat);
  S.iterations += 1;
  S.tokens += tokens;
  U.iters += 1;
  U.entries += S.np + S.nd;
  // peak_kv holds the peak allocated units until the unit ends (the division by
  // total_units is monotone, so max of the quotients = quotient of the max)
  const double alloc = (double)S.allocated;
  S.peak_kv = S.peak_kv < alloc ? alloc : S.peak_kv;
  U.flops = __dadd_rn(U.flops, flops);
  S.ev_kind = 2;
  S.ev_time = __dadd_rn(U.clock, lat);
  S.ev_seq = U.seq++;
  return true;
}

// Token tables: one thread per (table, t).  Same device arithmetic as the
// full per-batch path, so every entry equals what batch_latency would compute.
__global__ void k_build_tables(const SimConfig* __restrict__ cfgs, int32_t n, int32_t stride,
                               const SsgEstView* __restrict__ ests, double* __restrict__ pool,
                               uint8_t* __restrict__ valid) {
  const int32_t i = blockIdx.y;
  const int32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n || t >= stride) return;
  const SimConfig& c = cfgs[i];
  const SsgEstView E = ests[c.est];
  double* tab = pool + c.tab_off;
  const double tokens = (double)t;
  double s6 = 0.0, f6 = 0.0, cm[3] = {0.0, 0.0, 0.0}, p0 = 0.0, p0f = 0.0;
  bool ok_tok = t >= 1, ok_pre = t >= 1;
  int k = 0;
  for (int oi = 0; oi < c.nops; ++oi) {
    const SimOp& o = c.ops[oi];
    double pred = 0.0;
    int bad = 0;
    if (o.cls == SSG_CLS_TOKEN) {
      if (ssg_predict_one(E, o.slot, tokens, 0.0, &pred, &bad) != SSG_OK) ok_tok = false;
      s6 = __dadd_rn(s6, __dmul_rn(o.count, pred));
      double fl;
      if (o.flop_kind == 0)
        fl = __dmul_rn(__dmul_rn(__dmul_rn(2.0, tokens), o.fa), o.fb);
      else if (o.flop_kind == 1)
        fl = __dmul_rn(tokens, o.fa);
      else
        fl = __dmul_rn(__dmul_rn(8.0, tokens), o.fa);
      f6 = __dadd_rn(f6, __dmul_rn(o.count, fl));
    } else if (o.cls == SSG_CLS_COMM) {
      if (ssg_predict_one(E, o.slot, __dmul_rn(tokens, o.payload), 0.0, &pred, &bad) != SSG_OK)
        ok_tok = false;
      if (k < 3) cm[k++] = __dmul_rn(o.count, pred);
    } else if (o.flop_kind == 3) {
      const double v1 = __dmul_rn(0.0, o.kvb);
      const double ctx_tokens = v1 / o.kvb;
      if (ssg_predict_one(E, o.slot, tokens, v1, &pred, &bad) != SSG_OK) ok_pre = false;
      p0 = __dmul_rn(o.count, pred);
      p0f = __dmul_rn(o.count, __dmul_rn(__dmul_rn(__dmul_rn(4.0, tokens), __dadd_rn(tokens, ctx_tokens)), o.fa));
    }
  }
  tab[t] = s6;
  tab[(int64_t)stride + t] = f6;
  tab[2LL * stride + t] = cm[0];
  tab[3LL * stride + t] = cm[1];
  tab[4LL * stride + t] = cm[2];
  tab[5LL * stride + t] = p0;
  tab[6LL * stride + t] = p0f;
  if (c.tab_cells) {
    // axis-0 interp cells of the attention models at v0 = t (same device code
    // as ssg_interp: log1p of the host's glibc variant, then ssg_axis_cell)
    const double x0 = E.math_fma ? ssg_log1p(tokens, 1) : ssg_log1p(tokens, 0);
    const int idx[2] = {c.idx_dec, c.idx_pre};
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const SsgModelDesc& md = E.models[c.ops[idx[q]].slot];
      int32_t lo = 0;
      double f = 0.0;
      ssg_axis_cell(E.dpool + md.axis_off[0], md.axis_len[0], x0, &lo, &f);
      tab[(7LL + 2 * q) * stride + t] = f;
      tab[(8LL + 2 * q) * stride + t] = (double)lo;
    }
  }
  valid[(int64_t)i * stride + t] = (ok_tok ? 1 : 0) | (ok_pre ? 2 : 0);
}

// ---------------------------------------------------------------- fast-forward
// Pure-decode stretches of a lone replica (vLLM / Orca+ / LightLLM / Sarathi).
// While nothing can change the batch -- no request waits, or the batch is
// full (either way admission cannot run), every runner is past its prefill and
// stays unfinished, its block shortfalls fit in free memory (so nothing is
// preempted), the token budget
// covers one decode per runner, and no arrival lands before the batch
// completes -- each reference iteration is: every runner decodes (in running
// order), reserves kv+1 tokens, the batch costs predict_batch(...) and
// completes one token per runner.  Within such a stretch nd is constant, so
// the token-table terms, log1p(nd) and the interp cell along the batch-size
// axis are loop invariants, and each microbatch's context sum grows by its
// size per iteration.  The loop performs exactly the reference's steps on
// those quantities; it stops *before* any iteration that would break a
// condition (or raise) and hands it to the normal path, so every decision,
// clock value and counter stays identical.  Returns iterations executed.
#ifndef SSG_FF_MAX_PP
// the fast-forward keeps per-microbatch state in registers, unrolled over this
// many microbatches (deeper pipelines take the exact event-loop path).  4 covers
// the search space's pp in {1, 2, 4}; 8 measured slower (bigger unrolled body:
// 1/2 cfg #4 shard 0.696 vs 0.74 s, full sweep 1.128 vs 1.155 s)
#define SSG_FF_MAX_PP 4
#endif
#ifndef SSG_FF_RUNNERS
// runners of a fast-forwarded batch: one per lane, and with 64 a second slot
// per lane (runner lane + 32)
#define SSG_FF_RUNNERS 64
#endif
#ifndef SSG_FF_ARRIVE_ONE
#define SSG_FF_ARRIVE_ONE 1  // a batch that is not full still runs the iteration an arrival lands in
#endif
//
// Arrivals.  A request arriving during an iteration (at or before its
// completion: arrivals carry the lower sequence numbers) is routed to the lone
// replica and enqueued while the replica is busy, so the batch in flight is
// unaffected.  A full batch stays the same batch afterwards (every policy admits
// only while running < max_batch_size), so the stretch goes on with the queue
// longer; a batch that is not full ends the stretch after that iteration, and
// the next BatchStart (admission) is the event loop's.  An arrival whose
// enqueue would raise (KV capacity) ends the stretch before its iteration.
//
// Lane-parallel over iterations.  Inside a stretch, iteration k's schedule and
// cost are functions of k alone: runner r reserves kv_r+k+1 tokens holding
// max(held_r, units(kv_r+k)) (k >= 1), microbatch m's context sum is
// ctx_m + k*nd_m.  So lane i evaluates iteration done+i of a 32-iteration
// chunk -- block needs, the decode-attention interpolation per microbatch,
// the makespan -- all at once; only the order-dependent parts are chained:
// the allocation (an exact integer prefix scan), and the clock, busy time and
// flops (fp64 adds performed one iteration after the other, in iteration
// order, as the reference does).  The committed prefix ends before the first
// iteration that breaks a condition, exactly where the one-iteration loop
// stopped.
template <int FMA, int LONE>
__device__ __forceinline__ int fast_forward_t(Unit& U, RepState& S, int32_t* next_arrival,
                                              double* next_arrival_time, double* flops_acc) {
  const SimConfig& c = *U.cfg;
  const int nd = S.run_n, pp = c.pp;
  if (pp > SSG_FF_MAX_PP) return 0;  // deeper pipelines take the normal path
  const int nm = nd < pp ? nd : pp;  // non-empty microbatches
  // cheapest exit first: iteration 0 completes no earlier than
  // clock + S6[size of microbatch 0] + cpu overhead (every further term of
  // the latency is a non-negative prediction, and round-to-nearest adds of
  // non-negative terms never decrease), so an arrival at or before that
  // point stops the stretch before it starts.  The same bound holds for every
  // iteration of the stretch (same microbatch sizes).
  const double lb = __dadd_rn(U.tables[c.tab_off + (nd + pp - 1) / pp], c.cpu_overhead);
  const bool arrivals_end = nd < c.max_batch;  // an arrival ends the stretch
  if (!SSG_FF_ARRIVE_ONE && arrivals_end && *next_arrival < U.u->n &&
      *next_arrival_time <= __dadd_rn(U.clock, lb)) {
    FFSTAT(9);
    return 0;
  }
  const int lane = U.lane;
  const bool mine = lane < nd;
  // runner state (running order == decode entry order): runner lane, and
  // runner lane + 32 in the second slot
  int32_t j = 0, kv = 0, held = 0, rem = 0x7fffffff;
  if (mine) {
    j = RUN(U, 0)[lane];
    const ReqHot h = U.hot[j];
    kv = h.kv;
    held = h.held;
    rem = (h.done < h.target) ? 0 : h.decode - h.emitted;
  }
  const bool mine2 = SSG_FF_RUNNERS > 32 && lane + 32 < nd;
  int32_t j2 = 0, kv2 = 0, held2 = 0;
  if (mine2) {
    j2 = RUN(U, 0)[lane + 32];
    const ReqHot h = U.hot[j2];
    kv2 = h.kv;
    held2 = h.held;
    const int32_t rem2 = (h.done < h.target) ? 0 : h.decode - h.emitted;
    rem = rem2 < rem ? rem2 : rem;
  }
  // iterations before any runner would finish (the finishing one is left to the normal path)
  int min_rem = rem;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const int t = __shfl_xor_sync(SSG_FULL, min_rem, o);
    min_rem = t < min_rem ? t : min_rem;
  }
  const int max_iters = min_rem - 1;
  if (max_iters < 1) { FFSTAT(10); return 0; }
  const SimOp& od = c.ops[c.idx_dec];
  const SsgModelDesc& md = U.E.models[od.slot];
  if (md.kind != SSG_KIND_INTERP || !c.tab_cells) return 0;
  // contexts and block counts below 2^25: every 64-runner sum below fits 31 bits
  if (!__all_sync(SSG_FULL, ((kv | kv2) >> 25) == 0) || c.total_units >= (1LL << 25)) return 0;
  // lane layout of a round: P lanes per iteration (lane = it * P + m), one
  // lane per microbatch, so each lane makes one attention query per round
  const int P = pp == 1 ? 1 : (pp == 2 ? 2 : 4);
  const int lgP = pp == 1 ? 0 : (pp == 2 ? 1 : 2);
  const int KI = 32 >> lgP;  // iterations per round
  const int q_m = lane & (P - 1), q_it = lane >> lgP;
  const bool q_on = q_m < nm;
  // microbatch q_m's invariants: size, context sum, token-table terms, axis-0 cell
  int64_t ctx_q = 0;
  const int run_m = lane % pp, run_m2 = (lane + 32) % pp;  // runner -> its microbatch
#pragma unroll 1
  for (int m = 0; m < nm; ++m) {
    const unsigned cm = __reduce_add_sync(SSG_FULL, (mine && run_m == m ? (unsigned)kv + 1u : 0u) +
                                                        (mine2 && run_m2 == m ? (unsigned)kv2 + 1u : 0u));
    if (q_m == m) ctx_q = cm;
  }
  const int nd_q = q_on ? (nd - q_m + pp - 1) / pp : 0;
  const double* tab = U.tables + c.tab_off;
  const int T1 = c.tab_stride;
  double tok_s = 0.0, tok_f = 0.0, comm_q = 0.0;
  int32_t lo0 = 0;
  double f0 = 0.0;
  bool ok = true;
  if (q_on) {
    tok_s = tab[nd_q];
    tok_f = tab[(int64_t)T1 + nd_q];
    const double v0 = (double)nd_q;
    ok = v0 >= md.lower[0] && v0 <= md.upper[0];
    // the axis-0 cell at v0 = nd_q from the token tables (k_build_tables computes
    // ssg_axis_cell(log1p(t)) with the same code; tab_cells is checked on entry)
    f0 = tab[7LL * T1 + nd_q];
    lo0 = (int32_t)tab[8LL * T1 + nd_q];
  }
  if (!__all_sync(SSG_FULL, ok)) { FFSTAT(11); return 0; }
  const bool emit_times = (U.u->flags & SSG_UF_EMISSIONS) != 0;
  const bool logging = !LONE && (U.u->flags & SSG_UF_BATCH_LOG) != 0;
  const double fa4 = od.fa;
  // emission slot of this runner's next token
  // (every runner's prefill is complete here: rem = decode - emitted)
  const int64_t ebase = (mine && emit_times) ? U.emit_base[j] + U.hot[j].emitted : 0;
  const int64_t ebase2 = (mine2 && emit_times) ? U.emit_base[j2] + U.hot[j2].emitted : 0;
  const int64_t free0 = c.total_units;
  const double tp_pp = (double)(c.tp * c.pp);
  // block needs in closed form when units(x) = ceil(x / B) through the block
  // magic and every kv + k (< 2^31) and held * B stay below 2^32
  const int64_t B = c.block_size;
  const bool closed_needs = c.bs_magic != 0 && c.total_units * B < (1LL << 31);
  int done = 0;
  while (done < max_iters) {
    // iterations this round: at most KI, and (when an arrival ends the stretch)
    // no more than can complete before the next arrival, each lasting >= lb
    int KIr = max_iters - done < KI ? max_iters - done : KI;
    if (arrivals_end && *next_arrival < U.u->n) {
      // (a cap only: rounds split where it is low, so an approximate quotient is enough)
      const float est = __fdividef((float)__dsub_rn(*next_arrival_time, U.clock), (float)lb) + 2.0f;
      if (est < (float)KIr) KIr = est < 1.0f ? 1 : (int)est;
    }
    const int k = done + q_it;  // this lane's iteration
    const bool active = q_it < KIr;
    // ---- schedule: every runner reserves kv+k+1 tokens (no preemption allowed)
    int64_t need = 0;
    if (closed_needs) {
      // runner (kv, held) needs units(kv+1) - held blocks at k = 0 (if positive)
      // and, at k >= 1, one block exactly when kv + k is a multiple of B and
      // kv + k >= held * B (units(kv+k+1) exceeds both held and units(kv+k));
      // each runner adds its needs of the round to per-iteration counters
      int32_t* cnt = reinterpret_cast<int32_t*>(U.smem_stats);
      cnt[lane] = 0;
      __syncwarp();
#pragma unroll
      for (int sl = 0; sl < (SSG_FF_RUNNERS > 32 ? 2 : 1); ++sl) {
        if (sl == 0 ? mine : mine2) {
          const int64_t kvs = sl == 0 ? kv : kv2, hs = sl == 0 ? held : held2;
          if (done == 0) {
            const int64_t s0 = units_for(c, kvs + 1) - hs;
            if (s0 > 0) atomicAdd(&cnt[0], (int32_t)s0);
          }
          int64_t kmin = done > 1 ? done : 1;
          if (hs * B - kvs > kmin) kmin = hs * B - kvs;
          const uint64_t x = (uint64_t)(kvs + kmin);
          const int64_t rr = (int64_t)(x - __umul64hi(x, c.bs_magic) * (uint64_t)B);
#pragma unroll 1
          for (int64_t k = rr == 0 ? kmin : kmin + (B - rr); k < done + KIr; k += B)
            atomicAdd(&cnt[k - done], 1);
        }
      }
      __syncwarp();
      need = cnt[q_it];
      __syncwarp();
    } else
#pragma unroll 1
    for (int i = 0; i < KIr; ++i) {
      const int ki = done + i;
      uint32_t sr = 0;
#pragma unroll
      for (int sl = 0; sl < (SSG_FF_RUNNERS > 32 ? 2 : 1); ++sl) {
        if (sl == 0 ? mine : mine2) {
          const int32_t kvs = sl == 0 ? kv : kv2, hs = sl == 0 ? held : held2;
          int64_t hk = hs;
          if (ki > 0) {
            const int64_t u = units_for(c, (int64_t)kvs + ki);
            hk = hk < u ? u : hk;
          }
          const int64_t s = units_for(c, (int64_t)kvs + ki + 1) - hk;
          sr += s > 0 ? (uint32_t)s : 0u;
        }
      }
      const unsigned tot = __reduce_add_sync(SSG_FULL, sr);
      if (q_it == i) need = tot;
    }
    // ---- cost: lane (it, m) queries microbatch m's decode attention of iteration it
    double tim_l = 0.0, fl_l = 0.0;
    bool good_l = true;
    if (active && q_on) {
      const double v1 = __dmul_rn((double)(ctx_q + (int64_t)k * nd_q), od.kvb);
      // the batch latency's attention query (one out-of-line copy); v0 = nd_q
      // passed the bounding box on entry
      const AttnQuery aq = ssg_attn_interp<FMA>(U.E.dpool, &md, (double)nd_q, v1, lo0, f0, U.ax1_hint);
      U.ax1_hint = aq.hint;
      if (aq.code != SSG_OK) {
        good_l = false;
      } else {
        double acc = __dadd_rn(tok_s, __dmul_rn(od.count, aq.pred));
        // comm ops (at most 3), op order
        const double* comm = tab + 2 * (int64_t)T1 + nd_q;
        if (c.ncomm > 0) acc = __dadd_rn(acc, comm[0]);
        if (c.ncomm > 1) acc = __dadd_rn(acc, comm[T1]);
        if (c.ncomm > 2) acc = __dadd_rn(acc, comm[2 * (int64_t)T1]);
        const double ctx_tokens = v1 / od.kvb;
        fl_l = __dadd_rn(tok_f, __dmul_rn(od.count, __dmul_rn(__dmul_rn(4.0, ctx_tokens), fa4)));
        good_l = acc > 0.0;
        tim_l = acc;
      }
    }
    // ---- per iteration (its P lanes): flops in microbatch order, makespan
    const int base = lane & ~(P - 1);
    const unsigned badm = __ballot_sync(SSG_FULL, !good_l);
    const bool good = ((badm >> base) & ((1u << P) - 1u)) == 0u;
    double tim[SSG_FF_MAX_PP];
    double fl_tot = 0.0;
#pragma unroll
    for (int m = 0; m < SSG_FF_MAX_PP; ++m) {
      const double tm = __shfl_sync(SSG_FULL, tim_l, (base + m) & 31);
      const double fm = __shfl_sync(SSG_FULL, fl_l, (base + m) & 31);
      tim[m] = tm;
      if (m < nm) fl_tot = pp == 1 ? __dmul_rn(fm, (double)c.tp) : __dadd_rn(fl_tot, __dmul_rn(fm, tp_pp));
    }
    double lat;
    if (pp == 1) {
      lat = tim[0];
    } else {
      // synchronous pipeline finish times (scheduler.hpp:566-579), in registers
      double fin[SSG_FF_MAX_PP];
#pragma unroll
      for (int m = 0; m < SSG_FF_MAX_PP; ++m) fin[m] = 0.0;
#pragma unroll 1
      for (int st = 0; st < pp; ++st) {
        double prev = 0.0;
#pragma unroll
        for (int m = 0; m < SSG_FF_MAX_PP; ++m) {
          if (m < nm) {
            const double start = fin[m] < prev ? prev : fin[m];
            prev = __dadd_rn(start, tim[m]);
            fin[m] = prev;
          }
        }
      }
      lat = fin[0];
#pragma unroll
      for (int m = 1; m < SSG_FF_MAX_PP; ++m)
        if (m < nm) lat = fin[m];
    }
    lat = __dadd_rn(lat, c.cpu_overhead);
    // ---- the order-dependent parts, in iteration order
    // allocation before this lane's iteration: exclusive prefix of the needs
    // (a scan over the iteration groups: shifts by multiples of P)
    int64_t incl = need;
#pragma unroll 1
    for (int o = P; o < 32; o <<= 1) {
      const int64_t t = __shfl_up_sync(SSG_FULL, incl, o);
      if (lane >= o) incl += t;
    }
    const int64_t alloc_after = S.allocated + incl;
    const bool fits = need <= free0 - (alloc_after - need);
    // iterations that can happen as far as memory and the cost go
    const bool pre = active && fits && good && lat > 0.0;
    const unsigned bad = __ballot_sync(SSG_FULL, !pre);
    const int C = bad ? (__ffs(bad) - 1) >> lgP : KI;
    if (C == 0) { if (done == 0) FFSTAT(12); break; }
    // clock / busy time / flops: one fp64 add per iteration, in order; the
    // chain (warp-uniform) stops at the first completion at or after the next
    // arrival: an arrival at or before a completion is processed between the
    // batch's start and completion events, so that iteration is the loop's
    double clk = U.clock, busy = S.busy_time, fla = *flops_acc;
    double t_done = 0.0;  // on lane i: completion of the round's iteration i
    int K = 0;
    const int32_t na0 = *next_arrival;
    int32_t na = na0;                  // arrivals up to the last committed completion
    // (the event loop keeps the last arrival's time once every arrival is in)
    double ta = na0 < U.u->n ? *next_arrival_time : INFINITY;
    bool ends = false;                 // an arrival ends the stretch after iteration K
    for (; K < C; ++K) {
      const double li = __shfl_sync(SSG_FULL, lat, K << lgP);
      const double fi = __shfl_sync(SSG_FULL, fl_tot, K << lgP);
      const double c2 = __dadd_rn(clk, li);
      int32_t na2 = na;
      double ta2 = ta;
      bool reject = false;
      while (ta2 <= c2) {  // arrivals during iteration K
        const int32_t ja = arrival_slot<LONE>(U, na2);
        const ReqHot h = U.hot[ja];
        if (units_for(c, (int64_t)h.prefill + h.decode) > c.total_units) {
          reject = true;  // enqueue raises: the event loop's
          break;
        }
        ++na2;
        ta2 = na2 < U.u->n ? U.tm[arrival_slot<LONE>(U, na2)].arrival : INFINITY;
      }
      if (reject) break;
      clk = c2;
      busy = __dadd_rn(busy, li);
      fla = __dadd_rn(fla, fi);
      if (lane == K) t_done = clk;
      const bool arrived = na2 != na;
      na = na2;
      ta = ta2;
      if (arrived && arrivals_end) {
        ends = true;
        ++K;
        break;
      }
    }
    if (K == 0) { if (done == 0) FFSTAT(13); break; }
    const int last = K - 1;
    // ---- commit iterations done .. done+K-1 (from here on lane i <-> iteration done+i)
    const int kit = done + lane;
    if (logging) {
      const int64_t need_w = 6 + 2LL * nd;
      const int64_t used = U.out->log_used;
      int64_t fit = 0;
      if (used >= 0) {
        fit = (U.u->log_cap - used) / need_w;
        fit = fit < 0 ? 0 : (fit > K ? K : fit);
      }
      const int64_t a_it = __shfl_sync(SSG_FULL, alloc_after, (lane << lgP) & 31);
      const double lat_it = __shfl_sync(SSG_FULL, lat, (lane << lgP) & 31);
      if (lane < fit) {
        int64_t* L = U.log + used + lane * need_w;
        L[0] = 0;
        L[2] = a_it;
        L[3] = 0;
        L[4] = nd;
        L[5] = __double_as_longlong(lat_it);
      }
      // batch start clock of iteration i = completion of iteration i-1
      const double t_prev = __shfl_up_sync(SSG_FULL, t_done, 1);
      if (lane < fit) U.log[used + lane * need_w + 1] = __double_as_longlong(lane == 0 ? U.clock : t_prev);
#pragma unroll 1
      for (int r = 0; r < nd; ++r) {
        const int64_t id_r = U.ids[__shfl_sync(SSG_FULL, r < 32 ? j : j2, r & 31)];
        const int32_t kv_r = __shfl_sync(SSG_FULL, r < 32 ? kv : kv2, r & 31);
        if (lane < fit) {
          int64_t* L = U.log + used + lane * need_w;
          L[6 + 2 * r] = id_r;
          L[7 + 2 * r] = (int64_t)kv_r + kit + 1;
        }
      }
      __syncwarp();
      wput(U, &U.out->log_used, used >= 0 && fit == K ? used + K * need_w : (int64_t)-1);
    }
    if (emit_times) {
      // runner lanes write their token of each committed iteration
#pragma unroll 1
      for (int k = 0; k < K; ++k) {
        const double tk = __shfl_sync(SSG_FULL, t_done, k);
        if (mine) U.emissions[ebase + done + k] = tk;
        if (mine2) U.emissions[ebase2 + done + k] = tk;
      }
    }
    // peak allocated units of the committed iterations (below 2^25 here)
    const double pk = (double)__reduce_max_sync(SSG_FULL, q_it < K ? (unsigned)alloc_after : 0u);
    S.peak_kv = S.peak_kv < pk ? pk : S.peak_kv;
    S.allocated = __shfl_sync(SSG_FULL, alloc_after, last << lgP);
    S.busy_time = busy;
    *flops_acc = fla;
    U.clock = clk;
    U.serial += K;
    S.iterations += K;
    S.tokens += (int64_t)nd * K;
    U.iters += K;
    U.entries += (int64_t)nd * K;
    U.qbytes += (int64_t)K * nm * (c.qb_fixed + c.qb_dec);
    done += K;
    // the arrivals of the committed iterations: routed to the lone replica and
    // enqueued (sim.hpp:211-220); the replica is busy, so nothing starts
    for (int32_t q = na0; q < na; ++q) enqueue(U, S, 0, arrival_slot<LONE>(U, q));
    *next_arrival = na;
    *next_arrival_time = ta;
    if (ends || K < KIr) break;
  }
  if (done > 0 && mine) {
    ReqHot& h = U.hot[j];
    const int64_t u = units_for(c, (int64_t)kv + done);
    h.kv = kv + done;
    h.held = held < u ? (int32_t)u : held;
    h.emitted = h.emitted + done;
  }
  if (done > 0 && mine2) {
    ReqHot& h = U.hot[j2];
    const int64_t u = units_for(c, (int64_t)kv2 + done);
    h.kv = kv2 + done;
    h.held = held2 < u ? (int32_t)u : held2;
    h.emitted = h.emitted + done;
  }
  __syncwarp();
  return done;
}

template <int FMA, int LONE>
__device__ SSG_FFWD int fast_forward(Unit& U, RepState& S, int32_t* next_arrival,
                                     double* next_arrival_time, double* flops_acc) {
  const SimConfig& c = *U.cfg;
  if (c.policy != SSG_POL_VLLM && c.policy != SSG_POL_ORCA && c.policy != SSG_POL_LIGHTLLM &&
      c.policy != SSG_POL_SARATHI)
    return 0;
  // requests may wait only while the batch is full: every policy's admission
  // loop requires running < max_batch_size before it looks at the queue
  // (scheduler.hpp:360-361, 387-388, 425-427)
  if ((S.wait_n != 0 && S.run_n < c.max_batch) || S.run_n < 1 || S.run_n > SSG_FF_RUNNERS || c.tab_off < 0 ||
      c.idx_dec < 0)
    return 0;
  const int nd = S.run_n, pp = c.pp;
  if (c.policy == SSG_POL_SARATHI ? nd > c.chunk : nd > c.max_tokens) return 0;
  // microbatch 0 (ceil(nd / pp) runners) within the token tables: nd <= tab_tmax * pp
  if (nd > c.max_batch || nd > (int64_t)c.tab_tmax * pp) return 0;
  return fast_forward_t<FMA, LONE>(U, S, next_arrival, next_arrival_time, flops_acc);
}

// LONE = 1: every unit of the launch is one replica with round-robin or
// least-outstanding routing, without batch log or arrival permutation (the
// sweep's decoupled probes), so the multi-replica event selection, routing
// argmins, deferred pool, replica-state spills and log writers are compiled out
// of the body (the kernel is instruction-fetch bound).
template <int FMA, int FOREST, int FAST, int LONE>
__device__ void run_unit(Unit& U) {
  const long long t_start = clock64();
  const SimUnit& u = *U.u;
  const SimConfig& c = *U.cfg;
  const int R = LONE ? 1 : u.R;
  // ---- reset per-request state and replicas
#pragma unroll 1
  for (int32_t j = U.lane; j < u.n; j += 32) {
    ReqHot& h = U.hot[j];
    h.target = 0;
    h.done = 0;
    h.emitted = 0;
    h.kv = 0;
    h.held = 0;
    h.planned = 0;
    ReqTimes& t = U.tm[j];
    t.first_sched = -1.0;
    t.first_tok = -1.0;
    t.completion = -1.0;
    U.restarts[j] = 0;
  }
#pragma unroll 1
  for (int r = U.lane; r < R; r += 32) {
    RepState s;
    memset(&s, 0, sizeof s);
    U.reps[r] = s;
  }
  if (U.lane == 0) {
    POOL_HEAD(U)[0] = 0;
    POOL_HEAD(U)[1] = 0;
    SimUnitOut o;
    memset(&o, 0, sizeof o);
    *U.out = o;
  }
  __syncwarp();
  U.flops = 0.0;
  U.clock = 0.0;
  U.seq = (uint64_t)u.n;
  U.serial = 0;
  U.qbytes = 0;
  U.qb_lane = 0;
  U.iters = 0;
  U.entries = 0;
  int32_t next_arrival = 0;
  int32_t rr_next = 0;
  int64_t events = 0;
  double next_arrival_time =
      u.n > 0 ? U.tm[arrival_slot<LONE>(U, 0)].arrival : INFINITY;
  // a lone replica (no deferred pool) keeps its scheduler state in registers
  const bool reg1 = LONE ? true : (R == 1 && c.routing != SSG_ROUTE_DEFERRED);
  RepState S1;
  memset(&S1, 0, sizeof S1);
  // a lone replica's BatchStart queued by BatchComplete at the same clock is the
  // next event unless an arrival is due at or before it (arrivals carry lower
  // seq numbers): then the event selection is skipped (one call site each)
  bool direct = false;
  int since_check = 0;  // BatchStarts since the last speculation-group check
  while (true) {
    // ---- next event: (time, seq) argmin over the arrival head and replica slots
    double bt = INFINITY;
    uint64_t bs = ~0ull;
    int bw = -2;  // -1 arrival, r >= 0 replica
    if (direct) {
      direct = false;
      bt = U.clock;
      bw = 0;
      goto replica_event;
    }
    if (next_arrival < u.n) {
      bt = next_arrival_time;
      bs = (uint64_t)next_arrival;
      bw = -1;
    }
    if (R == 1) {
      // one replica: its pending event vs the next arrival, no warp reduction
      const RepState s0 = reg1 ? S1 : U.reps[0];
      if (s0.ev_kind != 0) {
        const double t = s0.ev_time;
        const uint64_t q = s0.ev_seq;
        if (t < bt || (t == bt && q < bs)) {
          bt = t;
          bs = q;
          bw = 0;
        }
      }
    } else
#pragma unroll 1
    for (int r0 = 0; r0 < R; r0 += 32) {
      const int r = r0 + U.lane;
      double t = INFINITY;
      uint64_t q = ~0ull;
      if (r < R && U.reps[r].ev_kind != 0) {
        t = U.reps[r].ev_time;
        q = U.reps[r].ev_seq;
      }
      int w = r;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double t2 = __shfl_xor_sync(SSG_FULL, t, o);
        const uint64_t q2 = __shfl_xor_sync(SSG_FULL, q, o);
        const int w2 = __shfl_xor_sync(SSG_FULL, w, o);
        if (t2 < t || (t2 == t && q2 < q)) {
          t = t2;
          q = q2;
          w = w2;
        }
      }
      if (q != ~0ull && (t < bt || (t == bt && q < bs))) {
        bt = t;
        bs = q;
        bw = w;
      }
    }
    if (bw == -2) break;
  replica_event:
    if (bt < U.clock) {
      set_error(U, SSG_ERR_INTERNAL, 6, 0, 0, bt);  // event time regression
      break;
    }
    U.clock = bt;
    ++events;
    if (bw == -1) {
      // ---- Arrival: route, enqueue, start_if_idle (sim.hpp:211-220)
      const int32_t j = arrival_slot<LONE>(U, next_arrival);
      ++next_arrival;
      if (next_arrival < u.n)
        next_arrival_time = U.tm[arrival_slot<LONE>(U, next_arrival)].arrival;
      int dest = 0;
      if (LONE) {
        // the lone replica takes every arrival
      } else if (c.routing == SSG_ROUTE_RR) {
        dest = rr_next;
        rr_next = (rr_next + 1) % R;
      } else if (c.routing == SSG_ROUTE_LO) {
        // argmin outstanding, ties to the lowest index
        int64_t key = INT64_MAX;
#pragma unroll 1
        for (int r0 = 0; r0 < R; r0 += 32) {
          const int r = r0 + U.lane;
          int64_t k2 = r < R ? (((int64_t)U.reps[r].outstanding) << 16 | r) : INT64_MAX;
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) {
            const int64_t t2 = __shfl_xor_sync(SSG_FULL, k2, o);
            k2 = t2 < k2 ? t2 : k2;
          }
          key = k2 < key ? k2 : key;
        }
        dest = (int)(key & 0xffff);
      } else {
        // deferred: pool the request, then drain
        int32_t* ph = POOL_HEAD(U);
        const int32_t head = ph[0], size = ph[1];
        wput(U, &POOL(U)[(head + size) & (U.WC - 1)], j);
        wput(U, &ph[1], size + 1);
        drain_pool(U);
        if (failed(U)) break;
        continue;
      }
      RepState S = reg1 ? S1 : load_rep(U, dest);
      SSG_PH_BEGIN(ph_a);
      const bool ok = enqueue(U, S, dest, j);
      if (ok) start_if_idle(U, S);
      SSG_PH_END(ph_a, 4);
      if (reg1)
        S1 = S;
      else
        store_rep(U, dest, S);
      if (!ok) break;
      continue;
    }
    const int r = bw;
    RepState S = reg1 ? S1 : load_rep(U, r);
#ifdef SSG_FF_STATS
    if (FAST && S.ev_kind == 1 && reg1) {
      if (S.run_n > SSG_FF_RUNNERS) FFSTAT(14);
      else if (!(S.wait_n == 0 || S.run_n >= c.max_batch)) FFSTAT(15);
    }
#endif
#ifdef SSG_PHASE_CYCLES
    if (FAST && S.ev_kind == 1 && reg1) {
      if (S.run_n > SSG_FF_RUNNERS) U.ph[12] += 1;
      else if (!(S.wait_n == 0 || S.run_n >= c.max_batch)) U.ph[13] += 1;
    }
#endif
    if (FAST && S.ev_kind == 1 && reg1 && (S.wait_n == 0 || S.run_n >= c.max_batch) &&
        S.run_n >= 1 && S.run_n <= SSG_FF_RUNNERS) {
      // pure-decode stretch: iterations that end at the same state the event
      // loop would reach; afterwards the replica is again "BatchStart at clock"
      double fl = U.flops;
      const int32_t na_before = next_arrival;
      SSG_PH_BEGIN(ph_f);
      const int k = fast_forward<FMA, LONE>(U, S, &next_arrival, &next_arrival_time, &fl);
      SSG_PH_END(ph_f, 3);
#ifdef SSG_PHASE_CYCLES
      U.ph[5] += k;
      U.ph[7] += 1;
      U.ph[14] += k == 0;
#endif
#ifdef SSG_FF_STATS
      if (U.lane == 0) {
        atomicAdd(&g_ff_stats[0], 1ull);
        atomicAdd(&g_ff_stats[1], (unsigned long long)k);
        atomicAdd(&g_ff_stats[2 + (k == 0 ? 0 : min(6, 32 - __clz(k)))], 1ull);
      }
#endif
      if (k > 0) {
        U.flops = fl;
        events += 2 * k + (next_arrival - na_before);
        S.ev_time = U.clock;
        S.ev_seq = U.seq++;
        S1 = S;
        continue;
      }
    }
    if (S.ev_kind == 1) {
      // a speculative probe the capacity replay can no longer ask for (a probe
      // it is only asked after, on a feasible outcome, failed): stop, result unused
      if (U.group_fail && ++since_check >= 64 &&
          (since_check = 0, (*(volatile const uint32_t*)U.group_fail & u.kill) != 0)) {
        wput(U, &U.out->aborted, 2);
        break;
      }
      S.ev_kind = 0;
      const bool ok = batch_start<FMA, FOREST, LONE>(U, S, r);
      if (reg1)
        S1 = S;
      else
        store_rep(U, r, S);
      if (!ok) break;
    } else {
      // ---- BatchComplete (sim.hpp:284-293)
      S.ev_kind = 0;
      SSG_PH_BEGIN(ph_c);
      complete_batch(U, S, r);
      SSG_PH_END(ph_c, 2);
      S.np = 0;
      S.nd = 0;
      S.busy = 0;
      if (failed(U)) {
        if (reg1)
          S1 = S;
        else
          store_rep(U, r, S);
        break;
      }
      start_if_idle(U, S);
      if (reg1) {
        S1 = S;
        direct = !FAST && S.ev_kind == 1 && !(next_arrival < u.n && next_arrival_time <= U.clock);
      } else if (!LONE) {
        store_rep(U, r, S);
        drain_pool(U);
      }
      if (failed(U)) break;
    }
  }
  if (reg1) store_rep(U, 0, S1);
  __syncwarp();
#pragma unroll 1
  for (int r = U.lane; r < R; r += 32) {
    const double p = U.reps[r].peak_kv;  // 0 stays 0 (no units ever allocated)
    if (p > 0.0) U.reps[r].peak_kv = p / (double)c.total_units;
  }
  // an aborted or failed probe cancels the speculative probes behind its feasible branch
  if (U.group_fail && U.lane == 0 && (U.out->aborted == 1 || U.out->code != SSG_OK))
    atomicOr(U.group_fail, 1u << u.rung);
  U.qbytes += warp_sum64(U.qb_lane);
  if (U.lane == 0) {
    U.out->flops = U.flops;
    U.out->span = U.clock;
    U.out->events = events;
    U.out->iterations = U.iters;
    U.out->entries = U.entries;
    U.out->qbytes = U.qbytes;
    U.out->cycles = clock64() - t_start;
  }
#ifdef SSG_PHASE_CYCLES
  U.ph[6] = clock64() - t_start;
#endif
  __syncwarp();
  if (!failed(U) && !U.out->aborted) {
    // "simulation drained with unfinished request" (sim.hpp:305-306)
    int32_t first_bad = INT32_MAX;
#pragma unroll 1
    for (int32_t j = U.lane; j < u.n; j += 32) {
      const ReqHot h = U.hot[j];
      if (h.emitted < h.decode && j < first_bad) first_bad = j;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const int32_t t = __shfl_xor_sync(SSG_FULL, first_bad, o);
      first_bad = t < first_bad ? t : first_bad;
    }
    if (first_bad != INT32_MAX) set_error(U, SSG_ERR_INTERNAL, 7, U.ids[first_bad], 0, 0.0);
  }
}

#ifndef SSG_SIM_FAST_MINB
#define SSG_SIM_FAST_MINB 1  // fast-forward kernels run lone simulations: registers over occupancy
#endif
#ifndef SSG_SIM_MINB
#define SSG_SIM_MINB 6  // 6 blocks x 2 warps per SM: <= 168 registers (measured best, DESIGN 6.4)
#endif
#ifdef SSG_FAST_MAXNREG
// diagnostic builds: a register cap for the fast-forward variant between the
// launch-bounds steps (A/B of occupancy against spills)
#define SSG_SIM_BOUNDS(FAST) __launch_bounds__(SSG_SIM_WARPS * 32) __maxnreg__(FAST ? SSG_FAST_MAXNREG : 168)
#else
#define SSG_SIM_BOUNDS(FAST) __launch_bounds__(SSG_SIM_WARPS * 32, FAST ? SSG_SIM_FAST_MINB : SSG_SIM_MINB)
#endif
#ifdef SSG_PHASE_CYCLES
#define SSG_PHASE_MAX_UNITS 16384
__device__ long long g_phase[SSG_PHASE_MAX_UNITS][SSG_PH_N];
#endif

template <int FMA, int FOREST, int FAST, int LONE>
__global__ void SSG_SIM_BOUNDS(FAST) k_simulate(SimLaunch L) {
  __shared__ int64_t stats[SSG_SIM_WARPS][SSG_MAX_PP * 6];
  __shared__ double part[SSG_SIM_WARPS][4 * SSG_MAX_PP];
  __shared__ SimConfig cfg_s[SSG_SIM_WARPS];  // the unit's config, read every event
  const int wib = threadIdx.x >> 5;
  const int64_t w = (int64_t)blockIdx.x * SSG_SIM_WARPS + wib;
  if (w >= L.nunits) return;
  const int32_t uid = L.order ? L.order[w] : (int32_t)w;
  Unit U;
  U.u = L.units + uid;
  {
    const int lane = threadIdx.x & 31;
    const uint32_t* src = reinterpret_cast<const uint32_t*>(L.configs + U.u->config);
    uint32_t* dst = reinterpret_cast<uint32_t*>(&cfg_s[wib]);
    for (int k = lane; k < (int)(sizeof(SimConfig) / 4); k += 32) dst[k] = src[k];
    __syncwarp();
  }
  U.cfg = &cfg_s[wib];
  U.E = L.ests[U.cfg->est];
  U.hot = L.hot + U.u->req_off;
  U.tm = L.tm + U.u->req_off;
  U.ids = L.ids + U.u->req_off;
  U.restarts = L.restarts + U.u->req_off;
  U.emit_base = L.emit_base ? L.emit_base + U.u->req_off : nullptr;
  U.emissions = L.emissions;
  U.arr_order = L.arr_order ? L.arr_order + U.u->req_off : nullptr;
  U.reps = L.reps + U.u->rep_off;
  U.ws = L.ws + U.u->ws_off;
  U.log = L.log ? L.log + U.u->log_off : nullptr;
  U.out = L.out + uid;
  U.smem_stats = stats[wib];
  U.smem_part = part[wib];
  U.pcap = SSG_MAX_PP;
  U.tables = L.tables;
  U.fast = L.fast_forward;
  U.group_fail = (L.group_fail && U.u->group >= 0) ? L.group_fail + U.u->group : nullptr;
  U.lane = threadIdx.x & 31;
  U.ax1_hint = 0;
  U.MB = U.u->mb_ws;
  U.WC = U.u->wait_cap;
  U.rep_stride = 6LL * U.MB + U.WC;
  if (U.cfg->pp > SSG_MAX_PP) {
    // deep pipelines: microbatch scratch after the unit's queues and pool
    // (SSG_PP_SCRATCH_WORDS; the host sizes and 8-byte aligns it)
    int32_t* x = U.ws + (int64_t)U.u->R * U.rep_stride + U.WC + 2;
    U.smem_stats = reinterpret_cast<int64_t*>(x);
    U.smem_part = reinterpret_cast<double*>(x + 12LL * U.cfg->pp);
    U.pcap = U.cfg->pp;
  }
#ifdef SSG_PHASE_CYCLES
  for (int k = 0; k < SSG_PH_N; ++k) U.ph[k] = 0;
#endif
  run_unit<FMA, FOREST, FAST, LONE>(U);
#ifdef SSG_PHASE_CYCLES
  if (U.lane == 0 && uid < SSG_PHASE_MAX_UNITS)
    for (int k = 0; k < SSG_PH_N; ++k) g_phase[uid][k] = U.ph[k];
#endif
}

// predict_batch / batch_device_flops for standalone compositions (the
// estimator.hpp:294-380 API): one warp per composition, same device code path
// as the engine's per-iteration latency.
template <int FMA>
__global__ void __launch_bounds__(SSG_SIM_WARPS * 32)
    k_predict_batch(const SimConfig* cfgs, const SsgEstView* ests, const int32_t* comp_cfg,
                    int64_t n, int32_t MB, int32_t* ws, const int32_t* np_nd, double* seconds,
                    double* flops, SimUnitOut* out) {
  __shared__ int64_t stats[SSG_SIM_WARPS][SSG_MAX_PP * 6];
  __shared__ double part[SSG_SIM_WARPS][4 * SSG_MAX_PP];
  const int wib = threadIdx.x >> 5;
  const int64_t c = (int64_t)blockIdx.x * SSG_SIM_WARPS + wib;
  if (c >= n) return;
  Unit U;
  SimUnit dummy;
  memset(&dummy, 0, sizeof dummy);
  dummy.R = 1;
  U.u = &dummy;
  U.cfg = cfgs + comp_cfg[c];
  U.E = ests[U.cfg->est];
  U.MB = MB;
  U.WC = 2;
  U.rep_stride = 6LL * MB + 2;
  U.ws = ws + c * (U.rep_stride + 4);
  U.out = out + c;
  U.smem_stats = stats[wib];
  U.smem_part = part[wib];
  U.pcap = SSG_MAX_PP;
  U.tables = nullptr;
  U.lane = threadIdx.x & 31;
  U.ax1_hint = 0;
  U.clock = 0.0;
  U.qbytes = 0;
  U.qb_lane = 0;
  if (U.lane == 0) {
    SimUnitOut o;
    memset(&o, 0, sizeof o);
    *U.out = o;
  }
  __syncwarp();
  RepState S;
  memset(&S, 0, sizeof S);
  S.np = np_nd[2 * c];
  S.nd = np_nd[2 * c + 1];
  double lat = 0.0, fl = 0.0;
  if (batch_latency<FMA, 1>(U, S, 0, &lat, &fl) == SSG_OK && U.lane == 0) {
    seconds[c] = lat;
    flops[c] = fl;
  }
}

}  // namespace ssgk
#ifdef SSG_FF_STATS
extern "C" void ssg_debug_ff_stats(unsigned long long* out, int reset) {
  cudaMemcpyFromSymbol(out, ssgk::g_ff_stats, sizeof(ssgk::g_ff_stats));
  if (reset) {
    unsigned long long z[16] = {};
    cudaMemcpyToSymbol(ssgk::g_ff_stats, z, sizeof z);
  }
}
#endif

namespace ssg {

void launch_build_tables(const SimConfig* d_cfgs, int32_t n, int32_t stride,
                         const SsgEstView* d_ests, double* d_pool, uint8_t* d_valid, cudaStream_t s) {
  if (n <= 0) return;
  dim3 grid((stride + 127) / 128, n);
  ssgk::k_build_tables<<<grid, 128, 0, s>>>(d_cfgs, n, stride, d_ests, d_pool, d_valid);
  cuda_check(cudaGetLastError(), "k_build_tables launch");
  stats().launches_setup += 1;
}

bool phase_cycles(long long* dst, int64_t n) {
#ifdef SSG_PHASE_CYCLES
  n = n < SSG_PHASE_MAX_UNITS ? n : SSG_PHASE_MAX_UNITS;
  cuda_check(cudaMemcpyFromSymbol(dst, ssgk::g_phase, n * SSG_PH_N * sizeof(long long)), "phase cycles");
  return true;
#else
  (void)dst;
  (void)n;
  return false;
#endif
}

int fast_forward_enabled() {
  static const int on = std::getenv("SSG_NO_FASTFWD") == nullptr ? 1 : 0;
  return on;
}

int sweep_fast_forward_enabled() {
  static const int on = std::getenv("SSG_SWEEP_FASTFWD") != nullptr ? 1 : 0;
  return on;
}

void launch_simulate(const SimLaunch& L, cudaStream_t s) {
  if (L.nunits <= 0) return;
  const int64_t blocks = (L.nunits + SSG_SIM_WARPS - 1) / SSG_SIM_WARPS;
  // one instantiation per glibc variant x (interp-only | with forests) x
  // (decode fast-forward compiled in | out): the kernel is instruction-fetch
  // bound, so each launch runs the smallest body that covers it
  const int fma = context().math_fma;
  const int key = (fma ? 4 : 0) | (L.has_forest ? 2 : 0) | (L.fast_forward ? 1 : 0);
  const unsigned grid = (unsigned)blocks, block = SSG_SIM_WARPS * 32;
  // diagnostic: SSG_SIM_SMEM bytes of dynamic shared memory per block caps
  // the resident warps per SM (A/B of occupancy vs instruction-cache reuse)
  static const int smem = [] {
    const char* e = std::getenv("SSG_SIM_SMEM");
    return e ? std::atoi(e) : 0;
  }();
  auto go = [&](auto kern) {
    if (smem > 48 * 1024)
      cuda_check(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem),
                 "k_simulate smem");
    kern<<<grid, block, smem, s>>>(L);
  };
  if (L.all_lone) {
    switch (key) {
      case 0: go(ssgk::k_simulate<0, 0, 0, 1>); break;
      case 1: go(ssgk::k_simulate<0, 0, 1, 1>); break;
      case 2: go(ssgk::k_simulate<0, 1, 0, 1>); break;
      case 3: go(ssgk::k_simulate<0, 1, 1, 1>); break;
      case 4: go(ssgk::k_simulate<1, 0, 0, 1>); break;
      case 5: go(ssgk::k_simulate<1, 0, 1, 1>); break;
      case 6: go(ssgk::k_simulate<1, 1, 0, 1>); break;
      default: go(ssgk::k_simulate<1, 1, 1, 1>); break;
    }
  } else {
    switch (key) {
      case 0: go(ssgk::k_simulate<0, 0, 0, 0>); break;
      case 1: go(ssgk::k_simulate<0, 0, 1, 0>); break;
      case 2: go(ssgk::k_simulate<0, 1, 0, 0>); break;
      case 3: go(ssgk::k_simulate<0, 1, 1, 0>); break;
      case 4: go(ssgk::k_simulate<1, 0, 0, 0>); break;
      case 5: go(ssgk::k_simulate<1, 0, 1, 0>); break;
      case 6: go(ssgk::k_simulate<1, 1, 0, 0>); break;
      default: go(ssgk::k_simulate<1, 1, 1, 0>); break;
    }
  }
  cuda_check(cudaGetLastError(), "k_simulate launch");
}

}  // namespace ssg

namespace ssg {

void predict_batches_multi(const std::vector<SimConfig>& cfgs_in, const std::vector<SsgEstView>& ests,
                           const std::vector<int32_t>& comp_cfg, int64_t n, const int64_t* p_off,
                           const int64_t* p_len, const int64_t* p_prior, const int64_t* d_off,
                           const int64_t* d_ctx, double* seconds, double* flops,
                           std::vector<SimUnitOut>& status) {
  using namespace servesim;
  status.assign(static_cast<std::size_t>(std::max<int64_t>(n, 0)), SimUnitOut{});
  if (n <= 0) return;
  auto& ctx = context();
  cudaStream_t s = ctx.stream;
  std::vector<SimConfig> cfgs = cfgs_in;
  for (auto& c : cfgs) {  // predict_batch on the whole composition: no microbatches, no tp scaling
    c.pp = 1;
    c.tp = 1;
    c.cpu_overhead = 0.0;
  }
  int64_t MB = 1;
  for (int64_t c = 0; c < n; ++c) {
    const int64_t np = p_off[c + 1] - p_off[c], nd = d_off[c + 1] - d_off[c];
    require(np + nd > 0, "predict_batch: empty batch");
    for (int64_t k = p_off[c]; k < p_off[c + 1]; ++k)
      require(p_len[k] > 0, "equivalent_prefill_length: lengths must be positive");
    MB = std::max<int64_t>(MB, std::max(np, nd));
  }
  internal_check(MB < (1 << 24), "predict_batch: composition too large");
  const int64_t stride = 6 * MB + 2 + 4;
  std::vector<int32_t> ws(static_cast<std::size_t>(stride * n), 0), np_nd(2 * n);
  for (int64_t c = 0; c < n; ++c) {
    int32_t* w = ws.data() + c * stride;
    const int64_t np = p_off[c + 1] - p_off[c], nd = d_off[c + 1] - d_off[c];
    np_nd[2 * c] = static_cast<int32_t>(np);
    np_nd[2 * c + 1] = static_cast<int32_t>(nd);
    int32_t* pc = w + MB + 2 + MB;  // P_CHUNK = P_IDX + MB, P_IDX = MB + WC
    for (int64_t k = 0; k < np; ++k) {
      require(p_len[p_off[c] + k] < INT32_MAX && p_prior[p_off[c] + k] < INT32_MAX &&
                  p_prior[p_off[c] + k] >= 0,
              "ssg: prefill entry outside the device engine range");
      pc[k] = static_cast<int32_t>(p_len[p_off[c] + k]);
      pc[MB + k] = static_cast<int32_t>(p_prior[p_off[c] + k]);
    }
    int32_t* dc = w + MB + 2 + 4 * MB;  // D_CTX = P_IDX + 4 MB
    for (int64_t k = 0; k < nd; ++k) {
      require(d_ctx[d_off[c] + k] >= 0 && d_ctx[d_off[c] + k] < INT32_MAX,
              "ssg: decode context outside the device engine range");
      dc[k] = static_cast<int32_t>(d_ctx[d_off[c] + k]);
    }
  }
  DeviceBuffer<SimConfig> d_cfg;
  DeviceBuffer<SsgEstView> d_est;
  DeviceBuffer<int32_t> d_ws, d_npnd, d_cc;
  DeviceBuffer<double> d_sec, d_fl;
  DeviceBuffer<SimUnitOut> d_out;
  d_cfg.upload(cfgs, s);
  d_est.upload(ests, s);
  d_cc.upload(comp_cfg, s);
  d_ws.upload(ws, s);
  d_npnd.upload(np_nd, s);
  d_sec.resize(n);
  d_fl.resize(n);
  d_out.resize(n);
  const int64_t blocks = (n + SSG_SIM_WARPS - 1) / SSG_SIM_WARPS;
  if (context().math_fma)
    ssgk::k_predict_batch<1><<<(unsigned)blocks, SSG_SIM_WARPS * 32, 0, s>>>(
        d_cfg.ptr, d_est.ptr, d_cc.ptr, n, static_cast<int32_t>(MB), d_ws.ptr, d_npnd.ptr, d_sec.ptr,
        d_fl.ptr, d_out.ptr);
  else
    ssgk::k_predict_batch<0><<<(unsigned)blocks, SSG_SIM_WARPS * 32, 0, s>>>(
        d_cfg.ptr, d_est.ptr, d_cc.ptr, n, static_cast<int32_t>(MB), d_ws.ptr, d_npnd.ptr, d_sec.ptr,
        d_fl.ptr, d_out.ptr);
  cuda_check(cudaGetLastError(), "k_predict_batch launch");
  stats().launches_batch += 1;
  d_out.download(status.data(), n, s);
  d_sec.download(seconds, n, s);
  d_fl.download(flops, n, s);
  cuda_check(cudaStreamSynchronize(s), "predict_batch");
}

void predict_batches(const servesim::EstimatorModel& est, const SimConfig& cfg_in, int64_t n,
                     const int64_t* p_off, const int64_t* p_len, const int64_t* p_prior,
                     const int64_t* d_off, const int64_t* d_ctx, double* seconds, double* flops) {
  SimConfig cfg = cfg_in;
  cfg.est = 0;
  std::vector<SimUnitOut> status;
  predict_batches_multi({cfg}, {est.device().view}, std::vector<int32_t>(n, 0), n, p_off, p_len,
                        p_prior, d_off, d_ctx, seconds, flops, status);
  for (int64_t c = 0; c < n; ++c)
    if (status[c].code != SSG_OK) raise_unit_error(status[c], cfg, est);
}

}  // namespace ssg
