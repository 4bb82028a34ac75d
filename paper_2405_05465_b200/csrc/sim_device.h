// sim_device.h -- POD layouts of the replica-simulation engine (engine.cu).
//
// A "unit" is what one warp simulates: R_u replicas of one cluster config over
// a request stream.  Round-robin clusters are split into R independent
// single-replica units (replica r owns arrivals r, r+R, ... -- the reference's
// RR router hands them out in exactly that order, scheduler.hpp:506-510);
// least-outstanding / deferred routing couple replicas and run as one unit.
#pragma once
#include <stdint.h>

// SchedulerPolicy order (scheduler.hpp:20)
#define SSG_POL_FT 0
#define SSG_POL_ORCA 1
#define SSG_POL_VLLM 2
#define SSG_POL_SARATHI 3
#define SSG_POL_LIGHTLLM 4
// RoutingPolicy order (scheduler.hpp:21)
#define SSG_ROUTE_RR 0
#define SSG_ROUTE_LO 1
#define SSG_ROUTE_DEFERRED 2
// OpClass order (model_spec.hpp:49)
#define SSG_CLS_TOKEN 0
#define SSG_CLS_SEQ 1
#define SSG_CLS_COMM 2

#define SSG_MAX_OPS 11
#define SSG_MAX_PP 16  // microbatch m uses lanes 2m, 2m + 1 of the batch-latency step; deeper
                       // pipelines take the general latency path with per-unit scratch in HBM
// int32 words of per-unit microbatch scratch (6 int64 sums + 4 doubles per
// microbatch) appended to a unit's workspace when pp exceeds the shared-memory
// scratch
#define SSG_PP_SCRATCH_WORDS(pp) ((pp) > SSG_MAX_PP ? 20LL * (pp) : 0LL)

// Unit flags
#define SSG_UF_EMISSIONS 1  // write per-token emission times (CSR)
#define SSG_UF_BATCH_LOG 2  // record every scheduled batch (SimObserver payload)
#define SSG_UF_ABORT 4      // capacity probe: stop once late schedules exceed the bound
#define SSG_UF_OBSERVER 8   // batch log carries the SimObserver's scheduler view (needs BATCH_LOG)
#define SSG_PH_N 16         // phase counters per unit of -DSSG_PHASE_CYCLES builds (engine.cuh)

#define SSG_TAB_ROWS 11     // token-table rows per table (see SimConfig)

// One operator of the per-stage operator set, with everything predict_batch /
// batch_device_flops need (estimator.hpp:294-380, op_cost.hpp:21-73).
struct SimOp {
  int32_t slot;   // estimator model slot
  int32_t cls;    // SSG_CLS_*
  int32_t op;     // OpName
  int32_t flop_kind;  // 0 matmul, 1 act_fn, 2 add_norm, 3 attn prefill, 4 attn decode, 5 none
  double count;   // double(d.count)
  double kvb;     // 2.0 * e * double(kv_heads_per_device * head_dim)
  double payload; // double(payload_bytes_per_token)
  double fa, fb;  // flop operands: matmul in/out, act/add_norm in, attention hq
  int64_t qbytes; // algorithmic bytes of one prediction of this op's model
};

struct SimConfig {
  int32_t policy, max_batch, max_tokens, chunk;
  int32_t token_granular, pp, tp, est;
  int64_t block_size;
  int64_t total_units, watermark_units;
  double cpu_overhead;
  int32_t nops, routing, defer_threshold, tab_stride;  // tab_stride: entries per table array
  // Token tables (predict_batch terms that depend only on the microbatch's
  // token count t, precomputed by the same device code for t in [1, tab_tmax]):
  //   S6[t] = fp64 sum of count*pred over the token-level ops, in op order
  //   F6[t] = same for their flops;  C_k[t] = count*pred of the k-th comm op
  //   P0[t], P0F[t] = prefill attention at n_eq = t with no prior context
  //   DF[t], DL[t] / PF[t], PL[t] = the interp cell (clamped fraction, lower
  //     index as a double) along axis 0 of the decode / prefill attention model
  //     at v0 = t, i.e. ssg_axis_cell(log1p(t)) -- only when tab_cells is set
  // Layout at `tab_off` in the table pool: S6 | F6 | C0 | C1 | C2 | P0 | P0F |
  // DF | DL | PF | PL, each tab_stride doubles.  tab_off < 0: no tables (full path).
  int64_t tab_off;
  int32_t tab_tmax;   // every token op and comm op is valid for t <= tab_tmax
  int32_t tab_pmax;   // prefill attention at prior 0 is valid for n_eq <= tab_pmax
  // derived once on the host (fill_sim_ops) so the per-batch path never scans ops
  int32_t idx_pre, idx_dec;  // op indices of attention prefill / decode (-1 if absent)
  int32_t ncomm, bs_shift;   // comm ops (<= 3); log2(block_size) if a power of two, else -1
  int32_t tab_cells;         // DF/DL/PF/PL rows valid: both attention models are 2-D interp
  int32_t tab_pad;
  uint64_t bs_magic;         // ceil(2^64 / block_size) when it is not a power of two
  int64_t qb_fixed;          // qbytes of token + comm ops (queried every non-empty microbatch)
  int64_t qb_pre, qb_dec;    // qbytes of the attention queries
  SimOp ops[SSG_MAX_OPS];
};

// Multiplier of the device's block count ceil(t / b) = mulhi(t + b - 1, magic)
// (engine.cuh units_for): 0 for one unit per token (token-granular LightLLM, or
// b = 1); 2^64 / b for a power of two (exact for every t); ceil(2^64 / b)
// otherwise (exact for t + b - 1 < 2^32).  Host only.
static inline uint64_t block_magic(int64_t block_size, bool token_granular) {
  if (token_granular || block_size <= 1) return 0;
  if ((block_size & (block_size - 1)) == 0) {
    int k = 0;
    while ((int64_t(1) << k) != block_size) ++k;
    return uint64_t(1) << (64 - k);
  }
  const unsigned __int128 one = static_cast<unsigned __int128>(1) << 64;
  return static_cast<uint64_t>(one / static_cast<uint64_t>(block_size)) + 1;
}

// Per-request hot state (32 B, one sector).  Indices are unit-local and
// ordered by (arrival, id), so "sorted by arrival then id" (scheduler.hpp:236)
// is plain integer order on the device.
struct __attribute__((aligned(16))) ReqHot {
  int32_t target;   // prefill_target
  int32_t done;     // prefill_done
  int32_t emitted;
  int32_t kv;       // kv_context
  int32_t held;     // KV units held (BlockManager::held_)
  int32_t planned;  // schedule serial that last planned it (planned_ set)
  int32_t decode;   // req.decode_tokens
  int32_t prefill;  // req.prefill_tokens
};

struct __attribute__((aligned(16))) ReqTimes {
  double arrival, first_sched, first_tok, completion;
};

struct SimUnit {
  int32_t config;
  int32_t n;          // requests in this unit
  int32_t R;          // replicas simulated together
  int32_t flags;
  int64_t req_off;    // into the request arena (ReqHot/ReqTimes/ids/...)
  int64_t ws_off;     // into the int32 workspace
  int64_t rep_off;    // into the RepState / RepOut arrays
  int32_t wait_cap;   // ring capacity, power of two > n
  int32_t abort_max_late;
  double abort_thr;
  int64_t log_off;    // into the batch-log arena (int64 words)
  int64_t log_cap;
  int32_t group;      // speculation group (a candidate's probes of one launch), -1: none
  int32_t rung;       // this probe's bit in its group's failure mask
  uint32_t kill;      // group failure bits that make this probe unnecessary
  int32_t mb_ws;      // workspace entries per queue / plan array: min(max_batch, n)
                      // (no replica ever runs or plans more than the unit's requests)
};

struct RepState {
  int32_t run_n, wait_head, wait_n, busy;
  int32_t ft_inflight, np, nd, outstanding;
  int64_t allocated;
  int64_t preemptions;
  double ev_time;
  uint64_t ev_seq;
  int32_t ev_kind;  // 0 none, 1 BatchStart, 2 BatchComplete
  int32_t pad;
  double busy_time;
  int64_t iterations, tokens;
  double peak_kv;
};

struct SimUnitOut {
  int32_t code;       // SSG_OK / SSG_ERR_*
  int32_t aborted;    // 1: probe stopped, late schedules exceeded the bound;
                      // 2: cancelled (the capacity replay cannot ask for it any more)
  int32_t late;       // late first-schedules counted (probe units)
  int32_t err_i32;    // error operand: op slot / replica
  int64_t err_i64[2]; // error operands: request id, needed units / feature index
  double err_f64;     // error operand: feature value
  double err_time;    // sim clock of the error
  double span;        // clock of the last event
  double flops;       // total_model_flops
  int64_t log_used;   // batch-log words written
  int64_t events;
  int64_t iterations; // batches executed (all replicas of the unit)
  int64_t entries;    // batch entries (prefill chunks + decodes)
  int64_t qbytes;     // algorithmic predictor bytes touched
  int64_t cycles;     // SM clock cycles the unit's warp ran (diagnostics)
};
