/* ssg.h -- C ABI of the B200 servesim hot path ("ssg" = servesim-gpu).
 *
 * Plain pointers and sizes only; no C++ or torch types cross this boundary.
 * Every entry point is synchronous on the library's own stream unless its
 * name ends in _device (those enqueue on the caller's stream and return).
 * Each entry point names the reference interface it replaces
 * (paths relative to /root/reference/proj/include/servesim/).
 *
 * Status codes (ssg_status.code and return value):
 *   0 SSG_STATUS_OK
 *   1 SSG_STATUS_INPUT     servesim::Error      -- bad input; message is the
 *                                                 reference's message verbatim
 *   2 SSG_STATUS_INTERNAL  servesim::InternalError (violated invariant)
 *   3 SSG_STATUS_CUDA      CUDA runtime failure (no device, launch error, OOM)
 * There is no CPU fallback: without a B200 every compute entry returns 3.
 */
#ifndef SSG_H
#define SSG_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SSG_STATUS_OK 0
#define SSG_STATUS_INPUT 1
#define SSG_STATUS_INTERNAL 2
#define SSG_STATUS_CUDA 3

typedef struct ssg_status {
  int32_t code;
  char message[4096];
} ssg_status;

typedef struct ssg_estimator ssg_estimator;

/* ---- runtime ------------------------------------------------------------ */
/* Selects the GPU and probes which glibc exp/log1p contraction this host's
 * libm runs (the device then reproduces exactly that one). */
int ssg_init(int device, ssg_status* st);
int ssg_shutdown(void);
/* 1 if the host libm is the FMA-contracted glibc variant, 0 if plain, -1 before init. */
int ssg_math_variant(void);
/* Self-check of the device libm restatement (glibc_math.h) against this
 * host's glibc: evaluates fn (0 = log1p, 1 = exp) on the GPU, with the libm
 * variant ssg_init selected, at every x_k = base + k * step, k in [0, n), and
 * counts the results whose bits differ from the host's std::log1p / std::exp.
 * The predictor's log1p inputs are integer multiples of one quantum per
 * feature (estimator.hpp:300-341), so a progression with base 0 covers a
 * feature's whole domain.  reference: estimator.hpp:120-122 (log1p, exp). */
int ssg_math_check(int fn, double base, double step, int64_t n, int64_t* mismatches,
                   double* first_bad_x, ssg_status* st);
/* Library build identifier (sm arch, git-independent). */
const char* ssg_version(void);
/* Frees any buffer this library returned (JSON/CSV text). */
void ssg_free(void* p);

/* ---- estimator (predictor plugin) --------------------------------------- */
/* EstimatorModel::from_json (estimator.hpp:158-177). */
int ssg_estimator_from_json(const char* json, size_t len, ssg_estimator** out, ssg_status* st);
/* generate_synthetic_profile + train (profiler.hpp:314-347, estimator.hpp:201-275):
 * regressor is "interp" or "forest"; tps lists the tp degrees to profile. */
int ssg_estimator_train(const char* model_spec_json, const char* device_json, const int64_t* tps,
                        size_t n_tps, const char* regressor, uint64_t seed, ssg_estimator** out,
                        ssg_status* st);
/* EstimatorModel::to_json (estimator.hpp:137-156); free *out with ssg_free. */
int ssg_estimator_to_json(const ssg_estimator* e, char** out, size_t* len, ssg_status* st);
void ssg_estimator_free(ssg_estimator* e);
/* Dense model slot of (op, tp) for the *_mixed/_device calls; -1 if untrained.
 * op follows servesim::OpName order (qkv_proj = 0 ... send_recv = 10). */
int32_t ssg_estimator_slot(const ssg_estimator* e, int32_t op, int64_t tp);
/* Bytes the estimator occupies in HBM (uploads on first call). */
int64_t ssg_estimator_device_bytes(const ssg_estimator* e, ssg_status* st);

/* EstimatorModel::predict (estimator.hpp:105-123) over n queries of one
 * (op, tp).  f0 = num_tokens | payload_bytes, f1 = kv_read_bytes (attention
 * only, else may be NULL).  HOST buffers; copies are part of the call.  On a
 * guard violation returns 1 with the reference's message for the
 * lowest-index failing query. */
int ssg_predict(const ssg_estimator* e, int32_t op, int64_t tp, size_t n, const double* f0,
                const double* f1, double* out, ssg_status* st);
/* Same over mixed models: slots[i] from ssg_estimator_slot. HOST buffers. */
int ssg_predict_mixed(const ssg_estimator* e, size_t n, const int32_t* slots, const double* f0,
                      const double* f1, double* out, ssg_status* st);
/* Device-pointer form, enqueued on `stream` (cudaStream_t, may be NULL for
 * the legacy stream).  d_slots may be NULL to use uniform_slot.  d_first_error
 * must hold ~0ull on entry and receives (index << 8 | code) of the first
 * failure. Returns after enqueueing. */
int ssg_predict_device(const ssg_estimator* e, size_t n, const int32_t* d_slots,
                       int32_t uniform_slot, const double* d_f0, const double* d_f1, double* d_out,
                       unsigned long long* d_first_error, void* stream, ssg_status* st);

/* predict_batch over many batch compositions (estimator.hpp:294-348), CSR
 * layout: composition c owns prefill entries [p_off[c], p_off[c+1]) of
 * (p_len, p_prior) and decode entries [d_off[c], d_off[c+1]) of d_ctx.  The
 * operator set is derive_operators(model, {tp, pp=1}) of `model_spec_json`.
 * Also returns batch_device_flops (estimator.hpp:353-380) when flops != NULL. */
int ssg_predict_batch(const ssg_estimator* e, const char* model_spec_json, int64_t tp, size_t n,
                      const int64_t* p_off, const int64_t* p_len, const int64_t* p_prior,
                      const int64_t* d_off, const int64_t* d_ctx, double* seconds,
                      double* flops, ssg_status* st);

/* ---- workload (host) ---------------------------------------------------- */
/* The inputs that feed simulations and probes, bit-identical to the
 * reference's libstdc++ draws.  Host code: these run once per trace. */
/* synth_trace (workload.hpp:213-247) from a DistConfig document
 * (parse_dist_config, workload.hpp:169-210): n request lengths, ids 0..n-1. */
int ssg_synth_trace(const char* dist_json, size_t n, uint64_t seed, int64_t* prefill,
                    int64_t* decode, ssg_status* st);
/* poisson_arrivals (workload.hpp:93-104): the arrival times of n requests. */
int ssg_poisson_arrivals(size_t n, double rate_qps, uint64_t seed, double* arrivals,
                         ssg_status* st);
/* cap_total_length (workload.hpp:109-121), in place over n requests. */
int ssg_cap_total_length(size_t n, int64_t* prefill, int64_t* decode, int64_t max_total,
                         ssg_status* st);
/* load_trace (workload.hpp:33-78) of CSV text: *out receives JSON
 * {"id": [...], "arrival": [...] | null, "prefill": [...], "decode": [...]}
 * in the reference's order (stable-sorted by arrival); free with ssg_free. */
int ssg_load_trace(const char* csv_text, char** out, ssg_status* st);

/* ---- engine ------------------------------------------------------------ */
/* run_simulation + build_report (sim.hpp:135-320, metrics.hpp:106-126) of one
 * cluster over one trace (arrays in trace order).  cluster_json is a cluster
 * document with the model spec and device embedded:
 *   {"model_spec": {...}, "device": {...}, "parallelism": {...},
 *    "scheduler": {...}, "routing": {"policy": ...}, "cpu_overhead_per_iter": x}
 * abort_delay > 0 turns on the capacity-probe abort (SimOptions, sim.hpp:99-107).
 * *out receives a JSON document (requests, replicas, iterations, report, and
 * the per-batch log when record_batches); free with ssg_free. */
int ssg_simulate(const char* cluster_json, const ssg_estimator* e, size_t n, const int64_t* ids,
                 const double* arrivals, const int64_t* prefill, const int64_t* decode,
                 int record_batches, double abort_delay, size_t abort_max_late, int static_mode,
                 char** out, ssg_status* st);

/* MetricSummary (metrics.hpp:17-25) and the report of one simulation
 * (MetricsReport + ClusterMetrics, metrics.hpp:27-60) in fixed layout. */
typedef struct ssg_metric_summary {
  double mean, p50, p90, p95, p99;
} ssg_metric_summary;
typedef struct ssg_sim_report {
  double simulated_span, total_model_flops;
  int64_t num_devices;
  ssg_metric_summary scheduling_delay, ttft, tbt, e2e, normalized;
  double mfu, kv_utilization_peak, busy_fraction;
  int64_t preemptions;
} ssg_sim_report;
/* run_simulation + build_report (sim.hpp:135-320, metrics.hpp:106-126) with
 * binary outputs: the call a C/C++ caller makes (no JSON).  Per-request arrays
 * are in trace order and each may be NULL; emissions receives request i's
 * decode[i] emission times back to back in trace order (sum(decode) slots) or
 * may be NULL.  Errors as ssg_simulate; a run that hits the probe abort
 * returns status 1 with the reference's ProbeInfeasible message. */
int ssg_simulate_run(const char* cluster_json, const ssg_estimator* e, size_t n, const int64_t* ids,
                     const double* arrivals, const int64_t* prefill, const int64_t* decode,
                     int static_mode, double* first_scheduled, double* first_token,
                     double* completion, int64_t* restarts, double* emissions,
                     ssg_sim_report* report, ssg_status* st);

/* ---- search (Vidur-Search) --------------------------------------------- */
/* One evaluated candidate, fixed-size so shards can be all-gathered as bytes.
 * Fields as ConfigResult (search.hpp:182-194); `index` is the enumeration
 * position (enumerate_configs order, search.hpp:76-129). */
typedef struct ssg_config_record {
  int64_t index;
  double capacity_qps, qps_per_dollar, ttft_p90, tbt_p99, delay_p99, makespan;
  int32_t slo_pass;
  int32_t reserved;
  char error[960];
} ssg_config_record;

size_t ssg_search_record_size(void);
/* load_search_config + run_search + writers (config.hpp:111, search.hpp:369-486)
 * over the whole grid: shard must be 0 and num_shards 1 (else status 1 --
 * shards go through ssg_search_shard + ssg_search_finalize).
 * *out: JSON {results_csv, frontier_ttft_csv, frontier_tbt_csv, summary,
 * configs, best}; free with ssg_free. */
int ssg_search(const char* config_path, int shard, int num_shards, char** out, ssg_status* st);
/* Evaluates this shard's configs into `records`.  The capacity objective
 * assigns configs to shards by a longest-processing-time split on their
 * initial QPS guesses (the same on every rank, so the shards partition the
 * grid); the makespan objective strides i % num_shards.  A shard may hold any
 * number of configs up to N: capacity >= N is always enough, and *count is
 * the number written.  Each record carries its enumeration index. */
int ssg_search_shard(const char* config_path, int shard, int num_shards, ssg_config_record* records,
                     size_t capacity, size_t* count, ssg_status* st);
/* Ranking, Pareto frontiers and writers over the gathered records of every
 * shard (search.hpp:395-486); byte-identical to the single-GPU outcome. */
int ssg_search_finalize(const char* config_path, const ssg_config_record* records, size_t n,
                        char** out, ssg_status* st);

/* A prepared sweep (SearchSession): config loaded, estimators trained and
 * resident in HBM, probe workload built.  ssg_search_run evaluates this
 * shard's configs (the timed hot path) and may be called repeatedly. */
typedef struct ssg_search_session ssg_search_session;
int ssg_search_open(const char* config_path, ssg_search_session** out, ssg_status* st);
int ssg_search_run(ssg_search_session* s, int shard, int num_shards, ssg_config_record* records,
                   size_t capacity, size_t* count, ssg_status* st);
int64_t ssg_search_num_configs(const ssg_search_session* s);
void ssg_search_close(ssg_search_session* s);

/* ---- counters over the library's kernels (bench / roofline evidence) ----- */
typedef struct ssg_run_stats {
  int64_t launches_simulate, launches_select, launches_predict, launches_batch;
  int64_t units, iterations, entries, events;
  int64_t predictor_bytes; /* algorithmic predictor bytes */
  int64_t entry_bytes;     /* 48 B per batch entry (request progress r/w) */
  int64_t queries;         /* k_predict queries */
  double simulate_ms;      /* k_simulate device time (CUDA events, library stream) */
  int64_t h2d_bytes, d2h_bytes; /* host<->device copies issued by the library */
  int64_t launches_setup;  /* probe-stream setup and SLO sample kernels */
  double simulate_busy_ms; /* union of k_simulate intervals: sweep launches of candidate groups
                              overlap on separate streams, so this is <= simulate_ms */
  /* the sweep work the sequential reference search would do: the probes its
     find_capacity replay asks for plus each SLO / static run (the rest of
     iterations / entries is speculation) */
  int64_t useful_iterations, useful_entries, useful_bytes;
  int64_t cancelled_probes; /* speculative probes stopped once a lower rate of their candidate failed */
  /* SLO runs taken in the round that settles a capacity, one per capacity it can end
     with; spec_slo_used of them are the runs the sequential search makes next */
  int64_t spec_slo_runs, spec_slo_used;
} ssg_run_stats;
void ssg_stats_reset(void);
void ssg_stats_get(ssg_run_stats* out);

#ifdef __cplusplus
}
#endif
#endif /* SSG_H */
