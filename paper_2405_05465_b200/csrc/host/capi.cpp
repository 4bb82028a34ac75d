// capi.cpp -- the extern "C" boundary (include/ssg.h) over the C++ drop-in API.
//
// Exceptions never cross the ABI: servesim::Error -> 1 (message verbatim),
// InternalError -> 2, CUDA failures -> 3.
#include "ssg.h"

#include <cmath>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <functional>
#include <memory>
#include <vector>

#include "json.hpp"
#include "runtime.h"
#include "servesim_b200.hpp"
#include "sim_host.h"
#include "sweep.h"

using namespace servesim;

namespace servesim {
ClusterConfig parse_cluster_inline(const std::string& text);  // config.cpp
}

struct ssg_estimator {
  EstimatorModel model;
};

namespace ssg {
void launch_predict(const DeviceEstimator& de, int64_t n, const int32_t* slots, int32_t uniform,
                    const double* f0, const double* f1, double* out,
                    unsigned long long* first_error, cudaStream_t s,
                    unsigned long long* invalid = nullptr, unsigned long long* flag_f1 = nullptr);
[[noreturn]] void raise_predict_error(const EstimatorModel& est, unsigned long long word,
                                      const int32_t* slots_host, int32_t uniform,
                                      const double* f0_host, const double* f1_host);
}  // namespace ssg

namespace {

void set_status(ssg_status* st, int code, const char* msg) {
  if (!st) return;
  st->code = code;
  std::strncpy(st->message, msg ? msg : "", sizeof(st->message) - 1);
  st->message[sizeof(st->message) - 1] = '\0';
}

int guarded(ssg_status* st, const std::function<void()>& body) {
  try {
    body();
    set_status(st, SSG_STATUS_OK, "");
    return SSG_STATUS_OK;
  } catch (const Error& e) {
    set_status(st, SSG_STATUS_INPUT, e.what());
    return SSG_STATUS_INPUT;
  } catch (const ssg::CudaError& e) {
    set_status(st, SSG_STATUS_CUDA, e.what());
    return SSG_STATUS_CUDA;
  } catch (const InternalError& e) {
    set_status(st, SSG_STATUS_INTERNAL, e.what());
    return SSG_STATUS_INTERNAL;
  } catch (const std::exception& e) {
    set_status(st, SSG_STATUS_INTERNAL, e.what());
    return SSG_STATUS_INTERNAL;
  }
}

char* dup_text(const std::string& s, size_t* len) {
  char* p = static_cast<char*>(std::malloc(s.size() + 1));
  if (!p) throw InternalError("out of host memory");
  std::memcpy(p, s.data(), s.size());
  p[s.size()] = '\0';
  if (len) *len = s.size();
  return p;
}

// Grow-only staging buffers for the host-buffer entry points.
struct Staging {
  ssg::DeviceBuffer<int32_t> slots;
  ssg::DeviceBuffer<double> f0, f1, out;
  ssg::DeviceBuffer<unsigned long long> err;
  cudaStream_t side[2] = {nullptr, nullptr};  // chunk streams besides the context stream
  cudaEvent_t ready = nullptr;
};
Staging& staging() {
  static Staging s;
  return s;
}

bool pinned(const void* p) {
  if (!p) return true;
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeHost;
}

// Host-buffer predictions.  From pinned host memory the queries stream through
// in chunks on three streams, so chunk k's copy-in, chunk k-1's kernel and
// chunk k-2's copy-out overlap (PCIe both ways and the SMs at once); pageable
// buffers take one copy-in, one launch, one copy-out.  Slot validation runs in
// the kernel (validate), and errors are raised in the reference's order: an
// invalid slot first, then a missing second feature, then the first failing
// query.
void predict_host(const EstimatorModel& est, size_t n, const int32_t* slots, int32_t uniform,
                  const double* f0, const double* f1, double* out, bool validate) {
  if (n == 0) return;
  // one staging set per process: concurrent host-buffer predictions serialise
  static std::mutex mu;
  std::lock_guard<std::mutex> lk(mu);
  const auto& de = est.device();
  auto& ctx = ssg::context();
  auto& S = staging();
  if (!S.ready) {
    for (auto& x : S.side)
      ssg::cuda_check(cudaStreamCreateWithFlags(&x, cudaStreamNonBlocking), "predict stream");
    ssg::cuda_check(cudaEventCreateWithFlags(&S.ready, cudaEventDisableTiming), "event");
  }
  const bool chunked = n > (1u << 20) && pinned(f0) && pinned(f1) && pinned(out) && pinned(slots);
  const size_t chunk = chunked ? (size_t(1) << 20) : n;
  const size_t nch = (n + chunk - 1) / chunk;
  cudaStream_t s0 = ctx.stream;
  if (slots) S.slots.resize(n);
  S.f0.resize(n);
  if (f1) S.f1.resize(n);
  S.out.resize(n);
  // per chunk: first failing query, first invalid slot; then the missing-f1 flag
  S.err.resize(2 * nch + 1);
  ssg::cuda_check(cudaMemsetAsync(S.err.ptr, 0xff, 2 * nch * sizeof(unsigned long long), s0), "memset");
  ssg::cuda_check(cudaMemsetAsync(S.err.ptr + 2 * nch, 0, sizeof(unsigned long long), s0), "memset");
  ssg::cuda_check(cudaEventRecord(S.ready, s0), "event");
  cudaStream_t streams[3] = {s0, S.side[0], S.side[1]};
  for (int k = 1; k < 3; ++k) ssg::cuda_check(cudaStreamWaitEvent(streams[k], S.ready, 0), "wait");
  auto h2d = [&](void* d, const void* h, size_t bytes, cudaStream_t st) {
    ssg::cuda_check(cudaMemcpyAsync(d, h, bytes, cudaMemcpyHostToDevice, st), "H2D");
    ssg::stats().h2d_bytes += static_cast<int64_t>(bytes);
  };
  for (size_t c = 0; c < nch; ++c) {
    cudaStream_t st = streams[c % 3];
    const size_t b = c * chunk, m = std::min(chunk, n - b);
    if (slots) h2d(S.slots.ptr + b, slots + b, m * sizeof(int32_t), st);
    h2d(S.f0.ptr + b, f0 + b, m * sizeof(double), st);
    if (f1) h2d(S.f1.ptr + b, f1 + b, m * sizeof(double), st);
    ssg::launch_predict(de, static_cast<int64_t>(m), slots ? S.slots.ptr + b : nullptr, uniform,
                        S.f0.ptr + b, f1 ? S.f1.ptr + b : nullptr, S.out.ptr + b, S.err.ptr + c, st,
                        validate ? S.err.ptr + nch + c : nullptr, S.err.ptr + 2 * nch);
    ssg::cuda_check(cudaMemcpyAsync(out + b, S.out.ptr + b, m * sizeof(double), cudaMemcpyDeviceToHost, st),
                    "D2H");
    ssg::stats().d2h_bytes += static_cast<int64_t>(m * sizeof(double));
  }
  std::vector<unsigned long long> words(2 * nch + 1);
  for (int k = 1; k < 3; ++k) {
    ssg::cuda_check(cudaEventRecord(S.ready, streams[k]), "event");
    ssg::cuda_check(cudaStreamWaitEvent(s0, S.ready, 0), "wait");
  }
  ssg::cuda_check(cudaMemcpyAsync(words.data(), S.err.ptr, words.size() * sizeof(unsigned long long),
                                  cudaMemcpyDeviceToHost, s0), "D2H");
  ssg::cuda_check(cudaStreamSynchronize(s0), "predict");
  for (size_t c = 0; validate && c < nch; ++c)  // chunk-local index, re-based
    if (words[nch + c] != SSG_NO_ERROR)
      throw Error("predict: query " + std::to_string(words[nch + c] + c * chunk) +
                  " has no trained model slot");
  if (validate && words[2 * nch] != 0) throw Error("predict: two-feature models need f1");
  for (size_t c = 0; c < nch; ++c) {
    if (words[c] == SSG_NO_ERROR) continue;
    // re-base the chunk-local query index
    const unsigned long long word = ((words[c] >> 8) + c * chunk) << 8 | (words[c] & 0xff);
    ssg::raise_predict_error(est, word, slots, uniform, f0, f1);
  }
}

}  // namespace

extern "C" {

int ssg_init(int device, ssg_status* st) {
  return guarded(st, [&] { ssg::init_context(device); });
}

int ssg_shutdown(void) {
  ssg::release_sweep_lanes();
  ssg::shutdown_context();
  return SSG_STATUS_OK;
}

int ssg_math_check(int fn, double base, double step, int64_t n, int64_t* mismatches,
                   double* first_bad_x, ssg_status* st) {
  return guarded(st, [&] {
    require(fn == 0 || fn == 1, "ssg_math_check: fn must be 0 (log1p) or 1 (exp)");
    require(n >= 0, "ssg_math_check: n must be >= 0");
    auto& ctx = ssg::context();
    const int variant = ctx.math_fma;
    const int64_t chunk = int64_t(1) << 24;
    ssg::DeviceBuffer<double> d(static_cast<std::size_t>(std::min(n, chunk) + 1));
    std::vector<double> dev(static_cast<std::size_t>(std::min(n, chunk) + 1));
    int64_t bad = 0;
    double first = std::nan("");
    for (int64_t k0 = 0; k0 < n; k0 += chunk) {
      const int64_t m = std::min(chunk, n - k0);
      ssg::launch_math_eval(fn, variant, base, step, k0, m, d.ptr, ctx.stream);
      d.download(dev.data(), m, ctx.stream);
      ssg::cuda_check(cudaStreamSynchronize(ctx.stream), "math check");
      for (int64_t i = 0; i < m; ++i) {
        // the same x as the device: base + k * step, two roundings, no contraction
        const double x = base + static_cast<double>(k0 + i) * step;
        const double h = fn == 0 ? std::log1p(x) : std::exp(x);
        const bool dev_nan = std::isnan(dev[i]);
        if ((fn == 1 && dev_nan) || std::memcmp(&h, &dev[i], sizeof h) != 0) {
          if (fn == 1 && dev_nan && !(std::fabs(x) < 512.0)) continue;  // outside the guarded range
          if (bad == 0) first = x;
          ++bad;
        }
      }
    }
    *mismatches = bad;
    if (first_bad_x) *first_bad_x = first;
  });
}

int ssg_math_variant(void) {
  try {
    return ssg::probe_host_math_variant();
  } catch (...) {
    return -1;
  }
}

const char* ssg_version(void) { return "ssg 0.1 sm_100a"; }

void ssg_free(void* p) { std::free(p); }

int ssg_estimator_from_json(const char* json, size_t len, ssg_estimator** out, ssg_status* st) {
  return guarded(st, [&] {
    nlohmann::json doc;
    try {
      doc = nlohmann::json::parse(std::string(json, len));
    } catch (const nlohmann::json::exception& ex) {
      throw Error(std::string("estimator file: invalid JSON: ") + ex.what());
    }
    auto* e = new ssg_estimator{EstimatorModel::from_json(doc)};
    *out = e;
  });
}

int ssg_estimator_train(const char* model_spec_json, const char* device_json, const int64_t* tps,
                        size_t n_tps, const char* regressor, uint64_t seed, ssg_estimator** out,
                        ssg_status* st) {
  return guarded(st, [&] {
    ModelSpec spec = parse_model_spec(model_spec_json);
    DeviceProfile dev = parse_device_profile(device_json);
    std::vector<std::int64_t> tp(tps, tps + n_tps);
    TrainConfig cfg;
    cfg.seed = seed;
    cfg.regressor = regressor ? regressor : "interp";
    std::vector<ProfileRecord> profile;
    {
      ssg::PhaseTimer t("train: synthetic profile");
      profile = generate_synthetic_profile(spec, dev, tp);
    }
    ssg::PhaseTimer t("train: fit");
    auto* e = new ssg_estimator{train(profile, cfg)};
    *out = e;
  });
}

int ssg_estimator_to_json(const ssg_estimator* e, char** out, size_t* len, ssg_status* st) {
  return guarded(st, [&] { *out = dup_text(e->model.to_json().dump(), len); });
}

void ssg_estimator_free(ssg_estimator* e) { delete e; }

int32_t ssg_estimator_slot(const ssg_estimator* e, int32_t op, int64_t tp) {
  try {
    return e->model.device().slot(static_cast<OpName>(op), tp);
  } catch (...) {
    return -1;
  }
}

int64_t ssg_estimator_device_bytes(const ssg_estimator* e, ssg_status* st) {
  int64_t b = -1;
  guarded(st, [&] { b = static_cast<int64_t>(e->model.device().bytes); });
  return b;
}

int ssg_predict(const ssg_estimator* e, int32_t op, int64_t tp, size_t n, const double* f0,
                const double* f1, double* out, ssg_status* st) {
  return guarded(st, [&] {
    const auto& m = e->model.find(static_cast<OpName>(op), tp);
    require(m.schema.size() == 1 || f1 != nullptr,
            "estimator: query for " + to_string(OpModelKey{static_cast<OpName>(op), tp}) +
                " missing feature " + m.schema.back());
    const int32_t slot = e->model.device().slot(static_cast<OpName>(op), tp);
    predict_host(e->model, n, nullptr, slot, f0, m.schema.size() > 1 ? f1 : nullptr, out, false);
  });
}

int ssg_predict_mixed(const ssg_estimator* e, size_t n, const int32_t* slots, const double* f0,
                      const double* f1, double* out, ssg_status* st) {
  return guarded(st, [&] {
    predict_host(e->model, n, slots, 0, f0, f1, out, true);
  });
}

int ssg_predict_device(const ssg_estimator* e, size_t n, const int32_t* d_slots,
                       int32_t uniform_slot, const double* d_f0, const double* d_f1, double* d_out,
                       unsigned long long* d_first_error, void* stream, ssg_status* st) {
  return guarded(st, [&] {
    const auto& de = e->model.device();
    require(d_slots || (uniform_slot >= 0 && uniform_slot < de.view.nmodels),
            "predict: invalid model slot");
    ssg::launch_predict(de, static_cast<int64_t>(n), d_slots, uniform_slot, d_f0, d_f1, d_out,
                        d_first_error, static_cast<cudaStream_t>(stream));
  });
}

int ssg_predict_batch(const ssg_estimator* e, const char* model_spec_json, int64_t tp, size_t n,
                      const int64_t* p_off, const int64_t* p_len, const int64_t* p_prior,
                      const int64_t* d_off, const int64_t* d_ctx, double* seconds, double* flops,
                      ssg_status* st) {
  return guarded(st, [&] {
    ModelSpec spec = parse_model_spec(model_spec_json);
    auto ops = derive_operators(spec, ParallelismConfig{tp, 1, 1});
    for (const auto& d : ops) e->model.find(d.op, d.tp_degree);
    SimConfig cfg{};
    ssg::fill_sim_ops(cfg, ops, e->model.device());
    std::vector<double> fl(n);
    ssg::predict_batches(e->model, cfg, static_cast<int64_t>(n), p_off, p_len, p_prior, d_off, d_ctx,
                         seconds, flops ? flops : fl.data());
  });
}

int ssg_simulate(const char* cluster_json, const ssg_estimator* e, size_t n, const int64_t* ids,
                 const double* arrivals, const int64_t* prefill, const int64_t* decode,
                 int record_batches, double abort_delay, size_t abort_max_late, int static_mode,
                 char** out, ssg_status* st) {
  return guarded(st, [&] {
    ClusterConfig cluster = parse_cluster_inline(cluster_json);
    std::vector<Request> trace(n);
    for (size_t i = 0; i < n; ++i) trace[i] = Request{ids[i], arrivals[i], prefill[i], decode[i]};
    SimOptions o;
    o.record_iterations = true;
    o.record_batches = record_batches != 0;
    o.abort_delay_threshold = abort_delay;
    o.abort_max_late = abort_max_late;
    nlohmann::json j;
    SimulationOutput so;
    try {
      so = run_simulation_logged(cluster, trace, e->model, o);
    } catch (const ProbeInfeasible&) {
      j["probe_infeasible"] = true;
      *out = dup_text(j.dump(), nullptr);
      return;
    }
    const SimulationResult& r = so.result;
    ssg::PhaseTimer timer("ssg_simulate: json");
    nlohmann::json reqs = nlohmann::json::array();
    for (const auto& q : r.requests)
      reqs.push_back({{"id", q.id},
                      {"arrival", q.arrival},
                      {"first_scheduled", q.first_scheduled},
                      {"first_token", q.first_token},
                      {"completion", q.completion},
                      {"restarts", q.restarts},
                      {"emissions", q.emission_times}});
    nlohmann::json reps = nlohmann::json::array();
    for (const auto& a : r.replicas)
      reps.push_back({{"busy_time", a.busy_time},
                      {"iterations", a.iterations},
                      {"tokens_processed", a.tokens_processed},
                      {"peak_kv_utilization", a.peak_kv_utilization},
                      {"preemptions", a.preemptions}});
    nlohmann::json iters = nlohmann::json::array();
    for (const auto& it : r.iterations)
      iters.push_back({it.start, it.latency, it.replica, it.batch_requests, it.current_tokens,
                       it.prefill_entries, it.decode_entries, it.kv_utilization});
    auto rep = build_report(r, static_mode != 0);
    auto summ = [](const MetricSummary& s) {
      return nlohmann::json{{"mean", s.mean}, {"p50", s.p50}, {"p90", s.p90}, {"p95", s.p95}, {"p99", s.p99}};
    };
    j["requests"] = std::move(reqs);
    j["replicas"] = std::move(reps);
    j["iterations"] = std::move(iters);
    j["simulated_span"] = r.simulated_span;
    j["total_model_flops"] = r.total_model_flops;
    j["num_devices"] = r.num_devices;
    j["report"] = {{"scheduling_delay", summ(rep.scheduling_delay)},
                   {"ttft", summ(rep.ttft)},
                   {"tbt", summ(rep.tbt)},
                   {"e2e", summ(rep.e2e)},
                   {"normalized", summ(rep.normalized)},
                   {"mfu", rep.cluster.mfu},
                   {"kv_utilization_peak", rep.cluster.kv_utilization_peak},
                   {"busy_fraction", rep.cluster.busy_fraction},
                   {"preemptions", rep.cluster.preemptions}};
    j["requests_csv"] = request_metrics_to_csv(rep);
    if (record_batches) {
      nlohmann::json log = nlohmann::json::array();
      for (const auto& b : so.batches) {
        nlohmann::json ent = nlohmann::json::array();
        for (const auto& en : b.entries) ent.push_back({en.prefill ? 1 : 0, en.request_id, en.tokens, en.context});
        log.push_back({{"replica", b.replica}, {"now", b.now}, {"kv", b.kv_allocated_units}, {"entries", ent}});
      }
      j["batches"] = std::move(log);
    }
    *out = dup_text(j.dump(), nullptr);
  });
}

int ssg_synth_trace(const char* dist_json, size_t n, uint64_t seed, int64_t* prefill,
                    int64_t* decode, ssg_status* st) {
  return guarded(st, [&] {
    const auto reqs = synth_trace(parse_dist_config_text(dist_json), n, seed);
    for (size_t i = 0; i < n; ++i) {
      prefill[i] = reqs[i].prefill_tokens;
      decode[i] = reqs[i].decode_tokens;
    }
  });
}

int ssg_poisson_arrivals(size_t n, double rate_qps, uint64_t seed, double* arrivals, ssg_status* st) {
  return guarded(st, [&] {
    const auto reqs = poisson_arrivals(std::vector<Request>(n), rate_qps, seed);
    for (size_t i = 0; i < n; ++i) arrivals[i] = reqs[i].arrival_time;
  });
}

int ssg_cap_total_length(size_t n, int64_t* prefill, int64_t* decode, int64_t max_total,
                         ssg_status* st) {
  return guarded(st, [&] {
    std::vector<Request> reqs(n);
    for (size_t i = 0; i < n; ++i) {
      reqs[i].prefill_tokens = prefill[i];
      reqs[i].decode_tokens = decode[i];
    }
    reqs = cap_total_length(std::move(reqs), max_total);
    for (size_t i = 0; i < n; ++i) {
      prefill[i] = reqs[i].prefill_tokens;
      decode[i] = reqs[i].decode_tokens;
    }
  });
}

int ssg_load_trace(const char* csv_text, char** out, ssg_status* st) {
  return guarded(st, [&] {
    const auto reqs = load_trace(csv_text);
    nlohmann::json j;
    std::vector<int64_t> id, pre, dec;
    std::vector<double> arr;
    for (const auto& r : reqs) {
      id.push_back(r.id);
      pre.push_back(r.prefill_tokens);
      dec.push_back(r.decode_tokens);
      arr.push_back(r.arrival_time);
    }
    j["id"] = id;
    j["prefill"] = pre;
    j["decode"] = dec;
    if (!reqs.empty() && !std::isnan(reqs.front().arrival_time))
      j["arrival"] = arr;
    else
      j["arrival"] = nullptr;
    *out = dup_text(j.dump(), nullptr);
  });
}

int ssg_simulate_run(const char* cluster_json, const ssg_estimator* e, size_t n, const int64_t* ids,
                     const double* arrivals, const int64_t* prefill, const int64_t* decode,
                     int static_mode, double* first_scheduled, double* first_token,
                     double* completion, int64_t* restarts, double* emissions,
                     ssg_sim_report* report, ssg_status* st) {
  return guarded(st, [&] {
    ClusterConfig cluster = parse_cluster_inline(cluster_json);
    std::vector<Request> trace(n);
    for (size_t i = 0; i < n; ++i) trace[i] = Request{ids[i], arrivals[i], prefill[i], decode[i]};
    SimulationResult r;
    try {
      r = run_simulation(cluster, trace, e->model, SimOptions{});
    } catch (const ProbeInfeasible& p) {
      throw Error(p.what());
    }
    size_t at = 0;
    for (size_t i = 0; i < n; ++i) {
      const RequestRecord& q = r.requests[i];
      if (first_scheduled) first_scheduled[i] = q.first_scheduled;
      if (first_token) first_token[i] = q.first_token;
      if (completion) completion[i] = q.completion;
      if (restarts) restarts[i] = q.restarts;
      if (emissions) {
        std::memcpy(emissions + at, q.emission_times.data(), q.emission_times.size() * sizeof(double));
        at += q.emission_times.size();
      }
    }
    if (report) {
      const MetricsReport rep = build_report(r, static_mode != 0);
      auto put = [](ssg_metric_summary& d, const MetricSummary& m) {
        d = ssg_metric_summary{m.mean, m.p50, m.p90, m.p95, m.p99};
      };
      report->simulated_span = r.simulated_span;
      report->total_model_flops = r.total_model_flops;
      report->num_devices = r.num_devices;
      put(report->scheduling_delay, rep.scheduling_delay);
      put(report->ttft, rep.ttft);
      put(report->tbt, rep.tbt);
      put(report->e2e, rep.e2e);
      put(report->normalized, rep.normalized);
      report->mfu = rep.cluster.mfu;
      report->kv_utilization_peak = rep.cluster.kv_utilization_peak;
      report->busy_fraction = rep.cluster.busy_fraction;
      report->preemptions = static_cast<int64_t>(rep.cluster.preemptions);
    }
  });
}

size_t ssg_search_record_size(void) { return sizeof(ssg_config_record); }

namespace {

nlohmann::json outcome_json(const SearchOutcome& o, const std::string& objective) {
  nlohmann::json j;
  j["results_csv"] = search_results_to_csv(o);
  j["frontier_ttft_csv"] = frontier_to_csv(o, o.frontier_ttft, true);
  j["frontier_tbt_csv"] = frontier_to_csv(o, o.frontier_tbt, false);
  j["summary"] = search_summary_text(o, objective);
  j["configs"] = o.results.size();
  if (o.best) j["best"] = o.results[*o.best].config.id;
  return j;
}

}  // namespace

int ssg_search(const char* config_path, int shard, int num_shards, char** out, ssg_status* st) {
  return guarded(st, [&] {
    // one process, whole grid: shards are ssg_search_shard + ssg_search_finalize
    require(num_shards == 1 && shard == 0,
            "ssg_search: evaluates the whole grid (num_shards must be 1); shard with "
            "ssg_search_shard and merge with ssg_search_finalize");
    ssg::PhaseTimer timer("ssg_search_shard");
    auto cfg = load_search_config(config_path);
    auto results = evaluate_configs_shard(cfg.spec, cfg.workload, cfg.options, shard, num_shards);
    auto o = finalize_search(cfg.spec, cfg.options, std::move(results));
    *out = dup_text(outcome_json(o, cfg.options.objective).dump(), nullptr);
  });
}

namespace {
void to_records(const std::vector<ConfigResult>& results, const std::vector<size_t>& owned,
                ssg_config_record* records, size_t capacity, size_t* count) {
    size_t k = 0;
    for (size_t i : owned) {
      require(k < capacity, "ssg_search_shard: record buffer too small");
      const ConfigResult& r = results[i];
      ssg_config_record& rec = records[k++];
      std::memset(&rec, 0, sizeof rec);
      rec.index = static_cast<int64_t>(i);
      rec.capacity_qps = r.capacity_qps;
      rec.qps_per_dollar = r.qps_per_dollar;
      rec.ttft_p90 = r.ttft_p90;
      rec.tbt_p99 = r.tbt_p99;
      rec.delay_p99 = r.delay_p99;
      rec.makespan = r.makespan;
      rec.slo_pass = r.slo_pass ? 1 : 0;
      internal_check(r.error.size() < sizeof(rec.error), "error message longer than a record");
      std::memcpy(rec.error, r.error.data(), r.error.size());
    }
    *count = k;
}
}  // namespace

int ssg_search_shard(const char* config_path, int shard, int num_shards, ssg_config_record* records,
                     size_t capacity, size_t* count, ssg_status* st) {
  return guarded(st, [&] {
    require(num_shards >= 1 && shard >= 0 && shard < num_shards, "ssg_search_shard: bad shard");
    ssg::PhaseTimer timer("ssg_search_shard");
    auto cfg = [&] {
      ssg::PhaseTimer t("ssg_search_shard: load config");
      return load_search_config(config_path);
    }();
    std::vector<size_t> owned;
    auto results =
        evaluate_configs_shard(cfg.spec, cfg.workload, cfg.options, shard, num_shards, &owned);
    to_records(results, owned, records, capacity, count);
  });
}

struct ssg_search_session {
  std::unique_ptr<SearchSession> session;
};

int ssg_search_open(const char* config_path, ssg_search_session** out, ssg_status* st) {
  return guarded(st, [&] {
    auto cfg = load_search_config(config_path);
    auto* s = new ssg_search_session{std::make_unique<SearchSession>(cfg.spec, cfg.workload, cfg.options)};
    *out = s;
  });
}

int ssg_search_run(ssg_search_session* s, int shard, int num_shards, ssg_config_record* records,
                   size_t capacity, size_t* count, ssg_status* st) {
  return guarded(st, [&] {
    require(num_shards >= 1 && shard >= 0 && shard < num_shards, "ssg_search_run: bad shard");
    std::vector<size_t> owned;
    auto results = s->session->evaluate(shard, num_shards, &owned);
    to_records(results, owned, records, capacity, count);
  });
}

int64_t ssg_search_num_configs(const ssg_search_session* s) {
  return static_cast<int64_t>(s->session->num_configs());
}

void ssg_search_close(ssg_search_session* s) { delete s; }

void ssg_stats_reset(void) { ssg::stats() = ssg::RunStats{}; }

void ssg_stats_get(ssg_run_stats* out) {
  const ssg::RunStats& r = ssg::stats();
  out->launches_simulate = r.launches_simulate;
  out->launches_select = r.launches_select;
  out->launches_predict = r.launches_predict;
  out->launches_batch = r.launches_batch;
  out->units = r.units;
  out->iterations = r.iterations;
  out->entries = r.entries;
  out->events = r.events;
  out->predictor_bytes = r.predictor_bytes;
  out->entry_bytes = r.entry_bytes;
  out->queries = r.queries;
  out->simulate_ms = r.simulate_ms;
  out->h2d_bytes = r.h2d_bytes;
  out->launches_setup = r.launches_setup;
  out->d2h_bytes = r.d2h_bytes;
  out->simulate_busy_ms = r.simulate_busy_ms;
  out->useful_iterations = r.useful_iterations;
  out->useful_entries = r.useful_entries;
  out->useful_bytes = r.useful_bytes;
  out->cancelled_probes = r.cancelled_probes;
  out->spec_slo_runs = r.spec_slo_runs;
  out->spec_slo_used = r.spec_slo_used;
}

int ssg_search_finalize(const char* config_path, const ssg_config_record* records, size_t n,
                        char** out, ssg_status* st) {
  return guarded(st, [&] {
    auto cfg = load_search_config(config_path);
    PolicyConfig base;
    auto configs = enumerate_configs(cfg.spec, cfg.options.space, base);
    std::vector<ConfigResult> results(configs.size());
    std::vector<char> seen(configs.size(), 0);
    for (size_t k = 0; k < n; ++k) {
      const ssg_config_record& rec = records[k];
      require(rec.index >= 0 && static_cast<size_t>(rec.index) < configs.size(),
              "ssg_search_finalize: record index out of range");
      ConfigResult& r = results[rec.index];
      seen[rec.index] = 1;
      r.config = configs[rec.index];
      r.sku_name = cfg.options.space.skus[r.config.sku_index].sku_name;
      r.capacity_qps = rec.capacity_qps;
      r.qps_per_dollar = rec.qps_per_dollar;
      r.ttft_p90 = rec.ttft_p90;
      r.tbt_p99 = rec.tbt_p99;
      r.delay_p99 = rec.delay_p99;
      r.makespan = rec.makespan;
      r.slo_pass = rec.slo_pass != 0;
      r.error.assign(rec.error, strnlen(rec.error, sizeof(rec.error)));
    }
    for (size_t i = 0; i < seen.size(); ++i)
      require(seen[i], "ssg_search_finalize: missing result for config " + configs[i].id);
    auto o = finalize_search(cfg.spec, cfg.options, std::move(results));
    *out = dup_text(outcome_json(o, cfg.options.objective).dump(), nullptr);
  });
}

}  // extern "C"
