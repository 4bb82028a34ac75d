// ref_driver.cpp -- TEST INFRASTRUCTURE ONLY (the parity oracle).
//
// Compiles the UNMODIFIED reference headers from /root/reference/proj/include
// (header-only C++20) into oracle/_ref/libservesim_ref.so and exposes a small
// extern "C" surface so the pytest parity suite and bench.py's cpu_baseline /
// --impl reference legs can call the reference's own code path:
//
//   ref_train            generate_synthetic_profile + train     (profiler.hpp:314, estimator.hpp:201)
//   ref_predict          EstimatorModel::predict per query       (estimator.hpp:105)
//   ref_predict_timed    the same over host threads (cpu baseline for the predictor bench)
//   ref_predict_batch    predict_batch + batch_device_flops      (estimator.hpp:294,353)
//   ref_simulate         run_simulation + build_report + batch log (sim.hpp:135, metrics.hpp:106)
//   ref_search           load_search_config + run_search + writers (config.hpp:111, search.hpp:369)
//   ref_evaluate_sample  evaluate_config over a subset of configs (search.hpp:294), timed
//   ref_workload         synth_trace / poisson_arrivals / cap_total_length / load_trace
//                        (workload.hpp:33-247); request and answer as JSON
//
// Nothing in the product (paper_2405_05465_b200/) links or loads this file.
// Built with the reference's own flags: -std=gnu++20 -O3 -DNDEBUG, no -march.
#include <atomic>
#include <chrono>
#include <cstdlib>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "servesim/config.hpp"
#include "servesim/estimator.hpp"
#include "servesim/metrics.hpp"
#include "servesim/search.hpp"
#include "servesim/sim.hpp"
#include "servesim/workload.hpp"

using namespace servesim;
using nlohmann::json;

namespace {

char* dup(const std::string& s) {
  char* p = static_cast<char*>(std::malloc(s.size() + 1));
  std::memcpy(p, s.data(), s.size());
  p[s.size()] = 0;
  return p;
}

std::string error_json(const char* kind, const char* what) {
  json j;
  j["error"] = what;
  j["kind"] = kind;
  return j.dump();
}

template <typename F>
char* wrap(F&& f) {
  try {
    return dup(f());
  } catch (const Error& e) {
    return dup(error_json("Error", e.what()));
  } catch (const InternalError& e) {
    return dup(error_json("InternalError", e.what()));
  } catch (const std::exception& e) {
    return dup(error_json("exception", e.what()));
  }
}

// Cluster document with the model spec and device inline:
// {"model_spec": {...}, "device": {...}, "parallelism": {...}, "scheduler": {...},
//  "routing": {"policy": ..., "deferred_threshold": ...}, "cpu_overhead_per_iter": x}
ClusterConfig cluster_from(const json& j) {
  ClusterConfig c;
  c.spec = parse_model_spec(j.at("model_spec").dump());
  c.dev = parse_device_profile(j.at("device").dump());
  const auto& par = j.at("parallelism");
  c.par.tp_degree = par.at("tp_degree").get<std::int64_t>();
  c.par.pp_degree = par.at("pp_degree").get<std::int64_t>();
  c.par.num_replicas = par.at("num_replicas").get<std::int64_t>();
  c.policy = parse_policy_config(j.at("scheduler"));
  if (j.contains("routing")) {
    c.routing = routing_policy_from_string(j.at("routing").at("policy").get<std::string>());
    c.deferred_threshold = j.at("routing").value("deferred_threshold", std::int64_t(0));
  }
  c.cpu_overhead_per_iter = j.value("cpu_overhead_per_iter", 0.0);
  return c;
}

struct BatchLogger : SimObserver {
  json log = json::array();
  void on_batch(std::size_t replica, double now, const BatchPlan& plan,
                const ReplicaScheduler& sched) override {
    json b;
    b["replica"] = replica;
    b["now"] = now;
    b["kv"] = sched.memory().allocated_units();
    json e = json::array();
    for (const auto& p : plan.prefills)
      e.push_back({1, p.request->req.id, p.chunk_tokens, p.prior_context});
    for (const auto& d : plan.decodes) e.push_back({0, d.request->req.id, 1, d.context_tokens});
    b["entries"] = std::move(e);
    log.push_back(std::move(b));
  }
};

}  // namespace

extern "C" {

void ref_free(void* p) { std::free(p); }

char* ref_train(const char* model_spec_json, const char* device_json, const int64_t* tps,
                size_t n_tps, const char* regressor, uint64_t seed) {
  return wrap([&] {
    auto spec = parse_model_spec(model_spec_json);
    auto dev = parse_device_profile(device_json);
    std::vector<std::int64_t> tp(tps, tps + n_tps);
    TrainConfig cfg;
    cfg.seed = seed;
    cfg.regressor = regressor;
    return train(generate_synthetic_profile(spec, dev, tp), cfg).to_json().dump();
  });
}

void* ref_estimator_load(const char* est_json) {
  try {
    return new EstimatorModel(EstimatorModel::from_json(json::parse(est_json)));
  } catch (...) {
    return nullptr;
  }
}
void ref_estimator_free(void* e) { delete static_cast<EstimatorModel*>(e); }

// Returns -1 when every query succeeded, else the index of the first query
// that threw (its message in err).
long ref_predict(void* est, const int32_t* ops, const int64_t* tps, size_t n, const double* f0,
                 const double* f1, double* out, char* err, size_t errlen) {
  const auto& e = *static_cast<EstimatorModel*>(est);
  for (size_t i = 0; i < n; ++i) {
    try {
      const OpName op = static_cast<OpName>(ops[i]);
      FeatureMap f;
      const auto& m = e.find(op, tps[i]);
      f[m.schema[0]] = f0[i];
      if (m.schema.size() > 1) f[m.schema[1]] = f1[i];
      out[i] = e.predict(op, tps[i], f);
    } catch (const std::exception& ex) {
      std::snprintf(err, errlen, "%s", ex.what());
      return static_cast<long>(i);
    }
  }
  return -1;
}

// cpu baseline: the same queries through EstimatorModel::predict on `threads`
// host threads (static interleaved split); returns wall seconds.
double ref_predict_timed(void* est, const int32_t* ops, const int64_t* tps, size_t n,
                         const double* f0, const double* f1, double* out, int threads) {
  const auto& e = *static_cast<EstimatorModel*>(est);
  auto work = [&](int t) {
    for (size_t i = static_cast<size_t>(t); i < n; i += static_cast<size_t>(threads)) {
      const OpName op = static_cast<OpName>(ops[i]);
      const auto& m = e.find(op, tps[i]);
      FeatureMap f;
      f[m.schema[0]] = f0[i];
      if (m.schema.size() > 1) f[m.schema[1]] = f1[i];
      out[i] = e.predict(op, tps[i], f);
    }
  };
  auto t0 = std::chrono::steady_clock::now();
  std::vector<std::thread> pool;
  for (int t = 1; t < threads; ++t) pool.emplace_back(work, t);
  work(0);
  for (auto& th : pool) th.join();
  return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

char* ref_predict_batch(void* est, const char* model_spec_json, int64_t tp, size_t n,
                        const int64_t* p_off, const int64_t* p_len, const int64_t* p_prior,
                        const int64_t* d_off, const int64_t* d_ctx, double* seconds,
                        double* flops) {
  return wrap([&] {
    const auto& e = *static_cast<EstimatorModel*>(est);
    auto spec = parse_model_spec(model_spec_json);
    auto ops = derive_operators(spec, ParallelismConfig{tp, 1, 1});
    for (size_t c = 0; c < n; ++c) {
      BatchComposition b;
      for (int64_t k = p_off[c]; k < p_off[c + 1]; ++k) {
        b.prefill_lengths.push_back(p_len[k]);
        b.prefill_prior_context.push_back(p_prior[k]);
      }
      for (int64_t k = d_off[c]; k < d_off[c + 1]; ++k) b.decode_context_lengths.push_back(d_ctx[k]);
      try {
        seconds[c] = predict_batch(e, ops, b);
        flops[c] = batch_device_flops(ops, b);
      } catch (const Error& ex) {
        json j;
        j["error"] = ex.what();
        j["index"] = c;
        return j.dump();
      }
    }
    return std::string("{}");
  });
}

// run_simulation on an inline cluster document; trace arrays in trace order.
char* ref_simulate(const char* cluster_json, void* est, size_t n, const int64_t* ids,
                   const double* arrivals, const int64_t* prefill, const int64_t* decode,
                   int record_batches, double abort_delay, size_t abort_max_late,
                   int static_mode) {
  return wrap([&] {
    ClusterConfig c = cluster_from(json::parse(cluster_json));
    std::vector<Request> trace(n);
    for (size_t i = 0; i < n; ++i) trace[i] = Request{ids[i], arrivals[i], prefill[i], decode[i]};
    BatchLogger logger;
    SimOptions o;
    o.record_iterations = true;
    o.observer = record_batches ? &logger : nullptr;
    o.abort_delay_threshold = abort_delay;
    o.abort_max_late = abort_max_late;
    json out;
    SimulationResult r;
    try {
      r = run_simulation(c, trace, *static_cast<EstimatorModel*>(est), o);
    } catch (const ProbeInfeasible&) {
      out["probe_infeasible"] = true;
      return out.dump();
    }
    json reqs = json::array();
    for (const auto& q : r.requests)
      reqs.push_back({{"id", q.id},
                      {"arrival", q.arrival},
                      {"first_scheduled", q.first_scheduled},
                      {"first_token", q.first_token},
                      {"completion", q.completion},
                      {"restarts", q.restarts},
                      {"emissions", q.emission_times}});
    json reps = json::array();
    for (const auto& a : r.replicas)
      reps.push_back({{"busy_time", a.busy_time},
                      {"iterations", a.iterations},
                      {"tokens_processed", a.tokens_processed},
                      {"peak_kv_utilization", a.peak_kv_utilization},
                      {"preemptions", a.preemptions}});
    json iters = json::array();
    for (const auto& it : r.iterations)
      iters.push_back({it.start, it.latency, it.replica, it.batch_requests, it.current_tokens,
                       it.prefill_entries, it.decode_entries, it.kv_utilization});
    auto rep = build_report(r, static_mode != 0);
    auto summ = [](const MetricSummary& s) {
      return json{{"mean", s.mean}, {"p50", s.p50}, {"p90", s.p90}, {"p95", s.p95}, {"p99", s.p99}};
    };
    out["requests"] = std::move(reqs);
    out["replicas"] = std::move(reps);
    out["iterations"] = std::move(iters);
    out["simulated_span"] = r.simulated_span;
    out["total_model_flops"] = r.total_model_flops;
    out["num_devices"] = r.num_devices;
    out["report"] = {{"scheduling_delay", summ(rep.scheduling_delay)},
                     {"ttft", summ(rep.ttft)},
                     {"tbt", summ(rep.tbt)},
                     {"e2e", summ(rep.e2e)},
                     {"normalized", summ(rep.normalized)},
                     {"mfu", rep.cluster.mfu},
                     {"kv_utilization_peak", rep.cluster.kv_utilization_peak},
                     {"busy_fraction", rep.cluster.busy_fraction},
                     {"preemptions", rep.cluster.preemptions}};
    out["requests_csv"] = request_metrics_to_csv(rep);
    if (record_batches) out["batches"] = std::move(logger.log);
    return out.dump();
  });
}

// run_simulation (default SimOptions) + build_report, timed on one thread: the
// CPU baseline of a single simulation.  Returns the seconds, the report and the
// per-request completion times as IEEE-754 bit patterns.
char* ref_simulate_timed(const char* cluster_json, void* est, size_t n, const int64_t* ids,
                         const double* arrivals, const int64_t* prefill, const int64_t* decode) {
  return wrap([&] {
    ClusterConfig c = cluster_from(json::parse(cluster_json));
    std::vector<Request> trace(n);
    for (size_t i = 0; i < n; ++i) trace[i] = Request{ids[i], arrivals[i], prefill[i], decode[i]};
    const auto t0 = std::chrono::steady_clock::now();
    SimulationResult r = run_simulation(c, trace, *static_cast<EstimatorModel*>(est), SimOptions{});
    auto rep = build_report(r, false);
    const double secs = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    std::vector<std::uint64_t> done;
    for (const auto& q : r.requests) {
      std::uint64_t u;
      std::memcpy(&u, &q.completion, 8);
      done.push_back(u);
    }
    json out;
    out["seconds"] = secs;
    out["completion_bits"] = done;
    out["ttft_p90"] = rep.ttft.p90;
    out["tbt_p99"] = rep.tbt.p99;
    out["scheduling_delay_p99"] = rep.scheduling_delay.p99;
    out["simulated_span"] = r.simulated_span;
    return out.dump();
  });
}

// Full search from a search-config file; workers host threads.
char* ref_search(const char* search_config_path, int workers) {
  return wrap([&] {
    auto cfg = load_search_config(search_config_path);
    cfg.options.workers = workers;
    auto t0 = std::chrono::steady_clock::now();
    auto outcome = run_search(cfg.spec, cfg.workload, cfg.options);
    double secs = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    json j;
    j["results_csv"] = search_results_to_csv(outcome);
    j["frontier_ttft_csv"] = frontier_to_csv(outcome, outcome.frontier_ttft, true);
    j["frontier_tbt_csv"] = frontier_to_csv(outcome, outcome.frontier_tbt, false);
    j["summary"] = search_summary_text(outcome, cfg.options.objective);
    j["seconds"] = secs;
    j["configs"] = outcome.results.size();
    return j.dump();
  });
}

// cpu baseline for the sweep: evaluate_config on the configs whose enumeration
// index is listed, over `workers` threads (estimators built first, untimed).
char* ref_evaluate_sample(const char* search_config_path, const int64_t* idx, size_t n,
                          int workers) {
  return wrap([&] {
    auto cfg = load_search_config(search_config_path);
    PolicyConfig base;
    auto configs = enumerate_configs(cfg.spec, cfg.options.space, base);
    auto ests = detail::build_estimators(cfg.spec, cfg.options.space, cfg.options.train);
    std::vector<ConfigResult> res(n);
    std::atomic<size_t> next{0};
    auto work = [&] {
      for (size_t k; (k = next.fetch_add(1)) < n;) {
        const auto& c = configs.at(static_cast<size_t>(idx[k]));
        res[k] = evaluate_config(cfg.spec, c, cfg.options.space.skus[c.sku_index],
                                 *ests.at(c.sku_index), cfg.workload, cfg.options);
      }
    };
    auto t0 = std::chrono::steady_clock::now();
    std::vector<std::thread> pool;
    for (int w = 1; w < workers; ++w) pool.emplace_back(work);
    work();
    for (auto& t : pool) t.join();
    double secs = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    json rows = json::array();
    for (const auto& r : res)
      rows.push_back({{"id", r.config.id},
                      {"capacity_qps", r.capacity_qps},
                      {"qps_per_dollar", r.qps_per_dollar},
                      {"ttft_p90", r.ttft_p90},
                      {"tbt_p99", r.tbt_p99},
                      {"delay_p99", r.delay_p99},
                      {"slo_pass", r.slo_pass},
                      {"error", r.error}});
    json j;
    j["results"] = std::move(rows);
    j["seconds"] = secs;
    j["num_configs_total"] = configs.size();
    return j.dump();
  });
}

// {"op": "synth", "dist": {...}, "n": n, "seed": s} -> {"prefill": [...], "decode": [...]}
// {"op": "poisson", "n": n, "rate": q, "seed": s}  -> {"arrivals": [...]}
// {"op": "cap", "prefill": [...], "decode": [...], "max_total": m} -> {"prefill", "decode"}
// {"op": "load_trace", "text": csv} -> {"id", "arrival" (null when absent), "prefill", "decode"}
// Doubles travel as their IEEE-754 bit patterns (uint64) so they compare exactly.
char* ref_workload(const char* request_json) {
  return wrap([&] {
    const json q = json::parse(request_json);
    const std::string op = q.at("op").get<std::string>();
    std::vector<Request> reqs;
    json out;
    auto lengths = [&](const std::vector<Request>& rs) {
      std::vector<std::int64_t> pre, dec, ids;
      for (const auto& r : rs) {
        pre.push_back(r.prefill_tokens);
        dec.push_back(r.decode_tokens);
        ids.push_back(r.id);
      }
      out["prefill"] = pre;
      out["decode"] = dec;
      out["id"] = ids;
    };
    auto bits = [](double v) {
      std::uint64_t u;
      std::memcpy(&u, &v, 8);
      return u;
    };
    if (op == "synth") {
      lengths(synth_trace(parse_dist_config(q.at("dist")), q.at("n").get<std::size_t>(),
                          q.at("seed").get<std::uint64_t>()));
    } else if (op == "poisson") {
      std::vector<Request> rs(q.at("n").get<std::size_t>());
      rs = poisson_arrivals(std::move(rs), q.at("rate").get<double>(), q.at("seed").get<std::uint64_t>());
      std::vector<std::uint64_t> a;
      for (const auto& r : rs) a.push_back(bits(r.arrival_time));
      out["arrivals"] = a;
    } else if (op == "cap") {
      const auto pre = q.at("prefill").get<std::vector<std::int64_t>>();
      const auto dec = q.at("decode").get<std::vector<std::int64_t>>();
      for (std::size_t i = 0; i < pre.size(); ++i) {
        Request r;
        r.id = static_cast<std::int64_t>(i);
        r.prefill_tokens = pre[i];
        r.decode_tokens = dec[i];
        reqs.push_back(r);
      }
      lengths(cap_total_length(std::move(reqs), q.at("max_total").get<std::int64_t>()));
    } else if (op == "load_trace") {
      const auto rs = load_trace(q.at("text").get<std::string>());
      lengths(rs);
      if (!rs.empty() && rs.front().has_arrival()) {
        std::vector<std::uint64_t> a;
        for (const auto& r : rs) a.push_back(bits(r.arrival_time));
        out["arrival"] = a;
      } else {
        out["arrival"] = nullptr;
      }
    } else {
      throw Error("ref_workload: unknown op " + op);
    }
    return out.dump();
  });
}

}  // extern "C"
