// metrics.cpp -- request/cluster metrics and the report of one simulation.
//
// reference: metrics.hpp:17-231, stats.hpp:15-43
//
// Percentiles are nearest-rank order statistics, taken with the device select
// kernel (select.cu) -- an exact selection, so bit-identical to the
// reference's sort-then-index.  Means are fp64 sums in sample order.
#include <algorithm>
#include <cmath>
#include <sstream>

#include "json.hpp"
#include "runtime.h"
#include "select.h"
#include "servesim_b200.hpp"


namespace servesim {

double percentile(const std::vector<double>& samples, double q) {
  require(!samples.empty(), "percentile: empty sample set");
  require(q > 0.0 && q <= 1.0, "percentile: q must be in (0, 1]");
  return ssg::device_percentiles(samples, {q})[0];
}

namespace {

double mean_of(const std::vector<double>& v) {
  require(!v.empty(), "mean: empty sample set");
  double s = 0.0;
  for (double x : v) s += x;
  return s / static_cast<double>(v.size());
}

MetricSummary summarize(const std::vector<double>& v) {
  MetricSummary s;
  if (v.empty()) return s;
  s.mean = mean_of(v);
  auto p = ssg::device_percentiles(v, {0.50, 0.90, 0.95, 0.99});
  s.p50 = p[0];
  s.p90 = p[1];
  s.p95 = p[2];
  s.p99 = p[3];
  return s;
}

}  // namespace

MetricsReport build_report(const SimulationResult& result, bool static_mode) {
  ssg::PhaseTimer timer("build_report");
  MetricsReport rep;
  std::vector<double> delays, ttfts, tbts, e2es, norms;
  for (const auto& r : result.requests) {
    RequestMetrics m;
    m.id = r.id;
    m.scheduling_delay = r.first_scheduled - r.arrival;
    m.ttft = r.first_token - r.arrival;
    m.prefill_completion = r.first_token - r.arrival;
    m.e2e_latency = r.completion - r.arrival;
    require(r.completion >= 0, "normalized_latency: request not completed");
    const double start = static_mode ? r.first_scheduled : r.arrival;
    m.normalized_latency = (r.completion - start) / static_cast<double>(r.decode_tokens);
    m.prefill_tokens = r.prefill_tokens;
    m.decode_tokens = r.decode_tokens;
    m.restarts = r.restarts;
    for (std::size_t i = 1; i < r.emission_times.size(); ++i)
      m.tbt_samples.push_back(r.emission_times[i] - r.emission_times[i - 1]);
    delays.push_back(m.scheduling_delay);
    ttfts.push_back(m.ttft);
    e2es.push_back(m.e2e_latency);
    norms.push_back(m.normalized_latency);
    for (double t : m.tbt_samples) tbts.push_back(t);
    rep.requests.push_back(std::move(m));
  }
  rep.scheduling_delay = summarize(delays);
  rep.ttft = summarize(ttfts);
  rep.tbt = summarize(tbts);
  rep.e2e = summarize(e2es);
  rep.normalized = summarize(norms);
  ClusterMetrics& c = rep.cluster;
  if (result.simulated_span > 0.0)
    c.mfu = result.total_model_flops /
            (result.simulated_span * result.peak_device_flops * static_cast<double>(result.num_devices));
  double busy = 0.0;
  for (const auto& a : result.replicas) {
    c.kv_utilization_peak = std::max(c.kv_utilization_peak, a.peak_kv_utilization);
    busy += a.busy_time;
    c.preemptions += a.preemptions;
  }
  if (result.simulated_span > 0 && !result.replicas.empty())
    c.busy_fraction = busy / (result.simulated_span * static_cast<double>(result.replicas.size()));
  rep.simulated_span = result.simulated_span;
  return rep;
}

std::string request_metrics_to_csv(const MetricsReport& rep) {
  std::ostringstream out;
  out << "request_id,prefill_tokens,decode_tokens,scheduling_delay_s,ttft_s,e2e_s,"
         "normalized_s_per_token,restarts\n";
  for (const auto& m : rep.requests)
    out << m.id << ',' << m.prefill_tokens << ',' << m.decode_tokens << ','
        << fmt_double(m.scheduling_delay) << ',' << fmt_double(m.ttft) << ','
        << fmt_double(m.e2e_latency) << ',' << fmt_double(m.normalized_latency) << ',' << m.restarts
        << "\n";
  return out.str();
}

nlohmann::ordered_json summary_to_json(const MetricsReport& rep) {  // metrics.hpp:173-197
  auto metric = [](const MetricSummary& s) {
    nlohmann::ordered_json j;
    j["mean"] = s.mean;
    j["p50"] = s.p50;
    j["p90"] = s.p90;
    j["p95"] = s.p95;
    j["p99"] = s.p99;
    return j;
  };
  nlohmann::ordered_json j;
  j["num_requests"] = rep.requests.size();
  j["simulated_span_s"] = rep.simulated_span;
  j["scheduling_delay_s"] = metric(rep.scheduling_delay);
  j["ttft_s"] = metric(rep.ttft);
  j["tbt_s"] = metric(rep.tbt);
  j["e2e_s"] = metric(rep.e2e);
  j["normalized_s_per_token"] = metric(rep.normalized);
  j["cluster"] = {{"mfu", rep.cluster.mfu},
                  {"kv_utilization_peak", rep.cluster.kv_utilization_peak},
                  {"busy_fraction", rep.cluster.busy_fraction},
                  {"preemptions", rep.cluster.preemptions}};
  return j;
}

std::vector<std::string> export_metrics(const MetricsReport& rep, const std::string& out_dir,
                                        const std::string& format) {  // metrics.hpp:200-231
  require(format == "csv" || format == "json", "export: format must be csv or json");
  std::vector<std::string> written;
  if (format == "csv") {
    written.push_back(out_dir + "/requests.csv");
    write_text_file(written.back(), request_metrics_to_csv(rep));
  } else {
    nlohmann::ordered_json rows = nlohmann::ordered_json::array();
    for (const auto& m : rep.requests) {
      nlohmann::ordered_json r;
      r["request_id"] = m.id;
      r["prefill_tokens"] = m.prefill_tokens;
      r["decode_tokens"] = m.decode_tokens;
      r["scheduling_delay_s"] = m.scheduling_delay;
      r["ttft_s"] = m.ttft;
      r["e2e_s"] = m.e2e_latency;
      r["normalized_s_per_token"] = m.normalized_latency;
      r["restarts"] = m.restarts;
      rows.push_back(std::move(r));
    }
    written.push_back(out_dir + "/requests.json");
    write_text_file(written.back(), rows.dump(2) + "\n");
  }
  written.push_back(out_dir + "/summary.json");
  write_text_file(written.back(), summary_to_json(rep).dump(2) + "\n");
  return written;
}

}  // namespace servesim
