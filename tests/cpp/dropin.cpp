// dropin.cpp -- one caller program, compiled twice: against the reference's
// headers (-DSSG_REFERENCE, oracle/Makefile -> oracle/_ref/dropin_ref) and
// against include/servesim_b200.hpp + libssg.so (paper_2405_05465_b200/csrc/
// Makefile -> build/dropin_ssg).  Nothing below differs between the two builds
// except the include lines, so the same source exercising the reference's
// plugin and entry-point API (scheduler, router, observer, regressor, capacity
// search, evaluate_config, run_simulation, run_search, the writers) is the
// drop-in proof; tests/test_dropin_gpu.py runs both and compares every output
// byte for byte.  Test infrastructure: this file is not part of the library.
//
// Modes (argv[1]):
//   scheduler                         scheduler/router known answers + a
//                                     randomised step-by-step trace per policy
//   simulate CLUSTER TRACE EST OUT FORMAT QPS SEED STATIC EVENTLOG
//                                     a cmd_simulate clone (servesim_cli.cpp:96-136)
//   search SEARCH OUT SEED            a cmd_search clone (servesim_cli.cpp:138-178)
//   invariants MODEL DEVICE           acceptance criterion 4 (acceptance.cpp:201-310)
//   capacity MODEL DEVICE             find_capacity, evaluate_config, Regressor
#ifdef SSG_REFERENCE
#include "servesim/config.hpp"
#include "servesim/csv.hpp"
#include "servesim/estimator.hpp"
#include "servesim/metrics.hpp"
#include "servesim/profiler.hpp"
#include "servesim/scheduler.hpp"
#include "servesim/search.hpp"
#include "servesim/sim.hpp"
#include "servesim/workload.hpp"
#else
#include "servesim_b200.hpp"
#endif

#include <algorithm>
#include <cstdio>
#include <filesystem>
#include <fstream>
#include <iostream>
#include <map>
#include <memory>
#include <random>
#include <sstream>
#include <string>
#include <vector>

using namespace servesim;

namespace {

int g_failed = 0, g_passed = 0;
#define EXPECT(cond)                                                   \
  do {                                                                 \
    if (cond) {                                                        \
      ++g_passed;                                                      \
    } else {                                                           \
      ++g_failed;                                                      \
      std::cout << "FAIL line " << __LINE__ << ": " #cond << "\n";     \
    }                                                                  \
  } while (0)

std::shared_ptr<RequestState> req(std::int64_t id, double arrival, std::int64_t prefill,
                                  std::int64_t decode) {
  auto r = std::make_shared<RequestState>();
  r->req = Request{id, arrival, prefill, decode};
  return r;
}

MemoryPlan blocks_plan(std::int64_t blocks, std::int64_t watermark, std::int64_t block_size = 16) {
  MemoryPlan p;
  p.block_size = block_size;
  p.num_blocks = blocks;
  p.kv_capacity_tokens = blocks * block_size;
  p.watermark_blocks = watermark;
  return p;
}

BatchPlan cycle(ReplicaScheduler& s, double now) {
  s.set_now(now);
  BatchPlan p = s.schedule_iteration();
  if (!p.empty()) s.complete_iteration(p, now + 0.01);
  return p;
}

std::string plan_text(const BatchPlan& p) {
  std::ostringstream o;
  o << "[";
  bool first = true;
  for (const auto& e : p.prefills) {
    o << (first ? "" : ",") << "p:" << e.request->req.id << ":" << e.chunk_tokens << ":" << e.prior_context;
    first = false;
  }
  for (const auto& e : p.decodes) {
    o << (first ? "" : ",") << "d:" << e.request->req.id << ":" << e.context_tokens;
    first = false;
  }
  o << "]";
  return o.str();
}

// ---------------------------------------------------------------- scheduler
void scheduler_known_answers() {
  {  // sarathi: decodes first, then one chunk filling the budget
    PolicyConfig c;
    c.policy = SchedulerPolicy::SarathiServe;
    c.chunk_size = 512;
    ReplicaScheduler s(c, blocks_plan(4096, 4));
    for (int i = 0; i < 10; ++i) s.enqueue(req(i, 0.1 * i, 1, 5));
    cycle(s, 1.0);
    s.enqueue(req(100, 1.5, 2000, 5));
    s.set_now(2.0);
    BatchPlan p = s.schedule_iteration();
    EXPECT(p.decodes.size() == 10);
    EXPECT(p.prefills.size() == 1 && p.prefills[0].chunk_tokens == 502);
    EXPECT(p.total_current_tokens() == 512);
  }
  {  // sarathi chunks carry their prior context
    PolicyConfig c;
    c.policy = SchedulerPolicy::SarathiServe;
    c.chunk_size = 512;
    c.max_batch_size = 8;
    ReplicaScheduler s(c, blocks_plan(4096, 4));
    s.enqueue(req(0, 0.0, 1300, 3));
    BatchPlan a = cycle(s, 0.0), b = cycle(s, 0.1), d = cycle(s, 0.2), e = cycle(s, 0.3);
    EXPECT(a.prefills.size() == 1 && a.prefills[0].chunk_tokens == 512 && a.prefills[0].prior_context == 0);
    EXPECT(b.prefills.size() == 1 && b.prefills[0].chunk_tokens == 512 && b.prefills[0].prior_context == 512);
    EXPECT(d.prefills.size() == 1 && d.prefills[0].chunk_tokens == 276 && d.prefills[0].prior_context == 1024);
    EXPECT(e.decodes.size() == 1 && e.prefills.empty());
  }
  {  // vllm: an admission below the watermark preempts the latest runner
    PolicyConfig c;
    c.max_batch_size = 8;
    ReplicaScheduler s(c, blocks_plan(10, 2));
    auto a = req(0, 0.0, 100, 10);
    s.enqueue(a);
    cycle(s, 0.0);
    EXPECT(s.memory().allocated_units() == 7);
    cycle(s, 0.1);
    EXPECT(a->emitted == 2);
    s.enqueue(req(1, 0.5, 33, 5));
    s.set_now(1.0);
    BatchPlan p = s.schedule_iteration();
    EXPECT(p.prefills.size() == 1 && p.prefills[0].request->req.id == 1);
    EXPECT(s.preemption_count() == 1);
    EXPECT(s.outstanding() == 2);
    EXPECT(a->restarts == 1 && a->kv_context == 0 && a->prefill_target == 102);
  }
  {  // faster_transformer: membership frozen until the batch drains
    PolicyConfig c;
    c.policy = SchedulerPolicy::FasterTransformer;
    c.max_batch_size = 4;
    ReplicaScheduler s(c, blocks_plan(4096, 4));
    s.enqueue(req(0, 0.0, 10, 2));
    s.enqueue(req(1, 0.1, 10, 4));
    cycle(s, 0.0);
    const auto members = s.ft_member_ids();
    EXPECT((members == std::vector<std::int64_t>{0, 1}));
    s.enqueue(req(2, 0.2, 10, 2));
    cycle(s, 0.2);
    EXPECT(s.ft_member_ids() == members);
    for (int i = 0; i < 3; ++i) {
      BatchPlan p = cycle(s, 0.3 + 0.1 * i);
      for (const auto& d : p.decodes) EXPECT(d.request->req.id != 2);
    }
    EXPECT(s.ft_member_ids().empty());
    BatchPlan f = cycle(s, 1.0);
    EXPECT(f.prefills.size() == 1 && f.prefills[0].request->req.id == 2);
  }
  {  // faster_transformer reserves the final context at admission
    PolicyConfig c;
    c.policy = SchedulerPolicy::FasterTransformer;
    c.max_batch_size = 4;
    ReplicaScheduler s(c, blocks_plan(6, 0));
    s.enqueue(req(0, 0.0, 30, 50));
    s.enqueue(req(1, 0.1, 30, 50));
    cycle(s, 0.0);
    EXPECT((s.ft_member_ids() == std::vector<std::int64_t>{0}));
  }
  {  // orca+: prefills take the budget first, decodes fill the rest
    PolicyConfig c;
    c.policy = SchedulerPolicy::OrcaPlus;
    c.max_batch_size = 64;
    c.max_tokens_per_iter = 100;
    ReplicaScheduler s(c, blocks_plan(4096, 4));
    for (int i = 0; i < 20; ++i) s.enqueue(req(i, 0.01 * i, 1, 5));
    cycle(s, 0.0);
    s.enqueue(req(100, 0.5, 95, 5));
    s.set_now(1.0);
    BatchPlan p = s.schedule_iteration();
    EXPECT(p.prefills.size() == 1 && p.prefills[0].chunk_tokens == 95);
    EXPECT(p.decodes.size() == 5 && p.total_current_tokens() == 100);
  }
  {  // lightllm holds tokens, orca+ whole blocks
    PolicyConfig orca;
    orca.policy = SchedulerPolicy::OrcaPlus;
    PolicyConfig light = orca;
    light.policy = SchedulerPolicy::LightLLM;
    ReplicaScheduler a(orca, blocks_plan(4096, 4)), b(light, blocks_plan(4096, 4));
    a.enqueue(req(0, 0.0, 20, 5));
    b.enqueue(req(0, 0.0, 20, 5));
    a.set_now(0.0);
    b.set_now(0.0);
    a.schedule_iteration();
    b.schedule_iteration();
    EXPECT(a.memory().held_units(0) == 2);
    EXPECT(b.memory().held_units(0) == 20);
  }
  {  // router
    Router rr(RoutingPolicy::RoundRobin, 3, 1);
    auto zero = [](std::size_t) { return std::size_t(0); };
    std::vector<std::size_t> got;
    for (int i = 0; i < 5; ++i) got.push_back(*rr.route(req(i, 0.0, 1, 1), zero));
    EXPECT((got == std::vector<std::size_t>{0, 1, 2, 0, 1}));
    Router lo(RoutingPolicy::LeastOutstanding, 3, 1);
    std::vector<std::size_t> counts = {4, 1, 4};
    auto load = [&](std::size_t i) { return counts[i]; };
    EXPECT(*lo.route(req(0, 0.0, 1, 1), load) == 1);
    counts = {2, 2, 5};
    EXPECT(*lo.route(req(1, 0.0, 1, 1), load) == 0);
    Router df(RoutingPolicy::Deferred, 2, 3);
    counts = {3, 3};
    EXPECT(!df.route(req(0, 0.0, 1, 1), load).has_value());
    EXPECT(df.drain(load).empty() && df.pooled() == 1);
    counts = {3, 2};
    auto assigned = df.drain(load);
    EXPECT(assigned.size() == 1 && assigned[0].first == 1 && df.pooled() == 0);
  }
  std::cout << "known answers: " << g_passed << " passed, " << g_failed << " failed\n";
}

// Step-by-step traces: random arrivals (some enqueued out of arrival order),
// tight memory so preemption paths run, every plan and the scheduler's view
// printed after each call.
void scheduler_traces() {
  const SchedulerPolicy pols[] = {SchedulerPolicy::FasterTransformer, SchedulerPolicy::OrcaPlus,
                                  SchedulerPolicy::VLLM, SchedulerPolicy::SarathiServe,
                                  SchedulerPolicy::LightLLM};
  for (auto pol : pols) {
    for (int variant = 0; variant < 2; ++variant) {
      PolicyConfig c;
      c.policy = pol;
      c.max_batch_size = variant ? 48 : 12;
      c.max_tokens_per_iter = variant ? 4096 : 700;
      c.chunk_size = variant ? 512 : 256;
      c.block_size = variant ? 16 : 7;
      ReplicaScheduler s(c, blocks_plan(variant ? 160 : 90, variant ? 2 : 1, c.block_size));
      std::mt19937_64 rng(1000 + 10 * static_cast<int>(pol) + variant);
      std::uniform_int_distribution<std::int64_t> plen(1, variant ? 600 : 200), dlen(1, 60);
      std::uniform_real_distribution<double> jitter(-0.5, 0.5);
      std::vector<std::shared_ptr<RequestState>> all;
      double now = 0.0;
      std::int64_t next_id = 0;
      std::cout << "trace policy=" << static_cast<int>(pol) << " variant=" << variant << "\n";
      for (int it = 0; it < 400; ++it) {
        // a few arrivals; arrival times may precede requests already queued
        const int k = static_cast<int>(rng() % 3);
        for (int q = 0; q < k && next_id < 120; ++q) {
          auto r = req(next_id++, std::max(0.0, now + jitter(rng)), plen(rng), dlen(rng));
          all.push_back(r);
          s.enqueue(r);
        }
        s.set_now(now);
        BatchPlan p = s.schedule_iteration();
        std::cout << it << " t=" << fmt_double(now) << " " << plan_text(p)
                  << " alloc=" << s.memory().allocated_units() << " out=" << s.outstanding()
                  << " pre=" << s.preemption_count() << " ft=" << s.ft_member_ids().size();
        if (!p.empty()) {
          auto done = s.complete_iteration(p, now + 0.05);
          std::cout << " done=";
          for (const auto& d : done) std::cout << d->req.id << ";";
        }
        std::cout << "\n";
        now += 0.1;
        if (!s.has_work() && next_id >= 120) break;
      }
      for (const auto& r : all)
        std::cout << "r " << r->req.id << " " << r->emitted << " " << r->restarts << " "
                  << r->prefill_target << " " << r->prefill_done << " " << r->kv_context << " "
                  << fmt_double(r->first_scheduled_time) << " " << fmt_double(r->first_token_time)
                  << " " << fmt_double(r->completion_time) << " " << r->emission_times.size()
                  << " " << s.memory().held_units(r->req.id) << "\n";
    }
  }
}

// ---------------------------------------------------------------- simulate
class EventLog : public SimObserver {
 public:
  explicit EventLog(const std::string& path) : out_(path, std::ios::binary) {}
  void on_batch(std::size_t replica, double now, const BatchPlan& plan,
                const ReplicaScheduler& sched) override {
    out_ << "t=" << fmt_double(now) << " replica=" << replica << " tokens=" << plan.total_current_tokens()
         << " kv_used=" << sched.memory().allocated_units() << "/" << sched.memory().total_units()
         << " batch=" << plan_text(plan) << "\n";
  }

 private:
  std::ofstream out_;
};

int cmd_simulate(char** a) {
  const std::string cluster_path = a[0], trace_path = a[1], est_path = a[2], out_dir = a[3],
                    format = a[4];
  const double qps = std::stod(a[5]);
  const std::uint64_t seed = std::stoull(a[6]);
  const bool static_mode = std::stoi(a[7]) != 0, event_log = std::stoi(a[8]) != 0;
  auto loaded = load_cluster_config(cluster_path);
  auto estimator = EstimatorModel::from_json(load_json_file(est_path));
  auto trace = load_trace(read_text_file(trace_path));
  if (qps > 0.0)
    trace = poisson_arrivals(std::move(trace), qps, seed);
  else if (static_mode)
    for (auto& r : trace) r.arrival_time = 0.0;
  std::filesystem::create_directories(out_dir);
  SimOptions opts;
  std::unique_ptr<EventLog> log;
  if (event_log) {
    log = std::make_unique<EventLog>(out_dir + "/events.log");
    opts.observer = log.get();
  }
  auto result = run_simulation(loaded.cluster, trace, estimator, opts);
  auto report = build_report(result, static_mode);
  export_metrics(report, out_dir, format);
  std::cout << result.requests.size() << " requests simulated, span " << fmt_double(result.simulated_span)
            << " s\n";
  return 0;
}

// ---------------------------------------------------------------- search
int cmd_search(char** a) {
  const std::string path = a[0], out_dir = a[1];
  const std::uint64_t seed = std::stoull(a[2]);
  auto loaded = load_search_config(path);
  loaded.options.workers = 4;
  loaded.options.capacity.seed = seed;
  loaded.options.train.seed = seed;
  std::filesystem::create_directories(out_dir);
  auto outcome = run_search(loaded.spec, loaded.workload, loaded.options);
  write_text_file(out_dir + "/results.csv", search_results_to_csv(outcome));
  nlohmann::ordered_json rows = nlohmann::ordered_json::array();
  for (const auto& r : outcome.results) {
    nlohmann::ordered_json j;
    j["config_id"] = r.config.id;
    j["capacity_qps"] = r.capacity_qps;
    j["qps_per_dollar"] = r.qps_per_dollar;
    j["ttft_p90_s"] = r.ttft_p90;
    j["tbt_p99_s"] = r.tbt_p99;
    j["delay_p99_s"] = r.delay_p99;
    j["makespan_s"] = r.makespan;
    j["slo_pass"] = r.slo_pass;
    j["error"] = r.error;
    rows.push_back(std::move(j));
  }
  write_text_file(out_dir + "/results.json", rows.dump(2) + "\n");
  write_text_file(out_dir + "/frontier_ttft.csv", frontier_to_csv(outcome, outcome.frontier_ttft, true));
  write_text_file(out_dir + "/frontier_tbt.csv", frontier_to_csv(outcome, outcome.frontier_tbt, false));
  write_text_file(out_dir + "/summary.txt", search_summary_text(outcome, loaded.options.objective));
  std::cout << search_summary_text(outcome, loaded.options.objective);
  return 0;
}

// ---------------------------------------------------------------- invariants
class InvariantCheck : public SimObserver {
 public:
  explicit InvariantCheck(const PolicyConfig& c) : cfg(c) {}
  void on_batch(std::size_t replica, double now, const BatchPlan& plan,
                const ReplicaScheduler& sched) override {
    if (sched.memory().allocated_units() > sched.memory().total_units()) ++memory;
    if (plan.batch_size() > cfg.max_batch_size) ++batch;
    const std::int64_t t = plan.total_current_tokens();
    if (cfg.policy == SchedulerPolicy::SarathiServe ? t > cfg.chunk_size
                                                    : cfg.policy != SchedulerPolicy::FasterTransformer &&
                                                          t > cfg.max_tokens_per_iter)
      ++tokens;
    for (const auto& e : plan.prefills)
      if (e.request->req.arrival_time > now + 1e-12) ++causality;
    for (const auto& e : plan.decodes)
      if (e.request->req.arrival_time > now + 1e-12) ++causality;
    if (cfg.policy == SchedulerPolicy::FasterTransformer) {
      auto m = sched.ft_member_ids();
      auto it = members.find(replica);
      if (it != members.end() && it->second != m)
        for (auto id : m)
          if (std::find(it->second.begin(), it->second.end(), id) != it->second.end()) ++ft;
      members[replica] = std::move(m);
    }
    ++batches;
    checksum = checksum * 1000003 + static_cast<std::size_t>(t) + 7 * sched.outstanding() +
               13 * sched.preemption_count() + 31 * static_cast<std::size_t>(sched.memory().allocated_units());
  }
  PolicyConfig cfg;
  std::size_t batches = 0, memory = 0, batch = 0, tokens = 0, causality = 0, ft = 0, checksum = 0;
  std::map<std::size_t, std::vector<std::int64_t>> members;
};

int cmd_invariants(char** a) {
  auto spec = load_model_spec_file(a[0]);
  auto dev = load_device_file(a[1]);
  dev.device_mem = 30e9;
  TrainConfig tc;
  tc.seed = 42;
  auto est = train(generate_synthetic_profile(spec, dev, {1}), tc);
  DistConfig dist;
  dist.kind = "lognormal";
  dist.prefill_median = 300;
  dist.prefill_sigma = 1.0;
  dist.decode_median = 40;
  dist.decode_sigma = 0.9;
  dist.max_total = 2048;
  for (auto pol : {SchedulerPolicy::FasterTransformer, SchedulerPolicy::OrcaPlus, SchedulerPolicy::VLLM,
                   SchedulerPolicy::SarathiServe, SchedulerPolicy::LightLLM}) {
    ClusterConfig cl;
    cl.spec = spec;
    cl.par = {1, 1, 2};
    cl.dev = dev;
    cl.policy.policy = pol;
    cl.policy.max_batch_size = 64;
    cl.policy.max_tokens_per_iter = 4096;
    cl.policy.chunk_size = 512;
    auto trace = poisson_arrivals(synth_trace(dist, 10000, 404), 60.0, 405);
    InvariantCheck obs(cl.policy);
    SimOptions opts;
    opts.observer = &obs;
    auto res = run_simulation(cl, trace, est, opts);
    std::size_t conserve = 0, order = 0, pre = 0;
    for (const auto& r : res.requests) {
      if (r.emission_times.size() != static_cast<std::size_t>(r.decode_tokens)) ++conserve;
      for (std::size_t i = 1; i < r.emission_times.size(); ++i)
        if (r.emission_times[i] <= r.emission_times[i - 1]) ++order;
    }
    for (const auto& rep : res.replicas) pre += rep.preemptions;
    std::cout << "policy " << static_cast<int>(pol) << " batches=" << obs.batches << " mem=" << obs.memory
              << " batch=" << obs.batch << " tokens=" << obs.tokens << " causality=" << obs.causality
              << " ft=" << obs.ft << " conserve=" << conserve << " order=" << order
              << " preemptions=" << pre << " checksum=" << obs.checksum
              << " span=" << fmt_double(res.simulated_span) << "\n";
  }
  return 0;
}

// ---------------------------------------------------------------- capacity, evaluate_config, regressor
int cmd_capacity(char** a) {
  auto spec = load_model_spec_file(a[0]);
  auto dev = load_device_file(a[1]);
  {
    std::vector<double> asked;
    CapacitySearchOptions o;
    o.initial_guess = 3.0;
    const double cap = find_capacity([&](double q) { asked.push_back(q); return q <= 37.3; }, o);
    std::cout << "find_capacity " << fmt_double(cap) << " probes";
    for (double q : asked) std::cout << " " << fmt_double(q);
    std::cout << "\n";
    asked.clear();
    o.initial_guess = 100.0;
    const double cap2 = find_capacity([&](double q) { asked.push_back(q); return q <= 0.7; }, o);
    std::cout << "find_capacity " << fmt_double(cap2) << " probes " << asked.size() << "\n";
  }
  TrainConfig tc;
  tc.seed = 11;
  auto est = train(generate_synthetic_profile(spec, dev, {1, 2}), tc);
  TrainConfig tf = tc;
  tf.regressor = "forest";
  auto forest = train(generate_synthetic_profile(spec, dev, {1}), tf);
  // Regressor plugin: from the serialized handoff, evaluated on transformed features
  for (const auto* e : {&est, &forest}) {
    auto doc = e->to_json();
    for (const auto& [key, mj] : doc.at("ops").items()) {
      auto r = regressor_from_json(mj.at("regressor"));
      const std::size_t nf = mj.at("schema").size();
      std::mt19937_64 rng(5);
      std::uniform_real_distribution<double> u(0.0, 14.0);
      std::cout << "regressor " << key;
      for (int q = 0; q < 4; ++q) {
        std::vector<double> x(nf);
        for (auto& v : x) v = u(rng);
        std::cout << " " << fmt_double(r->predict(x));
      }
      std::cout << " json=" << (r->to_json() == mj.at("regressor")) << "\n";
    }
  }
  // evaluate_config on a few candidates (error rows included)
  DistConfig dist;
  dist.kind = "lognormal";
  dist.prefill_median = 600;
  dist.prefill_sigma = 0.8;
  dist.decode_median = 250;
  dist.decode_sigma = 0.7;
  dist.max_total = 4096;
  auto workload = synth_trace(dist, 1500, 9);
  SearchOptions so;
  so.capacity.probe_requests = 1500;
  so.cost[dev.sku_name] = 2.5;
  std::vector<CandidateConfig> cands;
  for (auto pol : {SchedulerPolicy::VLLM, SchedulerPolicy::SarathiServe, SchedulerPolicy::OrcaPlus}) {
    for (std::int64_t tp : {1, 2}) {
      CandidateConfig c;
      c.id = std::string(to_string(pol)) + "_tp" + std::to_string(tp);
      c.par = {tp, 1, 2};
      c.policy.policy = pol;
      c.policy.max_batch_size = 64;
      cands.push_back(c);
    }
  }
  CandidateConfig bad;
  bad.id = "tp4_untrained";
  bad.par = {4, 1, 1};
  cands.push_back(bad);
  for (const auto& c : cands) {
    ConfigResult r = evaluate_config(spec, c, dev, est, workload, so);
    std::cout << "evaluate " << r.config.id << " " << r.sku_name << " cap=" << fmt_double(r.capacity_qps)
              << " qpd=" << fmt_double(r.qps_per_dollar) << " ttft=" << fmt_double(r.ttft_p90)
              << " tbt=" << fmt_double(r.tbt_p99) << " delay=" << fmt_double(r.delay_p99)
              << " slo=" << r.slo_pass << " err=" << r.error << "\n";
  }
  so.objective = "makespan";
  ConfigResult m = evaluate_config(spec, cands[1], dev, est, workload, so);
  std::cout << "makespan " << fmt_double(m.makespan) << " ttft=" << fmt_double(m.ttft_p90) << "\n";
  std::cout << "initial_qps_guess "
            << fmt_double(initial_qps_guess(spec, cands[0], est,
                                            ClusterConfig{spec, cands[0].par, dev, cands[0].policy}))
            << "\n";
  return 0;
}

}  // namespace

int main(int argc, char** argv) {
  if (argc < 2) {
    std::cerr << "usage: dropin scheduler|simulate|search|invariants|capacity ...\n";
    return 2;
  }
  const std::string mode = argv[1];
  try {
    if (mode == "scheduler") {
      scheduler_known_answers();
      scheduler_traces();
      return g_failed ? 1 : 0;
    }
    if (mode == "simulate" && argc >= 11) return cmd_simulate(argv + 2);
    if (mode == "search" && argc >= 5) return cmd_search(argv + 2);
    if (mode == "invariants" && argc >= 4) return cmd_invariants(argv + 2);
    if (mode == "capacity" && argc >= 4) return cmd_capacity(argv + 2);
  } catch (const Error& e) {
    std::cout << "error: " << e.what() << "\n";
    return 1;
  }
  std::cerr << "bad arguments\n";
  return 2;
}
