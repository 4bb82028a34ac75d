// search.cpp -- Vidur-Search on the GPU: every candidate's capacity search
// advances in lock-step rounds of speculative probes, each round one
// k_simulate launch over (config, probe QPS, replica) units; then one launch
// of SLO runs and one segmented select for their percentiles.
//
// reference: search.hpp:76-428 (enumerate_configs, find_capacity,
//            initial_qps_guess, evaluate_config, run_search, pareto_frontier,
//            writers), workload.hpp:93-104 (poisson_arrivals)
//
// Exactness of the capacity search.  find_capacity is deterministic given the
// answers of feasible(q), and every q it can ask for is an exact double built
// by the same arithmetic (hi *= 2, hi / 2, 0.5 * (lo + hi)).  Each round
// replays find_capacity from the start against a memo of answered q; the
// first unanswered q, plus the values the search could ask next (the doubling
// ladder, or a bisection sub-tree), become the round's probes.  The replay
// then selects exactly the capacity the sequential reference would.
#include <algorithm>
#include <cmath>
#include <map>
#include <sstream>
#include <unordered_map>

#include "engine_limits.h"
#include "select.h"
#include "servesim_b200.hpp"
#include "sim_host.h"

namespace servesim {

using namespace ssg;

// ------------------------------------------------------------------ enumerate
std::vector<CandidateConfig> enumerate_configs(const ModelSpec& spec, const SearchSpace& space,
                                               const PolicyConfig& base,
                                               std::vector<SkippedConfig>* skipped) {
  require(!space.skus.empty(), "search space: no SKUs");
  require(!space.schedulers.empty(), "search space: no schedulers");
  std::vector<CandidateConfig> out;
  for (std::size_t si = 0; si < space.skus.size(); ++si) {
    const DeviceProfile& dev = space.skus[si];
    for (auto tp : space.tp_degrees) {
      for (auto pp : space.pp_degrees) {
        const std::string stem =
            dev.sku_name + "_tp" + std::to_string(tp) + "_pp" + std::to_string(pp);
        auto skip = [&](const char* why) {
          if (skipped) skipped->push_back({stem, why});
        };
        if (tp * pp > space.max_gpus_total) {
          skip("needs more GPUs than the budget");
          continue;
        }
        ParallelismConfig par{tp, pp, space.max_gpus_total / (tp * pp)};
        if (spec.num_kv_heads % tp != 0) {
          skip("num_kv_heads not divisible by tp_degree");
          continue;
        }
        if (spec.num_layers % pp != 0) {
          skip("num_layers not divisible by pp_degree");
          continue;
        }
        for (auto sched : space.schedulers) {
          const bool chunked = sched == SchedulerPolicy::SarathiServe;
          const std::vector<std::int64_t> no_chunk{0};
          const auto& chunks = chunked ? space.chunk_sizes : no_chunk;
          for (auto bs : space.batch_sizes) {
            for (auto cs : chunks) {
              CandidateConfig c;
              c.sku_index = si;
              c.par = par;
              c.policy = base;
              c.policy.policy = sched;
              c.policy.max_batch_size = bs;
              if (cs > 0) c.policy.chunk_size = cs;
              std::ostringstream id;
              id << dev.sku_name << "_tp" << tp << "_pp" << pp << "_r" << par.num_replicas << "_"
                 << to_string(sched) << "_bs" << bs;
              if (chunked) id << "_cs" << c.policy.chunk_size;
              c.id = id.str();
              out.push_back(std::move(c));
            }
          }
        }
      }
    }
  }
  return out;
}

double qps_per_dollar(double capacity_qps, std::int64_t gpus_used, double rate_per_gpu_hr) {
  require(rate_per_gpu_hr > 0, "qps_per_dollar: rate must be positive");
  require(gpus_used >= 1, "qps_per_dollar: need at least one GPU");
  return capacity_qps / (static_cast<double>(gpus_used) * rate_per_gpu_hr);
}

static double hourly_rate(const CostTable& cost, const std::string& sku) {
  auto it = cost.find(sku);
  require(it != cost.end(), "cost table: unknown SKU '" + sku + "'");
  require(it->second > 0, "cost table: rate for '" + sku + "' must be positive");
  return it->second;
}

std::vector<std::size_t> pareto_frontier(const std::vector<ParetoPoint>& pts) {
  require(!pts.empty(), "pareto_frontier: empty point set");
  std::vector<std::size_t> out;
  for (std::size_t i = 0; i < pts.size(); ++i) {
    bool dominated = false;
    for (std::size_t j = 0; j < pts.size() && !dominated; ++j) {
      if (j == i) continue;
      const bool no_worse = pts[j].latency <= pts[i].latency && pts[j].value >= pts[i].value;
      const bool better = pts[j].latency < pts[i].latency || pts[j].value > pts[i].value;
      dominated = no_worse && better;
    }
    if (!dominated) out.push_back(i);
  }
  return out;
}

// ------------------------------------------------------------------ capacity replay
namespace {

struct NeedProbe {
  double q;
  int phase;  // 0 doubling, 1 halving, 2 bisection
  double lo, hi;
};

// The reference's find_capacity (search.hpp:145-174) against a memo; throws
// NeedProbe on the first unanswered rate.
double replay_capacity(const std::unordered_map<double, bool>& memo, const CapacitySearchOptions& o) {
  auto ask = [&](double q, int phase, double lo, double hi) {
    auto it = memo.find(q);
    if (it == memo.end()) throw NeedProbe{q, phase, lo, hi};
    return it->second;
  };
  require(o.initial_guess > 0 && o.tolerance > 0, "find_capacity: bad options");
  double lo = 0.0, hi = o.initial_guess;
  while (ask(hi, 0, lo, hi)) {
    lo = hi;
    hi *= 2.0;
    require(hi <= o.max_qps,
            "capacity probe never saturated (delay threshold unreachable); increase probe_requests");
  }
  if (lo == 0.0) {
    while (hi > o.min_qps && !ask(hi / 2.0, 1, lo, hi)) hi /= 2.0;
    if (hi <= o.min_qps) return 0.0;
    lo = hi / 2.0;
  }
  while (hi - lo > o.tolerance * hi) {
    const double mid = 0.5 * (lo + hi);
    if (ask(mid, 2, lo, hi))
      lo = mid;
    else
      hi = mid;
  }
  return lo;
}

// Rates the search may ask right after `need` (speculation; never affects
// the answer, only how many rounds it takes).
void speculate(const NeedProbe& need, const CapacitySearchOptions& o, int ladder, int depth,
               std::vector<double>& out) {
  out.push_back(need.q);
  if (need.phase == 0) {
    double q = need.q;
    for (int k = 1; k < ladder; ++k) {
      q *= 2.0;
      if (q > o.max_qps) break;
      out.push_back(q);
    }
  } else if (need.phase == 1) {
    double hi = need.hi / 2.0;
    for (int k = 1; k < ladder && hi > o.min_qps; ++k) {
      out.push_back(hi / 2.0);
      hi /= 2.0;
    }
  } else {
    // bisection sub-tree below (lo, hi) to `depth` levels
    std::vector<std::pair<double, double>> level{{need.lo, need.hi}}, next;
    for (int d = 0; d < depth; ++d) {
      next.clear();
      for (auto [lo, hi] : level) {
        if (!(hi - lo > o.tolerance * hi)) continue;
        const double mid = 0.5 * (lo + hi);
        if (d > 0) out.push_back(mid);
        next.push_back({lo, mid});
        next.push_back({mid, hi});
      }
      level.swap(next);
    }
  }
}

struct Workload {
  std::vector<Request> lengths;  // probe trace (ids 0..n-1)
  std::vector<double> unit_exp;  // E_i of the probe seed
};

// Arrivals of one probe: t += max(E_i / qps, 1e-12) (workload.hpp:96-103).
void probe_arrivals(const Workload& w, double qps, std::vector<Request>& out) {
  out = w.lengths;
  double t = 0.0;
  for (std::size_t i = 0; i < out.size(); ++i) {
    t += std::max(w.unit_exp[i] / qps, 1e-12);
    out[i].arrival_time = t;
  }
}

struct Candidate {
  std::size_t index;  // enumeration index
  CandidateConfig cand;
  ClusterConfig cluster;
  const EstimatorModel* est = nullptr;
  int32_t est_slot = 0;
  SimConfig sim{};
  bool sim_ok = false;  // make_sim_config succeeded (else the first probe raises)
  std::string sim_error;
  int sim_error_kind = 0;  // 1 Error, 2 InternalError
  double guess = 0;
  CapacitySearchOptions copts;
  std::unordered_map<double, bool> memo;
  bool done = false;
  ConfigResult res;
};

// One probe = one full arrival sequence at `qps` for one candidate.
struct ProbeSlot {
  std::size_t cand;
  double qps;
  int32_t first_unit, nunits;
  bool coupled;
};

// Adds a probe (or an SLO / static run) of candidate C to `jobs`.
ProbeSlot add_probe(SimJobs& jobs, const Candidate& C, int32_t config_index,
                    const std::vector<Request>& trace, int flags, double thr, int32_t max_late,
                    bool coupled) {
  ProbeSlot p{};
  p.first_unit = static_cast<int32_t>(jobs.units.size());
  const int R = static_cast<int>(C.cluster.par.num_replicas);
  UnitSpec us;
  us.config = config_index;
  us.flags = flags;
  us.abort_thr = thr;
  us.abort_max_late = max_late;
  // arrivals are strictly increasing and ids ascend with the trace index, so
  // (arrival, id) order == trace order == arrival-event order
  if (C.cluster.routing == RoutingPolicy::RoundRobin && !coupled) {
    us.R = 1;
    for (int r = 0; r < R; ++r) {
      std::vector<Request> sub;
      for (std::size_t i = r; i < trace.size(); i += R) sub.push_back(trace[i]);
      jobs.add_unit(us, sub, {});
    }
    p.nunits = R;
  } else {
    us.R = R;
    jobs.add_unit(us, trace, {});
    p.nunits = 1;
    p.coupled = true;
  }
  return p;
}

}  // namespace

double initial_qps_guess(const ModelSpec& spec, const CandidateConfig& cand,
                         const EstimatorModel& est, const ClusterConfig& cluster) {
  auto ops = derive_operators(spec, cand.par);
  SimConfig cfg{};
  // predict's find() order over the two compositions (prefill: attn_decode is
  // skipped before any lookup; decode: attn_prefill is)
  for (int pass = 0; pass < 2; ++pass)
    for (const auto& d : ops) {
      if (pass == 0 && d.op == OpName::AttnDecode) continue;
      if (pass == 1 && d.op == OpName::AttnPrefill) continue;
      est.find(d.op, d.tp_degree);
    }
  fill_sim_ops(cfg, ops, est.device());
  const std::int64_t len = std::min<std::int64_t>(512, spec.max_context);
  const int64_t p_off[3] = {0, 1, 1}, d_off[3] = {0, 0, 1};
  const int64_t p_len[1] = {len}, p_prior[1] = {0}, d_ctx[1] = {len};
  double secs[2], fl[2];
  predict_batches(est, cfg, 2, p_off, p_len, p_prior, d_off, d_ctx, secs, fl);
  const double service = secs[0] + 64.0 * secs[1];
  const double per_replica = 1.0 / std::max(service, 1e-9);
  return std::max(1e-3, per_replica * static_cast<double>(cluster.par.num_replicas));
}

double find_capacity_replay(const std::function<bool(double)>& feasible,
                            const CapacitySearchOptions& opts) {
  std::unordered_map<double, bool> memo;
  while (true) {
    try {
      return replay_capacity(memo, opts);
    } catch (const NeedProbe& n) {
      memo[n.q] = feasible(n.q);
    }
  }
}

// ------------------------------------------------------------------ the sweep
namespace {

struct SweepKnobs {
  int ladder = 4;  // doubling / halving rates probed per round
  int depth = 3;   // bisection levels probed per round (2^depth - 1 rates)
};

SweepKnobs knobs_from_env() {
  SweepKnobs k;
  if (const char* s = std::getenv("SSG_SPEC_LADDER")) k.ladder = std::max(1, std::atoi(s));
  if (const char* s = std::getenv("SSG_SPEC_DEPTH")) k.depth = std::max(1, std::atoi(s));
  return k;
}

// Runs one launch of probes; answers are written into the candidates' memos.
// Errors inside a probe end that candidate's evaluation (as the reference's
// exception would), unless the probe aborted first.
void run_probe_round(std::vector<Candidate>& cands, const std::vector<std::size_t>& active,
                     const std::vector<std::vector<double>>& rates, const Workload& w,
                     const CapacitySearchOptions& base) {
  SimJobs jobs;
  std::unordered_map<const EstimatorModel*, int32_t> est_index;
  std::vector<ProbeSlot> slots;
  const std::size_t n = w.lengths.size();
  const int32_t max_late =
      static_cast<int32_t>(n - static_cast<std::size_t>(std::ceil(0.99 * static_cast<double>(n))));
  std::vector<Request> trace;
  for (std::size_t a = 0; a < active.size(); ++a) {
    Candidate& C = cands[active[a]];
    auto it = est_index.find(C.est);
    if (it == est_index.end()) {
      it = est_index.emplace(C.est, static_cast<int32_t>(jobs.ests.size())).first;
      jobs.ests.push_back(C.est->device().view);
    }
    SimConfig sc = C.sim;
    sc.est = it->second;
    const int32_t ci = static_cast<int32_t>(jobs.configs.size());
    jobs.configs.push_back(sc);
    for (double q : rates[a]) {
      probe_arrivals(w, q, trace);
      ProbeSlot p = add_probe(jobs, C, ci, trace, SSG_UF_ABORT, base.delay_p99_threshold, max_late, false);
      p.cand = active[a];
      p.qps = q;
      slots.push_back(p);
    }
  }
  SimResults res;
  run_jobs(jobs, res, false);
  std::vector<std::size_t> redo;  // probes needing the exact coupled event order
  for (std::size_t k = 0; k < slots.size(); ++k) {
    const ProbeSlot& p = slots[k];
    Candidate& C = cands[p.cand];
    int64_t late = 0;
    int errors = 0;
    bool aborted = false;
    for (int32_t u = p.first_unit; u < p.first_unit + p.nunits; ++u) {
      late += res.out[u].late;
      aborted |= res.out[u].aborted != 0;
      errors += res.out[u].code != SSG_OK;
    }
    if (errors == 0) {
      C.memo[p.qps] = !aborted && late <= max_late;
      continue;
    }
    if (!p.coupled && static_cast<int>(C.cluster.par.num_replicas) <= kMaxCoupledReplicas) {
      redo.push_back(k);
      continue;
    }
    // coupled unit: exact reference order -- an abort ends the probe before any
    // later error; otherwise the error is the probe's (and the config's) outcome
    const SimUnitOut* e = nullptr;
    for (int32_t u = p.first_unit; u < p.first_unit + p.nunits; ++u)
      if (res.out[u].code != SSG_OK && (!e || res.out[u].err_time < e->err_time)) e = &res.out[u];
    if (aborted && p.coupled) {
      C.memo[p.qps] = false;
      continue;
    }
    try {
      raise_unit_error(*e, C.sim, *C.est);
    } catch (const Error& ex) {
      C.res.error = ex.what();
      C.done = true;
    }
  }
  if (redo.empty()) return;
  // replay the ambiguous probes with all replicas in one unit
  SimJobs j2;
  j2.ests = jobs.ests;
  std::vector<ProbeSlot> s2;
  for (std::size_t k : redo) {
    const ProbeSlot& p = slots[k];
    Candidate& C = cands[p.cand];
    const int32_t ci = static_cast<int32_t>(j2.configs.size());
    j2.configs.push_back(jobs.configs[jobs.units[p.first_unit].config]);
    probe_arrivals(w, p.qps, trace);
    ProbeSlot q = add_probe(j2, C, ci, trace, SSG_UF_ABORT, base.delay_p99_threshold, max_late, true);
    q.cand = p.cand;
    q.qps = p.qps;
    s2.push_back(q);
  }
  SimResults r2;
  run_jobs(j2, r2, false);
  for (const auto& p : s2) {
    Candidate& C = cands[p.cand];
    const SimUnitOut& o = r2.out[p.first_unit];
    if (o.aborted) {
      C.memo[p.qps] = false;
    } else if (o.code == SSG_OK) {
      C.memo[p.qps] = o.late <= max_late;
    } else {
      try {
        raise_unit_error(o, C.sim, *C.est);
      } catch (const Error& ex) {
        C.res.error = ex.what();
        C.done = true;
      }
    }
  }
}

// Full runs (SLO measurement or the static makespan run) of several
// candidates in one launch, then their TTFT p90 / TBT p99 / delay p99 by one
// segmented select.  `qps` <= 0 means the static run (all arrivals at 0).
void run_measurements(std::vector<Candidate>& cands, const std::vector<std::size_t>& which,
                      const std::vector<double>& qps, const Workload& w, bool static_run) {
  if (which.empty()) return;
  SimJobs jobs;
  std::unordered_map<const EstimatorModel*, int32_t> est_index;
  std::vector<ProbeSlot> slots;
  std::vector<Request> trace;
  for (std::size_t a = 0; a < which.size(); ++a) {
    Candidate& C = cands[which[a]];
    auto it = est_index.find(C.est);
    if (it == est_index.end()) {
      it = est_index.emplace(C.est, static_cast<int32_t>(jobs.ests.size())).first;
      jobs.ests.push_back(C.est->device().view);
    }
    SimConfig sc = C.sim;
    sc.est = it->second;
    const int32_t ci = static_cast<int32_t>(jobs.configs.size());
    jobs.configs.push_back(sc);
    if (static_run) {
      trace = w.lengths;
      for (auto& r : trace) r.arrival_time = 0.0;
    } else {
      probe_arrivals(w, qps[a], trace);
    }
    // static runs put every arrival at t=0: the event order is the trace
    // order and RR still splits by position, so replicas stay independent
    ProbeSlot p = add_probe(jobs, C, ci, trace, SSG_UF_EMISSIONS, 0.0, 0, false);
    p.cand = which[a];
    slots.push_back(p);
  }
  SimResults res;
  auto& ctx = context();
  cudaStream_t s = ctx.stream;
  run_jobs(jobs, res, true);
  // errors first (a failing SLO run fails the config)
  std::vector<char> ok(slots.size(), 1);
  for (std::size_t k = 0; k < slots.size(); ++k) {
    const ProbeSlot& p = slots[k];
    const SimUnitOut* e = nullptr;
    for (int32_t u = p.first_unit; u < p.first_unit + p.nunits; ++u)
      if (res.out[u].code != SSG_OK && (!e || res.out[u].err_time < e->err_time)) e = &res.out[u];
    if (!e) continue;
    ok[k] = 0;
    Candidate& C = cands[p.cand];
    try {
      raise_unit_error(*e, C.sim, *C.est);
    } catch (const Error& ex) {
      C.res.error = ex.what();
      C.done = true;
    }
  }
  // samples: per request delay and TTFT; per emission gap (first emission of
  // each request marked +inf, which sorts last and never reaches the ranks)
  const std::size_t nreq = jobs.tm.size();
  std::vector<double> delay(nreq), ttft(nreq), tbt(static_cast<std::size_t>(jobs.emissions));
  for (std::size_t g = 0; g < nreq; ++g) {
    delay[g] = res.tm[g].first_sched - res.tm[g].arrival;
    ttft[g] = res.tm[g].first_tok - res.tm[g].arrival;
  }
  for (std::size_t g = 0; g < nreq; ++g) {
    const int64_t b = jobs.emit_base[g];
    const int64_t d = jobs.hot[g].decode;
    tbt[b] = INFINITY;
    for (int64_t k = 1; k < d; ++k) tbt[b + k] = res.emissions[b + k] - res.emissions[b + k - 1];
  }
  // segments: [delay of probe k] [ttft of probe k] [tbt of probe k]
  std::vector<double> pool;
  std::vector<int64_t> off{0};
  std::vector<SelectTask> tasks;
  std::vector<int64_t> tbt_count(slots.size());
  for (std::size_t k = 0; k < slots.size(); ++k) {
    const ProbeSlot& p = slots[k];
    const SimUnit& u0 = jobs.units[p.first_unit];
    const SimUnit& u1 = jobs.units[p.first_unit + p.nunits - 1];
    const int64_t r0 = u0.req_off, r1 = u1.req_off + u1.n;
    const int64_t e0 = jobs.emit_base[r0], e1 = jobs.emit_base[r1 - 1] + jobs.hot[r1 - 1].decode;
    const int64_t nr = r1 - r0, nt = (e1 - e0) - nr;
    tbt_count[k] = nt;
    pool.insert(pool.end(), delay.begin() + r0, delay.begin() + r1);
    off.push_back(static_cast<int64_t>(pool.size()));
    pool.insert(pool.end(), ttft.begin() + r0, ttft.begin() + r1);
    off.push_back(static_cast<int64_t>(pool.size()));
    pool.insert(pool.end(), tbt.begin() + e0, tbt.begin() + e1);
    off.push_back(static_cast<int64_t>(pool.size()));
    const int64_t seg = 3 * static_cast<int64_t>(k);
    tasks.push_back({seg + 0, nearest_rank_index(nr, 0.99)});
    tasks.push_back({seg + 1, nearest_rank_index(nr, 0.90)});
    tasks.push_back({seg + 2, nt > 0 ? nearest_rank_index(nt, 0.99) : 0});
  }
  DeviceBuffer<double> d_pool, d_out;
  DeviceBuffer<int64_t> d_off;
  DeviceBuffer<SelectTask> d_tasks;
  d_pool.upload(pool, s);
  d_off.upload(off, s);
  d_tasks.upload(tasks, s);
  d_out.resize(tasks.size());
  launch_select(d_pool.ptr, d_off.ptr, d_tasks.ptr, static_cast<int64_t>(tasks.size()), d_out.ptr, s);
  std::vector<double> sel(tasks.size());
  d_out.download(sel.data(), sel.size(), s);
  cuda_check(cudaStreamSynchronize(s), "slo select");
  for (std::size_t k = 0; k < slots.size(); ++k) {
    if (!ok[k]) continue;
    Candidate& C = cands[slots[k].cand];
    const bool has_tbt = tbt_count[k] > 0;
    C.res.delay_p99 = sel[3 * k + 0];
    C.res.ttft_p90 = sel[3 * k + 1];
    C.res.tbt_p99 = has_tbt ? sel[3 * k + 2] : 0.0;  // summarize({}) leaves 0
    if (static_run) {
      double span = 0.0;
      for (int32_t u = slots[k].first_unit; u < slots[k].first_unit + slots[k].nunits; ++u)
        span = std::max(span, res.out[u].span);
      C.res.makespan = span;
    }
  }
}

}  // namespace

struct SearchSession::State {
  ModelSpec spec;
  SearchOptions opts;
  std::vector<CandidateConfig> configs;
  std::vector<EstimatorModel> ests;
  Workload w;
};

SearchSession::SearchSession(const ModelSpec& spec, const std::vector<Request>& workload,
                             const SearchOptions& opts)
    : st_(std::make_unique<State>()) {
  State& S = *st_;
  S.spec = spec;
  S.opts = opts;
  PolicyConfig base;
  S.configs = enumerate_configs(spec, opts.space, base);
  require(!S.configs.empty(), "search: empty configuration space");
  // one shared estimator per SKU over every valid tp (search.hpp:248-260)
  std::vector<std::int64_t> tps;
  for (auto tp : opts.space.tp_degrees)
    if (spec.num_kv_heads % tp == 0) tps.push_back(tp);
  require(!tps.empty(), "search: no valid tp degree for this model");
  for (const auto& sku : opts.space.skus)
    S.ests.push_back(train(generate_synthetic_profile(spec, sku, tps), opts.train));
  for (const auto& e : S.ests) e.device();  // resident in HBM before any timed work
  require(!workload.empty(), "search: empty workload");
  for (std::size_t i = 0; i < opts.capacity.probe_requests; ++i) {
    Request r = workload[i % workload.size()];
    r.id = static_cast<std::int64_t>(i);
    S.w.lengths.push_back(r);
  }
  S.w.unit_exp = unit_exponentials(S.w.lengths.size(), opts.capacity.seed);
}

SearchSession::~SearchSession() = default;

std::size_t SearchSession::num_configs() const { return st_->configs.size(); }

std::vector<ConfigResult> evaluate_configs_shard(const ModelSpec& spec,
                                                 const std::vector<Request>& workload,
                                                 const SearchOptions& opts, int shard,
                                                 int num_shards) {
  SearchSession session(spec, workload, opts);
  return session.evaluate(shard, num_shards);
}

std::vector<ConfigResult> SearchSession::evaluate(int shard, int num_shards) {
  const State& S = *st_;
  const ModelSpec& spec = S.spec;
  const SearchOptions& opts = S.opts;
  const auto& configs = S.configs;
  const auto& ests = S.ests;
  const Workload& w = S.w;
  std::vector<ConfigResult> results(configs.size());
  std::vector<Candidate> cands;
  for (std::size_t i = 0; i < configs.size(); ++i) {
    if (static_cast<int>(i % static_cast<std::size_t>(num_shards)) != shard) continue;
    const CandidateConfig& cand = configs[i];
    Candidate C;
    C.index = i;
    C.cand = cand;
    C.res.config = cand;
    C.res.sku_name = opts.space.skus[cand.sku_index].sku_name;
    C.cluster = ClusterConfig{spec, cand.par, opts.space.skus[cand.sku_index], cand.policy,
                              opts.routing, 0, opts.cpu_overhead_per_iter};
    C.est = &ests[cand.sku_index];
    C.copts = opts.capacity;
    try {
      C.sim = make_sim_config(C.cluster, *C.est, 0);
      C.sim_ok = true;
    } catch (const Error& e) {
      C.sim_error = e.what();
      C.sim_error_kind = 1;
    }
    cands.push_back(std::move(C));
  }

  const bool makespan = opts.objective == "makespan";
  std::vector<std::size_t> live;
  for (std::size_t k = 0; k < cands.size(); ++k) {
    Candidate& C = cands[k];
    if (makespan) {
      // the static run is the first simulation: its preamble errors surface
      if (!C.sim_ok) {
        C.res.error = C.sim_error;
        C.done = true;
      }
      continue;
    }
    try {
      C.guess = initial_qps_guess(spec, C.cand, *C.est, C.cluster);
      C.copts.initial_guess = C.guess;
      require(C.copts.initial_guess > 0 && C.copts.tolerance > 0, "find_capacity: bad options");
      // the first probe's run_simulation preamble (validation, plan_memory)
      if (!C.sim_ok) throw Error(C.sim_error);
      live.push_back(k);
    } catch (const Error& e) {
      C.res.error = e.what();
      C.done = true;
    }
  }

  if (makespan) {
    std::vector<std::size_t> ok;
    for (std::size_t k = 0; k < cands.size(); ++k)
      if (!cands[k].done) ok.push_back(k);
    run_measurements(cands, ok, {}, w, true);
    for (auto k : ok) {
      Candidate& C = cands[k];
      if (!C.res.failed()) {
        C.res.slo_pass = true;
        C.res.qps_per_dollar = 0.0;
      }
    }
  } else {
    const SweepKnobs knobs = knobs_from_env();
    // ---- capacity rounds
    while (!live.empty()) {
      std::vector<std::size_t> active;
      std::vector<std::vector<double>> rates;
      for (auto k : live) {
        Candidate& C = cands[k];
        if (C.done) continue;
        try {
          const double cap = replay_capacity(C.memo, C.copts);
          C.res.capacity_qps = cap;
          C.done = true;  // capacity known
        } catch (const NeedProbe& need) {
          std::vector<double> qs;
          speculate(need, C.copts, knobs.ladder, knobs.depth, qs);
          std::vector<double> fresh;
          for (double q : qs)
            if (!C.memo.count(q) && std::find(fresh.begin(), fresh.end(), q) == fresh.end())
              fresh.push_back(q);
          active.push_back(k);
          rates.push_back(fresh);
        } catch (const Error& e) {
          C.res.error = e.what();
          C.res.capacity_qps = 0.0;
          C.done = true;
        }
      }
      if (active.empty()) break;
      run_probe_round(cands, active, rates, w, opts.capacity);
      std::vector<std::size_t> still;
      for (auto k : active)
        if (!cands[k].done) still.push_back(k);
      live.swap(still);
    }
    // ---- SLO runs at evaluation_fraction of capacity
    std::vector<std::size_t> measure;
    std::vector<double> eval_qps;
    for (std::size_t k = 0; k < cands.size(); ++k) {
      Candidate& C = cands[k];
      if (C.res.failed()) continue;
      if (C.res.capacity_qps <= C.copts.min_qps) {
        C.res.capacity_qps = 0.0;
        C.res.error = "no feasible arrival rate (scheduling delay above threshold)";
        continue;
      }
      measure.push_back(k);
      eval_qps.push_back(opts.evaluation_fraction * C.res.capacity_qps);
    }
    for (double q : eval_qps) require(q > 0.0, "poisson_arrivals: rate must be positive");
    run_measurements(cands, measure, eval_qps, w, false);
    for (auto k : measure) {
      Candidate& C = cands[k];
      if (C.res.failed()) continue;
      C.res.slo_pass = C.res.ttft_p90 <= opts.slos.ttft_p90_max &&
                       C.res.tbt_p99 <= opts.slos.tbt_p99_max &&
                       C.res.delay_p99 <= opts.slos.delay_p99_max;
      try {
        C.res.qps_per_dollar = qps_per_dollar(C.res.capacity_qps, C.cluster.gpus_used(),
                                              hourly_rate(opts.cost, C.res.sku_name));
      } catch (const Error& e) {
        C.res.error = e.what();
      }
    }
  }
  for (auto& C : cands) results[C.index] = std::move(C.res);
  for (std::size_t i = 0; i < configs.size(); ++i)
    if (results[i].config.id.empty()) results[i].config = configs[i];
  return results;
}

SearchOutcome finalize_search(const ModelSpec& spec, const SearchOptions& opts,
                              std::vector<ConfigResult> results) {
  SearchOutcome outcome;
  PolicyConfig base;
  enumerate_configs(spec, opts.space, base, &outcome.skipped);
  outcome.results = std::move(results);
  for (std::size_t i = 0; i < outcome.results.size(); ++i)
    if (!outcome.results[i].failed() && outcome.results[i].slo_pass) outcome.ranking.push_back(i);
  const bool by_makespan = opts.objective == "makespan";
  std::sort(outcome.ranking.begin(), outcome.ranking.end(), [&](std::size_t a, std::size_t b) {
    const auto& ra = outcome.results[a];
    const auto& rb = outcome.results[b];
    if (by_makespan) {
      if (ra.makespan != rb.makespan) return ra.makespan < rb.makespan;
    } else if (ra.qps_per_dollar != rb.qps_per_dollar) {
      return ra.qps_per_dollar > rb.qps_per_dollar;
    }
    return ra.config.id < rb.config.id;
  });
  if (!outcome.ranking.empty()) outcome.best = outcome.ranking.front();
  std::vector<ParetoPoint> ttft, tbt;
  std::vector<std::size_t> ok;
  for (std::size_t i = 0; i < outcome.results.size(); ++i) {
    const auto& r = outcome.results[i];
    if (r.failed() || r.capacity_qps <= 0) continue;
    ok.push_back(i);
    ttft.push_back({r.ttft_p90, r.qps_per_dollar});
    tbt.push_back({r.tbt_p99, r.qps_per_dollar});
  }
  if (!ok.empty()) {
    for (auto k : pareto_frontier(ttft)) outcome.frontier_ttft.push_back(ok[k]);
    for (auto k : pareto_frontier(tbt)) outcome.frontier_tbt.push_back(ok[k]);
  }
  return outcome;
}

SearchOutcome run_search(const ModelSpec& spec, const std::vector<Request>& workload,
                         const SearchOptions& opts) {
  return finalize_search(spec, opts, evaluate_configs_shard(spec, workload, opts, 0, 1));
}

// ------------------------------------------------------------------ writers
std::string search_results_to_csv(const SearchOutcome& outcome) {
  std::ostringstream out;
  out << "config_id,sku,tp,pp,replicas,policy,max_batch_size,chunk_size,capacity_qps,"
         "qps_per_dollar,ttft_p90_s,tbt_p99_s,delay_p99_s,makespan_s,slo_pass,error\n";
  for (const auto& r : outcome.results) {
    const auto& c = r.config;
    out << c.id << ',' << r.sku_name << ',' << c.par.tp_degree << ',' << c.par.pp_degree << ','
        << c.par.num_replicas << ',' << to_string(c.policy.policy) << ',' << c.policy.max_batch_size
        << ','
        << (c.policy.policy == SchedulerPolicy::SarathiServe ? std::to_string(c.policy.chunk_size)
                                                             : std::string())
        << ',' << fmt_double(r.capacity_qps) << ',' << fmt_double(r.qps_per_dollar) << ','
        << fmt_double(r.ttft_p90) << ',' << fmt_double(r.tbt_p99) << ',' << fmt_double(r.delay_p99)
        << ',' << fmt_double(r.makespan) << ',' << (r.slo_pass ? "true" : "false") << ','
        << r.error << "\n";
  }
  return out.str();
}

std::string frontier_to_csv(const SearchOutcome& outcome, const std::vector<std::size_t>& frontier,
                            bool use_ttft) {
  std::ostringstream out;
  out << "config_id,latency_metric,qps_per_dollar,slo_pass\n";
  for (auto i : frontier) {
    const auto& r = outcome.results[i];
    out << r.config.id << ',' << fmt_double(use_ttft ? r.ttft_p90 : r.tbt_p99) << ','
        << fmt_double(r.qps_per_dollar) << ',' << (r.slo_pass ? "true" : "false") << "\n";
  }
  return out.str();
}

std::string search_summary_text(const SearchOutcome& outcome, const std::string& objective) {
  std::ostringstream out;
  std::size_t failed = 0;
  for (const auto& r : outcome.results) failed += r.failed() ? 1 : 0;
  out << "configs evaluated: " << outcome.results.size() << " (" << failed << " failed, "
      << outcome.skipped.size() << " skipped)\n";
  for (const auto& s : outcome.skipped) out << "  skipped " << s.id << ": " << s.reason << "\n";
  if (outcome.best) {
    const auto& b = outcome.results[*outcome.best];
    out << "optimum (" << objective << "): " << b.config.id;
    if (objective == "makespan")
      out << " makespan " << fmt_double(b.makespan) << " s\n";
    else
      out << " capacity " << fmt_double(b.capacity_qps) << " qps, " << fmt_double(b.qps_per_dollar)
          << " qps per dollar-hour\n";
  } else {
    out << "no configuration satisfied the SLOs\n";
  }
  return out.str();
}

}  // namespace servesim
