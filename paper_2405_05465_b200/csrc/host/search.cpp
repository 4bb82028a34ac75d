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
#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <exception>
#include <map>
#include <memory>
#include <mutex>
#include <sstream>
#include <thread>
#include <unordered_map>

#include "engine_limits.h"
#include "select.h"
#include "servesim_b200.hpp"
#include "sim_host.h"
#include "sweep.h"

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

// A probe rate's answer: feasible / infeasible, or the Error its simulation
// raised.  Errors are memoised like answers and surface only when the replay
// actually asks for that rate: a speculative rate the sequential search never
// reaches cannot turn a successful evaluation into an error row.
struct ProbeAnswer {
  bool feasible = false;
  bool error = false;
  SimUnitOut err{};  // the failing unit (error == true)
  // device work of the probe's simulation (its units summed): the sequential
  // search's share of the sweep is the work of the rates its replay asks for
  int64_t iters = 0, entries = 0, bytes = 0;
};
using ProbeMemo = std::unordered_map<double, ProbeAnswer>;

struct ProbeError {
  SimUnitOut err;
};

void add_work(ProbeAnswer& a, const SimUnitOut& o) {
  a.iters += o.iterations;
  a.entries += o.entries;
  a.bytes += o.qbytes + 48 * o.entries;  // predictor bytes + 48 B per entry
}

// The reference's find_capacity (search.hpp:145-174) against a memo; throws
// NeedProbe on the first unanswered rate and ProbeError when the asked rate's
// simulation raised (the reference's feasible(q) throwing out of find_capacity).
double replay_capacity(const ProbeMemo& memo, const CapacitySearchOptions& o,
                       std::vector<const ProbeAnswer*>* asked = nullptr) {
  auto ask = [&](double q, int phase, double lo, double hi) {
    auto it = memo.find(q);
    if (it == memo.end()) throw NeedProbe{q, phase, lo, hi};
    if (asked) asked->push_back(&it->second);
    if (it->second.error) throw ProbeError{it->second.err};
    return it->second.feasible;
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
// the answer, only how many rounds it takes), each with the indices (into
// `out`) of the earlier rates that must come out feasible for the replay to
// ask it: a failure of any of them cancels it on the device (SimUnit::kill).
struct SpecRate {
  double q;
  std::vector<int> after_feasible;
};

// One candidate's unanswered rates for a round, with their cancel masks.
struct SpecProbes {
  std::size_t k = 0;  // candidate
  std::vector<double> rates;
  std::vector<uint32_t> kill;
};

// Bisection sub-tree below (lo, hi) to `depth` levels: an interval's mid is
// asked once the interval is reached; its upper half is reached only when the
// mid is feasible (its lower half when it is not, which no early failure can
// tell, so that half inherits its parent's conditions only).  `root` is the
// index of the root's mid when it is already in `out` (-1: add it).
void speculate_subtree(double lo, double hi, const std::vector<int>& cond, int root, int depth,
                       const CapacitySearchOptions& o, std::vector<SpecRate>& out) {
  struct Interval {
    double lo, hi;
    std::vector<int> cond;  // indices into out that must be feasible
  };
  std::vector<Interval> level{{lo, hi, cond}}, next;
  for (int d = 0; d < depth; ++d) {
    next.clear();
    for (const Interval& iv : level) {
      if (!(iv.hi - iv.lo > o.tolerance * iv.hi)) continue;
      const double mid = 0.5 * (iv.lo + iv.hi);
      int idx = root;
      if (d > 0 || root < 0) {
        idx = static_cast<int>(out.size());
        out.push_back({mid, iv.cond});
      }
      next.push_back({iv.lo, mid, iv.cond});
      std::vector<int> up = iv.cond;
      up.push_back(idx);
      next.push_back({mid, iv.hi, up});
    }
    level.swap(next);
  }
}

void speculate(const NeedProbe& need, const CapacitySearchOptions& o, int ladder, int depth,
               int pre_depth, std::vector<SpecRate>& out) {
  out.push_back({need.q, {}});
  if (need.phase == 0) {
    // doubling: rung k is asked only after rungs 0..k-1 were feasible
    double q = need.q;
    std::vector<int> rung{0};
    for (int k = 1; k < ladder; ++k) {
      q *= 2.0;
      if (q > o.max_qps) break;
      std::vector<int> prev(out.size());
      for (std::size_t i = 0; i < prev.size(); ++i) prev[i] = static_cast<int>(i);
      rung.push_back(static_cast<int>(out.size()));
      out.push_back({q, prev});
    }
    // under-loaded sweeps: the first bisection levels of every bracket the ladder
    // can end in (rung k-1 feasible, rung k not), asked after rungs 0..k-1; the
    // bracket below rung 0 exists once an earlier round found a feasible rate
    if (pre_depth <= 0) return;
    if (need.lo > 0.0) speculate_subtree(need.lo, need.q, {}, -1, pre_depth, o, out);
    for (std::size_t k = 1; k < rung.size(); ++k) {
      std::vector<int> cond(rung.begin(), rung.begin() + static_cast<std::ptrdiff_t>(k));
      speculate_subtree(out[rung[k - 1]].q, out[rung[k]].q, cond, -1, pre_depth, o, out);
    }
  } else if (need.phase == 1) {
    // halving: each deeper rate is the slowest probe of its round (iterations
    // grow ~1/qps), and the first halving usually suffices -- no speculation
  } else {
    speculate_subtree(need.lo, need.hi, {}, 0, depth, o, out);
  }
}

struct Workload {
  std::vector<Request> lengths;  // probe trace (ids 0..n-1)
  std::vector<double> unit_exp;  // E_i of the probe seed
};

struct Candidate {
  std::size_t index;  // enumeration index
  CandidateConfig cand;
  ClusterConfig cluster;
  const EstimatorModel* est = nullptr;
  SimConfig sim{};
  bool sim_ok = false;  // make_sim_config succeeded (else the first probe raises)
  std::string sim_error;
  CapacitySearchOptions copts;
  ProbeMemo memo;
  bool done = false;       // evaluation finished (capacity known, or failed)
  bool measured = false;   // SLO / static run taken
  int64_t probe_iters = 0; // longest probe unit so far (iterations): speculation budget
  int rounds = 0;          // rounds with probes so far
  int bisect_from = -1;    // rounds before its first bisection round
  // speculative SLO runs: taken in the round whose probes settle the capacity, at
  // evaluation_fraction x every capacity the replay can still end with; the one the
  // replay does end with is the SLO run the sequential search would make next
  struct SpecFull {
    std::vector<SimUnitOut> out;  // the run's units (ProbeDesc::first_unit = 0)
    ProbeDesc p;
    double sel3[3];
  };
  std::unordered_map<double, SpecFull> spec_full;
  ProbeAnswer full_run;    // work of the SLO / static run (iters, entries, bytes)
  ConfigResult res;
};

// Persistent (grow-only) device buffers of the sweep's launches.
struct SweepBuffers {
  DeviceBuffer<SimConfig> cfg;
  DeviceBuffer<SsgEstView> est;
  DeviceBuffer<SimUnit> units;
  DeviceBuffer<ProbeDesc> probes, mprobes;
  DeviceBuffer<int32_t> order, ws, restarts;
  DeviceBuffer<ReqHot> hot;
  DeviceBuffer<ReqTimes> tm;
  DeviceBuffer<int64_t> ids, emit_base, seg_off;
  DeviceBuffer<double> emis, samples, sel;
  DeviceBuffer<RepState> reps;
  DeviceBuffer<SimUnitOut> out;
  DeviceBuffer<SelectTask> tasks;
  DeviceBuffer<uint32_t> group_fail;  // per speculation group: bits of its failed probes
};

// A launch under construction: per-candidate configs, probes and their units.
struct ProbeLaunch {
  std::vector<SimConfig> configs;
  std::vector<SsgEstView> ests;
  std::unordered_map<const EstimatorModel*, int32_t> est_index;
  std::vector<SimUnit> units;
  std::vector<ProbeDesc> probes;
  std::vector<std::size_t> probe_cand;
  std::vector<int32_t> measured;  // probe indices of full (measured) runs, slot order
  bool has_forest = false;
  int64_t nreq = 0, ws_words = 0, nreps = 0;

  int32_t add_config(const Candidate& C) {
    auto it = est_index.find(C.est);
    if (it == est_index.end()) {
      it = est_index.emplace(C.est, static_cast<int32_t>(ests.size())).first;
      ests.push_back(C.est->device().view);
      has_forest = has_forest || C.est->device().has_forest;
    }
    SimConfig sc = C.sim;
    sc.est = it->second;
    configs.push_back(sc);
    return static_cast<int32_t>(configs.size() - 1);
  }

  // One probe of candidate `cand` (config `ci`): RR replicas become independent
  // units (replica r owns trace positions r, r+R, ...), otherwise one coupled unit.
  int32_t ngroups = 0;  // speculation groups (SimUnit::group)

  void add_probe(std::size_t cand, const Candidate& C, int32_t ci, double qps, int32_t n, int flags,
                 double thr, int32_t max_late, bool coupled, bool static_run, int64_t emis_base,
                 int32_t group = -1, int32_t rung = 0, uint32_t kill = 0) {
    const SimConfig& cfg = configs[ci];
    const int R = static_cast<int>(C.cluster.par.num_replicas);
    ProbeDesc p{};
    p.qps = qps;
    p.R = R;
    p.first_unit = static_cast<int32_t>(units.size());
    p.decoupled = (C.cluster.routing == RoutingPolicy::RoundRobin && !coupled) ? 1 : 0;
    p.static_run = static_run ? 1 : 0;
    p.emis_base = emis_base;
    const int nu = p.decoupled ? R : 1;
    for (int r = 0; r < nu; ++r) {
      SimUnit u{};
      u.config = ci;
      u.n = p.decoupled ? (n - r + R - 1) / R : n;
      u.R = p.decoupled ? 1 : R;
      u.flags = flags;
      u.req_off = nreq;
      nreq += u.n;
      int64_t wc = 2;
      while (wc <= u.n) wc <<= 1;
      u.wait_cap = static_cast<int32_t>(wc);
      u.mb_ws = static_cast<int32_t>(std::min<int64_t>(cfg.max_batch, std::max<int32_t>(u.n, 1)));
      u.ws_off = ws_words;
      ws_words += static_cast<int64_t>(u.R) * (6LL * u.mb_ws + wc) + wc + 2 +
                  SSG_PP_SCRATCH_WORDS(cfg.pp);
      u.rep_off = nreps;
      nreps += u.R;
      u.abort_thr = thr;
      u.abort_max_late = max_late;
      u.group = group;
      u.rung = rung;
      u.kill = kill;
      units.push_back(u);
    }
    if (emis_base >= 0) measured.push_back(static_cast<int32_t>(probes.size()));
    probes.push_back(p);
    probe_cand.push_back(cand);
  }
  int64_t next_emis_base(int64_t per_probe) const {
    return static_cast<int64_t>(measured.size()) * per_probe;
  }
};

// Runs a launch entirely on the device: request streams built from the resident
// workload, simulation, and (measure) the SLO samples + their percentiles.
// Returns the per-unit outputs; `sel` gets delay p99, TTFT p90, TBT p99 per probe.
// Runs a launch entirely on the device: request streams built from the resident
// workload, simulation, and for the measured (full) runs the SLO samples and
// their percentiles.  `sel` gets delay p99, TTFT p90, TBT p99 per measured run
// (in L.measured order).
// A sweep lane: one stream and its launch buffers.  Candidate groups advance
// their capacity searches on separate lanes, so one group's long probes do not
// hold the others' next rounds (their launches overlap on the device).
struct SweepLane {
  struct Stream {
    cudaStream_t s = nullptr;
    Stream() { cuda_check(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking), "lane stream"); }
    ~Stream() {
      if (s) cudaStreamDestroy(s);
    }
  } stream;          // declared first: destroyed after the buffers freed on it
  SweepBuffers B;
  HostStaging staging;             // pinned: this lane's copies never touch pageable memory
  const double* tables = nullptr;  // token tables (session-wide, read-only)
  cudaEvent_t origin = nullptr;    // sweep start, for k_simulate busy intervals
  std::vector<std::pair<float, float>> intervals;
};

std::mutex g_dump_mu;

// Lanes outlive sessions: a process that opens search after search (the e2e
// bench, a service) reuses the streams, grow-only HBM buffers and pinned
// staging of earlier sessions instead of paying fresh allocations (+300 ms on
// a sweep's first launch, measured).  Sessions borrow lanes and give them back.
struct LanePool {
  std::mutex mu;
  std::vector<std::unique_ptr<SweepLane>> free;
};
LanePool& lane_pool() {
  static LanePool* pool = new LanePool;  // never destroyed: lanes may outlive static teardown
  return *pool;
}
std::unique_ptr<SweepLane> borrow_lane() {
  LanePool& p = lane_pool();
  {
    std::lock_guard<std::mutex> lk(p.mu);
    if (!p.free.empty()) {
      auto lane = std::move(p.free.back());
      p.free.pop_back();
      return lane;
    }
  }
  return std::make_unique<SweepLane>();
}

void run_launch(SweepLane& lane, ProbeLaunch& L, const ResidentWorkload& w,
                std::vector<SimUnitOut>& out, std::vector<double>& sel) {
  PhaseTimer timer("search: launch");
  SweepBuffers& B = lane.B;
  cudaStream_t s = lane.stream.s;
  const int32_t np = static_cast<int32_t>(L.probes.size());
  const int32_t nm = static_cast<int32_t>(L.measured.size());
  const bool emissions = nm > 0;
  B.cfg.upload(L.configs, s, lane.staging);
  B.est.upload(L.ests, s, lane.staging);
  B.units.upload(L.units, s, lane.staging);
  B.probes.upload(L.probes, s, lane.staging);
  B.hot.resize(std::max<int64_t>(1, L.nreq));
  B.tm.resize(std::max<int64_t>(1, L.nreq));
  B.ids.resize(std::max<int64_t>(1, L.nreq));
  B.restarts.resize(std::max<int64_t>(1, L.nreq));
  B.ws.resize(std::max<int64_t>(1, L.ws_words));
  B.reps.resize(std::max<int64_t>(1, L.nreps));
  B.out.resize(std::max<std::size_t>(1, L.units.size()));
  if (emissions) {
    B.emit_base.resize(std::max<int64_t>(1, L.nreq));
    B.emis.resize(std::max<int64_t>(1, w.emis_per_probe * nm));
  }
  // longest units first (fewest replicas share the trace => most requests per unit)
  std::vector<int32_t> order(L.units.size());
  for (std::size_t u = 0; u < order.size(); ++u) order[u] = static_cast<int32_t>(u);
  static const int sort_mode = [] {
    const char* e = std::getenv("SSG_UNIT_SORT");
    return e ? std::atoi(e) : 0;
  }();
  if (sort_mode == 1) {
    // length, then policy: co-resident warps share their scheduler's code
    std::stable_sort(order.begin(), order.end(), [&](int32_t a, int32_t b) {
      const auto& ua = L.units[a];
      const auto& ub = L.units[b];
      if (ua.n != ub.n) return ua.n > ub.n;
      return L.configs[ua.config].policy < L.configs[ub.config].policy;
    });
  } else {
    std::stable_sort(order.begin(), order.end(),
                     [&](int32_t a, int32_t b) { return L.units[a].n > L.units[b].n; });
  }
  B.order.upload(order, s, lane.staging);
  launch_probe_setup(B.probes.ptr, np, B.units.ptr, w, B.hot.ptr, B.tm.ptr, B.ids.ptr,
                     emissions ? B.emit_base.ptr : nullptr, s);
  SimLaunch K{};
  K.configs = B.cfg.ptr;
  K.units = B.units.ptr;
  K.order = B.order.ptr;
  K.nunits = static_cast<int64_t>(L.units.size());
  K.ests = B.est.ptr;
  K.hot = B.hot.ptr;
  K.tm = B.tm.ptr;
  K.ids = B.ids.ptr;
  K.restarts = B.restarts.ptr;
  K.emit_base = emissions ? B.emit_base.ptr : nullptr;
  K.emissions = emissions ? B.emis.ptr : nullptr;
  K.arr_order = nullptr;
  K.reps = B.reps.ptr;
  K.ws = B.ws.ptr;
  K.log = nullptr;
  K.out = B.out.ptr;
  K.tables = lane.tables;
  // decode fast-forward variant for every launch with at most SSG_FF_UNITS
  // units (default 54 per SM).  Measured on cfg #4 shards since the
  // fast-forward runs lane-parallel over iterations and through arrivals: it
  // beats the earlier threshold of 16 units per SM at every shard count (1/2
  // shard 0.944 -> 0.742 s), and only the two most loaded rounds of the full
  // sweep (~10K units: its 240-register body fits 8 warps per SM, the other
  // 12) still run faster without it (full sweep 1.188 -> 1.158 s with the cap).
  const int64_t ff_units = [] {
    const char* e = std::getenv("SSG_FF_UNITS");
    return e ? std::atoll(e) : 54LL * context().num_sms;
  }();
  K.fast_forward = sweep_fast_forward_enabled() ||
                   static_cast<int64_t>(L.units.size()) <= ff_units ? 1 : 0;
  K.has_forest = L.has_forest ? 1 : 0;
  K.all_lone = all_lone_units(K, L.units, L.configs) ? 1 : 0;
  K.group_fail = nullptr;
  if (L.ngroups > 0) {
    B.group_fail.resize(L.ngroups);
    cuda_check(cudaMemsetAsync(B.group_fail.ptr, 0, L.ngroups * sizeof(uint32_t), s), "memset");
    K.group_fail = B.group_fail.ptr;
  }
  cudaEvent_t e0, e1;
  cuda_check(cudaEventCreate(&e0), "event");
  cuda_check(cudaEventCreate(&e1), "event");
  cuda_check(cudaEventRecord(e0, s), "event");
  launch_simulate(K, s);
  cuda_check(cudaEventRecord(e1, s), "event");
  const double* sel_staged = nullptr;
  if (emissions) {
    // samples per measured run m: [delay | ttft] (n each), then TBT gaps (E each)
    std::vector<ProbeDesc> mp;
    for (int32_t k : L.measured) mp.push_back(L.probes[k]);
    B.mprobes.upload(mp, s, lane.staging);
    const int64_t n = w.n, E = w.emis_per_probe;
    B.samples.resize(std::max<int64_t>(1, nm * (2 * n + E)));
    double* delay = B.samples.ptr;
    double* ttft = delay + nm * n;
    double* gaps = ttft + nm * n;
    launch_slo_samples(B.mprobes.ptr, nm, B.units.ptr, B.tm.ptr, w, B.emis.ptr, delay, ttft, gaps, s);
    std::vector<int64_t> off;
    std::vector<SelectTask> tasks;
    for (int32_t k = 0; k < nm; ++k) off.push_back(k * n);                // delay segments
    for (int32_t k = 0; k < nm; ++k) off.push_back(nm * n + k * n);       // ttft segments
    for (int32_t k = 0; k < nm; ++k) off.push_back(2 * nm * n + k * E);   // tbt segments
    off.push_back(2 * nm * n + nm * E);
    const int64_t n_tbt = E - n;  // decode_tokens - 1 samples per request
    for (int32_t k = 0; k < nm; ++k) {
      tasks.push_back({k, nearest_rank_index(n, 0.99)});
      tasks.push_back({nm + k, nearest_rank_index(n, 0.90)});
      tasks.push_back({2 * nm + k, n_tbt > 0 ? nearest_rank_index(n_tbt, 0.99) : 0});
    }
    B.seg_off.upload(off, s, lane.staging);
    B.tasks.upload(tasks, s, lane.staging);
    B.sel.resize(tasks.size());
    launch_select(B.samples.ptr, B.seg_off.ptr, B.tasks.ptr, static_cast<int64_t>(tasks.size()),
                  B.sel.ptr, s);
    sel.resize(tasks.size());
    sel_staged = B.sel.download_staged(sel.size(), s, lane.staging);
  }
  out.resize(L.units.size());
  const SimUnitOut* out_staged = B.out.download_staged(out.size(), s, lane.staging);
  cuda_check(cudaStreamSynchronize(s), "sweep launch");
  std::memcpy(out.data(), out_staged, out.size() * sizeof(SimUnitOut));
  if (sel_staged) std::memcpy(sel.data(), sel_staged, sel.size() * sizeof(double));
  lane.staging.reset();
  float ms = 0.f;
  cuda_check(cudaEventElapsedTime(&ms, e0, e1), "event");
  if (lane.origin) {
    float a = 0.f, b = 0.f;
    cuda_check(cudaEventElapsedTime(&a, lane.origin, e0), "event");
    cuda_check(cudaEventElapsedTime(&b, lane.origin, e1), "event");
    lane.intervals.push_back({a, b});
  }
  if (std::getenv("SSG_TRACE_LANES")) {
    int64_t alg = 0, iters = 0;
    for (const auto& o : out) {
      alg += o.qbytes + 48 * o.entries;
      iters += o.iterations;
    }
    std::fprintf(stderr, "lane %p launch %.3f ms units %zu iterations %lld alg_bytes %lld\n",
                 (void*)&lane, ms, L.units.size(), (long long)iters, (long long)alg);
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  if (const char* dump = std::getenv("SSG_DUMP_UNITS")) {
    std::lock_guard<std::mutex> lk(g_dump_mu);
    // diagnostics: one line per unit (launch, unit, config, n, R, iterations, cycles, qps)
    FILE* f = std::fopen(dump, "a");
    if (f) {
      static int launch_no = 0;
      std::vector<double> qps_of(L.units.size(), 0.0);
      for (const auto& p : L.probes)
        for (int u = p.first_unit; u < p.first_unit + (p.decoupled ? p.R : 1); ++u) qps_of[u] = p.qps;
      std::vector<long long> ph(out.size() * SSG_PH_N, 0);
      const bool have_ph = phase_cycles(ph.data(), static_cast<int64_t>(out.size()));
      for (std::size_t u = 0; u < out.size(); ++u) {
        const SimConfig& cf = L.configs[L.units[u].config];
        if (have_ph && u < 16384) {
          std::fprintf(f, "P %d %zu", launch_no, u);
          for (int k = 0; k < SSG_PH_N; ++k) std::fprintf(f, " %lld", ph[u * SSG_PH_N + k]);
          std::fprintf(f, "\n");
        }
        std::fprintf(f, "%d %zu %d %d %d %lld %lld %.17g %d %d %lld %d %d %d %lld %d\n", launch_no, u,
                     L.units[u].config, L.units[u].n, L.units[u].R, (long long)out[u].iterations,
                     (long long)out[u].cycles, qps_of[u], cf.policy, cf.max_batch,
                     (long long)out[u].entries, cf.tp, cf.pp, cf.chunk, (long long)out[u].events,
                     out[u].aborted);
      }
      std::fprintf(f, "# launch %d ms %.3f\n", launch_no, ms);
      ++launch_no;
      std::fclose(f);
    }
  }
  RunStats& st = stats();
  st.launches_simulate += 1;
  st.simulate_ms += ms;
  st.units += static_cast<int64_t>(out.size());
  for (const auto& o : out) {
    st.iterations += o.iterations;
    st.entries += o.entries;
    st.events += o.events;
    st.predictor_bytes += o.qbytes;
    st.entry_bytes += 48 * o.entries;
  }
}

int32_t max_late_of(std::size_t n) {
  return static_cast<int32_t>(n - static_cast<std::size_t>(std::ceil(0.99 * static_cast<double>(n))));
}

// First error of a probe's units in simulated time.
const SimUnitOut* first_error(const std::vector<SimUnitOut>& out, const ProbeDesc& p) {
  const SimUnitOut* e = nullptr;
  const int nu = p.decoupled ? p.R : 1;
  for (int u = p.first_unit; u < p.first_unit + nu; ++u)
    if (out[u].code != SSG_OK && (!e || out[u].err_time < e->err_time)) e = &out[u];
  return e;
}

void fail(Candidate& C, const SimUnitOut& o) {
  try {
    raise_unit_error(o, C.sim, *C.est);
  } catch (const Error& ex) {
    C.res.error = ex.what();
    C.done = true;
  }
}

// Capacities find_capacity can return once `rates` are answered, over every
// feasible / infeasible outcome of them.  False when some outcome asks a rate
// outside `rates` (the search would go on past this round) or more than `max`
// capacities are possible.  `memo` is restored on return.
bool possible_capacities(ProbeMemo& memo, const CapacitySearchOptions& o,
                         const std::vector<double>& rates, std::size_t max, std::vector<double>& caps) {
  try {
    const double c = replay_capacity(memo, o);
    if (std::find(caps.begin(), caps.end(), c) == caps.end()) caps.push_back(c);
    return caps.size() <= max;
  } catch (const NeedProbe& need) {
    if (std::find(rates.begin(), rates.end(), need.q) == rates.end()) return false;
    for (int f = 1; f >= 0; --f) {
      ProbeAnswer a;
      a.feasible = f != 0;
      memo.emplace(need.q, a);
      const bool ok = possible_capacities(memo, o, rates, max, caps);
      memo.erase(need.q);
      if (!ok) return false;
    }
    return true;
  } catch (const ProbeError&) {
    return true;  // no capacity on this branch
  } catch (const Error&) {
    return true;
  }
}

// Live candidates of every sweep in flight in this process (concurrent sessions,
// e.g. cfg #5's twelve sweeps): the under-loaded test of the speculation knobs.
std::atomic<int64_t> g_live_candidates{0};
struct LiveCandidates {
  int64_t n;
  explicit LiveCandidates(int64_t k) : n(k) { g_live_candidates += n; }
  ~LiveCandidates() { g_live_candidates -= n; }
};
std::atomic<int> g_sweeps_in_flight{0};
struct SweepInFlight {
  SweepInFlight() { ++g_sweeps_in_flight; }
  ~SweepInFlight() { --g_sweeps_in_flight; }
};

// ~4 probes per live candidate fit the SMs' warp slots (8 per SM)
bool sweeps_underloaded() {
  return g_live_candidates.load() * 4 <= 8 * static_cast<int64_t>(context().num_sms);
}

struct SweepKnobs {
  int ladder = -1;  // doubling rates probed per round (-1: auto, 4; 6 when under-loaded:
                    // cfg #4 1/2 shard 0.352 -> 0.333 s, 1/4 0.249 -> 0.241 s, DESIGN 6.7)
  int depth = 2;   // bisection levels probed per round (2^depth - 1 rates); 3 until the
                   // kernel diet (DESIGN 6.4): 0.83 s vs 0.96 s at 3, 0.94 s at 1
  int crit_extra = -1;  // extra levels for the candidates with the longest probes (-1: auto,
                        // 1; 2 when under-loaded -- v9: full sweep 0.433-0.436 s at 1 vs
                        // 0.439-0.445 at 2, 1/2 shard 0.315 at 2 vs 0.319 at 1)
  int crit_pct = 95;   // "longest": probes within this % of the group's longest (A/B: DESIGN 6.4)
  int lanes = -1;  // candidate groups advancing independently (streams): one group's
                   // launch tail overlaps the other's next round.  1 until the round-2
                   // v5 kernels (no gain then); now 2 lanes 0.453 s, 3: 0.462, 4: 0.461,
                   // 1: 0.474 (DESIGN 6.7).  -1 = auto: 2 for a sweep running alone, 1
                   // when other sweeps are in flight (cfg #5's twelve: 1/8 shards 3.99 s
                   // on 2 lanes, 2.95 s on 1)
  bool block = false;  // groups = contiguous blocks of the capacity order (else dealt)
  // Under-loaded sweeps (a multi-GPU rank's shard: few candidates, chain-bound
  // rounds) trade work for rounds; -1 = auto: on when the live candidates' ~4
  // probes each fit the SMs' warp slots (8 per SM), off for a full one-GPU sweep
  // (DESIGN 6.7: 1/8 shard 0.254 -> 0.212 s, full sweep 0.455 -> 0.51 s if forced on).
  int spec_slo = -1;     // speculative SLO runs per candidate and round (0: off, auto 8)
  int slo_pct = 0;       // for candidates whose probes are within this % of the longest
  int64_t slo_bytes = int64_t(1) << 31;  // device bytes of a launch's measured runs
  int pre = 0;           // bisection levels speculated under every ladder bracket in the
                         // ladder's own round (-1: auto, 1 when under-loaded).  Measured
                         // (DESIGN 6.7): 1/2 shard 0.342 -> 0.332 s at 1, 1/4 and 1/8 shards
                         // unchanged at 1, mixed at 2, slower at 3: off by default
  int lag = -1;          // extra bisection levels for candidates whose bisection started
                         // this many rounds late at most (they set the sweep's round
                         // count; auto 2)
};

SweepKnobs knobs_from_env() {
  SweepKnobs k;
  if (const char* s = std::getenv("SSG_SPEC_LADDER")) k.ladder = std::atoi(s) >= 1 ? std::atoi(s) : -1;
  if (const char* s = std::getenv("SSG_SPEC_DEPTH")) k.depth = std::max(1, std::atoi(s));
  if (const char* s = std::getenv("SSG_SPEC_CRIT")) k.crit_extra = std::atoi(s);
  if (const char* s = std::getenv("SSG_SPEC_CRIT_PCT")) k.crit_pct = std::max(0, std::atoi(s));
  if (const char* s = std::getenv("SSG_LANES")) k.lanes = std::atoi(s) >= 1 ? std::atoi(s) : -1;
  if (const char* s = std::getenv("SSG_LANE_BLOCK")) k.block = s[0] == '1';
  if (const char* s = std::getenv("SSG_SPEC_SLO")) k.spec_slo = std::atoi(s);
  if (const char* s = std::getenv("SSG_SPEC_PRE")) k.pre = std::atoi(s);
  if (const char* s = std::getenv("SSG_SPEC_SLO_BYTES")) k.slo_bytes = std::atoll(s);
  if (const char* s = std::getenv("SSG_SPEC_SLO_PCT")) k.slo_pct = std::max(0, std::atoi(s));
  if (const char* s = std::getenv("SSG_SPEC_LAG")) k.lag = std::atoi(s);
  return k;
}

// Records a full run's SLO measurement (or an error) on its candidate.
void take_measurement(Candidate& C, const std::vector<SimUnitOut>& out, const ProbeDesc& p,
                      const double* sel3, const ResidentWorkload& w) {
  C.full_run = ProbeAnswer{};
  for (int u = p.first_unit; u < p.first_unit + (p.decoupled ? p.R : 1); ++u) add_work(C.full_run, out[u]);
  if (const SimUnitOut* e = first_error(out, p)) {
    fail(C, *e);
    return;
  }
  C.res.delay_p99 = sel3[0];
  C.res.ttft_p90 = sel3[1];
  C.res.tbt_p99 = (w.emis_per_probe - w.n) > 0 ? sel3[2] : 0.0;  // summarize({}) -> 0
  if (p.static_run) {
    double span = 0.0;
    const int nu = p.decoupled ? p.R : 1;
    for (int u = p.first_unit; u < p.first_unit + nu; ++u) span = std::max(span, out[u].span);
    C.res.makespan = span;
  }
  C.measured = true;
}

// One launch: capacity probes (answers into the candidates' memos) together
// with the full runs of candidates whose capacity is already known (SLO
// measurement at evaluation_fraction x capacity, or the static makespan run).
// An error inside a probe ends that candidate's evaluation (the reference's
// exception) unless the probe's abort came first in event order.
void run_round(SweepLane& lane, std::vector<Candidate>& cands, const std::vector<SpecProbes>& probes,
               const std::vector<std::pair<std::size_t, double>>& full, bool static_run,
               const ResidentWorkload& w, const CapacitySearchOptions& base,
               const std::vector<std::pair<std::size_t, double>>& spec = {}) {
  const int32_t n = w.n;
  const int32_t max_late = max_late_of(static_cast<std::size_t>(n));
  ProbeLaunch L;
  for (const SpecProbes& sp : probes) {
    const std::size_t k = sp.k;
    const int32_t ci = L.add_config(cands[k]);
    // a candidate's probes form one speculation group: once a probe fails
    // (abort or error), the probes the replay would only ask after it came out
    // feasible are cancelled on the device (SimUnit::kill).  Safe by
    // construction: a cancelled rate stays unanswered in the memo, so a replay
    // that does ask for it probes it in a later round.
    const int32_t g = sp.rates.size() > 1 && sp.rates.size() <= 32 ? L.ngroups++ : -1;
    for (std::size_t i = 0; i < sp.rates.size(); ++i)
      L.add_probe(k, cands[k], ci, sp.rates[i], n, SSG_UF_ABORT, base.delay_p99_threshold, max_late,
                  false, false, -1, g, static_cast<int32_t>(i), g >= 0 ? sp.kill[i] : 0u);
  }
  for (const auto& [k, q] : full) {
    const int32_t ci = L.add_config(cands[k]);
    L.add_probe(k, cands[k], ci, static_run ? 0.0 : q, n, SSG_UF_EMISSIONS, 0.0, 0, false,
                static_run, L.next_emis_base(w.emis_per_probe));
  }
  for (const auto& [k, q] : spec) {  // measured after the real ones (L.measured order)
    const int32_t ci = L.add_config(cands[k]);
    L.add_probe(k, cands[k], ci, q, n, SSG_UF_EMISSIONS, 0.0, 0, false, false,
                L.next_emis_base(w.emis_per_probe));
  }
  if (L.probes.empty()) return;
  std::vector<SimUnitOut> out;
  std::vector<double> sel;
  run_launch(lane, L, w, out, sel);
  // Full runs: the first error in simulated time is the one the reference
  // raises, but independent round-robin units cannot order two errors at the
  // same clock (the makespan run queues every arrival at t = 0) -- the
  // reference raises for the event first in its global (time, seq) order.
  // A full run with more than one failing unit is replayed with all its
  // replicas in one unit, in exact event order (as sim.cpp does for single runs).
  ProbeLaunch redo_full;
  for (std::size_t m = 0; m < L.measured.size(); ++m) {
    const ProbeDesc& p = L.probes[L.measured[m]];
    Candidate& C = cands[L.probe_cand[L.measured[m]]];
    int errors = 0;
    for (int u = p.first_unit; u < p.first_unit + (p.decoupled ? p.R : 1); ++u)
      errors += out[u].code != SSG_OK ? 1 : 0;
    if (m >= full.size()) {
      // speculative SLO run: kept for the replay (a run that would need the coupled
      // redo is dropped; the sequential order then takes it in a later round)
      if (errors > 1 && p.decoupled) continue;
      Candidate::SpecFull sf;
      const int nu = p.decoupled ? p.R : 1;
      sf.out.assign(out.begin() + p.first_unit, out.begin() + p.first_unit + nu);
      sf.p = p;
      sf.p.first_unit = 0;
      std::copy(sel.begin() + 3 * m, sel.begin() + 3 * m + 3, sf.sel3);
      C.spec_full[p.qps] = std::move(sf);
      continue;
    }
    if (errors > 1 && p.decoupled && p.R <= kMaxCoupledReplicas) {
      const int32_t ci = redo_full.add_config(C);
      redo_full.add_probe(L.probe_cand[L.measured[m]], C, ci, p.qps, n, SSG_UF_EMISSIONS, 0.0, 0,
                          true, p.static_run != 0, redo_full.next_emis_base(w.emis_per_probe));
      continue;
    }
    take_measurement(C, out, p, sel.data() + 3 * m, w);
  }
  if (!redo_full.probes.empty()) {
    std::vector<SimUnitOut> out2;
    std::vector<double> sel2;
    run_launch(lane, redo_full, w, out2, sel2);
    for (std::size_t m = 0; m < redo_full.measured.size(); ++m) {
      const ProbeDesc& p = redo_full.probes[redo_full.measured[m]];
      take_measurement(cands[redo_full.probe_cand[redo_full.measured[m]]], out2, p,
                       sel2.data() + 3 * m, w);
    }
  }
  ProbeLaunch redo;
  for (std::size_t k = 0; k < L.probes.size(); ++k) {
    const ProbeDesc& p = L.probes[k];
    if (p.emis_base >= 0) continue;  // measured run, handled above
    Candidate& C = cands[L.probe_cand[k]];
    int64_t late = 0, iters = 0;
    bool aborted = false, cancelled = false;
    const int nu = p.decoupled ? p.R : 1;
    ProbeAnswer work;
    for (int u = p.first_unit; u < p.first_unit + nu; ++u) {
      late += out[u].late;
      aborted |= out[u].aborted == 1;
      cancelled |= out[u].aborted == 2;
      iters = std::max<int64_t>(iters, out[u].iterations);
      add_work(work, out[u]);
    }
    if (cancelled) {  // not needed by the replay; leave the rate unanswered
      stats().cancelled_probes += 1;
      continue;
    }
    C.probe_iters = std::max(C.probe_iters, iters);
    const SimUnitOut* e = first_error(out, p);
    if (!e) {
      work.feasible = !aborted && late <= max_late;
      C.memo[p.qps] = work;
    } else if (p.decoupled && p.R <= kMaxCoupledReplicas) {
      // independent replicas cannot order an error against the global abort:
      // replay this probe with every replica in one unit
      const int32_t ci = redo.add_config(C);
      redo.add_probe(L.probe_cand[k], C, ci, p.qps, n, SSG_UF_ABORT, base.delay_p99_threshold,
                     max_late, true, false, -1);
    } else if (aborted && !p.decoupled) {
      C.memo[p.qps] = work;
    } else {
      work.error = true;
      work.err = *e;
      C.memo[p.qps] = work;
    }
  }
  if (redo.probes.empty()) return;
  run_launch(lane, redo, w, out, sel);
  for (std::size_t k = 0; k < redo.probes.size(); ++k) {
    const ProbeDesc& p = redo.probes[k];
    Candidate& C = cands[redo.probe_cand[k]];
    const SimUnitOut& o = out[p.first_unit];
    ProbeAnswer work;
    add_work(work, o);
    if (o.aborted) {
    } else if (o.code == SSG_OK) {
      work.feasible = o.late <= max_late;
    } else {
      work.error = true;
      work.err = o;
    }
    C.memo[p.qps] = work;
  }
}

// One candidate group's capacity searches and SLO runs, round after round on
// its lane.  Rounds: every live candidate's find_capacity is replayed;
// unanswered rates (plus speculative successors) become probes, and candidates
// whose capacity resolved get their SLO run in the same launch.
void run_group(SweepLane& lane, std::vector<Candidate>& cands, const std::vector<std::size_t>& live,
               const SearchOptions& opts, const ResidentWorkload& w, const SweepKnobs& knobs,
               std::vector<std::size_t>& measured) {
  while (true) {
    std::vector<SpecProbes> probes;
    std::vector<std::pair<std::size_t, double>> full, spec;
    int64_t longest = 1;
    for (auto k : live) longest = std::max(longest, cands[k].probe_iters);
    const bool under =
        (knobs.spec_slo < 0 || knobs.lag < 0 || knobs.pre < 0 || knobs.ladder < 0 || knobs.crit_extra < 0) &&
        sweeps_underloaded();
    const int crit_extra = knobs.crit_extra >= 0 ? knobs.crit_extra : (under ? 2 : 1);
    const int ladder = knobs.ladder >= 1 ? knobs.ladder : (under ? 6 : 4);
    const int spec_slo = knobs.spec_slo >= 0 ? knobs.spec_slo : (under ? 8 : 0);
    const int lag = knobs.lag >= 0 ? knobs.lag : (under ? 2 : 0);
    const int pre = knobs.pre >= 0 ? knobs.pre : (under ? 1 : 0);
    for (auto k : live) {
      Candidate& C = cands[k];
      if (C.res.failed() || C.measured) continue;
      if (!C.done) {
        try {
          C.res.capacity_qps = replay_capacity(C.memo, C.copts);
          C.done = true;  // capacity known
        } catch (const NeedProbe& need) {
          // candidates on the critical path (longest probes) speculate deeper,
          // so their bisection finishes in one round
          const bool critical = C.probe_iters * 100 >= longest * knobs.crit_pct;
          std::vector<SpecRate> qs;
          int depth = critical ? knobs.depth + crit_extra : knobs.depth;
          if (need.phase == 2) {
            if (C.bisect_from < 0) C.bisect_from = C.rounds;
            // the first ladder round settles most candidates' brackets; one that is
            // still climbing then would need an extra round at the end
            depth = std::max(depth, knobs.depth + std::min(lag, C.bisect_from - 1));
          }
          speculate(need, C.copts, ladder, depth, pre, qs);
          // unanswered rates; each one's cancel mask over the others' positions
          std::vector<int> pos(qs.size(), -1);
          SpecProbes sp;
          sp.k = k;
          for (std::size_t i = 0; i < qs.size(); ++i) {
            const double q = qs[i].q;
            if (C.memo.count(q) || std::find(sp.rates.begin(), sp.rates.end(), q) != sp.rates.end()) continue;
            pos[i] = static_cast<int>(sp.rates.size());
            uint32_t kill = 0;
            for (int a : qs[i].after_feasible)
              if (pos[a] >= 0 && pos[a] < 32) kill |= 1u << pos[a];
            sp.rates.push_back(q);
            sp.kill.push_back(kill);
          }
          C.rounds += 1;
          if (spec_slo > 0 && C.probe_iters * 100 >= longest * knobs.slo_pct) {
            // this round may settle the capacity: SLO runs at every capacity it can end with
            std::vector<double> caps;
            const bool ok = possible_capacities(C.memo, C.copts, sp.rates, spec_slo, caps);
            if (std::getenv("SSG_SPEC_DEBUG"))
              std::fprintf(stderr, "try %zu round %d ok %d caps %zu rates %zu\n", C.index, C.rounds, ok ? 1 : 0,
                           caps.size(), sp.rates.size());
            if (ok)
              for (double cap : caps) {
                const double q = opts.evaluation_fraction * cap;
                if (cap > C.copts.min_qps && q > 0.0 && !C.spec_full.count(q)) spec.push_back({k, q});
              }
          }
          probes.push_back(std::move(sp));
          continue;
        } catch (const ProbeError& pe) {
          fail(C, pe.err);
          continue;
        } catch (const Error& e) {
          C.res.error = e.what();
          C.res.capacity_qps = 0.0;
          C.done = true;
          continue;
        }
      }
      // capacity known: the SLO measurement run at evaluation_fraction of it
      if (C.res.capacity_qps <= C.copts.min_qps) {
        C.res.capacity_qps = 0.0;
        C.res.error = "no feasible arrival rate (scheduling delay above threshold)";
        continue;
      }
      const double q = opts.evaluation_fraction * C.res.capacity_qps;
      try {
        require(q > 0.0, "poisson_arrivals: rate must be positive");
      } catch (const Error& e) {
        C.res.error = e.what();
        continue;
      }
      if (auto it = C.spec_full.find(q); it != C.spec_full.end()) {
        // taken speculatively in the round that settled the capacity
        take_measurement(C, it->second.out, it->second.p, it->second.sel3, w);
        stats().spec_slo_used += 1;
        C.spec_full.clear();
        measured.push_back(k);
        continue;
      }
      if (std::getenv("SSG_SPEC_DEBUG")) {
        std::fprintf(stderr, "miss %zu rounds %d bisect_from %d iters %lld q %.17g spec", C.index, C.rounds,
                     C.bisect_from, static_cast<long long>(C.probe_iters), q);
        for (const auto& kv : C.spec_full) std::fprintf(stderr, " %.17g", kv.first);
        std::fprintf(stderr, "\n");
      }
      full.push_back({k, q});
      measured.push_back(k);
    }
    if (probes.empty() && full.empty()) break;
    if (std::getenv("SSG_ROUND_LOG")) {
      int ph[3] = {0, 0, 0}, rates = 0;
      for (const SpecProbes& sp : probes) rates += static_cast<int>(sp.rates.size());
      for (auto k : live) {
        const Candidate& C = cands[k];
        if (C.done || C.res.failed()) continue;
        try {
          replay_capacity(C.memo, C.copts);
        } catch (const NeedProbe& nd) {
          ph[nd.phase] += 1;
        } catch (...) {
        }
      }
      std::fprintf(stderr, "round lane %p cands %zu ladder %d halving %d bisect %d rates %d full %zu longest %lld\n",
                   static_cast<void*>(&lane), probes.size(), ph[0], ph[1], ph[2], rates, full.size(),
                   static_cast<long long>(longest));
    }
    // every measured run keeps its emission times and SLO samples on the device
    // (~16 B per decode token): speculative runs stay within a per-launch budget,
    // longest-probe candidates first (the group's order)
    if (!spec.empty()) {
      const int64_t per_run = 16 * std::max<int64_t>(1, w.emis_per_probe + 2 * w.n);
      const int64_t room = knobs.slo_bytes / per_run - static_cast<int64_t>(full.size());
      spec.resize(static_cast<std::size_t>(std::clamp<int64_t>(room, 0, static_cast<int64_t>(spec.size()))));
    }
    stats().spec_slo_runs += static_cast<int64_t>(spec.size());
    run_round(lane, cands, probes, full, false, w, opts.capacity, spec);
  }
}

bool shard_split_by_cost() {  // SSG_SHARD_SPLIT=stride: i % num_shards (A/B)
  const char* e = std::getenv("SSG_SHARD_SPLIT");
  return !(e && std::strcmp(e, "stride") == 0);
}

// Greedy LPT: configs by cost descending (ties by enumeration index) onto the
// least-loaded shard (ties to the lowest shard).  Deterministic on every rank.
std::vector<int> lpt_split(const std::vector<Candidate>& cands, int num_shards) {
  std::vector<double> cost(cands.size(), 0.0);
  for (std::size_t k = 0; k < cands.size(); ++k)
    if (!cands[k].done) cost[k] = 1.0 / cands[k].copts.initial_guess;
  std::vector<std::size_t> order(cands.size());
  for (std::size_t k = 0; k < order.size(); ++k) order[k] = k;
  std::stable_sort(order.begin(), order.end(), [&](std::size_t a, std::size_t b) {
    return cost[a] > cost[b];
  });
  std::vector<double> load(static_cast<std::size_t>(num_shards), 0.0);
  std::vector<int> count(static_cast<std::size_t>(num_shards), 0);
  std::vector<int> owner(cands.size(), 0);
  for (auto k : order) {
    int best = 0;
    for (int r = 1; r < num_shards; ++r)
      if (load[r] < load[best] || (load[r] == load[best] && count[r] < count[best])) best = r;
    owner[k] = best;
    load[best] += cost[k];
    count[best] += 1;
  }
  return owner;
}

}  // namespace

struct SearchSession::State {
  ModelSpec spec;
  SearchOptions opts;
  std::vector<CandidateConfig> configs;
  std::vector<EstimatorModel> owned;        // trained by the session (run_search)
  std::vector<const EstimatorModel*> ests;  // per SKU index: owned or the caller's
  Workload w;
  ResidentWorkload rw;
  DeviceBuffer<double> tables;                    // token tables (context stream)
  std::vector<std::unique_ptr<SweepLane>> lanes;  // borrowed from the lane pool
  ~State() {
    LanePool& p = lane_pool();
    std::lock_guard<std::mutex> lk(p.mu);
    for (auto& l : lanes) p.free.push_back(std::move(l));
  }
};

SearchSession::SearchSession(const ModelSpec& spec, const std::vector<Request>& workload,
                             const SearchOptions& opts)
    : st_(std::make_unique<State>()) {
  StatsScope stats_scope;  // sessions may be opened and run on several host threads at once
  PhaseTimer timer("search: session open");
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
  // SKUs are independent (own profile, own seed-identical training): build them
  // on host threads; errors surface in SKU order, as the reference's loop raises
  const std::size_t nsku = opts.space.skus.size();
  std::vector<EstimatorModel> built(nsku);
  std::vector<std::exception_ptr> err(nsku);
  {
    const int dev = context().device;
    auto one = [&](std::size_t k) {
      try {
        StatsScope scope;  // counters merge into the process totals under the lock
        cuda_check(cudaSetDevice(dev), "cudaSetDevice");
        PhaseTimer t("search: profile + train SKU");
        built[k] = train(generate_synthetic_profile(spec, opts.space.skus[k], tps), opts.train);
      } catch (...) {
        err[k] = std::current_exception();
      }
    };
    std::vector<std::thread> pool;
    for (std::size_t k = 1; k < nsku; ++k) pool.emplace_back(one, k);
    if (nsku) one(0);
    for (auto& t : pool) t.join();
  }
  for (auto& e : err)
    if (e) std::rethrow_exception(e);
  for (auto& e : built) S.owned.push_back(std::move(e));
  for (const auto& e : S.owned) S.ests.push_back(&e);
  open_workload(workload);
}

SearchSession::SearchSession(const ModelSpec& spec, std::vector<CandidateConfig> cands,
                             const std::vector<DeviceProfile>& skus,
                             const std::vector<const EstimatorModel*>& estimators,
                             const std::vector<Request>& workload, const SearchOptions& opts)
    : st_(std::make_unique<State>()) {
  StatsScope stats_scope;
  PhaseTimer timer("search: session open");
  State& S = *st_;
  S.spec = spec;
  S.opts = opts;
  S.opts.space.skus = skus;
  require(estimators.size() == skus.size(), "evaluate_configs: one estimator per SKU");
  for (const auto& c : cands)
    require(c.sku_index < skus.size(), "evaluate_configs: candidate " + c.id + " has no SKU");
  for (auto* e : estimators) internal_check(e != nullptr, "evaluate_configs: null estimator");
  S.configs = std::move(cands);
  S.ests = estimators;
  open_workload(workload);
}

void SearchSession::open_workload(const std::vector<Request>& workload) {
  PhaseTimer timer("search: open workload");
  State& S = *st_;
  const SearchOptions& opts = S.opts;
  for (const auto* e : S.ests) e->device();  // resident in HBM before any timed work
  require(!workload.empty(), "search: empty workload");
  for (std::size_t i = 0; i < opts.capacity.probe_requests; ++i) {
    Request r = workload[i % workload.size()];
    r.id = static_cast<std::int64_t>(i);
    S.w.lengths.push_back(r);
  }
  S.w.unit_exp = unit_exponentials(S.w.lengths.size(), opts.capacity.seed);
  // resident probe stream inputs
  auto& ctx = context();
  const std::size_t n = S.w.lengths.size();
  require(n < static_cast<std::size_t>(INT32_MAX), "search: probe_requests too large");
  std::vector<int32_t> pre(n), dec(n);
  std::vector<int64_t> prefix(n);
  int64_t acc = 0;
  for (std::size_t i = 0; i < n; ++i) {
    require(S.w.lengths[i].prefill_tokens < INT32_MAX / 2 && S.w.lengths[i].decode_tokens < INT32_MAX / 2,
            "ssg: request lengths above the device engine limit");
    pre[i] = static_cast<int32_t>(S.w.lengths[i].prefill_tokens);
    dec[i] = static_cast<int32_t>(S.w.lengths[i].decode_tokens);
    prefix[i] = acc;
    acc += dec[i];
  }
  std::vector<uint8_t> first(static_cast<std::size_t>(acc), 0);
  for (std::size_t i = 0; i < n; ++i) first[prefix[i]] = 1;
  S.rw.n = static_cast<int32_t>(n);
  S.rw.emis_per_probe = acc;
  S.rw.pre.upload(pre, ctx.stream);
  S.rw.dec.upload(dec, ctx.stream);
  S.rw.unit_exp.upload(S.w.unit_exp, ctx.stream);
  S.rw.dec_prefix.upload(prefix, ctx.stream);
  S.rw.first_emis.upload(first, ctx.stream);
  cuda_check(cudaStreamSynchronize(ctx.stream), "session upload");
}

SearchSession::~SearchSession() = default;

}  // namespace servesim

namespace ssg {
void release_sweep_lanes() {
  servesim::LanePool& p = servesim::lane_pool();
  std::lock_guard<std::mutex> lk(p.mu);
  p.free.clear();
}
}  // namespace ssg

namespace servesim {

std::size_t SearchSession::num_configs() const { return st_->configs.size(); }

std::vector<ConfigResult> evaluate_configs_shard(const ModelSpec& spec,
                                                 const std::vector<Request>& workload,
                                                 const SearchOptions& opts, int shard,
                                                 int num_shards, std::vector<std::size_t>* owned) {
  SearchSession session(spec, workload, opts);
  return session.evaluate(shard, num_shards, owned);
}

std::vector<ConfigResult> SearchSession::evaluate(int shard, int num_shards,
                                                  std::vector<std::size_t>* owned) {
  StatsScope stats_scope;  // counters merge into the process totals when the evaluation ends
  SweepInFlight in_flight;
  PhaseTimer timer("search: evaluate");
  const State& S = *st_;
  const ModelSpec& spec = S.spec;
  const SearchOptions& opts = S.opts;
  const auto& configs = S.configs;
  const auto& ests = S.ests;
  const ResidentWorkload& w = S.rw;
  State& SS = *st_;
  std::vector<ConfigResult> results(configs.size());
  std::vector<Candidate> cands;
  const bool makespan = opts.objective == "makespan";
  // The capacity objective computes every config's initial guess first (one
  // launch for the whole grid, identical on every rank) and splits the grid by
  // its cost; the makespan objective's static runs are alike, so it strides.
  const bool by_cost = !makespan && num_shards > 1 && shard_split_by_cost();
  for (std::size_t i = 0; i < configs.size(); ++i) {
    if (!by_cost && static_cast<int>(i % static_cast<std::size_t>(num_shards)) != shard) continue;
    const CandidateConfig& cand = configs[i];
    Candidate C;
    C.index = i;
    C.cand = cand;
    C.res.config = cand;
    C.res.sku_name = opts.space.skus[cand.sku_index].sku_name;
    C.cluster = ClusterConfig{spec, cand.par, opts.space.skus[cand.sku_index], cand.policy,
                              opts.routing, 0, opts.cpu_overhead_per_iter};
    C.est = ests[cand.sku_index];
    C.copts = opts.capacity;
    try {
      C.sim = make_sim_config(C.cluster, *C.est, 0);
      C.sim_ok = true;
    } catch (const Error& e) {
      C.sim_error = e.what();
    }
    cands.push_back(std::move(C));
  }

  std::vector<std::size_t> live;
  if (makespan) {
    // the static run is the first simulation: its preamble errors surface
    for (auto& C : cands)
      if (!C.sim_ok) {
        C.res.error = C.sim_error;
        C.done = true;
      }
  } else {
    // initial_qps_guess (search.hpp:278-290) for every candidate in one launch:
    // predict_batch of a 512-token prefill and of one 512-context decode
    std::vector<SimConfig> gcfg;
    std::vector<SsgEstView> gest;
    std::unordered_map<const EstimatorModel*, int32_t> gidx;
    std::vector<int32_t> comp_cfg;
    std::vector<std::size_t> who;
    std::vector<int64_t> p_off{0}, d_off{0}, p_len, p_prior, d_ctx;
    const std::int64_t len = std::min<std::int64_t>(512, spec.max_context);
    for (std::size_t k = 0; k < cands.size(); ++k) {
      Candidate& C = cands[k];
      try {
        auto ops = derive_operators(spec, C.cand.par);
        // predict()'s find() order over the two compositions (a missing model
        // raises the reference's message for the first op looked up)
        for (int pass = 0; pass < 2; ++pass)
          for (const auto& d : ops) {
            if (pass == 0 && d.op == OpName::AttnDecode) continue;
            if (pass == 1 && d.op == OpName::AttnPrefill) continue;
            C.est->find(d.op, d.tp_degree);
          }
        SimConfig g{};
        fill_sim_ops(g, ops, C.est->device());
        auto it = gidx.find(C.est);
        if (it == gidx.end()) {
          it = gidx.emplace(C.est, static_cast<int32_t>(gest.size())).first;
          gest.push_back(C.est->device().view);
        }
        g.est = it->second;
        gcfg.push_back(g);
        const int32_t ci = static_cast<int32_t>(gcfg.size() - 1);
        comp_cfg.push_back(ci);  // prefill composition
        p_len.push_back(len);
        p_prior.push_back(0);
        p_off.push_back(static_cast<int64_t>(p_len.size()));
        d_off.push_back(static_cast<int64_t>(d_ctx.size()));
        comp_cfg.push_back(ci);  // decode composition
        d_ctx.push_back(len);
        p_off.push_back(static_cast<int64_t>(p_len.size()));
        d_off.push_back(static_cast<int64_t>(d_ctx.size()));
        who.push_back(k);
      } catch (const Error& e) {
        C.res.error = e.what();
        C.done = true;
      }
    }
    const int64_t ncomp = static_cast<int64_t>(comp_cfg.size());
    std::vector<double> secs(ncomp), fl(ncomp);
    std::vector<SimUnitOut> status;
    predict_batches_multi(gcfg, gest, comp_cfg, ncomp, p_off.data(), p_len.data(), p_prior.data(),
                          d_off.data(), d_ctx.data(), secs.data(), fl.data(), status);
    for (std::size_t w2 = 0; w2 < who.size(); ++w2) {
      Candidate& C = cands[who[w2]];
      try {
        for (int q = 0; q < 2; ++q)
          if (status[2 * w2 + q].code != SSG_OK)
            raise_unit_error(status[2 * w2 + q], gcfg[w2], *C.est);
        const double service = secs[2 * w2] + 64.0 * secs[2 * w2 + 1];
        const double per_replica = 1.0 / std::max(service, 1e-9);
        C.copts.initial_guess =
            std::max(1e-3, per_replica * static_cast<double>(C.cluster.par.num_replicas));
        require(C.copts.initial_guess > 0 && C.copts.tolerance > 0, "find_capacity: bad options");
        // the first probe's run_simulation preamble (validation, plan_memory)
        if (!C.sim_ok) throw Error(C.sim_error);
        live.push_back(who[w2]);
      } catch (const Error& e) {
        C.res.error = e.what();
        C.done = true;
      }
    }
  }

  if (by_cost) {
    // Longest-processing-time split on the capacity search's critical chain:
    // a probe at rate q spans n / q seconds of simulated time, so 1 / guess
    // orders the configs by how long their probe chains run.  Failed configs
    // cost nothing but still belong to one shard (their error rows).
    const std::vector<int> owner = lpt_split(cands, num_shards);
    std::vector<Candidate> mine;
    for (std::size_t k = 0; k < cands.size(); ++k)
      if (owner[k] == shard) mine.push_back(std::move(cands[k]));
    cands.swap(mine);
    live.clear();
    for (std::size_t k = 0; k < cands.size(); ++k)
      if (!cands[k].done) live.push_back(k);
  }
  if (owned) {
    owned->clear();
    for (const auto& C : cands) owned->push_back(C.index);
  }
  {
    // token tables for every distinct (SKU, tp, pp) operator table
    std::vector<SimConfig> tcfg;
    std::vector<std::size_t> tk;
    std::vector<SsgEstView> tests;
    std::vector<const DeviceEstimator*> test_of;
    for (const auto* e : ests) {
      tests.push_back(e->device().view);
      test_of.push_back(&e->device());
    }
    for (std::size_t k = 0; k < cands.size(); ++k) {
      if (!cands[k].sim_ok) continue;
      SimConfig c = cands[k].sim;
      c.est = static_cast<int32_t>(cands[k].cand.sku_index);
      tcfg.push_back(c);
      tk.push_back(k);
    }
    PhaseTimer t("search: token tables");
    if (std::getenv("SSG_NO_TABLES") == nullptr)
      build_token_tables(tcfg, tests, test_of, SS.tables);
    for (std::size_t i = 0; i < tk.size(); ++i) {
      SimConfig& c = cands[tk[i]].sim;
      c.tab_off = tcfg[i].tab_off;
      c.tab_cells = tcfg[i].tab_cells;
      c.tab_stride = tcfg[i].tab_stride;
      c.tab_tmax = tcfg[i].tab_tmax;
      c.tab_pmax = tcfg[i].tab_pmax;
    }
  }


  PhaseTimer t_rounds("search: rounds");
  // lanes: streams + buffers; every lane waits for the token tables
  const SweepKnobs knobs = knobs_from_env();
  LiveCandidates live_scope(static_cast<int64_t>(live.size()));
  const std::size_t nlanes =
      makespan ? 1
               : std::max<std::size_t>(1, std::min<std::size_t>(
                                              knobs.lanes >= 0 ? knobs.lanes : (g_sweeps_in_flight.load() > 1 ? 1 : 2),
                                              live.size()));
  while (SS.lanes.size() < nlanes) SS.lanes.push_back(borrow_lane());
  auto& ctx = context();
  cudaEvent_t origin;
  cuda_check(cudaEventCreate(&origin), "event");
  cuda_check(cudaEventRecord(origin, ctx.stream), "event");
  for (std::size_t g = 0; g < nlanes; ++g) {
    SweepLane& lane = *SS.lanes[g];
    lane.tables = SS.tables.ptr;
    lane.origin = origin;
    lane.intervals.clear();
    cuda_check(cudaStreamWaitEvent(lane.stream.s, origin, 0), "lane wait");
  }

  if (makespan) {
    std::vector<std::pair<std::size_t, double>> full;
    for (std::size_t k = 0; k < cands.size(); ++k)
      if (!cands[k].done) full.push_back({k, 0.0});
    {
      StreamScope scope(SS.lanes[0]->stream.s);
      run_round(*SS.lanes[0], cands, {}, full, true, w, opts.capacity);
    }
    for (const auto& f : full) {
      Candidate& C = cands[f.first];
      if (!C.res.failed()) {
        C.res.slo_pass = true;
        C.res.qps_per_dollar = 0.0;
      }
    }
  } else {
    // candidate groups, one per lane: ordered by initial guess (lowest rate =
    // longest probes first), dealt round-robin or in contiguous blocks
    std::vector<std::size_t> order = live;
    std::stable_sort(order.begin(), order.end(), [&](std::size_t a, std::size_t b) {
      return cands[a].copts.initial_guess < cands[b].copts.initial_guess;
    });
    std::vector<std::vector<std::size_t>> groups(nlanes);
    for (std::size_t i = 0; i < order.size(); ++i) {
      const std::size_t g = knobs.block ? i * nlanes / order.size() : i % nlanes;
      groups[g].push_back(order[i]);
    }
    std::vector<std::vector<std::size_t>> measured(nlanes);
    std::vector<std::exception_ptr> errors(nlanes);
    auto body = [&](std::size_t g) {
      try {
        cuda_check(cudaSetDevice(ctx.device), "cudaSetDevice");
        StatsScope stats_scope;
        StreamScope scope(SS.lanes[g]->stream.s);
        run_group(*SS.lanes[g], cands, groups[g], opts, w, knobs, measured[g]);
      } catch (...) {
        errors[g] = std::current_exception();
      }
    };
    std::vector<std::thread> threads;
    for (std::size_t g = 1; g < nlanes; ++g) threads.emplace_back(body, g);
    body(0);
    for (auto& t : threads) t.join();
    for (auto& e : errors)
      if (e) std::rethrow_exception(e);
    for (const auto& m : measured)
      for (auto k : m) {
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
  // k_simulate busy time: the union of every lane's launch intervals
  {
    std::vector<std::pair<float, float>> iv;
    for (std::size_t g = 0; g < nlanes; ++g) {
      iv.insert(iv.end(), SS.lanes[g]->intervals.begin(), SS.lanes[g]->intervals.end());
      SS.lanes[g]->origin = nullptr;
    }
    std::sort(iv.begin(), iv.end());
    double busy = 0.0, a = 0.0, b = 0.0;
    bool open = false;
    for (auto [x, y] : iv) {
      if (!open || x > b) {
        if (open) busy += b - a;
        a = x;
        b = y;
        open = true;
      } else {
        b = std::max<double>(b, y);
      }
    }
    if (open) busy += b - a;
    stats().simulate_busy_ms += busy;
    cudaEventDestroy(origin);
  }
  {
    // the sequential search's share of the device work: the probes its
    // find_capacity replay asks for, plus each SLO / static run
    RunStats& st = stats();
    for (auto& C : cands) {
      std::vector<const ProbeAnswer*> asked;
      try {
        replay_capacity(C.memo, C.copts, &asked);
      } catch (...) {
        // errors, unfinished searches: the asked prefix is still the reference's work
      }
      for (const ProbeAnswer* a : asked) {
        st.useful_iterations += a->iters;
        st.useful_entries += a->entries;
        st.useful_bytes += a->bytes;
      }
      st.useful_iterations += C.full_run.iters;
      st.useful_entries += C.full_run.entries;
      st.useful_bytes += C.full_run.bytes;
    }
  }
  for (auto& C : cands) results[C.index] = std::move(C.res);
  for (std::size_t i = 0; i < configs.size(); ++i)
    if (results[i].config.id.empty()) results[i].config = configs[i];
  return results;
}

double find_capacity(const std::function<bool(double)>& feasible_at,
                     const CapacitySearchOptions& opts) {  // search.hpp:145-174
  // the sweep's replay against a memo, answering each rate it asks for from the
  // caller's probe as it is first needed: the probes run in the reference's order
  ProbeMemo memo;
  while (true) {
    try {
      return replay_capacity(memo, opts);
    } catch (const NeedProbe& need) {
      ProbeAnswer a;
      a.feasible = feasible_at(need.q);
      memo.emplace(need.q, a);
    }
  }
}

double find_capacity_replay(const std::function<bool(double)>& feasible,
                            const CapacitySearchOptions& opts) {
  return find_capacity(feasible, opts);
}

double initial_qps_guess(const ModelSpec& spec, const CandidateConfig& cand,
                         const EstimatorModel& estimator, const ClusterConfig& cluster) {  // search.hpp:278-290
  auto ops = derive_operators(spec, cand.par);
  const std::int64_t len = std::min<std::int64_t>(512, spec.max_context);
  BatchComposition prefill, decode;
  prefill.prefill_lengths = {len};
  prefill.prefill_prior_context = {0};
  decode.decode_context_lengths = {len};
  const double service =
      predict_batch(estimator, ops, prefill) + 64.0 * predict_batch(estimator, ops, decode);
  const double per_replica = 1.0 / std::max(service, 1e-9);
  return std::max(1e-3, per_replica * static_cast<double>(cluster.par.num_replicas));
}

std::vector<ConfigResult> evaluate_configs(const ModelSpec& spec,
                                           const std::vector<CandidateConfig>& cands,
                                           const std::vector<DeviceProfile>& skus,
                                           const std::vector<const EstimatorModel*>& estimators,
                                           const std::vector<Request>& workload,
                                           const SearchOptions& opts) {
  if (cands.empty()) return {};
  SearchSession session(spec, cands, skus, estimators, workload, opts);
  return session.evaluate();
}

ConfigResult evaluate_config(const ModelSpec& spec, const CandidateConfig& cand,
                             const DeviceProfile& dev, const EstimatorModel& estimator,
                             const std::vector<Request>& workload, const SearchOptions& opts) {
  CandidateConfig c = cand;
  c.sku_index = 0;
  ConfigResult r = evaluate_configs(spec, {c}, {dev}, {&estimator}, workload, opts).at(0);
  r.config = cand;
  return r;
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
