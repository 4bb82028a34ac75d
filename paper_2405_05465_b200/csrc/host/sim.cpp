// sim.cpp -- run_simulation on the GPU: config flattening, unit decomposition,
// launch, and reassembly of the reference's SimulationResult.
//
// reference: sim.hpp:135-320, scheduler.hpp:146-155 (enqueue capacity error),
//            model_spec.hpp:203-266 (operators), memory.hpp:21-46
#include <algorithm>
#include <cmath>
#include <map>
#include <numeric>
#include <string>
#include <unordered_map>

#include "sim_host.h"
#include "engine_limits.h"

namespace ssg {

using namespace servesim;

void fill_sim_ops(SimConfig& c, const std::vector<OperatorDescriptor>& ops, const DeviceEstimator& de) {
  internal_check(ops.size() <= SSG_MAX_OPS, "operator set larger than the device table");
  c.nops = static_cast<int32_t>(ops.size());
  c.tab_off = -1;  // no token tables unless a caller builds them (build_token_tables)
  c.tab_tmax = 0;
  c.tab_pmax = 0;
  c.tab_stride = 0;
  c.tab_cells = 0;
  c.idx_pre = c.idx_dec = -1;
  c.ncomm = 0;
  c.qb_fixed = c.qb_pre = c.qb_dec = 0;
  for (std::size_t i = 0; i < ops.size(); ++i) {
    const auto& d = ops[i];
    SimOp& o = c.ops[i];
    o.slot = de.slot(d.op, d.tp_degree);
    o.qbytes = o.slot >= 0 ? de.qbytes[o.slot] : 0;
    o.cls = static_cast<int32_t>(d.op_class);
    o.op = static_cast<int32_t>(d.op);
    o.count = static_cast<double>(d.count);
    o.kvb = 2.0 * static_cast<double>(d.elem_bytes) *
            static_cast<double>(d.kv_heads_per_device * d.head_dim);
    o.payload = static_cast<double>(d.payload_bytes_per_token);
    switch (d.op) {
      case OpName::QkvProj:
      case OpName::AttnOutProj:
      case OpName::MlpUpProj:
      case OpName::MlpDownProj:
        o.flop_kind = 0;
        o.fa = static_cast<double>(d.in_dim);
        o.fb = static_cast<double>(d.out_dim);
        break;
      case OpName::ActFn:
        o.flop_kind = 1;
        o.fa = static_cast<double>(d.in_dim);
        break;
      case OpName::AddNorm:
        o.flop_kind = 2;
        o.fa = static_cast<double>(d.in_dim);
        break;
      case OpName::AttnPrefill:
      case OpName::AttnDecode:
        o.flop_kind = d.op == OpName::AttnPrefill ? 3 : 4;
        o.fa = static_cast<double>(d.q_heads_per_device * d.head_dim);
        break;
      default:
        o.flop_kind = 5;
        break;
    }
  }
  bool seen_seq = false, seen_comm = false;
  for (int i = 0; i < c.nops; ++i) {
    const SimOp& o = c.ops[i];
    if (o.cls == SSG_CLS_TOKEN) {
      internal_check(!seen_seq && !seen_comm, "operator table: token ops must come first");
      c.qb_fixed += o.qbytes;
    } else if (o.cls == SSG_CLS_SEQ) {
      internal_check(!seen_comm, "operator table: attention before collectives");
      seen_seq = true;
      if (o.flop_kind == 3) {
        c.idx_pre = i;
        c.qb_pre = o.qbytes;
      } else {
        c.idx_dec = i;
        c.qb_dec = o.qbytes;
      }
    } else {
      seen_comm = true;
      c.qb_fixed += o.qbytes;
      c.ncomm += 1;
    }
  }
  internal_check(c.ncomm <= 3, "operator table: more than three collectives");
}

SimConfig make_sim_config(const ClusterConfig& cl, const EstimatorModel& est, int32_t est_index,
                          MemoryPlan* plan_out) {
  validate(cl.spec);
  validate(cl.spec, cl.par);
  validate(cl.dev);
  validate(cl.policy);
  auto ops = derive_operators(cl.spec, cl.par);
  for (const auto& d : ops) est.find(d.op, d.tp_degree);  // throws the reference's message
  MemoryPlan plan = plan_memory(cl.spec, cl.par, cl.dev, cl.policy.block_size,
                                cl.policy.watermark_fraction, cl.policy.activation_reserve_fraction);
  if (plan_out) *plan_out = plan;
  const std::int64_t threshold =
      cl.deferred_threshold > 0 ? cl.deferred_threshold : cl.policy.max_batch_size;
  require(cl.par.num_replicas >= 1, "router: need at least one replica");
  require(threshold >= 1, "router: deferred threshold must be >= 1");

  const auto& de = est.device();
  SimConfig c{};
  c.policy = static_cast<int32_t>(cl.policy.policy);
  // queues are sized by min(max_batch_size, requests) per unit (SimUnit::mb_ws), so
  // any batch cap is exact; one above INT32_MAX never binds (a unit holds fewer requests)
  c.max_batch = static_cast<int32_t>(std::min<std::int64_t>(cl.policy.max_batch_size, INT32_MAX));
  c.max_tokens = static_cast<int32_t>(std::min<std::int64_t>(cl.policy.max_tokens_per_iter, INT32_MAX));
  c.chunk = static_cast<int32_t>(std::min<std::int64_t>(cl.policy.chunk_size, INT32_MAX));
  c.token_granular = cl.policy.policy == SchedulerPolicy::LightLLM ? 1 : 0;
  c.pp = static_cast<int32_t>(cl.par.pp_degree);
  c.tp = static_cast<int32_t>(cl.par.tp_degree);
  c.est = est_index;
  c.block_size = plan.block_size;
  c.bs_shift = -1;
  for (int k = 0; k < 62; ++k)
    if ((int64_t(1) << k) == plan.block_size) c.bs_shift = k;
  // block counts on the device: token counts stay below 2^31 (request lengths
  // are checked), so ceil-division by a block size below 2^31 is one 64-bit
  // high multiply (block_magic), exact for numerators below 2^32
  require(plan.block_size < (int64_t(1) << 31), "ssg: block_size above the device engine limit");
  c.bs_magic = block_magic(plan.block_size, c.token_granular != 0);
  c.total_units = c.token_granular ? plan.kv_capacity_tokens : plan.num_blocks;
  c.watermark_units = c.token_granular ? plan.watermark_blocks * plan.block_size : plan.watermark_blocks;
  c.cpu_overhead = cl.cpu_overhead_per_iter;
  c.nops = static_cast<int32_t>(ops.size());
  c.routing = static_cast<int32_t>(cl.routing);
  c.defer_threshold = static_cast<int32_t>(std::min<std::int64_t>(threshold, INT32_MAX));
  fill_sim_ops(c, ops, de);
  return c;
}

void build_token_tables(std::vector<SimConfig>& cfgs, const std::vector<SsgEstView>& ests,
                        const std::vector<const DeviceEstimator*>& est_of,
                        DeviceBuffer<double>& pool) {
  if (cfgs.empty()) return;
  auto& ctx = context();
  cudaStream_t s = ctx.stream;
  // table key: estimator + the op table (slot, count, payload, kvb, flop operands)
  auto key_of = [](const SimConfig& c) {
    std::string k(reinterpret_cast<const char*>(&c.est), sizeof c.est);
    k.append(reinterpret_cast<const char*>(&c.nops), sizeof c.nops);
    for (int i = 0; i < c.nops; ++i) {
      SimOp o = c.ops[i];
      o.qbytes = 0;
      k.append(reinterpret_cast<const char*>(&o), sizeof o);
    }
    return k;
  };
  std::map<std::string, int32_t> table_of;
  std::vector<SimConfig> reps;  // one representative per table
  std::vector<int32_t> cap;
  std::vector<int32_t> which(cfgs.size());
  for (std::size_t i = 0; i < cfgs.size(); ++i) {
    auto [it, fresh] = table_of.emplace(key_of(cfgs[i]), static_cast<int32_t>(reps.size()));
    which[i] = it->second;
    if (!fresh) continue;
    // t can only be valid up to the smallest token-op bbox upper bound
    double up = 1e18;
    const DeviceEstimator& de = *est_of.at(cfgs[i].est);
    for (int k = 0; k < cfgs[i].nops; ++k)
      if (cfgs[i].ops[k].cls == SSG_CLS_TOKEN && cfgs[i].ops[k].slot >= 0)
        up = std::min(up, de.host_models[cfgs[i].ops[k].slot].upper[0]);
    cap.push_back(static_cast<int32_t>(std::min(up, 1.0e6)));
    // axis-0 cell rows need both attention models to be 2-D interpolators
    auto interp2 = [&](int32_t idx) {
      if (idx < 0) return false;
      const int32_t slot = cfgs[i].ops[idx].slot;
      if (slot < 0) return false;
      const SsgModelDesc& md = de.host_models[slot];
      return md.kind == SSG_KIND_INTERP && md.nf == 2;
    };
    reps.push_back(cfgs[i]);
    reps.back().tab_cells = interp2(cfgs[i].idx_pre) && interp2(cfgs[i].idx_dec) ? 1 : 0;
  }
  int32_t stride = 2;
  for (auto c : cap) stride = std::max(stride, c + 1);
  const int32_t n = static_cast<int32_t>(reps.size());
  for (int32_t t = 0; t < n; ++t) {
    reps[t].tab_off = static_cast<int64_t>(t) * SSG_TAB_ROWS * stride;
    reps[t].tab_stride = stride;
  }
  pool.resize(static_cast<std::size_t>(n) * SSG_TAB_ROWS * stride);
  DeviceBuffer<SimConfig> d_cfg;
  DeviceBuffer<SsgEstView> d_est;
  DeviceBuffer<uint8_t> d_valid(static_cast<std::size_t>(n) * stride);
  d_cfg.upload(reps, s);
  d_est.upload(ests, s);
  launch_build_tables(d_cfg.ptr, n, stride, d_est.ptr, pool.ptr, d_valid.ptr, s);
  std::vector<uint8_t> valid(static_cast<std::size_t>(n) * stride);
  d_valid.download(valid.data(), valid.size(), s);
  cuda_check(cudaStreamSynchronize(s), "token tables");
  for (int32_t t = 0; t < n; ++t) {
    int32_t tmax = 0, pmax = 0;
    while (tmax + 1 < stride && (valid[static_cast<std::size_t>(t) * stride + tmax + 1] & 1)) ++tmax;
    while (pmax + 1 < stride && (valid[static_cast<std::size_t>(t) * stride + pmax + 1] & 2)) ++pmax;
    reps[t].tab_tmax = tmax;
    reps[t].tab_pmax = std::min(pmax, tmax);
  }
  for (std::size_t i = 0; i < cfgs.size(); ++i) {
    const SimConfig& r = reps[which[i]];
    cfgs[i].tab_off = r.tab_tmax >= 1 ? r.tab_off : -1;
    cfgs[i].tab_stride = r.tab_stride;
    cfgs[i].tab_tmax = r.tab_tmax;
    cfgs[i].tab_pmax = r.tab_pmax;
    cfgs[i].tab_cells = r.tab_off >= 0 && r.tab_tmax >= 1 ? r.tab_cells : 0;
  }
}

static int32_t pow2_above(int64_t n) {
  int64_t c = 2;
  while (c <= n) c <<= 1;
  internal_check(c <= (int64_t(1) << 30), "unit too large for the device queue");
  return static_cast<int32_t>(c);
}

int32_t SimJobs::add_unit(const UnitSpec& spec, const std::vector<Request>& reqs,
                          const std::vector<int32_t>& event_order) {
  const SimConfig& cfg = configs.at(spec.config);
  SimUnit u{};
  u.config = spec.config;
  u.n = static_cast<int32_t>(reqs.size());
  u.R = spec.R;
  u.flags = spec.flags;
  u.req_off = static_cast<int64_t>(hot.size());
  u.wait_cap = pow2_above(u.n);
  u.mb_ws = static_cast<int32_t>(std::min<int64_t>(cfg.max_batch, std::max<int32_t>(u.n, 1)));
  u.ws_off = ws_words;
  ws_words += static_cast<int64_t>(u.R) * (6LL * u.mb_ws + u.wait_cap) + u.wait_cap + 2 +
              SSG_PP_SCRATCH_WORDS(cfg.pp);
  u.rep_off = nreps;
  nreps += u.R;
  u.abort_thr = spec.abort_thr;
  u.abort_max_late = spec.abort_max_late;
  u.log_off = log_words;
  u.log_cap = spec.log_cap;
  log_words += spec.log_cap;
  for (std::size_t j = 0; j < reqs.size(); ++j) {
    const Request& r = reqs[j];
    require(r.prefill_tokens < INT32_MAX / 2 && r.decode_tokens < INT32_MAX / 2,
            "ssg: request lengths above the device engine limit");
    ReqHot h{};
    h.prefill = static_cast<int32_t>(r.prefill_tokens);
    h.decode = static_cast<int32_t>(r.decode_tokens);
    hot.push_back(h);
    ReqTimes t{};
    t.arrival = r.arrival_time;
    tm.push_back(t);
    ids.push_back(r.id);
    if (spec.flags & SSG_UF_EMISSIONS) {
      emit_base.push_back(emissions);
      emissions += r.decode_tokens;
    } else {
      emit_base.push_back(-1);
    }
  }
  if (!event_order.empty()) {
    any_order = true;
    for (auto k : event_order) arr_order.push_back(k);
  } else {
    for (int32_t k = 0; k < u.n; ++k) arr_order.push_back(k);
  }
  units.push_back(u);
  return static_cast<int32_t>(units.size() - 1);
}

void run_jobs(const SimJobs& J, SimResults& R, bool want_requests) {
  auto& ctx = context();
  cudaStream_t s = ctx.stream;
  DeviceBuffer<SimConfig> d_cfg;
  DeviceBuffer<SsgEstView> d_est;
  DeviceBuffer<SimUnit> d_units;
  DeviceBuffer<ReqHot> d_hot;
  DeviceBuffer<ReqTimes> d_tm;
  DeviceBuffer<int64_t> d_ids, d_emit_base, d_log;
  DeviceBuffer<int32_t> d_restarts, d_order, d_ws, d_launch;
  DeviceBuffer<double> d_emis;
  DeviceBuffer<RepState> d_reps;
  DeviceBuffer<SimUnitOut> d_out;
  d_cfg.upload(J.configs, s);
  d_est.upload(J.ests, s);
  d_units.upload(J.units, s);
  d_hot.upload(J.hot, s);
  d_tm.upload(J.tm, s);
  d_ids.upload(J.ids, s);
  d_restarts.resize(std::max<std::size_t>(1, J.hot.size()));
  if (J.emissions > 0) {
    d_emit_base.upload(J.emit_base, s);
    d_emis.resize(static_cast<std::size_t>(J.emissions));
  }
  if (J.any_order) d_order.upload(J.arr_order, s);
  d_ws.resize(static_cast<std::size_t>(std::max<int64_t>(1, J.ws_words)));
  d_reps.resize(static_cast<std::size_t>(std::max<int64_t>(1, J.nreps)));
  if (J.log_words > 0) d_log.resize(static_cast<std::size_t>(J.log_words));
  d_out.resize(J.units.size());
  // longest units first: requests x decode length is a fair proxy
  std::vector<int32_t> order(J.units.size());
  std::iota(order.begin(), order.end(), 0);
  std::vector<int64_t> work(J.units.size(), 0);
  for (std::size_t u = 0; u < J.units.size(); ++u)
    for (int32_t j = 0; j < J.units[u].n; ++j) work[u] += J.hot[J.units[u].req_off + j].decode;
  std::stable_sort(order.begin(), order.end(), [&](int32_t a, int32_t b) { return work[a] > work[b]; });
  d_launch.upload(order, s);

  SimLaunch L{};
  L.configs = d_cfg.ptr;
  L.units = d_units.ptr;
  L.order = d_launch.ptr;
  L.nunits = static_cast<int64_t>(J.units.size());
  L.ests = d_est.ptr;
  L.hot = d_hot.ptr;
  L.tm = d_tm.ptr;
  L.ids = d_ids.ptr;
  L.restarts = d_restarts.ptr;
  L.emit_base = J.emissions > 0 ? d_emit_base.ptr : nullptr;
  L.emissions = J.emissions > 0 ? d_emis.ptr : nullptr;
  L.arr_order = J.any_order ? d_order.ptr : nullptr;
  L.reps = d_reps.ptr;
  L.ws = d_ws.ptr;
  L.log = J.log_words > 0 ? d_log.ptr : nullptr;
  L.out = d_out.ptr;
  L.tables = J.tables;
  bool observed = false;
  for (const auto& u : J.units) observed = observed || (u.flags & SSG_UF_OBSERVER);
  L.fast_forward = fast_forward_enabled() && !observed;
  L.has_forest = J.has_forest ? 1 : 0;
  L.all_lone = all_lone_units(L, J.units, J.configs) ? 1 : 0;
  cudaEvent_t ev0, ev1;
  cuda_check(cudaEventCreate(&ev0), "event");
  cuda_check(cudaEventCreate(&ev1), "event");
  cuda_check(cudaEventRecord(ev0, s), "event");
  launch_simulate(L, s);
  cuda_check(cudaEventRecord(ev1, s), "event");

  R.out.resize(J.units.size());
  d_out.download(R.out.data(), R.out.size(), s);
  R.reps.resize(static_cast<std::size_t>(J.nreps));
  d_reps.download(R.reps.data(), R.reps.size(), s);
  if (want_requests) {
    R.tm.resize(J.tm.size());
    d_tm.download(R.tm.data(), R.tm.size(), s);
    R.restarts.resize(J.hot.size());
    d_restarts.download(R.restarts.data(), R.restarts.size(), s);
  }
  if (J.emissions > 0) {
    R.emissions.resize(static_cast<std::size_t>(J.emissions));
    d_emis.download(R.emissions.data(), R.emissions.size(), s);
  }
  {
    PhaseTimer t("sim: kernel + downloads");
    cuda_check(cudaStreamSynchronize(s), "simulate");
  }
  if (J.log_words > 0) {
    // only the words each unit wrote (the arena is sized for the worst case)
    PhaseTimer t("sim: batch log download");
    R.log.resize(static_cast<std::size_t>(J.log_words));
    for (std::size_t u = 0; u < J.units.size(); ++u) {
      const int64_t used = R.out[u].log_used;
      if (used <= 0) continue;
      const int64_t off = J.units[u].log_off;
      cuda_check(cudaMemcpyAsync(R.log.data() + off, d_log.ptr + off,
                                 static_cast<std::size_t>(used) * sizeof(int64_t),
                                 cudaMemcpyDeviceToHost, s), "D2H");
      stats().d2h_bytes += used * static_cast<int64_t>(sizeof(int64_t));
    }
    cuda_check(cudaStreamSynchronize(s), "batch log");
  }
  float ms = 0.f;
  cuda_check(cudaEventElapsedTime(&ms, ev0, ev1), "event");
  cudaEventDestroy(ev0);
  cudaEventDestroy(ev1);
  RunStats& st = stats();
  st.launches_simulate += 1;
  st.simulate_ms += ms;
  st.units += static_cast<int64_t>(R.out.size());
  for (const auto& o : R.out) {
    st.iterations += o.iterations;
    st.entries += o.entries;
    st.events += o.events;
    st.predictor_bytes += o.qbytes;
    st.entry_bytes += 48 * o.entries;  // request progress read 32 B + write 16 B per entry
  }
}

[[noreturn]] void raise_unit_error(const SimUnitOut& o, const SimConfig& cfg,
                                   const EstimatorModel& est) {
  switch (o.code) {
    case SSG_ERR_ENQUEUE:
      throw Error("request " + std::to_string(o.err_i64[0]) + " needs " +
                  std::to_string(o.err_i64[1]) + " KV units but replica capacity is " +
                  std::to_string(cfg.total_units) + " (model/config cannot serve this request)");
    case SSG_ERR_BBOX: {
      const auto& de = est.device();
      const SsgModelDesc& d = de.host_models.at(o.err_i32);
      const OpModelKey key{static_cast<OpName>(d.op), d.tp};
      throw Error(bbox_error_message(est.find(key.op, key.tp_degree), key,
                                     static_cast<int>(o.err_i64[0]), o.err_f64));
    }
    case SSG_ERR_EXP_RANGE:
      throw InternalError("predict: regressor output outside exp fast path");
    default:
      break;
  }
  static const char* kInternal[] = {"?",
                                    "request not in waiting queue",
                                    "predict_batch: non-positive prediction",
                                    "non-positive iteration latency",
                                    "prefill progressed past its target",
                                    "sarathi: token budget exceeded",
                                    "event time regression",
                                    "simulation drained with unfinished request"};
  const int k = (o.err_i32 >= 1 && o.err_i32 <= 7) ? o.err_i32 : 0;
  std::string msg = kInternal[k];
  if (k == 7) msg += " " + std::to_string(o.err_i64[0]);
  throw InternalError(msg);
}

}  // namespace ssg

namespace servesim {

using namespace ssg;

// Read-only ReplicaScheduler views handed to SimObserver::on_batch: the
// replica's configuration plus the scheduler state the batch log recorded.
struct SchedulerView {
  static ReplicaScheduler make(const PolicyConfig& cfg, const MemoryPlan& plan) {
    ReplicaScheduler s;
    s.cfg_ = cfg;
    s.plan_ = plan;
    s.mem_ = BlockManager(plan, cfg.policy == SchedulerPolicy::LightLLM);
    return s;
  }
  static void set(ReplicaScheduler& s, const BatchLog& b) {
    s.mem_.allocated_ = b.kv_allocated_units;
    s.outstanding_ = static_cast<std::size_t>(b.outstanding);
    s.preemptions_ = static_cast<std::size_t>(b.preemptions);
    s.ft_members_ = b.ft_members;
  }
};

namespace {

struct Placement {
  DeviceBuffer<double> tables;
  SimJobs jobs;
  std::vector<std::pair<int32_t, int32_t>> where;  // trace index -> (unit, local)
  bool coupled = false;
};

// Units for one run_simulation call.  Round-robin replicas are independent
// (each owns the arrivals at event positions r, r+R, ...) and become one unit
// each; otherwise -- or when exact cross-replica event order matters -- all
// replicas share one coupled unit.
Placement place(const ClusterConfig& cluster, const std::vector<Request>& trace,
                const EstimatorModel& estimator, const SimOptions& opts, bool coupled) {
  Placement P;
  P.coupled = coupled;
  SimJobs& J = P.jobs;
  J.configs.push_back(make_sim_config(cluster, estimator, 0));
  J.ests.push_back(estimator.device().view);
  {
    PhaseTimer t("sim: token tables");
    build_token_tables(J.configs, J.ests, {&estimator.device()}, P.tables);
  }
  J.has_forest = estimator.device().has_forest;
  J.tables = P.tables.ptr;
  const int R = static_cast<int>(cluster.par.num_replicas);
  const std::size_t n = trace.size();
  std::vector<int32_t> ev(n);
  std::iota(ev.begin(), ev.end(), 0);
  std::stable_sort(ev.begin(), ev.end(), [&](int32_t a, int32_t b) {
    return trace[a].arrival_time < trace[b].arrival_time;
  });
  const bool want_log = opts.record_batches || opts.record_iterations || opts.observer;
  UnitSpec us;
  us.config = 0;
  us.flags = SSG_UF_EMISSIONS | (want_log ? SSG_UF_BATCH_LOG : 0) |
             (opts.observer ? SSG_UF_OBSERVER : 0) |
             (opts.abort_delay_threshold > 0.0 ? SSG_UF_ABORT : 0);
  us.abort_thr = opts.abort_delay_threshold;
  us.abort_max_late = static_cast<int32_t>(std::min<std::size_t>(opts.abort_max_late, INT32_MAX));
  std::vector<std::vector<int32_t>> members;
  if (!coupled) {
    members.resize(R);
    for (std::size_t p = 0; p < n; ++p) members[p % R].push_back(ev[p]);
    us.R = 1;
  } else {
    require(R <= kMaxCoupledReplicas, "ssg: least_outstanding/deferred routing supports up to " +
                                          std::to_string(kMaxCoupledReplicas) + " replicas");
    members.push_back(ev);
    us.R = R;
  }
  P.where.assign(n, {0, 0});
  for (std::size_t u = 0; u < members.size(); ++u) {
    const auto& m = members[u];
    std::vector<int32_t> rank(m);
    std::stable_sort(rank.begin(), rank.end(), [&](int32_t a, int32_t b) {
      if (trace[a].arrival_time != trace[b].arrival_time)
        return trace[a].arrival_time < trace[b].arrival_time;
      return trace[a].id < trace[b].id;
    });
    std::vector<Request> reqs;
    reqs.reserve(rank.size());
    int64_t tokens = 0;
    for (std::size_t k = 0; k < rank.size(); ++k) {
      P.where[rank[k]] = {static_cast<int32_t>(u), static_cast<int32_t>(k)};
      reqs.push_back(trace[rank[k]]);
      tokens += trace[rank[k]].prefill_tokens + trace[rank[k]].decode_tokens;
    }
    std::vector<int32_t> order;
    bool identity = true;
    for (std::size_t k = 0; k < m.size(); ++k) {
      order.push_back(P.where[m[k]].second);
      if (order.back() != static_cast<int32_t>(k)) identity = false;
    }
    if (identity) order.clear();
    UnitSpec s2 = us;
    if (want_log) s2.log_cap = 1024 + (opts.observer ? 24 : 16) * tokens;
    J.add_unit(s2, reqs, order);
  }
  return P;
}

}  // namespace

SimulationOutput run_simulation_logged(const ClusterConfig& cluster,
                                       const std::vector<Request>& trace,
                                       const EstimatorModel& estimator, const SimOptions& opts) {
  for (const auto& r : trace)
    require(r.has_arrival(), "trace request " + std::to_string(r.id) +
                                 " has no arrival time; assign arrivals before simulating");
  const int R = static_cast<int>(cluster.par.num_replicas);
  // probes with an abort bound need the global event order of late schedules
  // an observer sees every replica's batches in the global event order: one
  // coupled unit logs them in exactly that order
  bool coupled = cluster.routing != RoutingPolicy::RoundRobin ||
                 (opts.abort_delay_threshold > 0.0 && R > 1) || (opts.observer && R > 1);
  if (opts.observer)
    require(R <= kMaxCoupledReplicas, "ssg: an observed simulation supports up to " +
                                          std::to_string(kMaxCoupledReplicas) + " replicas");
  PhaseTimer total("sim: run_simulation");
  Placement P = place(cluster, trace, estimator, opts, coupled);
  SimResults res;
  {
    PhaseTimer t("sim: run_jobs");
    run_jobs(P.jobs, res, true);
  }
  PhaseTimer t_assemble("sim: reassemble");
  int errors = 0;
  for (const auto& o : res.out) errors += o.code != SSG_OK;
  if (errors > 1 && !coupled && R <= kMaxCoupledReplicas) {
    // several independent replicas failed: replay coupled for the exact first one
    P = place(cluster, trace, estimator, opts, true);
    run_jobs(P.jobs, res, true);
  }
  const SimJobs& J = P.jobs;
  const SimConfig& cfg = J.configs[0];
  const bool want_log = opts.record_batches || opts.record_iterations || opts.observer;
  SimulationOutput out;
  SimulationResult& r = out.result;
  std::vector<BatchLog> batches;
  if (want_log) {
    for (std::size_t u = 0; u < J.units.size(); ++u) {
      const SimUnit& su = J.units[u];
      const int64_t used = res.out[u].log_used;
      internal_check(used >= 0, "batch log overflow");
      for (int64_t p = 0; p < used;) {
        const int64_t* L = res.log.data() + su.log_off + p;
        BatchLog b;
        b.replica = !P.coupled ? u : static_cast<std::size_t>(L[0]);
        b.now = __builtin_bit_cast(double, L[1]);
        b.kv_allocated_units = L[2];
        const int64_t np = L[3], nd = L[4];
        const double lat = __builtin_bit_cast(double, L[5]);
        for (int64_t k = 0; k < np; ++k)
          b.entries.push_back(BatchEntryLog{true, L[6 + 3 * k], L[7 + 3 * k], L[8 + 3 * k]});
        for (int64_t k = 0; k < nd; ++k)
          b.entries.push_back(BatchEntryLog{false, L[6 + 3 * np + 2 * k], 1, L[7 + 3 * np + 2 * k]});
        int64_t extra = 0;
        if (su.flags & SSG_UF_OBSERVER) {
          const int64_t* X = L + 6 + 3 * np + 2 * nd;
          b.outstanding = X[0];
          b.preemptions = X[1];
          b.ft_members.assign(X + 4, X + 4 + X[3]);
          extra = 4 + X[3];
        }
        if (opts.record_iterations && lat > 0.0) {
          IterationRecord it;
          it.start = b.now;
          it.latency = lat;
          it.replica = b.replica;
          it.batch_requests = np + nd;
          int64_t tok = nd;
          for (int64_t k = 0; k < np; ++k) tok += L[7 + 3 * k];
          it.current_tokens = tok;
          it.prefill_entries = np;
          it.decode_entries = nd;
          it.kv_utilization =
              static_cast<double>(b.kv_allocated_units) / static_cast<double>(cfg.total_units);
          r.iterations.push_back(it);
        }
        batches.push_back(std::move(b));
        p += 6 + 3 * np + 2 * nd + extra;
      }
    }
    std::stable_sort(r.iterations.begin(), r.iterations.end(), [](const auto& a, const auto& b) {
      return a.start != b.start ? a.start < b.start : a.replica < b.replica;
    });
  }
  if (opts.observer) {
    // SimObserver::on_batch in event order (the coupled unit logged it so),
    // including the batches before an error or abort, as the reference calls it
    std::vector<RequestState> states(trace.size());
    std::unordered_map<std::int64_t, RequestState*> by_id;
    for (std::size_t i = 0; i < trace.size(); ++i) {
      states[i].req = trace[i];
      by_id.emplace(trace[i].id, &states[i]);
    }
    MemoryPlan plan = plan_memory(cluster.spec, cluster.par, cluster.dev, cluster.policy.block_size,
                                  cluster.policy.watermark_fraction,
                                  cluster.policy.activation_reserve_fraction);
    std::vector<ReplicaScheduler> views;
    for (int k = 0; k < R; ++k) views.push_back(SchedulerView::make(cluster.policy, plan));
    for (const auto& b : batches) {
      BatchPlan bp;
      for (const auto& e : b.entries) {
        RequestState* rs = by_id.at(e.request_id);
        if (e.prefill)
          bp.prefills.push_back({rs, e.tokens, e.context});
        else
          bp.decodes.push_back({rs, e.context});
      }
      ReplicaScheduler& v = views.at(b.replica);
      SchedulerView::set(v, b);
      opts.observer->on_batch(b.replica, b.now, bp, v);
    }
  }
  const SimUnitOut* first_err = nullptr;
  bool aborted = false;
  for (const auto& o : res.out) {
    if (o.code != SSG_OK && (!first_err || o.err_time < first_err->err_time)) first_err = &o;
    if (o.aborted) aborted = true;
  }
  if (first_err) raise_unit_error(*first_err, cfg, estimator);
  if (aborted) throw ProbeInfeasible();

  const std::size_t n = trace.size();
  r.num_devices = cluster.gpus_used();
  r.peak_device_flops = cluster.dev.peak_flops;
  r.replicas.resize(R);
  double span = 0.0, flops = 0.0;
  for (std::size_t u = 0; u < J.units.size(); ++u) {
    span = std::max(span, res.out[u].span);
    flops += res.out[u].flops;
  }
  r.simulated_span = span;
  r.total_model_flops = flops;
  for (int rep = 0; rep < R; ++rep) {
    const RepState& s = !P.coupled ? res.reps[J.units[rep].rep_off] : res.reps[J.units[0].rep_off + rep];
    ReplicaAggregate& a = r.replicas[rep];
    a.busy_time = s.busy_time;
    a.iterations = s.iterations;
    a.tokens_processed = s.tokens;
    a.peak_kv_utilization = s.peak_kv;
    a.preemptions = static_cast<std::size_t>(s.preemptions);
  }
  r.requests.resize(n);
  for (std::size_t i = 0; i < n; ++i) {
    const SimUnit& u = J.units[P.where[i].first];
    const int64_t g = u.req_off + P.where[i].second;
    RequestRecord& rec = r.requests[i];
    rec.id = trace[i].id;
    rec.arrival = trace[i].arrival_time;
    rec.first_scheduled = res.tm[g].first_sched;
    rec.first_token = res.tm[g].first_tok;
    rec.completion = res.tm[g].completion;
    rec.prefill_tokens = trace[i].prefill_tokens;
    rec.decode_tokens = trace[i].decode_tokens;
    rec.restarts = res.restarts[g];
    const int64_t b = J.emit_base[g];
    rec.emission_times.assign(res.emissions.begin() + b,
                              res.emissions.begin() + b + trace[i].decode_tokens);
  }
  if (opts.record_batches) out.batches = std::move(batches);
  return out;
}

double predict_batch(const EstimatorModel& model, const std::vector<OperatorDescriptor>& ops,
                     const BatchComposition& batch) {  // estimator.hpp:294-348, on the GPU
  require(batch.prefill_prior_context.empty() ||
              batch.prefill_prior_context.size() == batch.prefill_lengths.size(),
          "predict_batch: prefill_prior_context size mismatch");
  require(batch.total_current_tokens() > 0, "predict_batch: empty batch");
  // the models the reference would look up, in its order (a missing one raises first)
  for (const auto& d : ops) {
    if (d.op == OpName::AttnPrefill && batch.prefill_lengths.empty()) continue;
    if (d.op == OpName::AttnDecode && batch.decode_context_lengths.empty()) continue;
    model.find(d.op, d.tp_degree);
  }
  SimConfig cfg{};
  fill_sim_ops(cfg, ops, model.device());
  const int64_t np = static_cast<int64_t>(batch.prefill_lengths.size());
  const int64_t nd = static_cast<int64_t>(batch.decode_context_lengths.size());
  std::vector<int64_t> prior = batch.prefill_prior_context;
  prior.resize(static_cast<std::size_t>(np), 0);
  const int64_t p_off[2] = {0, np}, d_off[2] = {0, nd};
  double seconds = 0.0, flops = 0.0;
  predict_batches(model, cfg, 1, p_off, batch.prefill_lengths.data(), prior.data(), d_off,
                  batch.decode_context_lengths.data(), &seconds, &flops);
  return seconds;
}

SimulationResult run_simulation(const ClusterConfig& cluster, const std::vector<Request>& trace,
                                const EstimatorModel& estimator, const SimOptions& opts) {
  return run_simulation_logged(cluster, trace, estimator, opts).result;
}

}  // namespace servesim
