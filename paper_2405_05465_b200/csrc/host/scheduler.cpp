// scheduler.cpp -- the reference's scheduler plugin API (ReplicaScheduler,
// BlockManager; scheduler.hpp:136-233, memory.hpp:51-104) over HBM state.
//
// Every ReplicaScheduler call is one launch of k_sched_op (sched_api.cu): a
// warp runs the device scheduler -- the same functions k_simulate runs at each
// BatchStart -- on the replica's queues and block accounting, then the host
// copies back what the caller can observe: the plan, the replica counters and
// the fields of the caller's RequestStates the scheduler owns.
#include <algorithm>
#include <unordered_map>

#include "engine_limits.h"
#include "runtime.h"
#include "sched_api.h"

namespace servesim {

using ssg::DeviceBuffer;
using ssg::cuda_check;

// ------------------------------------------------------------------ BlockManager
bool BlockManager::try_reserve(std::int64_t request_id, std::int64_t tokens) {  // memory.hpp:82-89
  const std::int64_t need = shortfall(request_id, tokens);
  if (need > free_units()) return false;
  held_[request_id] += need;
  allocated_ += need;
  internal_check(allocated_ <= total_units(), "BlockManager: oversubscribed");
  return true;
}

void BlockManager::release(std::int64_t request_id) {  // memory.hpp:91-97
  auto it = held_.find(request_id);
  if (it == held_.end()) return;
  allocated_ -= it->second;
  held_.erase(it);
  internal_check(allocated_ >= 0, "BlockManager: negative allocation");
}

// ------------------------------------------------------------------ device state
namespace {

int32_t pow2_above(int64_t n) {
  int64_t c = 2;
  while (c <= n) c <<= 1;
  internal_check(c <= (int64_t(1) << 30), "scheduler: too many requests for the device queue");
  return static_cast<int32_t>(c);
}

// The scheduler-side fields of SimConfig (make_sim_config's, sim.cpp).
SimConfig sched_config(const PolicyConfig& p, const MemoryPlan& m) {
  require(p.max_batch_size >= 1 && p.max_batch_size <= ssg::kMaxBatchEntries,
          "ssg: max_batch_size above the device engine limit (" + std::to_string(ssg::kMaxBatchEntries) + ")");
  require(m.block_size >= 1 && m.block_size < (int64_t(1) << 31),
          "ssg: block_size outside the device engine range");
  SimConfig c{};
  c.policy = static_cast<int32_t>(p.policy);
  c.max_batch = static_cast<int32_t>(p.max_batch_size);
  c.max_tokens = static_cast<int32_t>(std::min<std::int64_t>(p.max_tokens_per_iter, INT32_MAX));
  c.chunk = static_cast<int32_t>(std::min<std::int64_t>(p.chunk_size, INT32_MAX));
  c.token_granular = p.policy == SchedulerPolicy::LightLLM ? 1 : 0;
  c.pp = 1;
  c.tp = 1;
  c.block_size = m.block_size;
  c.bs_shift = -1;
  for (int k = 0; k < 62; ++k)
    if ((int64_t(1) << k) == m.block_size) c.bs_shift = k;
  c.bs_magic = block_magic(m.block_size, c.token_granular != 0);
  c.total_units = c.token_granular ? m.kv_capacity_tokens : m.num_blocks;
  c.watermark_units = c.token_granular ? m.watermark_blocks * m.block_size : m.watermark_blocks;
  c.tab_off = -1;
  c.idx_pre = c.idx_dec = -1;
  return c;
}

}  // namespace

namespace {

[[noreturn]] void raise_sched_error(const SimUnitOut& o, const SimConfig& c) {
  if (o.code == SSG_ERR_ENQUEUE)
    throw Error("request " + std::to_string(o.err_i64[0]) + " needs " + std::to_string(o.err_i64[1]) +
                " KV units but replica capacity is " + std::to_string(c.total_units) +
                " (model/config cannot serve this request)");
  switch (o.err_i32) {
    case 1: throw InternalError("request not in waiting queue");
    case 4: throw InternalError("prefill progressed past its target");
    case 5: throw InternalError("sarathi: token budget exceeded");
    default: throw InternalError("scheduler: device invariant violated");
  }
}

}  // namespace

struct ReplicaScheduler::Device {
  SimConfig cfg{};
  SimUnit unit{};
  int32_t cap = 0;     // request slots allocated
  int32_t n = 0;       // slots in use, ordered by (arrival, id)
  int32_t serial = 0;  // schedule_iteration counter
  DeviceBuffer<SimConfig> d_cfg;
  DeviceBuffer<SimUnit> d_unit;
  DeviceBuffer<ReqHot> hot;
  DeviceBuffer<ReqTimes> tm;
  DeviceBuffer<int64_t> ids;
  DeviceBuffer<int32_t> restarts, ws;
  DeviceBuffer<RepState> rep;
  DeviceBuffer<SimUnitOut> out;
  std::vector<std::shared_ptr<RequestState>> slot;  // slot -> the caller's state
  std::unordered_map<const RequestState*, int32_t> where;
  // host copies after the last call
  RepState S{};
  std::vector<int32_t> run;
  std::vector<ReqHot> h_hot;
  std::vector<ReqTimes> h_tm;
  std::vector<int32_t> h_restarts;

  int64_t stride() const { return 6LL * cfg.max_batch + unit.wait_cap; }

  SchedArgs args(int32_t op) {
    SchedArgs a{};
    a.op = op;
    a.n = n;
    a.serial = serial;
    a.cfg = d_cfg.ptr;
    a.unit = d_unit.ptr;
    a.hot = hot.ptr;
    a.tm = tm.ptr;
    a.ids = ids.ptr;
    a.restarts = restarts.ptr;
    a.reps = rep.ptr;
    a.ws = ws.ptr;
    a.out = out.ptr;
    return a;
  }

  // Launches one op and copies back the replica, its running queue and every slot.
  void run_op(const SchedArgs& a) {
    cudaStream_t s = ssg::context().stream;
    ssg::launch_sched_op(a, s);
    SimUnitOut o{};
    out.download(&o, 1, s);
    rep.download(&S, 1, s);
    h_hot.resize(n);
    h_tm.resize(n);
    h_restarts.resize(n);
    hot.download(h_hot.data(), n, s);
    tm.download(h_tm.data(), n, s);
    restarts.download(h_restarts.data(), n, s);
    std::vector<int32_t> r(static_cast<std::size_t>(cfg.max_batch));
    ws.download(r.data(), r.size(), s);
    cuda_check(cudaStreamSynchronize(s), "scheduler op");
    if (o.code != SSG_OK) raise_sched_error(o, cfg);
    r.resize(static_cast<std::size_t>(S.run_n));
    run = std::move(r);
  }

  template <typename T>
  static void grow(DeviceBuffer<T>& b, std::size_t keep, std::size_t cap, cudaStream_t s) {
    DeviceBuffer<T> nb(cap);
    if (keep)
      cuda_check(cudaMemcpyAsync(nb.ptr, b.ptr, keep * sizeof(T), cudaMemcpyDeviceToDevice, s), "D2D");
    b = std::move(nb);
  }

  // Room for one more request: slots, and a waiting ring larger than every request.
  void reserve(int32_t need, cudaStream_t s) {
    if (need <= cap && need < unit.wait_cap) return;
    const int32_t ncap = std::max<int32_t>(64, std::max(need, 2 * cap));
    grow(hot, n, ncap, s);
    grow(tm, n, ncap, s);
    grow(ids, n, ncap, s);
    grow(restarts, n, ncap, s);
    // re-lay the workspace for the larger ring: running queue and plan arrays
    // keep their contents, the waiting ring is unwrapped to start at slot 0
    const int32_t MB = cfg.max_batch, old_wc = unit.wait_cap, wc = pow2_above(ncap);
    std::vector<int32_t> nws(static_cast<std::size_t>(6LL * MB + wc), 0);
    if (old_wc > 0) {
      std::vector<int32_t> ows(static_cast<std::size_t>(6LL * MB + old_wc));
      ws.download(ows.data(), ows.size(), s);
      rep.download(&S, 1, s);
      cuda_check(cudaStreamSynchronize(s), "scheduler relayout");
      std::copy(ows.begin(), ows.begin() + MB, nws.begin());
      for (int32_t k = 0; k < S.wait_n; ++k) nws[MB + k] = ows[MB + ((S.wait_head + k) & (old_wc - 1))];
      std::copy(ows.begin() + MB + old_wc, ows.end(), nws.begin() + MB + wc);
      S.wait_head = 0;
      rep.upload(&S, 1, s);
    }
    unit.wait_cap = wc;
    ws.upload(nws, s);
    d_unit.upload(&unit, 1, s);
    cap = ncap;
  }
};

ReplicaScheduler::ReplicaScheduler() = default;
ReplicaScheduler::~ReplicaScheduler() = default;
ReplicaScheduler::ReplicaScheduler(ReplicaScheduler&&) noexcept = default;
ReplicaScheduler& ReplicaScheduler::operator=(ReplicaScheduler&&) noexcept = default;

ReplicaScheduler::ReplicaScheduler(PolicyConfig cfg, MemoryPlan plan)
    : cfg_(cfg), plan_(plan), mem_(plan, cfg.policy == SchedulerPolicy::LightLLM),
      dev_(std::make_unique<Device>()) {
  auto& ctx = ssg::context();
  cudaStream_t s = ctx.stream;
  Device& d = *dev_;
  d.cfg = sched_config(cfg_, plan_);
  d.unit.R = 1;
  d.unit.abort_thr = INFINITY;  // no probe abort: mark_scheduled never counts late requests
  d.d_cfg.upload(&d.cfg, 1, s);
  d.rep.resize(1);
  cuda_check(cudaMemsetAsync(d.rep.ptr, 0, sizeof(RepState), s), "memset");
  d.out.resize(1);
  d.reserve(1, s);
  cuda_check(cudaStreamSynchronize(s), "scheduler init");
}


void ReplicaScheduler::enqueue(std::shared_ptr<RequestState> r) {  // scheduler.hpp:146-155
  internal_check(dev_ != nullptr, "ReplicaScheduler: observer views are read-only");
  internal_check(r != nullptr, "enqueue: null request");
  const std::int64_t need = mem_.units_for_tokens(r->req.prefill_tokens + r->req.decode_tokens);
  require(need <= mem_.total_units(),
          "request " + std::to_string(r->req.id) + " needs " + std::to_string(need) +
              " KV units but replica capacity is " + std::to_string(mem_.total_units()) +
              " (model/config cannot serve this request)");
  require(r->req.prefill_tokens < INT32_MAX / 2 && r->req.decode_tokens < INT32_MAX / 2 &&
              r->emitted < INT32_MAX / 2 && r->prefill_done < INT32_MAX / 2,
          "ssg: request lengths above the device engine limit");
  Device& d = *dev_;
  cudaStream_t s = ssg::context().stream;
  d.reserve(d.n + 1, s);
  // slot p: after every request with (arrival, id) <= r's (insert_sorted's upper_bound)
  auto key_less = [](const Request& a, const Request& b) {
    return a.arrival_time != b.arrival_time ? a.arrival_time < b.arrival_time : a.id < b.id;
  };
  const auto it = std::upper_bound(d.slot.begin(), d.slot.end(), r,
                                   [&](const std::shared_ptr<RequestState>& x,
                                       const std::shared_ptr<RequestState>& y) {
                                     return key_less(x->req, y->req);
                                   });
  const int32_t p = static_cast<int32_t>(it - d.slot.begin());
  if (p < d.n) {
    SchedArgs a = d.args(SSG_SCHED_RENUMBER);
    a.arg = p;
    ssg::launch_sched_op(a, s);
  }
  d.slot.insert(d.slot.begin() + p, r);
  for (int32_t k = p; k < static_cast<int32_t>(d.slot.size()); ++k) d.where[d.slot[k].get()] = k;
  ReqHot h{};
  h.done = static_cast<int32_t>(r->prefill_done);
  h.emitted = static_cast<int32_t>(r->emitted);
  h.kv = static_cast<int32_t>(r->kv_context);
  h.decode = static_cast<int32_t>(r->req.decode_tokens);
  h.prefill = static_cast<int32_t>(r->req.prefill_tokens);
  const ReqTimes t{r->req.arrival_time, r->first_scheduled_time, r->first_token_time, r->completion_time};
  const int64_t id = r->req.id;
  const int32_t rs = static_cast<int32_t>(r->restarts);
  cuda_check(cudaMemcpyAsync(d.hot.ptr + p, &h, sizeof h, cudaMemcpyHostToDevice, s), "H2D");
  cuda_check(cudaMemcpyAsync(d.tm.ptr + p, &t, sizeof t, cudaMemcpyHostToDevice, s), "H2D");
  cuda_check(cudaMemcpyAsync(d.ids.ptr + p, &id, sizeof id, cudaMemcpyHostToDevice, s), "H2D");
  cuda_check(cudaMemcpyAsync(d.restarts.ptr + p, &rs, sizeof rs, cudaMemcpyHostToDevice, s), "H2D");
  d.n += 1;
  d.unit.n = d.n;
  d.d_unit.upload(&d.unit, 1, s);
  SchedArgs a = d.args(SSG_SCHED_ENQUEUE);
  a.arg = p;
  d.run_op(a);
  refresh_();
}

BatchPlan ReplicaScheduler::schedule_iteration() {  // scheduler.hpp:184-194
  internal_check(dev_ != nullptr, "ReplicaScheduler: observer views are read-only");
  Device& d = *dev_;
  cudaStream_t s = ssg::context().stream;
  d.serial += 1;
  SchedArgs a = d.args(SSG_SCHED_SCHEDULE);
  a.now = now_;
  d.run_op(a);
  refresh_();
  // the plan arrays: P_IDX | P_CHUNK | P_PRIOR | D_IDX | D_CTX after RUN and WAIT
  const int32_t MB = d.cfg.max_batch, np = d.S.np, nd = d.S.nd;
  std::vector<int32_t> pl(static_cast<std::size_t>(5LL * MB));
  cuda_check(cudaMemcpyAsync(pl.data(), d.ws.ptr + MB + d.unit.wait_cap, pl.size() * sizeof(int32_t),
                             cudaMemcpyDeviceToHost, s), "D2H");
  cuda_check(cudaStreamSynchronize(s), "schedule_iteration");
  BatchPlan plan;
  plan.prefills.reserve(np);
  plan.decodes.reserve(nd);
  for (int32_t k = 0; k < np; ++k)
    plan.prefills.push_back({d.slot.at(pl[k]).get(), pl[MB + k], pl[2 * MB + k]});
  for (int32_t k = 0; k < nd; ++k)
    plan.decodes.push_back({d.slot.at(pl[3 * MB + k]).get(), pl[4 * MB + k]});
  return plan;
}

std::vector<std::shared_ptr<RequestState>> ReplicaScheduler::complete_iteration(const BatchPlan& plan,
                                                                                double now) {
  internal_check(dev_ != nullptr, "ReplicaScheduler: observer views are read-only");
  Device& d = *dev_;
  cudaStream_t s = ssg::context().stream;
  const int32_t MB = d.cfg.max_batch;
  const int64_t np = static_cast<int64_t>(plan.prefills.size()), nd = static_cast<int64_t>(plan.decodes.size());
  internal_check(np <= MB && nd <= MB, "complete_iteration: plan larger than the batch cap");
  std::vector<int32_t> pl(static_cast<std::size_t>(5LL * MB), 0);
  std::vector<int32_t> touched;
  auto slot_of = [&](const RequestState* r) {
    auto it = d.where.find(r);
    internal_check(it != d.where.end(), "complete_iteration: request not owned by this scheduler");
    return it->second;
  };
  for (int64_t k = 0; k < np; ++k) {
    const auto& e = plan.prefills[k];
    pl[k] = slot_of(e.request);
    pl[MB + k] = static_cast<int32_t>(e.chunk_tokens);
    pl[2 * MB + k] = static_cast<int32_t>(e.prior_context);
    touched.push_back(pl[k]);
  }
  for (int64_t k = 0; k < nd; ++k) {
    const auto& e = plan.decodes[k];
    pl[3 * MB + k] = slot_of(e.request);
    pl[4 * MB + k] = static_cast<int32_t>(e.context_tokens);
    touched.push_back(pl[3 * MB + k]);
  }
  cuda_check(cudaMemcpyAsync(d.ws.ptr + MB + d.unit.wait_cap, pl.data(), pl.size() * sizeof(int32_t),
                             cudaMemcpyHostToDevice, s), "H2D");
  std::vector<int32_t> emitted_before;
  for (auto j : touched) emitted_before.push_back(d.h_hot[j].emitted);
  const std::vector<int32_t> run_before = d.run;
  SchedArgs a = d.args(SSG_SCHED_COMPLETE);
  a.np = static_cast<int32_t>(np);
  a.nd = static_cast<int32_t>(nd);
  a.now = now;
  d.run_op(a);
  refresh_();
  // emit_token's emission_times (scheduler.hpp:254-260): one per token emitted now
  for (std::size_t k = 0; k < touched.size(); ++k)
    for (int32_t e = emitted_before[k]; e < d.h_hot[touched[k]].emitted; ++e)
      d.slot[touched[k]]->emission_times.push_back(now);
  // requests of the running queue that are finished (FT keeps them until it drains)
  std::vector<std::shared_ptr<RequestState>> done;
  for (auto j : run_before)
    if (d.h_hot[j].emitted >= d.h_hot[j].decode) done.push_back(d.slot[j]);
  return done;
}

// The counters and the caller-visible request fields after an op.
void ReplicaScheduler::refresh_() {
  Device& d = *dev_;
  outstanding_ = static_cast<std::size_t>(d.S.outstanding);
  preemptions_ = static_cast<std::size_t>(d.S.preemptions);
  ft_members_.clear();
  if (d.S.ft_inflight)
    for (auto j : d.run) ft_members_.push_back(d.slot[j]->req.id);
  mem_.allocated_ = d.S.allocated;
  mem_.held_.clear();
  for (int32_t j = 0; j < d.n; ++j) {
    const ReqHot& h = d.h_hot[j];
    RequestState& r = *d.slot[j];
    r.prefill_target = h.target;
    r.prefill_done = h.done;
    r.emitted = h.emitted;
    r.kv_context = h.kv;
    r.restarts = d.h_restarts[j];
    r.first_scheduled_time = d.h_tm[j].first_sched;
    r.first_token_time = d.h_tm[j].first_tok;
    r.completion_time = d.h_tm[j].completion;
    if (h.held > 0) mem_.held_[r.req.id] += h.held;
  }
}

}  // namespace servesim
