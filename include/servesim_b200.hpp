// servesim_b200.hpp -- the C++ drop-in surface of the B200 framework.
//
// A program written against the reference library (proj/include/servesim/*.hpp)
// keeps its types and calls: the declarations below carry the reference's
// names, field meanings, defaults and error behaviour (Error for bad input,
// InternalError for violated invariants), but the hot path underneath --
// predictor evaluation, replica simulation, capacity search, percentile
// selection -- runs in the sm_100a kernels behind the C ABI in ssg.h.  Host
// code here is configuration, training (once per SKU) and result formatting.
//
// Each declaration cites the reference symbol it stands in for.
#pragma once

#include <cstdint>
#include <deque>
#include <functional>
#include <map>
#include <memory>
#include <optional>
#include <span>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "json.hpp"  // nlohmann/json 3.11, as the reference (vendor/json.hpp)

namespace servesim {

// ---------------------------------------------------------------- errors
// reference: error.hpp:9-26
class Error : public std::runtime_error {
 public:
  explicit Error(const std::string& m) : std::runtime_error(m) {}
};
class InternalError : public std::logic_error {
 public:
  explicit InternalError(const std::string& m) : std::logic_error(m) {}
};
inline void require(bool ok, const std::string& msg) {
  if (!ok) throw Error(msg);
}
inline void internal_check(bool ok, const std::string& msg) {
  if (!ok) throw InternalError(msg);
}

// Shortest round-trip decimal (reference csv.hpp:17-22).
std::string fmt_double(double v);

// ---------------------------------------------------------------- model
// reference: model_spec.hpp:12-110
enum class AttentionVariant { MHA, GQA };

struct ModelSpec {
  std::string name;
  std::int64_t num_layers = 0, hidden_dim = 0, num_q_heads = 0, num_kv_heads = 0;
  std::int64_t head_dim = 0, mlp_dim = 0, vocab_size = 0, max_context = 0;
  std::int64_t param_bytes_per_element = 0;
  AttentionVariant attention_variant = AttentionVariant::MHA;
};

struct ParallelismConfig {
  std::int64_t tp_degree = 1;
  std::int64_t pp_degree = 1;
  std::int64_t num_replicas = 1;
};

enum class OpName {
  QkvProj, AttnOutProj, MlpUpProj, MlpDownProj, ActFn, AddNorm,
  AttnPrefill, AttnDecode, AllReduce, AllGather, SendRecv,
};
constexpr int kNumOps = 11;
enum class OpClass { TokenLevel, SequenceLevel, Communication };

const char* to_string(OpName op);
OpName op_name_from_string(const std::string& s);
OpClass triage(OpName op);  // reference profiler.hpp:33-51

struct OperatorDescriptor {
  OpName op = OpName::QkvProj;
  OpClass op_class = OpClass::TokenLevel;
  std::int64_t count = 1, tp_degree = 1;
  std::int64_t in_dim = 0, out_dim = 0;
  std::int64_t q_heads_per_device = 0, kv_heads_per_device = 0, head_dim = 0;
  std::int64_t payload_bytes_per_token = 0;
  std::int64_t elem_bytes = 2;
};

void validate(const ModelSpec& s);
void validate(const ModelSpec& s, const ParallelismConfig& p);
ModelSpec parse_model_spec(const std::string& json_text);
std::vector<OperatorDescriptor> derive_operators(const ModelSpec& s, const ParallelismConfig& p);
std::int64_t param_bytes_per_device(const ModelSpec& s, const ParallelismConfig& p);
std::int64_t kv_bytes_per_token_per_device(const ModelSpec& s, const ParallelismConfig& p);
std::int64_t kv_bytes_per_token_per_block(const ModelSpec& s, const ParallelismConfig& p);

// ---------------------------------------------------------------- device
// reference: device.hpp:13-61
struct DeviceProfile {
  std::string sku_name;
  double peak_flops = 0, mem_bandwidth = 0, link_bandwidth = 0, kernel_overhead = 0,
         device_mem = 0;
};
void validate(const DeviceProfile& d);
DeviceProfile parse_device_profile(const std::string& json_text);

// ---------------------------------------------------------------- workload
// reference: workload.hpp:19-247
struct Request {
  std::int64_t id = 0;
  double arrival_time = 0.0;  // NaN until assigned
  std::int64_t prefill_tokens = 0;
  std::int64_t decode_tokens = 0;
  bool has_arrival() const { return arrival_time == arrival_time; }
};
std::vector<Request> load_trace(const std::string& csv_text);
std::vector<Request> poisson_arrivals(std::vector<Request> reqs, double rate_qps,
                                      std::uint64_t seed);
// E_i = -log(1 - U_i) of poisson_arrivals' i-th draw; gap_i = E_i / rate
// (bit-identical to exponential_distribution(rate)).  Host side, once per seed.
std::vector<double> unit_exponentials(std::size_t n, std::uint64_t seed);
std::vector<Request> cap_total_length(std::vector<Request> reqs, std::int64_t max_total);

struct DistConfig {
  std::string kind;  // "lognormal" | "histogram"
  double prefill_median = 0, prefill_sigma = 0, decode_median = 0, decode_sigma = 0;
  struct Bin {
    std::int64_t prefill = 0, decode = 0;
    double weight = 0;
  };
  std::vector<Bin> bins;
  std::int64_t max_total = 0;
};
DistConfig parse_dist_config_text(const std::string& json_text);
std::vector<Request> synth_trace(const DistConfig& dist, std::size_t n, std::uint64_t seed);

// ---------------------------------------------------------------- profiler
// reference: profiler.hpp:18-347 (training-data generation, host side)
inline constexpr const char* kFeatNumTokens = "num_tokens";
inline constexpr const char* kFeatKvReadBytes = "kv_read_bytes";
inline constexpr const char* kFeatPayloadBytes = "payload_bytes";
inline constexpr const char* kFeatTpDegree = "tp_degree";
using FeatureMap = std::map<std::string, double>;

struct ProfileRecord {
  OpName op = OpName::QkvProj;
  FeatureMap features;
  double runtime = 0.0;
};
std::vector<std::string> feature_schema(OpClass c);
double synthetic_oracle(const OperatorDescriptor& d, const FeatureMap& f, const DeviceProfile& dev);
std::vector<ProfileRecord> generate_synthetic_profile(const ModelSpec& spec,
                                                      const DeviceProfile& dev,
                                                      const std::vector<std::int64_t>& tps);

// ---------------------------------------------------------------- estimator
// reference: regressor.hpp:19-386, estimator.hpp:20-380
struct ForestConfig {
  int num_trees = 48, max_depth = 16, min_samples_leaf = 0, threshold_draws = 8;
  std::uint64_t seed = 0;
};
struct TrainConfig {
  std::size_t min_points_per_op = 8;
  ForestConfig forest;
  std::uint64_t seed = 0;
  std::string regressor = "interp";  // "interp" | "forest"
};

// One trained per-(op, tp) predictor in the reference's serialized layout.
struct ForestTree {
  std::vector<int> feature;
  std::vector<double> threshold;
  std::vector<int> left, right;
  std::vector<std::vector<double>> leaf_weights;
};
struct RegressorData {
  std::string type;  // "forest" | "interp"
  // forest
  std::size_t num_features = 0;
  double y_lo = 0, y_hi = 0;
  std::vector<ForestTree> trees;
  // interp
  std::vector<std::vector<double>> axes;
  std::vector<double> values;
};

// Prediction backend for one operator (reference regressor.hpp:19-24): trained
// on log1p-transformed features.  predict() runs on the GPU -- the regressor is
// flattened to HBM on first use and evaluated by the same device code as the
// batched predictor (predictor.cuh); data() is the trained parameter set the
// upload flattens.
struct DeviceRegressor;  // HBM copy (predictor.cu)
class Regressor {
 public:
  virtual ~Regressor();
  virtual double predict(std::span<const double> x) const;
  virtual nlohmann::json to_json() const;
  const RegressorData& data() const { return data_; }

 protected:
  explicit Regressor(RegressorData d);
  RegressorData data_;

 private:
  mutable std::shared_ptr<DeviceRegressor> dev_;
};

// reference regressor.hpp:78-270 (random forest of piecewise-linear trees)
class ForestRegressor final : public Regressor {
 public:
  static ForestRegressor train(const std::vector<std::vector<double>>& x,
                               const std::vector<double>& y, const ForestConfig& cfg);
  static ForestRegressor from_json(const nlohmann::json& j);
  explicit ForestRegressor(RegressorData d);
};

// reference regressor.hpp:273-376 (multilinear interpolation over the profiled grid)
class GridInterpolator final : public Regressor {
 public:
  static GridInterpolator fit(const std::vector<std::vector<double>>& x,
                              const std::vector<double>& y);
  static GridInterpolator from_json(const nlohmann::json& j);
  explicit GridInterpolator(RegressorData d);
};

// reference regressor.hpp:379-386
std::unique_ptr<Regressor> regressor_from_json(const nlohmann::json& j);

struct OpModelKey {
  OpName op;
  std::int64_t tp_degree;
  bool operator<(const OpModelKey& o) const {
    return op != o.op ? op < o.op : tp_degree < o.tp_degree;
  }
};
std::string to_string(const OpModelKey& k);

struct DeviceEstimator;  // flattened SoA copy resident in HBM (predictor.cu)

class EstimatorModel {
 public:
  struct PerOpModel {
    std::vector<std::string> schema;
    std::vector<double> bbox_lo, bbox_hi;
    std::vector<std::vector<double>> levels;
    std::unique_ptr<Regressor> regressor;  // over log1p(features) -> log(runtime)
    double holdout_mape = 0.0;
    std::size_t n_points = 0;
  };
  static constexpr double kExtrapolationMargin = 0.10;

  EstimatorModel();
  ~EstimatorModel();
  EstimatorModel(EstimatorModel&&) noexcept;
  EstimatorModel& operator=(EstimatorModel&&) noexcept;

  bool has(OpName op, std::int64_t tp) const { return models_.count({op, tp}) > 0; }
  const PerOpModel& find(OpName op, std::int64_t tp) const;
  const std::map<OpModelKey, PerOpModel>& models() const { return models_; }
  void insert(const OpModelKey& k, PerOpModel m);

  // Single query (reference estimator.hpp:105-123), evaluated on the GPU.
  double predict(OpName op, std::int64_t tp, const FeatureMap& features) const;

  // reference estimator.hpp:137-177 (the serialized handoff format)
  nlohmann::json to_json() const;
  static EstimatorModel from_json(const nlohmann::json& j);

  // HBM-resident copy, built on first use and reused by every kernel.
  const DeviceEstimator& device() const;

 private:
  std::map<OpModelKey, PerOpModel> models_;
  mutable std::unique_ptr<DeviceEstimator> dev_;
};

EstimatorModel train(const std::vector<ProfileRecord>& records, const TrainConfig& cfg);

struct BatchComposition {
  std::vector<std::int64_t> prefill_lengths;
  std::vector<std::int64_t> prefill_prior_context;
  std::vector<std::int64_t> decode_context_lengths;
  std::int64_t num_decode_tokens() const { return (std::int64_t)decode_context_lengths.size(); }
  std::int64_t total_current_tokens() const {
    std::int64_t t = num_decode_tokens();
    for (auto p : prefill_lengths) t += p;
    return t;
  }
};
std::int64_t equivalent_prefill_length(const std::vector<std::int64_t>& prefill_lengths);
// Both evaluated on the GPU (one warp per composition).
double predict_batch(const EstimatorModel& model, const std::vector<OperatorDescriptor>& ops,
                     const BatchComposition& batch);
double batch_device_flops(const std::vector<OperatorDescriptor>& ops, const BatchComposition& b);

// ---------------------------------------------------------------- memory
// reference: memory.hpp:12-46
struct MemoryPlan {
  std::int64_t kv_capacity_tokens = 0, block_size = 0, num_blocks = 0, watermark_blocks = 0;
};
MemoryPlan plan_memory(const ModelSpec& spec, const ParallelismConfig& par,
                       const DeviceProfile& dev, std::int64_t block_size,
                       double watermark_fraction = 0.01, double activation_reserve_fraction = 0.10);

// ---------------------------------------------------------------- scheduling
// reference: scheduler.hpp:20-76
enum class SchedulerPolicy { FasterTransformer, OrcaPlus, VLLM, SarathiServe, LightLLM };
enum class RoutingPolicy { RoundRobin, LeastOutstanding, Deferred };
const char* to_string(SchedulerPolicy p);
const char* to_string(RoutingPolicy p);
SchedulerPolicy scheduler_policy_from_string(const std::string& s);
RoutingPolicy routing_policy_from_string(const std::string& s);

struct PolicyConfig {
  SchedulerPolicy policy = SchedulerPolicy::VLLM;
  std::int64_t max_batch_size = 128;
  std::int64_t max_tokens_per_iter = 4096;
  std::int64_t chunk_size = 512;
  std::int64_t block_size = 16;
  double watermark_fraction = 0.01;
  double activation_reserve_fraction = 0.10;
};
void validate(const PolicyConfig& c);

// ---------------------------------------------------------------- scheduler plugin
struct SchedulerView;  // builds the SimObserver's read-only scheduler views (sim.cpp)
// reference: scheduler.hpp:78-233, memory.hpp:51-104

// Per-request progress inside one replica (scheduler.hpp:81-96).
struct RequestState {
  Request req;
  std::int64_t prefill_target = 0, prefill_done = 0, emitted = 0, kv_context = 0, restarts = 0;
  double first_scheduled_time = -1.0, first_token_time = -1.0, completion_time = -1.0;
  std::vector<double> emission_times;
  bool prefill_complete() const { return prefill_done >= prefill_target; }
  bool finished() const { return emitted >= req.decode_tokens; }
};

struct PrefillEntry {
  RequestState* request;
  std::int64_t chunk_tokens;
  std::int64_t prior_context;
};
struct DecodeEntry {
  RequestState* request;
  std::int64_t context_tokens;
};

struct BatchPlan {
  std::vector<PrefillEntry> prefills;
  std::vector<DecodeEntry> decodes;
  bool empty() const { return prefills.empty() && decodes.empty(); }
  std::int64_t batch_size() const { return static_cast<std::int64_t>(prefills.size() + decodes.size()); }
  std::int64_t total_current_tokens() const {
    std::int64_t t = static_cast<std::int64_t>(decodes.size());
    for (const auto& p : prefills) t += p.chunk_tokens;
    return t;
  }
  BatchComposition composition() const {
    BatchComposition c;
    for (const auto& p : prefills) {
      c.prefill_lengths.push_back(p.chunk_tokens);
      c.prefill_prior_context.push_back(p.prior_context);
    }
    for (const auto& d : decodes) c.decode_context_lengths.push_back(d.context_tokens);
    return c;
  }
};

// Block accounting of one replica (memory.hpp:51-104).  Standalone it is the
// reference's integer bookkeeping; a ReplicaScheduler's memory() is a snapshot
// of the accounting its device state holds after the last call.
class BlockManager {
 public:
  BlockManager() = default;
  BlockManager(const MemoryPlan& plan, bool token_granular)
      : plan_(plan), token_granular_(token_granular) {}
  std::int64_t total_units() const {
    return token_granular_ ? plan_.kv_capacity_tokens : plan_.num_blocks;
  }
  std::int64_t free_units() const { return total_units() - allocated_; }
  std::int64_t allocated_units() const { return allocated_; }
  std::int64_t watermark_units() const {
    return token_granular_ ? plan_.watermark_blocks * plan_.block_size : plan_.watermark_blocks;
  }
  std::int64_t units_for_tokens(std::int64_t tokens) const {
    return token_granular_ ? tokens : (tokens + plan_.block_size - 1) / plan_.block_size;
  }
  std::int64_t held_units(std::int64_t request_id) const {
    auto it = held_.find(request_id);
    return it == held_.end() ? 0 : it->second;
  }
  std::int64_t shortfall(std::int64_t request_id, std::int64_t tokens) const {
    const std::int64_t s = units_for_tokens(tokens) - held_units(request_id);
    return s > 0 ? s : 0;
  }
  bool try_reserve(std::int64_t request_id, std::int64_t tokens);
  void release(std::int64_t request_id);

 private:
  friend class ReplicaScheduler;
  friend struct SchedulerView;
  MemoryPlan plan_;
  bool token_granular_ = false;
  std::int64_t allocated_ = 0;
  std::map<std::int64_t, std::int64_t> held_;
};

// Replica-tier scheduler: batching policy + paged KV management
// (scheduler.hpp:136-233).  The state lives in HBM and every call is one warp
// of the device scheduler (sched_api.cu) -- the code the simulation kernel runs
// per BatchStart -- so plans, preemptions and block counts are the engine's.
// Request states are shared with the caller: after each call the scheduler
// writes back the fields it owns (progress, restarts, times, emission_times).
class ReplicaScheduler {
 public:
  ReplicaScheduler();
  ReplicaScheduler(PolicyConfig cfg, MemoryPlan plan);
  ~ReplicaScheduler();
  ReplicaScheduler(ReplicaScheduler&&) noexcept;
  ReplicaScheduler& operator=(ReplicaScheduler&&) noexcept;

  const BlockManager& memory() const { return mem_; }
  const MemoryPlan& memory_plan() const { return plan_; }
  const PolicyConfig& config() const { return cfg_; }

  void enqueue(std::shared_ptr<RequestState> r);
  std::size_t outstanding() const { return outstanding_; }
  bool has_work() const { return outstanding_ > 0; }
  std::size_t preemption_count() const { return preemptions_; }
  // Members of the in-flight request-level batch (FasterTransformer only).
  std::vector<std::int64_t> ft_member_ids() const { return ft_members_; }
  void set_now(double now) { now_ = now; }
  BatchPlan schedule_iteration();
  std::vector<std::shared_ptr<RequestState>> complete_iteration(const BatchPlan& plan, double now);

 private:
  friend struct SchedulerView;  // the SimObserver's read-only views (sim.cpp)
  PolicyConfig cfg_;
  MemoryPlan plan_;
  BlockManager mem_;
  double now_ = 0.0;
  std::size_t outstanding_ = 0, preemptions_ = 0;
  std::vector<std::int64_t> ft_members_;
  struct Device;
  std::unique_ptr<Device> dev_;  // null for observer views
  void refresh_();
};

// Global-tier routing (scheduler.hpp:492-561).  The simulation kernel routes on
// the device (engine.cu); this is the same policy for callers that drive
// ReplicaSchedulers themselves.
class Router {
 public:
  Router(RoutingPolicy policy, std::size_t num_replicas, std::int64_t deferred_threshold)
      : policy_(policy), n_(num_replicas), threshold_(deferred_threshold) {
    require(n_ >= 1, "router: need at least one replica");
    require(threshold_ >= 1, "router: deferred threshold must be >= 1");
  }
  // Replica for `r`, or nullopt while the deferred policy pools it.
  template <typename OutstandingFn>
  std::optional<std::size_t> route(std::shared_ptr<RequestState> r, OutstandingFn&& outstanding) {
    if (policy_ == RoutingPolicy::RoundRobin) {
      const std::size_t k = next_;
      next_ = next_ + 1 == n_ ? 0 : next_ + 1;
      return k;
    }
    if (policy_ == RoutingPolicy::LeastOutstanding) {
      std::size_t best = 0, load = outstanding(std::size_t(0));
      for (std::size_t k = 1; k < n_; ++k) {
        const std::size_t c = outstanding(k);
        if (c < load) best = k, load = c;  // ties stay on the lowest index
      }
      return best;
    }
    pool_.push_back(std::move(r));
    return std::nullopt;
  }
  // Deferred policy: pooled requests to replicas below the threshold, least
  // loaded first (counts advance as requests are assigned).
  template <typename OutstandingFn>
  std::vector<std::pair<std::size_t, std::shared_ptr<RequestState>>> drain(OutstandingFn&& outstanding) {
    std::vector<std::pair<std::size_t, std::shared_ptr<RequestState>>> out;
    if (policy_ != RoutingPolicy::Deferred || pool_.empty()) return out;
    std::vector<std::int64_t> load(n_);
    for (std::size_t k = 0; k < n_; ++k) load[k] = static_cast<std::int64_t>(outstanding(k));
    while (!pool_.empty()) {
      std::size_t best = n_;
      for (std::size_t k = 0; k < n_; ++k)
        if (load[k] < threshold_ && (best == n_ || load[k] < load[best])) best = k;
      if (best == n_) break;
      out.emplace_back(best, std::move(pool_.front()));
      pool_.pop_front();
      ++load[best];
    }
    return out;
  }
  std::size_t pooled() const { return pool_.size(); }

 private:
  RoutingPolicy policy_;
  std::size_t n_;
  std::int64_t threshold_;
  std::size_t next_ = 0;
  std::deque<std::shared_ptr<RequestState>> pool_;
};

// ---------------------------------------------------------------- engine
// reference: sim.hpp:20-320
struct ClusterConfig {
  ModelSpec spec;
  ParallelismConfig par;
  DeviceProfile dev;
  PolicyConfig policy;
  RoutingPolicy routing = RoutingPolicy::RoundRobin;
  std::int64_t deferred_threshold = 0;
  double cpu_overhead_per_iter = 0.0;
  std::int64_t gpus_used() const { return par.tp_degree * par.pp_degree * par.num_replicas; }
};

struct RequestRecord {
  std::int64_t id = 0;
  double arrival = 0, first_scheduled = -1, first_token = -1, completion = -1;
  std::int64_t prefill_tokens = 0, decode_tokens = 0, restarts = 0;
  std::vector<double> emission_times;
};
struct IterationRecord {
  double start = 0, latency = 0;
  std::size_t replica = 0;
  std::int64_t batch_requests = 0, current_tokens = 0, prefill_entries = 0, decode_entries = 0;
  double kv_utilization = 0;
};
struct ReplicaAggregate {
  double busy_time = 0;
  std::int64_t iterations = 0, tokens_processed = 0;
  double peak_kv_utilization = 0;
  std::size_t preemptions = 0;
};
struct SimulationResult {
  std::vector<RequestRecord> requests;
  std::vector<ReplicaAggregate> replicas;
  std::vector<IterationRecord> iterations;
  double simulated_span = 0, total_model_flops = 0;
  std::int64_t num_devices = 0;
  double peak_device_flops = 0;
};

// Per-batch trace (the reference SimObserver::on_batch payload, sim.hpp:92-97),
// recorded on the device when SimOptions::record_batches is set.
struct BatchEntryLog {
  bool prefill;
  std::int64_t request_id, tokens, context;  // prefill: chunk, prior; decode: 1, context
};
struct BatchLog {
  std::size_t replica;
  double now;
  std::int64_t kv_allocated_units;
  std::vector<BatchEntryLog> entries;
  // observer runs only: the replica's scheduler state at this batch
  std::int64_t outstanding = 0, preemptions = 0;
  std::vector<std::int64_t> ft_members;
};

// Observation hook (sim.hpp:92-97): called with each scheduled batch, in the
// global event order, before it executes.  run_simulation with an observer runs
// the replicas in one coupled warp with the batch log enabled and replays the
// log through the callback after the kernel: `plan` points at RequestStates
// carrying each request's `req` (progress fields are the device's and are not
// mirrored), `sched` is a read-only view of the replica at that batch --
// memory() (allocated / total units), outstanding(), preemption_count(),
// ft_member_ids(), config(), memory_plan().
class SimObserver {
 public:
  virtual ~SimObserver() = default;
  virtual void on_batch(std::size_t replica, double now, const BatchPlan& plan,
                        const ReplicaScheduler& sched) = 0;
};

struct SimOptions {
  bool record_iterations = false;
  SimObserver* observer = nullptr;
  // capacity probes: stop once more than abort_max_late requests were first
  // scheduled later than abort_delay_threshold after arrival (sim.hpp:99-107)
  double abort_delay_threshold = 0.0;
  std::size_t abort_max_late = 0;
  bool record_batches = false;  // B200: return the device batch log (SimulationOutput::batches)
};
class ProbeInfeasible : public std::exception {
 public:
  const char* what() const noexcept override { return "probe aborted: delay threshold exceeded"; }
};

struct SimulationOutput {
  SimulationResult result;
  std::vector<BatchLog> batches;  // when record_batches
};

SimulationResult run_simulation(const ClusterConfig& cluster, const std::vector<Request>& trace,
                                const EstimatorModel& estimator, const SimOptions& opts = {});
SimulationOutput run_simulation_logged(const ClusterConfig& cluster,
                                       const std::vector<Request>& trace,
                                       const EstimatorModel& estimator, const SimOptions& opts);

// ---------------------------------------------------------------- metrics
// reference: metrics.hpp:17-126, stats.hpp:15-43
struct MetricSummary {
  double mean = 0, p50 = 0, p90 = 0, p95 = 0, p99 = 0;
};
struct ClusterMetrics {
  double mfu = 0, kv_utilization_peak = 0, busy_fraction = 0;
  std::size_t preemptions = 0;
};
struct RequestMetrics {
  std::int64_t id = 0;
  double scheduling_delay = 0, ttft = 0, prefill_completion = 0, e2e_latency = 0,
         normalized_latency = 0;
  std::vector<double> tbt_samples;
  std::int64_t prefill_tokens = 0, decode_tokens = 0, restarts = 0;
};
struct MetricsReport {
  std::vector<RequestMetrics> requests;
  MetricSummary scheduling_delay, ttft, tbt, e2e, normalized;
  ClusterMetrics cluster;
  double simulated_span = 0;
};
double percentile(const std::vector<double>& samples, double q);
MetricsReport build_report(const SimulationResult& result, bool static_mode = false);
std::string request_metrics_to_csv(const MetricsReport& rep);
nlohmann::ordered_json summary_to_json(const MetricsReport& rep);
// requests.csv (or requests.json) plus summary.json under out_dir
// (metrics.hpp:200-231); returns the files written.
std::vector<std::string> export_metrics(const MetricsReport& rep, const std::string& out_dir,
                                        const std::string& format);

// ---------------------------------------------------------------- search
// reference: search.hpp:25-486
struct SearchSpace {
  std::vector<DeviceProfile> skus;
  std::vector<std::int64_t> tp_degrees = {1, 2, 4};
  std::vector<std::int64_t> pp_degrees = {1, 2, 4};
  std::vector<SchedulerPolicy> schedulers;
  std::vector<std::int64_t> batch_sizes = {32, 64, 128, 256, 512};
  std::vector<std::int64_t> chunk_sizes = {512, 1024, 2048};
  std::int64_t max_gpus_total = 16;
};
struct SLOs {
  double ttft_p90_max = 2.0, tbt_p99_max = 0.2, delay_p99_max = 5.0;
};
using CostTable = std::map<std::string, double>;

struct CandidateConfig {
  std::string id;
  std::size_t sku_index = 0;
  ParallelismConfig par;
  PolicyConfig policy;
};
struct SkippedConfig {
  std::string id, reason;
};
std::vector<CandidateConfig> enumerate_configs(const ModelSpec& spec, const SearchSpace& space,
                                               const PolicyConfig& base,
                                               std::vector<SkippedConfig>* skipped = nullptr);

struct CapacitySearchOptions {
  double tolerance = 0.02, delay_p99_threshold = 5.0;
  std::size_t probe_requests = 2000;
  std::uint64_t seed = 1;
  double initial_guess = 1.0, min_qps = 1e-6, max_qps = 1e9;
};

struct ConfigResult {
  CandidateConfig config;
  std::string sku_name;
  double capacity_qps = 0, qps_per_dollar = 0, ttft_p90 = 0, tbt_p99 = 0, delay_p99 = 0,
         makespan = 0;
  bool slo_pass = false;
  std::string error;
  bool failed() const { return !error.empty(); }
};
struct ParetoPoint {
  double latency = 0, value = 0;
};
std::vector<std::size_t> pareto_frontier(const std::vector<ParetoPoint>& pts);

struct SearchOptions {
  SearchSpace space;
  SLOs slos;
  CostTable cost;
  CapacitySearchOptions capacity;
  double evaluation_fraction = 0.85;
  std::string objective = "qps_per_dollar";
  int workers = 1;  // accepted for API compatibility; the GPU runs every config at once
  RoutingPolicy routing = RoutingPolicy::RoundRobin;
  double cpu_overhead_per_iter = 0.0;
  TrainConfig train;
};
struct SearchOutcome {
  std::vector<ConfigResult> results;
  std::vector<SkippedConfig> skipped;
  std::vector<std::size_t> ranking, frontier_ttft, frontier_tbt;
  std::optional<std::size_t> best;
};

// ---------------------------------------------------------------- files and configs
// reference: csv.hpp:56-70, config.hpp:17-179 (paths resolve relative to the config file)
std::string read_text_file(const std::string& path);
void write_text_file(const std::string& path, const std::string& content);
nlohmann::json load_json_file(const std::string& path);
ModelSpec load_model_spec_file(const std::string& path);
DeviceProfile load_device_file(const std::string& path);
PolicyConfig parse_policy_config(const nlohmann::json& j);

struct LoadedSearchConfig {
  ModelSpec spec;
  std::vector<Request> workload;  // lengths; arrivals assigned per probe
  SearchOptions options;
  std::string model_spec_path;
  std::vector<std::string> device_paths;
  std::string trace_path;  // empty for synthetic workloads
};
LoadedSearchConfig load_search_config(const std::string& path);
struct LoadedClusterConfig {
  ClusterConfig cluster;
  std::string model_spec_path;
  std::string device_path;
};
LoadedClusterConfig load_cluster_config(const std::string& path);

// Maximum sustainable rate by doubling then bisection over a monotone
// feasibility callback (search.hpp:145-174); the feasible end is returned.
double find_capacity(const std::function<bool(double)>& feasible_at, const CapacitySearchOptions& opts);
double find_capacity_replay(const std::function<bool(double)>& feasible,
                            const CapacitySearchOptions& opts);  // same search (kept name)
double initial_qps_guess(const ModelSpec& spec, const CandidateConfig& cand,
                         const EstimatorModel& est, const ClusterConfig& cluster);
double qps_per_dollar(double capacity_qps, std::int64_t gpus_used, double rate_per_gpu_hr);

// One candidate end to end (search.hpp:294-363): capacity search, SLO run at
// evaluation_fraction of capacity (or the static run of the makespan
// objective).  Runs on the GPU as a one-config sweep.
ConfigResult evaluate_config(const ModelSpec& spec, const CandidateConfig& cand,
                             const DeviceProfile& dev, const EstimatorModel& estimator,
                             const std::vector<Request>& workload, const SearchOptions& opts);
// B200: any list of candidates in one sweep (every capacity search advances in
// the same rounds of speculative probes).  skus[cand.sku_index] and
// estimators[cand.sku_index] serve each candidate; results are in `cands` order
// and equal evaluate_config on each.  This is how axes the search config
// cannot express (watermark, replica count, block size) are swept.
std::vector<ConfigResult> evaluate_configs(const ModelSpec& spec,
                                           const std::vector<CandidateConfig>& cands,
                                           const std::vector<DeviceProfile>& skus,
                                           const std::vector<const EstimatorModel*>& estimators,
                                           const std::vector<Request>& workload,
                                           const SearchOptions& opts);

// The whole sweep on the local GPU: every config's capacity search advances
// in lock-step rounds of speculative probes (sweep.cu / search.cpp).
// `shard`/`num_shards` restrict evaluation to one shard of the grid for the
// multi-GPU driver (the other entries are left default; `owned` receives the
// enumeration indices this shard evaluated).  The capacity objective splits the
// grid by a longest-processing-time assignment on every config's initial QPS
// guess (identical on every rank); the makespan objective strides i % num_shards.
SearchOutcome run_search(const ModelSpec& spec, const std::vector<Request>& workload,
                         const SearchOptions& opts);
std::vector<ConfigResult> evaluate_configs_shard(const ModelSpec& spec,
                                                 const std::vector<Request>& workload,
                                                 const SearchOptions& opts, int shard,
                                                 int num_shards,
                                                 std::vector<std::size_t>* owned = nullptr);
SearchOutcome finalize_search(const ModelSpec& spec, const SearchOptions& opts,
                              std::vector<ConfigResult> results);

// A prepared sweep: configs enumerated, estimators trained and resident in
// HBM, probe workload and arrival exponentials built.  evaluate() is the hot
// path (repeatable; what the bench times).
class SearchSession {
 public:
  SearchSession(const ModelSpec& spec, const std::vector<Request>& workload,
                const SearchOptions& opts);
  // A session over the caller's candidates, SKUs and trained estimators
  // (estimators[k] serves skus[k]); evaluate_configs is built on it.
  SearchSession(const ModelSpec& spec, std::vector<CandidateConfig> cands,
                const std::vector<DeviceProfile>& skus,
                const std::vector<const EstimatorModel*>& estimators,
                const std::vector<Request>& workload, const SearchOptions& opts);
  ~SearchSession();
  std::vector<ConfigResult> evaluate(int shard = 0, int num_shards = 1,
                                     std::vector<std::size_t>* owned = nullptr);
  std::size_t num_configs() const;

 private:
  struct State;
  std::unique_ptr<State> st_;
  void open_workload(const std::vector<Request>& workload);
};

std::string search_results_to_csv(const SearchOutcome& outcome);
std::string frontier_to_csv(const SearchOutcome& outcome, const std::vector<std::size_t>& frontier,
                            bool use_ttft);
std::string search_summary_text(const SearchOutcome& outcome, const std::string& objective);

}  // namespace servesim
