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
#include <functional>
#include <map>
#include <memory>
#include <optional>
#include <stdexcept>
#include <string>
#include <vector>

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
    RegressorData regressor;
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

  std::string to_json() const;
  static EstimatorModel from_json(const std::string& text);

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
};

struct SimOptions {
  bool record_iterations = false;
  bool record_batches = false;
  double abort_delay_threshold = 0.0;
  std::size_t abort_max_late = 0;
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
std::string summary_to_json(const MetricsReport& rep);

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

// Loaded search config (reference config.hpp:101-179).
struct LoadedSearchConfig {
  ModelSpec spec;
  std::vector<Request> workload;
  SearchOptions options;
};
LoadedSearchConfig load_search_config(const std::string& path);
struct LoadedClusterConfig {
  ClusterConfig cluster;
};
LoadedClusterConfig load_cluster_config(const std::string& path);

double find_capacity_replay(const std::function<bool(double)>& feasible,
                            const CapacitySearchOptions& opts);
double initial_qps_guess(const ModelSpec& spec, const CandidateConfig& cand,
                         const EstimatorModel& est, const ClusterConfig& cluster);
double qps_per_dollar(double capacity_qps, std::int64_t gpus_used, double rate_per_gpu_hr);

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
  ~SearchSession();
  std::vector<ConfigResult> evaluate(int shard = 0, int num_shards = 1,
                                     std::vector<std::size_t>* owned = nullptr);
  std::size_t num_configs() const;

 private:
  struct State;
  std::unique_ptr<State> st_;
};

std::string search_results_to_csv(const SearchOutcome& outcome);
std::string frontier_to_csv(const SearchOutcome& outcome, const std::vector<std::size_t>& frontier,
                            bool use_ttft);
std::string search_summary_text(const SearchOutcome& outcome, const std::string& objective);

}  // namespace servesim
