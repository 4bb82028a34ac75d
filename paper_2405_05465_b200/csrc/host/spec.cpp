// spec.cpp -- model/device/policy configuration and the per-stage operator set.
//
// Host-side inputs of the hot path: the simulation kernels never see a JSON
// document or a ModelSpec, only the flattened operator table and memory plan
// computed here once per candidate config.
//
// reference: model_spec.hpp:112-307, device.hpp:22-61, memory.hpp:21-46,
//            scheduler.hpp:23-76, op_cost.hpp, csv.hpp:17-22
#include <charconv>
#include <cmath>

#include "json.hpp"
#include "servesim_b200.hpp"

namespace servesim {

using json = nlohmann::json;

std::string fmt_double(double v) {
  char buf[64];
  auto r = std::to_chars(buf, buf + sizeof buf, v);
  internal_check(r.ec == std::errc(), "fmt_double: to_chars failed");
  return std::string(buf, r.ptr);
}

// ------------------------------------------------------------------ op names
namespace {
struct OpInfo {
  OpName op;
  const char* name;
  OpClass cls;
};
constexpr OpInfo kOps[kNumOps] = {
    {OpName::QkvProj, "qkv_proj", OpClass::TokenLevel},
    {OpName::AttnOutProj, "attn_out_proj", OpClass::TokenLevel},
    {OpName::MlpUpProj, "mlp_up_proj", OpClass::TokenLevel},
    {OpName::MlpDownProj, "mlp_down_proj", OpClass::TokenLevel},
    {OpName::ActFn, "act_fn", OpClass::TokenLevel},
    {OpName::AddNorm, "add_norm", OpClass::TokenLevel},
    {OpName::AttnPrefill, "attn_prefill", OpClass::SequenceLevel},
    {OpName::AttnDecode, "attn_decode", OpClass::SequenceLevel},
    {OpName::AllReduce, "allreduce", OpClass::Communication},
    {OpName::AllGather, "allgather", OpClass::Communication},
    {OpName::SendRecv, "send_recv", OpClass::Communication},
};
}  // namespace

const char* to_string(OpName op) {
  int i = static_cast<int>(op);
  return (i >= 0 && i < kNumOps) ? kOps[i].name : "?";
}

OpClass triage(OpName op) {
  int i = static_cast<int>(op);
  if (i < 0 || i >= kNumOps) throw Error("triage: unknown operator");
  return kOps[i].cls;
}

OpName op_name_from_string(const std::string& s) {
  std::string known;
  for (const auto& o : kOps) {
    if (s == o.name) return o.op;
    if (!known.empty()) known += ", ";
    known += o.name;
  }
  throw Error("unknown op_name '" + s + "'; known ops: " + known);
}

std::string to_string(const OpModelKey& k) {
  return std::string(to_string(k.op)) + "@tp" + std::to_string(k.tp_degree);
}

// ------------------------------------------------------------------ model spec
void validate(const ModelSpec& s) {
  auto positive = [](std::int64_t v, const char* field) {
    require(v > 0, std::string("model spec: field '") + field + "' must be strictly positive");
  };
  require(!s.name.empty(), "model spec: field 'name' must be non-empty");
  positive(s.num_layers, "num_layers");
  positive(s.hidden_dim, "hidden_dim");
  positive(s.num_q_heads, "num_q_heads");
  positive(s.num_kv_heads, "num_kv_heads");
  positive(s.head_dim, "head_dim");
  positive(s.mlp_dim, "mlp_dim");
  positive(s.vocab_size, "vocab_size");
  positive(s.max_context, "max_context");
  positive(s.param_bytes_per_element, "param_bytes_per_element");
  require(s.num_q_heads * s.head_dim == s.hidden_dim,
          "model spec: invariant num_q_heads*head_dim == hidden_dim violated "
          "(fields 'num_q_heads', 'head_dim', 'hidden_dim')");
  require(s.num_q_heads % s.num_kv_heads == 0,
          "model spec: field 'num_kv_heads' must divide num_q_heads");
  const bool same = s.num_kv_heads == s.num_q_heads;
  if (s.attention_variant == AttentionVariant::MHA)
    require(same, "model spec: field 'attention_variant' is mha but num_kv_heads != num_q_heads");
  else
    require(!same, "model spec: field 'attention_variant' is gqa but num_kv_heads == num_q_heads");
}

void validate(const ModelSpec& s, const ParallelismConfig& p) {
  require(p.tp_degree > 0 && p.pp_degree > 0 && p.num_replicas > 0,
          "parallelism: tp_degree, pp_degree and num_replicas must be strictly positive");
  require(s.num_layers % p.pp_degree == 0,
          "parallelism: num_layers (" + std::to_string(s.num_layers) +
              ") not divisible by pp_degree (" + std::to_string(p.pp_degree) + ")");
  require(s.num_kv_heads % p.tp_degree == 0,
          "parallelism: num_kv_heads (" + std::to_string(s.num_kv_heads) +
              ") not divisible by tp_degree (" + std::to_string(p.tp_degree) + ")");
}

ModelSpec parse_model_spec(const std::string& text) {
  json j;
  try {
    j = json::parse(text);
  } catch (const json::exception& e) {
    throw Error(std::string("model spec: invalid document: ") + e.what());
  }
  auto field = [&](const char* key) -> const json& {
    require(j.contains(key), std::string("model spec: missing required field '") + key + "'");
    return j.at(key);
  };
  ModelSpec s;
  std::string variant;
  try {
    require(field("schema_version").get<int>() == 1, "model spec: unsupported schema_version");
    s.name = field("name").get<std::string>();
    auto count = [&](const char* key) {
      const json& v = field(key);
      require(v.is_number_integer(),
              std::string("model spec: field '") + key + "' must be an integer");
      return v.get<std::int64_t>();
    };
    s.num_layers = count("num_layers");
    s.hidden_dim = count("hidden_dim");
    s.num_q_heads = count("num_q_heads");
    s.num_kv_heads = count("num_kv_heads");
    s.head_dim = count("head_dim");
    s.mlp_dim = count("mlp_dim");
    s.vocab_size = count("vocab_size");
    s.max_context = count("max_context");
    s.param_bytes_per_element = count("param_bytes_per_element");
    variant = field("attention_variant").get<std::string>();
  } catch (const json::exception& e) {
    throw Error(std::string("model spec: malformed field: ") + e.what());
  }
  if (variant == "mha")
    s.attention_variant = AttentionVariant::MHA;
  else if (variant == "gqa")
    s.attention_variant = AttentionVariant::GQA;
  else
    throw Error("model spec: field 'attention_variant' must be 'mha' or 'gqa'");
  validate(s);
  return s;
}

std::vector<OperatorDescriptor> derive_operators(const ModelSpec& s, const ParallelismConfig& p) {
  validate(s);
  validate(s, p);
  const std::int64_t t = p.tp_degree, lps = s.num_layers / p.pp_degree;
  const std::int64_t q_width = s.num_q_heads * s.head_dim, kv_width = s.num_kv_heads * s.head_dim;
  const std::int64_t e = s.param_bytes_per_element;
  std::vector<OperatorDescriptor> ops;
  auto token_op = [&](OpName op, std::int64_t in, std::int64_t out) {
    OperatorDescriptor d;
    d.op = op;
    d.op_class = OpClass::TokenLevel;
    d.count = lps;
    d.tp_degree = t;
    d.in_dim = in;
    d.out_dim = out;
    d.elem_bytes = e;
    ops.push_back(d);
  };
  token_op(OpName::QkvProj, s.hidden_dim, (q_width + 2 * kv_width) / t);
  token_op(OpName::AttnOutProj, q_width / t, s.hidden_dim);
  token_op(OpName::MlpUpProj, s.hidden_dim, s.mlp_dim / t);
  token_op(OpName::MlpDownProj, s.mlp_dim / t, s.hidden_dim);
  token_op(OpName::ActFn, s.mlp_dim / t, s.mlp_dim / t);
  token_op(OpName::AddNorm, s.hidden_dim, s.hidden_dim);
  for (OpName op : {OpName::AttnPrefill, OpName::AttnDecode}) {
    OperatorDescriptor d;
    d.op = op;
    d.op_class = OpClass::SequenceLevel;
    d.count = lps;
    d.tp_degree = t;
    d.q_heads_per_device = s.num_q_heads / t;
    d.kv_heads_per_device = s.num_kv_heads / t;
    d.head_dim = s.head_dim;
    d.elem_bytes = e;
    ops.push_back(d);
  }
  auto comm_op = [&](OpName op, std::int64_t count, std::int64_t bytes_per_token) {
    OperatorDescriptor d;
    d.op = op;
    d.op_class = OpClass::Communication;
    d.count = count;
    d.tp_degree = t;
    d.payload_bytes_per_token = bytes_per_token;
    d.elem_bytes = e;
    ops.push_back(d);
  };
  if (t > 1) {
    comm_op(OpName::AllReduce, 2 * lps, s.hidden_dim * e);
    comm_op(OpName::AllGather, 1, (s.vocab_size / t) * e);
  }
  if (p.pp_degree > 1) comm_op(OpName::SendRecv, 1, s.hidden_dim * e);
  return ops;
}

std::int64_t param_bytes_per_device(const ModelSpec& s, const ParallelismConfig& p) {
  validate(s);
  validate(s, p);
  const std::int64_t t = p.tp_degree;
  const std::int64_t q_width = s.num_q_heads * s.head_dim, kv_width = s.num_kv_heads * s.head_dim;
  const std::int64_t layer = s.hidden_dim * ((q_width + 2 * kv_width) / t) +
                             (q_width / t) * s.hidden_dim + s.hidden_dim * (s.mlp_dim / t) +
                             (s.mlp_dim / t) * s.hidden_dim;
  const std::int64_t embed = ((s.vocab_size + t - 1) / t) * s.hidden_dim;
  std::int64_t elems = (s.num_layers / p.pp_degree) * layer;
  elems += (p.pp_degree == 1 ? 2 : 1) * embed;
  return elems * s.param_bytes_per_element;
}

std::int64_t kv_bytes_per_token_per_device(const ModelSpec& s, const ParallelismConfig& p) {
  validate(s);
  validate(s, p);
  require(p.tp_degree <= s.num_kv_heads, "kv sharding: tp_degree exceeds num_kv_heads");
  return 2 * (s.num_layers / p.pp_degree) * (s.num_kv_heads / p.tp_degree) * s.head_dim *
         s.param_bytes_per_element;
}

std::int64_t kv_bytes_per_token_per_block(const ModelSpec& s, const ParallelismConfig& p) {
  return kv_bytes_per_token_per_device(s, p) / (s.num_layers / p.pp_degree);
}

// ------------------------------------------------------------------ device
void validate(const DeviceProfile& d) {
  require(!d.sku_name.empty(), "device profile: field 'sku_name' must be non-empty");
  require(d.peak_flops > 0, "device profile: field 'peak_flops' must be positive");
  require(d.mem_bandwidth > 0, "device profile: field 'mem_bandwidth' must be positive");
  require(d.link_bandwidth > 0, "device profile: field 'link_bandwidth' must be positive");
  require(d.kernel_overhead > 0, "device profile: field 'kernel_overhead' must be positive");
  require(d.kernel_overhead < 1e-3, "device profile: field 'kernel_overhead' must be < 1e-3 s");
  require(d.device_mem > 0, "device profile: field 'device_mem' must be positive");
}

DeviceProfile parse_device_profile(const std::string& text) {
  json j;
  try {
    j = json::parse(text);
  } catch (const json::exception& e) {
    throw Error(std::string("device profile: invalid document: ") + e.what());
  }
  DeviceProfile d;
  try {
    auto field = [&](const char* key) -> const json& {
      require(j.contains(key),
              std::string("device profile: missing required field '") + key + "'");
      return j.at(key);
    };
    require(field("schema_version").get<int>() == 1, "device profile: unsupported schema_version");
    d.sku_name = field("sku_name").get<std::string>();
    d.peak_flops = field("peak_flops").get<double>();
    d.mem_bandwidth = field("mem_bandwidth").get<double>();
    d.link_bandwidth = field("link_bandwidth").get<double>();
    d.kernel_overhead = field("kernel_overhead").get<double>();
    d.device_mem = field("device_mem").get<double>();
  } catch (const json::exception& e) {
    throw Error(std::string("device profile: malformed field: ") + e.what());
  }
  validate(d);
  return d;
}

// ------------------------------------------------------------------ memory
MemoryPlan plan_memory(const ModelSpec& spec, const ParallelismConfig& par,
                       const DeviceProfile& dev, std::int64_t block_size,
                       double watermark_fraction, double activation_reserve_fraction) {
  require(block_size >= 1, "plan_memory: block_size must be >= 1");
  require(watermark_fraction >= 0.0 && watermark_fraction < 1.0,
          "plan_memory: watermark_fraction must be in [0, 1)");
  require(activation_reserve_fraction >= 0.0 && activation_reserve_fraction < 1.0,
          "plan_memory: activation_reserve_fraction must be in [0, 1)");
  const double params = static_cast<double>(param_bytes_per_device(spec, par));
  const double reserve = activation_reserve_fraction * dev.device_mem;
  const double free_bytes = dev.device_mem - params - reserve;
  const double per_token = static_cast<double>(kv_bytes_per_token_per_device(spec, par));
  MemoryPlan m;
  m.block_size = block_size;
  if (free_bytes > 0)
    m.num_blocks = static_cast<std::int64_t>(free_bytes / (static_cast<double>(block_size) * per_token));
  require(m.num_blocks >= 1, "insufficient device memory: " + spec.name + " on " + dev.sku_name +
                                 " (params " + std::to_string(static_cast<std::int64_t>(params)) +
                                 " B + reserve leave no room for KV blocks)");
  m.kv_capacity_tokens = m.num_blocks * block_size;
  m.watermark_blocks = static_cast<std::int64_t>(watermark_fraction * static_cast<double>(m.num_blocks));
  return m;
}

// ------------------------------------------------------------------ policies
const char* to_string(SchedulerPolicy p) {
  switch (p) {
    case SchedulerPolicy::FasterTransformer: return "faster_transformer";
    case SchedulerPolicy::OrcaPlus: return "orca_plus";
    case SchedulerPolicy::VLLM: return "vllm";
    case SchedulerPolicy::SarathiServe: return "sarathi_serve";
    case SchedulerPolicy::LightLLM: return "lightllm";
  }
  return "?";
}

SchedulerPolicy scheduler_policy_from_string(const std::string& s) {
  for (auto p : {SchedulerPolicy::FasterTransformer, SchedulerPolicy::OrcaPlus,
                 SchedulerPolicy::VLLM, SchedulerPolicy::SarathiServe, SchedulerPolicy::LightLLM})
    if (s == to_string(p)) return p;
  throw Error("unknown scheduler policy '" + s +
              "' (expected faster_transformer|orca_plus|vllm|sarathi_serve|lightllm)");
}

const char* to_string(RoutingPolicy p) {
  switch (p) {
    case RoutingPolicy::RoundRobin: return "round_robin";
    case RoutingPolicy::LeastOutstanding: return "least_outstanding";
    case RoutingPolicy::Deferred: return "deferred";
  }
  return "?";
}

RoutingPolicy routing_policy_from_string(const std::string& s) {
  for (auto p : {RoutingPolicy::RoundRobin, RoutingPolicy::LeastOutstanding,
                 RoutingPolicy::Deferred})
    if (s == to_string(p)) return p;
  throw Error("unknown routing policy '" + s +
              "' (expected round_robin|least_outstanding|deferred)");
}

void validate(const PolicyConfig& c) {
  require(c.max_batch_size >= 1, "policy: max_batch_size must be >= 1");
  require(c.max_tokens_per_iter >= 1, "policy: max_tokens_per_iter must be >= 1");
  require(c.chunk_size >= 1, "policy: chunk_size must be >= 1");
  require(c.block_size >= 1, "policy: block_size must be >= 1");
}

}  // namespace servesim
