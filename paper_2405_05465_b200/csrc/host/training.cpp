// training.cpp -- synthetic profiling and per-operator predictor fitting.
//
// Runs once per (model, SKU) on the host before any simulation: it is the
// "data loader" of the framework, producing the tables and tree ensembles the
// predictor kernels evaluate.  Arithmetic is kept operation-for-operation
// equal to the reference (built with -ffp-contract=off, libstdc++ RNG) so the
// trained models are bit-identical and the JSON handoff round-trips exactly.
//
// reference: op_cost.hpp:21-98, profiler.hpp:54-347, regressor.hpp:26-386,
//            estimator.hpp:137-275
#include <algorithm>
#include <cstdlib>
#include <exception>
#include <cmath>
#include <random>
#include <cstring>
#include <unordered_map>
#include <vector>

#include "json.hpp"
#include "runtime.h"
#include "servesim_b200.hpp"
#include "train.h"

namespace servesim {

using json = nlohmann::json;

// ------------------------------------------------------------------ costs
namespace {

struct Work {
  double flops = 0, bytes = 0, wire_bytes = 0;
  std::int64_t hops = 0;
};

Work token_work(const OperatorDescriptor& d, double n) {  // op_cost.hpp:21-48
  Work w;
  const double e = static_cast<double>(d.elem_bytes);
  const double in = static_cast<double>(d.in_dim), out = static_cast<double>(d.out_dim);
  switch (d.op) {
    case OpName::QkvProj:
    case OpName::AttnOutProj:
    case OpName::MlpUpProj:
    case OpName::MlpDownProj:
      w.flops = 2.0 * n * in * out;
      w.bytes = n > 0 ? e * (in * out + n * (in + out)) : 0.0;
      break;
    case OpName::ActFn:
      w.flops = n * in;
      w.bytes = 2.0 * e * n * in;
      break;
    case OpName::AddNorm:
      w.flops = 8.0 * n * in;
      w.bytes = 6.0 * e * n * in;
      break;
    default:
      throw InternalError("token_level_cost: not a token-level op");
  }
  return w;
}

Work attention_work(const OperatorDescriptor& d, double n, double kv_read) {  // op_cost.hpp:52-73
  Work w;
  const double e = static_cast<double>(d.elem_bytes);
  const double hq = static_cast<double>(d.q_heads_per_device * d.head_dim);
  const double hkv = static_cast<double>(d.kv_heads_per_device * d.head_dim);
  const double ctx = kv_read / (2.0 * e * hkv);
  if (d.op == OpName::AttnPrefill) {
    w.flops = 4.0 * n * (n + ctx) * hq;
    w.bytes = kv_read + e * n * (2.0 * hq + 2.0 * hkv);
  } else if (d.op == OpName::AttnDecode) {
    w.flops = 4.0 * ctx * hq;
    w.bytes = kv_read;
  } else {
    throw InternalError("attention_cost: not an attention op");
  }
  return w;
}

Work comm_work(const OperatorDescriptor& d, double payload) {  // op_cost.hpp:78-98
  Work w;
  const double t = static_cast<double>(d.tp_degree);
  switch (d.op) {
    case OpName::AllReduce:
      w.wire_bytes = payload * 2.0 * (t - 1.0) / t;
      w.hops = d.tp_degree - 1;
      break;
    case OpName::AllGather:
      w.wire_bytes = payload * (t - 1.0) / t;
      w.hops = d.tp_degree - 1;
      break;
    case OpName::SendRecv:
      w.wire_bytes = payload;
      w.hops = 1;
      break;
    default:
      throw InternalError("communication_cost: not a communication op");
  }
  return w;
}

double feature_or(const FeatureMap& f, const char* name, double fallback) {
  auto it = f.find(name);
  return it == f.end() ? fallback : it->second;
}

}  // namespace

std::vector<std::string> feature_schema(OpClass c) {
  switch (c) {
    case OpClass::TokenLevel: return {kFeatNumTokens};
    case OpClass::SequenceLevel: return {kFeatNumTokens, kFeatKvReadBytes};
    case OpClass::Communication: return {kFeatPayloadBytes};
  }
  throw InternalError("feature_schema: bad op class");
}

double synthetic_oracle(const OperatorDescriptor& d, const FeatureMap& f, const DeviceProfile& dev) {
  switch (d.op_class) {
    case OpClass::TokenLevel: {
      Work w = token_work(d, feature_or(f, kFeatNumTokens, 0.0));
      return std::max(w.flops / dev.peak_flops, w.bytes / dev.mem_bandwidth) + dev.kernel_overhead;
    }
    case OpClass::SequenceLevel: {
      Work w = attention_work(d, feature_or(f, kFeatNumTokens, 0.0),
                              feature_or(f, kFeatKvReadBytes, 0.0));
      return std::max(w.flops / dev.peak_flops, w.bytes / dev.mem_bandwidth) + dev.kernel_overhead;
    }
    case OpClass::Communication: {
      Work w = comm_work(d, feature_or(f, kFeatPayloadBytes, 0.0));
      return w.wire_bytes / dev.link_bandwidth + static_cast<double>(w.hops) * dev.kernel_overhead;
    }
  }
  throw InternalError("synthetic_oracle: bad op class");
}

// ------------------------------------------------------------------ grids
namespace {

// synthetic_oracle at a grid point given in feature_schema order, without
// building the FeatureMap (same Work functions, same arithmetic)
double oracle_at(const OperatorDescriptor& d, const std::vector<double>& pt, const DeviceProfile& dev) {
  switch (d.op_class) {
    case OpClass::TokenLevel: {
      Work w = token_work(d, pt[0]);
      return std::max(w.flops / dev.peak_flops, w.bytes / dev.mem_bandwidth) + dev.kernel_overhead;
    }
    case OpClass::SequenceLevel: {
      Work w = attention_work(d, pt[0], pt[1]);
      return std::max(w.flops / dev.peak_flops, w.bytes / dev.mem_bandwidth) + dev.kernel_overhead;
    }
    case OpClass::Communication: {
      Work w = comm_work(d, pt[0]);
      return w.wire_bytes / dev.link_bandwidth + static_cast<double>(w.hops) * dev.kernel_overhead;
    }
  }
  throw InternalError("synthetic_oracle: bad op class");
}

std::vector<std::int64_t> doubling_levels(std::int64_t lo, std::int64_t hi) {
  std::vector<std::int64_t> v;
  for (std::int64_t x = lo; x < hi; x *= 2) v.push_back(x);
  v.push_back(hi);
  return v;
}

std::vector<std::int64_t> ratio_levels(std::int64_t lo, std::int64_t hi, double ratio) {
  std::vector<std::int64_t> v;
  for (double x = static_cast<double>(lo); x < static_cast<double>(hi); x *= ratio) {
    const std::int64_t level = std::llround(x);
    if (v.empty() || level > v.back()) v.push_back(level);
  }
  if (v.empty() || v.back() != hi) v.push_back(hi);
  return v;
}

// Axis levels of the base profiling grid per op class (profiler.hpp:97-128).
std::vector<std::vector<double>> base_axes(OpClass c, std::int64_t max_context,
                                           std::int64_t kv_per_token_block) {
  std::vector<std::vector<double>> axes;
  switch (c) {
    case OpClass::TokenLevel: {
      std::vector<double> n;
      for (auto v : doubling_levels(1, max_context)) n.push_back(static_cast<double>(v));
      axes.push_back(n);
      break;
    }
    case OpClass::SequenceLevel: {
      require(kv_per_token_block > 0,
              "profile_grid: kv_bytes_per_token_block unset for sequence-level grid");
      const double r = std::sqrt(2.0);
      std::vector<double> n, kv;
      for (auto v : ratio_levels(1, max_context, r)) n.push_back(static_cast<double>(v));
      kv.push_back(0.0);
      for (auto k : ratio_levels(1, 512 * max_context, r))
        kv.push_back(static_cast<double>(k * kv_per_token_block));
      axes.push_back(n);
      axes.push_back(kv);
      break;
    }
    case OpClass::Communication: {
      std::vector<double> p;
      for (std::int64_t e = 10; e <= 30; ++e) p.push_back(static_cast<double>(std::int64_t(1) << e));
      axes.push_back(p);
      break;
    }
  }
  // sorted-unique already holds for these generators; keep the invariant explicit
  for (auto& ax : axes) {
    std::sort(ax.begin(), ax.end());
    ax.erase(std::unique(ax.begin(), ax.end()), ax.end());
  }
  return axes;
}

FeatureMap feature_point(const std::vector<std::string>& schema, const std::vector<double>& v) {
  FeatureMap f;
  for (std::size_t i = 0; i < schema.size(); ++i) f[schema[i]] = v[i];
  return f;
}

// Adaptive bisection of axis gaps where log-space interpolation of the oracle
// is worst (profiler.hpp:241-309); returns the refined per-axis levels.
std::vector<std::vector<double>> refine_axes(const OperatorDescriptor& d,
                                             std::vector<std::vector<double>> axes,
                                             const DeviceProfile& dev) {
  const double tol = 0.015;
  const int max_extra = 24;
  const auto schema = feature_schema(d.op_class);
  const std::size_t nf = axes.size();
  // the error of one (axis, gap, cross-section) never changes between rounds:
  // memoised by its exact coordinates, each round re-reads the old ones and
  // evaluates the oracle only where the last inserted level made new gaps or
  // sections (same errors, same scan order, same strict-max choice)
  struct KeyHash {
    std::size_t operator()(const std::vector<std::uint64_t>& k) const {
      std::uint64_t h = 0x9e3779b97f4a7c15ull;
      for (auto v : k) h = (h ^ v) * 0x100000001b3ull;
      return static_cast<std::size_t>(h ^ (h >> 29));
    }
  };
  std::unordered_map<std::vector<std::uint64_t>, double, KeyHash> memo;
  auto bits = [](double v) {
    std::uint64_t u;
    std::memcpy(&u, &v, sizeof u);
    return u;
  };
  std::vector<std::uint64_t> key;
  for (int round = 0; round < max_extra; ++round) {
    double worst = 0.0, worst_mid = 0.0;
    std::size_t worst_axis = 0;
    for (std::size_t f = 0; f < nf; ++f) {
      // cross sections over the other axes, earlier axes outermost
      std::vector<std::vector<double>> sections{std::vector<double>(nf, 0.0)};
      for (std::size_t g = 0; g < nf; ++g) {
        if (g == f) continue;
        std::vector<std::vector<double>> next;
        for (const auto& base : sections)
          for (double v : axes[g]) {
            auto m = base;
            m[g] = v;
            next.push_back(std::move(m));
          }
        sections = std::move(next);
      }
      for (std::size_t i = 0; i + 1 < axes[f].size(); ++i) {
        const double a = axes[f][i], b = axes[f][i + 1];
        const double mid = std::expm1(0.5 * (std::log1p(a) + std::log1p(b)));
        for (auto sec : sections) {
          key.assign({static_cast<std::uint64_t>(f), bits(a), bits(b)});
          for (std::size_t g = 0; g < nf; ++g)
            if (g != f) key.push_back(bits(sec[g]));
          auto it = memo.find(key);
          double err;
          if (it != memo.end()) {
            err = it->second;
          } else {
            sec[f] = a;
            const double ya = std::log(oracle_at(d, sec, dev));
            sec[f] = b;
            const double yb = std::log(oracle_at(d, sec, dev));
            sec[f] = mid;
            const double truth = oracle_at(d, sec, dev);
            err = std::fabs(std::exp(0.5 * (ya + yb)) - truth) / truth;
            memo.emplace(key, err);
          }
          if (err > worst) {
            worst = err;
            worst_axis = f;
            worst_mid = mid;
          }
        }
      }
    }
    if (worst <= tol) break;
    auto& ax = axes[worst_axis];
    ax.insert(std::upper_bound(ax.begin(), ax.end(), worst_mid), worst_mid);
  }
  return axes;
}

}  // namespace

std::vector<ProfileRecord> generate_synthetic_profile(const ModelSpec& spec,
                                                      const DeviceProfile& dev,
                                                      const std::vector<std::int64_t>& tps) {
  std::vector<ProfileRecord> out;
  for (std::int64_t tp : tps) {
    ParallelismConfig par{tp, 1, 1};
    validate(spec, par);
    auto ops = derive_operators(spec, par);
    OperatorDescriptor sr;
    sr.op = OpName::SendRecv;
    sr.op_class = OpClass::Communication;
    sr.count = 1;
    sr.tp_degree = tp;
    sr.payload_bytes_per_token = spec.hidden_dim * spec.param_bytes_per_element;
    sr.elem_bytes = spec.param_bytes_per_element;
    ops.push_back(sr);
    const std::int64_t kvb = kv_bytes_per_token_per_block(spec, par);
    for (const auto& d : ops) {
      const auto schema = feature_schema(d.op_class);
      auto axes = refine_axes(d, base_axes(d.op_class, spec.max_context, kvb), dev);
      std::size_t cells = 1;
      for (auto& ax : axes) cells *= ax.size();
      std::vector<double> pt(axes.size());
      for (std::size_t c = 0; c < cells; ++c) {  // last axis fastest
        std::size_t rem = c;
        for (std::size_t k = axes.size(); k-- > 0;) {
          pt[k] = axes[k][rem % axes[k].size()];
          rem /= axes[k].size();
        }
        ProfileRecord r;
        r.op = d.op;
        r.features = feature_point(schema, pt);
        r.runtime = oracle_at(d, pt, dev);
        r.features[kFeatTpDegree] = static_cast<double>(tp);
        out.push_back(std::move(r));
      }
    }
  }
  return out;
}

// Root-sum-square prefill length (estimator.hpp:38-46); the engine forms the
// same value on the device from integer sums of squares (exact below 2^53).
std::int64_t equivalent_prefill_length(const std::vector<std::int64_t>& prefill_lengths) {
  require(!prefill_lengths.empty(), "equivalent_prefill_length: empty prefill set");
  double sq = 0.0;
  for (auto p : prefill_lengths) {
    require(p > 0, "equivalent_prefill_length: lengths must be positive");
    sq += static_cast<double>(p) * static_cast<double>(p);
  }
  return static_cast<std::int64_t>(std::llround(std::sqrt(sq)));
}

// Model flops of one batch on one device (estimator.hpp:353-380): the MFU
// numerator for callers of the API; the engine accumulates the same terms on
// the device per iteration (engine.cuh batch_latency).
double batch_device_flops(const std::vector<OperatorDescriptor>& ops, const BatchComposition& batch) {
  const double total_tokens = static_cast<double>(batch.total_current_tokens());
  double flops = 0.0;
  for (const auto& d : ops) {
    const double count = static_cast<double>(d.count);
    if (d.op_class == OpClass::TokenLevel) {
      flops += count * token_work(d, total_tokens).flops;
    } else if (d.op_class == OpClass::SequenceLevel) {
      const double kvb = 2.0 * static_cast<double>(d.elem_bytes) *
                         static_cast<double>(d.kv_heads_per_device * d.head_dim);
      if (d.op == OpName::AttnPrefill && !batch.prefill_lengths.empty()) {
        const double n_eq = static_cast<double>(equivalent_prefill_length(batch.prefill_lengths));
        double prior = 0.0;
        for (auto c : batch.prefill_prior_context) prior += static_cast<double>(c);
        flops += count * attention_work(d, n_eq, prior * kvb).flops;
      } else if (d.op == OpName::AttnDecode && !batch.decode_context_lengths.empty()) {
        double ctx = 0.0;
        for (auto c : batch.decode_context_lengths) ctx += static_cast<double>(c);
        flops += count * attention_work(d, static_cast<double>(batch.num_decode_tokens()), ctx * kvb).flops;
      }
    }
  }
  return flops;
}

// ------------------------------------------------------------------ regressors
namespace {

using Rows = std::vector<std::vector<double>>;

RegressorData fit_interp(const Rows& x, const std::vector<double>& y) {  // regressor.hpp:278-306
  require(!x.empty() && x.size() == y.size(), "interp fit: empty or mismatched data");
  RegressorData g;
  g.type = "interp";
  const std::size_t nf = x.front().size();
  g.axes.resize(nf);
  for (std::size_t f = 0; f < nf; ++f) {
    auto& ax = g.axes[f];
    for (const auto& row : x) ax.push_back(row[f]);
    std::sort(ax.begin(), ax.end());
    ax.erase(std::unique(ax.begin(), ax.end()), ax.end());
  }
  std::size_t cells = 1;
  for (auto& ax : g.axes) cells *= ax.size();
  require(cells == x.size(), "interp fit: training points do not form a full grid (" +
                                 std::to_string(x.size()) + " points vs " + std::to_string(cells) +
                                 " cells); train scattered data with the forest regressor");
  g.values.assign(cells, 0.0);
  std::vector<char> seen(cells, 0);
  for (std::size_t i = 0; i < x.size(); ++i) {
    std::size_t flat = 0, stride = 1;
    for (std::size_t f = nf; f-- > 0;) {
      auto it = std::lower_bound(g.axes[f].begin(), g.axes[f].end(), x[i][f]);
      internal_check(it != g.axes[f].end() && *it == x[i][f], "interp fit: off-axis point");
      flat += static_cast<std::size_t>(it - g.axes[f].begin()) * stride;
      stride *= g.axes[f].size();
    }
    require(!seen[flat], "interp fit: duplicate grid point");
    seen[flat] = 1;
    g.values[flat] = y[i];
  }
  return g;
}

// Host evaluation used only for the training-time hold-out score (estimator.hpp:261-270);
// every runtime query goes through the device kernels.
double host_regress(const RegressorData& r, const std::vector<double>& x) {
  double sum = 0.0;
  for (const auto& t : r.trees) {
    int node = 0;
    while (t.feature[node] >= 0) node = x[t.feature[node]] <= t.threshold[node] ? t.left[node] : t.right[node];
    const auto& w = t.leaf_weights[-t.feature[node] - 1];
    double v = w[0];
    for (std::size_t f = 0; f < r.num_features; ++f) v += w[f + 1] * x[f];
    sum += std::clamp(v, r.y_lo, r.y_hi);
  }
  return sum / static_cast<double>(r.trees.size());
}

}  // namespace

EstimatorModel train(const std::vector<ProfileRecord>& records, const TrainConfig& cfg) {
  std::map<OpModelKey, std::vector<const ProfileRecord*>> groups;
  for (const auto& r : records) {
    auto it = r.features.find(kFeatTpDegree);
    require(it != r.features.end(), "train: record missing tp_degree feature");
    groups[{r.op, static_cast<std::int64_t>(it->second)}].push_back(&r);
  }
  require(!groups.empty(), "train: no records");
  const bool forest = cfg.regressor == "forest";
  // per (op, tp): transformed rows (x = log1p(feature), y = log(runtime)) and
  // the hold-out split (estimator.hpp:201-275); fitting happens afterwards
  struct Group {
    OpModelKey key;
    EstimatorModel::PerOpModel m;
    Rows x, xt;
    std::vector<double> y, yt;
    std::vector<std::size_t> held;
    ForestConfig fc;
  };
  std::vector<Group> todo;
  std::uint64_t group_index = 0;
  for (const auto& [key, recs] : groups) {
    require(recs.size() >= cfg.min_points_per_op,
            "train: op " + to_string(key) + " has only " + std::to_string(recs.size()) +
                " points (need " + std::to_string(cfg.min_points_per_op) + ")");
    Group G;
    G.key = key;
    EstimatorModel::PerOpModel& m = G.m;
    m.schema = feature_schema(triage(key.op));
    m.n_points = recs.size();
    const std::size_t nf = m.schema.size();
    m.levels.assign(nf, {});
    m.bbox_lo.assign(nf, 0.0);
    m.bbox_hi.assign(nf, 0.0);
    for (const auto* r : recs) {
      std::vector<double> row(nf);
      for (std::size_t f = 0; f < nf; ++f) {
        auto it = r->features.find(m.schema[f]);
        require(it != r->features.end(),
                "train: op " + to_string(key) + " record missing feature " + m.schema[f]);
        row[f] = std::log1p(it->second);
        m.levels[f].push_back(it->second);
      }
      G.x.push_back(std::move(row));
      G.y.push_back(std::log(r->runtime));
    }
    for (std::size_t f = 0; f < nf; ++f) {
      auto& lv = m.levels[f];
      std::sort(lv.begin(), lv.end());
      lv.erase(std::unique(lv.begin(), lv.end()), lv.end());
      m.bbox_lo[f] = lv.front();
      m.bbox_hi[f] = lv.back();
    }
    G.fc = cfg.forest;
    G.fc.seed = cfg.seed * 1000003ULL + group_index++;
    const bool can_hold = G.x.size() >= 2 * cfg.min_points_per_op;
    for (std::size_t i = 0; i < G.x.size(); ++i) {
      if (can_hold && i % 5 == 2) {
        G.held.push_back(i);
      } else {
        G.xt.push_back(G.x[i]);
        G.yt.push_back(G.y[i]);
      }
    }
    if (!forest) {
      // the interpolator is a grid reshape (host); its errors surface in group order
      if (cfg.regressor != "interp") throw Error("train: unknown regressor kind '" + cfg.regressor + "'");
      m.regressor = std::make_unique<GridInterpolator>(fit_interp(G.x, G.y));
    }
    todo.push_back(std::move(G));
  }
  if (forest) {
    // every forest of the call -- hold-out probes and final models -- grows in
    // one device launch, one warp per tree (train.cu)
    std::vector<ssg::ForestFit> fits;
    std::vector<std::pair<std::size_t, bool>> what;  // (group, is hold-out probe)
    for (std::size_t g = 0; g < todo.size(); ++g) {
      if (!todo[g].held.empty()) {
        fits.push_back({&todo[g].xt, &todo[g].yt, todo[g].fc});
        what.push_back({g, true});
      }
      fits.push_back({&todo[g].x, &todo[g].y, todo[g].fc});
      what.push_back({g, false});
    }
    std::vector<RegressorData> grown = ssg::grow_forests(fits);
    for (std::size_t k = 0; k < grown.size(); ++k) {
      Group& G = todo[what[k].first];
      if (what[k].second) {
        double ape = 0.0;
        for (auto i : G.held) {
          const double pred = std::exp(host_regress(grown[k], G.x[i]));
          const double truth = std::exp(G.y[i]);
          ape += std::fabs(pred - truth) / truth;
        }
        G.m.holdout_mape = ape / static_cast<double>(G.held.size());
      } else {
        G.m.regressor = std::make_unique<ForestRegressor>(std::move(grown[k]));
      }
    }
  }
  EstimatorModel model;
  for (auto& G : todo) model.insert(G.key, std::move(G.m));
  return model;
}

// ------------------------------------------------------------------ JSON
namespace {

json regressor_json(const RegressorData& r) {
  json j;
  j["type"] = r.type;
  if (r.type == "forest") {
    j["num_features"] = r.num_features;
    j["y_lo"] = r.y_lo;
    j["y_hi"] = r.y_hi;
    json trees = json::array();
    for (const auto& t : r.trees) {
      json tj;
      tj["feature"] = t.feature;
      tj["threshold"] = t.threshold;
      tj["left"] = t.left;
      tj["right"] = t.right;
      tj["leaf_weights"] = t.leaf_weights;
      trees.push_back(std::move(tj));
    }
    j["trees"] = std::move(trees);
  } else {
    j["axes"] = r.axes;
    j["values"] = r.values;
  }
  return j;
}

RegressorData regressor_from(const json& j) {
  RegressorData r;
  r.type = j.at("type").get<std::string>();
  if (r.type == "forest") {
    r.num_features = j.at("num_features").get<std::size_t>();
    r.y_lo = j.at("y_lo").get<double>();
    r.y_hi = j.at("y_hi").get<double>();
    for (const auto& tj : j.at("trees")) {
      ForestTree t;
      t.feature = tj.at("feature").get<std::vector<int>>();
      t.threshold = tj.at("threshold").get<std::vector<double>>();
      t.left = tj.at("left").get<std::vector<int>>();
      t.right = tj.at("right").get<std::vector<int>>();
      t.leaf_weights = tj.at("leaf_weights").get<std::vector<std::vector<double>>>();
      r.trees.push_back(std::move(t));
    }
    require(!r.trees.empty(), "forest model: no trees");
    return r;
  }
  if (r.type == "interp") {
    r.axes = j.at("axes").get<std::vector<std::vector<double>>>();
    r.values = j.at("values").get<std::vector<double>>();
    std::size_t cells = 1;
    for (auto& ax : r.axes) cells *= ax.size();
    require(cells == r.values.size(), "interp model: axes/value size mismatch");
    return r;
  }
  throw Error("unknown regressor type '" + r.type + "'");
}

}  // namespace

// ------------------------------------------------------------------ Regressor
Regressor::Regressor(RegressorData d) : data_(std::move(d)) {}
Regressor::~Regressor() = default;
json Regressor::to_json() const { return regressor_json(data_); }
ForestRegressor::ForestRegressor(RegressorData d) : Regressor(std::move(d)) {
  require(data_.type == "forest", "ForestRegressor: not a forest");
}
GridInterpolator::GridInterpolator(RegressorData d) : Regressor(std::move(d)) {
  require(data_.type == "interp", "GridInterpolator: not an interpolator");
}
ForestRegressor ForestRegressor::train(const std::vector<std::vector<double>>& x,
                                       const std::vector<double>& y, const ForestConfig& cfg) {
  return ForestRegressor(std::move(ssg::grow_forests({{&x, &y, cfg}}).at(0)));  // on the GPU
}
ForestRegressor ForestRegressor::from_json(const json& j) {
  require(j.at("type").get<std::string>() == "forest", "forest model: wrong type");
  return ForestRegressor(regressor_from(j));
}
GridInterpolator GridInterpolator::fit(const std::vector<std::vector<double>>& x,
                                       const std::vector<double>& y) {
  return GridInterpolator(fit_interp(x, y));
}
GridInterpolator GridInterpolator::from_json(const json& j) {
  require(j.at("type").get<std::string>() == "interp", "interp model: wrong type");
  return GridInterpolator(regressor_from(j));
}
std::unique_ptr<Regressor> regressor_from_json(const json& j) {
  RegressorData r = regressor_from(j);  // throws "unknown regressor type '...'"
  if (r.type == "forest") return std::make_unique<ForestRegressor>(std::move(r));
  return std::make_unique<GridInterpolator>(std::move(r));
}

json EstimatorModel::to_json() const {
  json j;
  j["schema_version"] = 1;
  j["kind"] = "estimator";
  json ops = json::object();
  for (const auto& [key, m] : models_) {
    json mj;
    mj["op"] = servesim::to_string(key.op);
    mj["tp_degree"] = key.tp_degree;
    mj["schema"] = m.schema;
    mj["bbox_lo"] = m.bbox_lo;
    mj["bbox_hi"] = m.bbox_hi;
    mj["levels"] = m.levels;
    mj["holdout_mape"] = m.holdout_mape;
    mj["n_points"] = m.n_points;
    mj["regressor"] = m.regressor->to_json();
    ops[servesim::to_string(key)] = std::move(mj);
  }
  j["ops"] = std::move(ops);
  return j;
}

EstimatorModel EstimatorModel::from_json(const json& j) {
  try {
    require(j.value("kind", "") == "estimator", "estimator file: wrong kind");
    require(j.at("schema_version").get<int>() == 1, "estimator file: unsupported schema_version");
    EstimatorModel e;
    for (const auto& [unused, mj] : j.at("ops").items()) {
      OpModelKey key{op_name_from_string(mj.at("op").get<std::string>()),
                     mj.at("tp_degree").get<std::int64_t>()};
      PerOpModel m;
      m.schema = mj.at("schema").get<std::vector<std::string>>();
      m.bbox_lo = mj.at("bbox_lo").get<std::vector<double>>();
      m.bbox_hi = mj.at("bbox_hi").get<std::vector<double>>();
      m.levels = mj.at("levels").get<std::vector<std::vector<double>>>();
      m.holdout_mape = mj.at("holdout_mape").get<double>();
      m.n_points = mj.at("n_points").get<std::size_t>();
      m.regressor = regressor_from_json(mj.at("regressor"));
      e.models_[key] = std::move(m);
    }
    return e;
  } catch (const json::exception& ex) {
    throw Error(std::string("estimator file: malformed: ") + ex.what());
  }
}

}  // namespace servesim
