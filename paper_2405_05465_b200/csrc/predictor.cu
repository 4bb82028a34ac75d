// predictor.cu -- K1/K2: batched operator-runtime prediction on sm_100a.
//
// Upload: each (op, tp) model of an EstimatorModel is flattened once into HBM
//   * interp axes + values  -> dpool (fp64)
//   * forest trees          -> nodes[] 16 B records in preorder (left = i + 1,
//                              leaves carry their plane weights inline) and
//                              roots[] per tree
// A whole SKU's estimator (all ops x tp degrees) is ~60 KB (interp) or a few MB
// (forest), so it stays resident in L2 across every kernel of a sweep.
//
// Kernel: one thread per query, grid-stride over 148 SMs x resident blocks.
// Queries are SoA (model slot, feature 0, feature 1) for coalesced loads.
//
// reference: estimator.hpp:105-131 (predict/find), regressor.hpp:103-108,
//            256-264, 308-341
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <mutex>

#include "predictor.cuh"
#include "runtime.h"

namespace servesim {

namespace {

// Re-layout one reference tree (arbitrary node numbering) into preorder
// 16-byte records appended to `out`; returns the root's absolute index.
int32_t append_tree(const ForestTree& t, std::size_t nf, std::vector<SsgNode>& out) {
  const int32_t root = static_cast<int32_t>(out.size());
  // explicit stack of (reference node, slot whose `right` must be patched)
  std::vector<std::pair<int, int32_t>> stack;
  stack.push_back({0, -1});
  while (!stack.empty()) {
    auto [ref, patch] = stack.back();
    stack.pop_back();
    const int32_t here = static_cast<int32_t>(out.size());
    if (patch >= 0) out[patch].right = here;
    internal_check(ref >= 0 && ref < static_cast<int>(t.feature.size()), "forest: bad child index");
    if (t.feature[ref] >= 0) {
      SsgNode n{};
      n.a = t.threshold[ref];
      n.feat = t.feature[ref];
      n.right = -1;
      out.push_back(n);
      // preorder: left subtree immediately follows, right is patched later
      stack.push_back({t.right[ref], here});
      stack.push_back({t.left[ref], -1});
    } else {
      const auto& w = t.leaf_weights.at(static_cast<std::size_t>(-t.feature[ref] - 1));
      internal_check(w.size() == nf + 1, "forest: leaf weight count mismatch");
      SsgNode n{};
      n.a = w[0];
      n.feat = -1;
      n.right = static_cast<int32_t>(nf);
      out.push_back(n);
      SsgNode tail{};
      double w12[2] = {nf > 0 ? w[1] : 0.0, nf > 1 ? w[2] : 0.0};
      std::memcpy(&tail, w12, sizeof w12);
      out.push_back(tail);
    }
  }
  return root;
}

// `invalid` (optional, host-buffer entry points): lowest query index with no
// trained model slot; *flag_f1 set if a two-feature model got no f1 --
// checked here instead of a host pass over every query before the copies.
// `perm` (optional): the queries arrive grouped (k_bucket_scatter); query k of
// the launch is the caller's query perm[k], which is where its answer goes and
// the index any error reports.
__global__ void k_predict(SsgEstView E, int64_t n, const int32_t* __restrict__ slot,
                          int32_t uniform_slot, const double* __restrict__ f0,
                          const double* __restrict__ f1, double* __restrict__ out,
                          unsigned long long* __restrict__ first_error,
                          unsigned long long* __restrict__ invalid,
                          unsigned long long* __restrict__ flag_f1,
                          const int32_t* __restrict__ perm) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += stride) {
    const int64_t i = perm ? (int64_t)__ldg(perm + k) : k;
    const int32_t m = slot ? __ldg(slot + k) : uniform_slot;
    if (invalid) {
      if (m < 0 || m >= E.nmodels) {
        atomicMin(invalid, (unsigned long long)i);
        out[i] = 0.0;
        continue;
      }
      if (!f1 && E.models[m].nf > 1) {
        *flag_f1 = 1ull;
        out[i] = 0.0;
        continue;
      }
    }
    const double v0 = __ldg(f0 + k);
    const double v1 = f1 ? __ldg(f1 + k) : 0.0;
    double r = 0.0;
    int bad = 0;
    const int code = ssg_predict_one(E, m, v0, v1, &r, &bad);
    out[i] = r;
    if (code != SSG_OK) atomicMin(first_error, ((unsigned long long)i << 8) | (unsigned)code);
  }
}

// ---- query grouping for mixed-model launches --------------------------------
// Queries of one model with nearby features walk the same tree nodes, so a
// warp of them shares cache lines and branches (measured: 10M mixed queries
// 8.2 ms as given, 4.4 ms grouped by model x 16 x 16 log-scale feature cells, 4.2 ms by
// 32 x 32; the histograms of 64 x 64 cost more than they save: 5.3 ms).
// A counting sort by that cell: per-block histograms, one scan, a scatter.
// The grouping only reorders work: every query is still answered by the same
// exact evaluation, at its own index.
#ifndef SSG_PRED_SIDE
#define SSG_PRED_SIDE 32  // A/B on cfg #3 (10M queries): 16: 2.27, 32: 2.39, 64: 1.89 G queries/s
#endif
constexpr int kSide = SSG_PRED_SIDE;      // log-scale cells per feature axis
constexpr int kCells = kSide * kSide;     // feature cells per model

__device__ __forceinline__ int feature_cell(double v, double lo, double hi) {
  const float l = log2f(fmaxf((float)lo, 0.f) + 1.f), h = log2f(fmaxf((float)hi, 0.f) + 1.f);
  const float x = log2f(fmaxf((float)v, 0.f) + 1.f);
  const int c = (int)((float)kSide * (x - l) / fmaxf(h - l, 1e-6f));
  return c < 0 ? 0 : (c > kSide - 1 ? kSide - 1 : c);
}

__device__ __forceinline__ int query_bucket(const SsgEstView& E, int32_t m, double v0, double v1,
                                            bool has_f1) {
  if (m < 0 || m >= E.nmodels) return E.nmodels * kCells;  // invalid slots: last bucket
  const SsgModelDesc& d = E.models[m];
  const int c0 = feature_cell(v0, d.lower[0], d.upper[0]);
  const int c1 = (d.nf > 1 && has_f1) ? feature_cell(v1, d.lower[1], d.upper[1]) : 0;
  return m * kCells + c0 * kSide + c1;
}

constexpr int kTile = 4096;  // queries per block in the grouping passes

__global__ void k_bucket_hist(SsgEstView E, int64_t n, const int32_t* __restrict__ slot,
                              const double* __restrict__ f0, const double* __restrict__ f1,
                              int nb, unsigned* __restrict__ hist) {
  extern __shared__ unsigned sh[];
  for (int b = threadIdx.x; b < nb; b += blockDim.x) sh[b] = 0;
  __syncthreads();
  const int64_t t0 = (int64_t)blockIdx.x * kTile;
  const int64_t t1 = t0 + kTile < n ? t0 + kTile : n;
  for (int64_t i = t0 + threadIdx.x; i < t1; i += blockDim.x)
    atomicAdd(&sh[query_bucket(E, __ldg(slot + i), __ldg(f0 + i), f1 ? __ldg(f1 + i) : 0.0, f1)], 1u);
  __syncthreads();
  for (int b = threadIdx.x; b < nb; b += blockDim.x)
    if (sh[b]) atomicAdd(&hist[b], sh[b]);
}

// exclusive scan of the bucket sizes into the scatter cursors (one block)
__global__ void k_bucket_scan(int nb, const unsigned* __restrict__ hist, unsigned* __restrict__ cursor) {
  __shared__ unsigned carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (int base = 0; base < nb; base += blockDim.x) {
    const int b = base + threadIdx.x;
    const unsigned v = b < nb ? hist[b] : 0u;
    // block-wide inclusive scan (warp scans, then the warp totals)
    unsigned x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned y = __shfl_up_sync(0xffffffffu, x, o);
      if ((threadIdx.x & 31) >= o) x += y;
    }
    __shared__ unsigned warp_tot[32];
    if ((threadIdx.x & 31) == 31) warp_tot[threadIdx.x >> 5] = x;
    __syncthreads();
    if (threadIdx.x < 32) {
      unsigned w = threadIdx.x < (blockDim.x >> 5) ? warp_tot[threadIdx.x] : 0u;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const unsigned y = __shfl_up_sync(0xffffffffu, w, o);
        if (threadIdx.x >= o) w += y;
      }
      warp_tot[threadIdx.x] = w;
    }
    __syncthreads();
    const unsigned before = (threadIdx.x >= 32 ? warp_tot[(threadIdx.x >> 5) - 1] : 0u) + x - v;
    if (b < nb) cursor[b] = carry + before;
    __syncthreads();
    if (threadIdx.x == blockDim.x - 1) carry += before + v;
    __syncthreads();
  }
}

__global__ void k_bucket_scatter(SsgEstView E, int64_t n, const int32_t* __restrict__ slot,
                                 const double* __restrict__ f0, const double* __restrict__ f1,
                                 int nb, unsigned* __restrict__ cursor, int32_t* __restrict__ perm,
                                 int32_t* __restrict__ sslot, double* __restrict__ sf0,
                                 double* __restrict__ sf1) {
  extern __shared__ unsigned sh[];
  for (int b = threadIdx.x; b < nb; b += blockDim.x) sh[b] = 0;
  __syncthreads();
  const int64_t t0 = (int64_t)blockIdx.x * kTile;
  const int64_t t1 = t0 + kTile < n ? t0 + kTile : n;
  for (int64_t i = t0 + threadIdx.x; i < t1; i += blockDim.x)
    atomicAdd(&sh[query_bucket(E, __ldg(slot + i), __ldg(f0 + i), f1 ? __ldg(f1 + i) : 0.0, f1)], 1u);
  __syncthreads();
  // reserve this block's range in every bucket it touches
  for (int b = threadIdx.x; b < nb; b += blockDim.x)
    if (sh[b]) sh[b] = atomicAdd(&cursor[b], sh[b]);
  __syncthreads();
  for (int64_t i = t0 + threadIdx.x; i < t1; i += blockDim.x) {
    const int32_t m = __ldg(slot + i);
    const double v0 = __ldg(f0 + i), v1 = f1 ? __ldg(f1 + i) : 0.0;
    const unsigned pos = atomicAdd(&sh[query_bucket(E, m, v0, v1, f1)], 1u);
    perm[pos] = (int32_t)i;
    sslot[pos] = m;
    sf0[pos] = v0;
    if (f1) sf1[pos] = v1;
  }
}

}  // namespace

std::string bbox_error_message(const EstimatorModel::PerOpModel& m, const OpModelKey& key,
                               int f, double v) {
  const double extent = m.bbox_hi[f] - m.bbox_lo[f];
  const double margin = EstimatorModel::kExtrapolationMargin * extent;
  return "estimator: feature " + m.schema[f] + "=" + std::to_string(v) + " for " +
         to_string(key) + " outside extrapolation margin [" +
         std::to_string(m.bbox_lo[f] - margin) + ", " + std::to_string(m.bbox_hi[f] + margin) + "]";
}

// ------------------------------------------------------------------ model
EstimatorModel::EstimatorModel() = default;
EstimatorModel::~EstimatorModel() = default;
EstimatorModel::EstimatorModel(EstimatorModel&&) noexcept = default;
EstimatorModel& EstimatorModel::operator=(EstimatorModel&&) noexcept = default;

const EstimatorModel::PerOpModel& EstimatorModel::find(OpName op, std::int64_t tp) const {
  auto it = models_.find({op, tp});
  require(it != models_.end(), "estimator: no trained model for op " + to_string(OpModelKey{op, tp}) +
                                   " (profile and train must cover the config's operators)");
  return it->second;
}

void EstimatorModel::insert(const OpModelKey& k, PerOpModel m) {
  models_[k] = std::move(m);
  dev_.reset();
}

namespace {

// Flattens one trained regressor into the device pools (interp axes + values
// in dpool; forest trees as preorder 16 B nodes) and fills the descriptor's
// regressor fields; returns the algorithmic bytes of one query:
// features + output, plus interp: 2^nf corner values + binary-search probes
// per axis; forest: per tree, visited nodes x 20 B + the leaf plane.
int64_t flatten_regressor(const RegressorData& r, SsgModelDesc& desc, std::vector<double>& dpool,
                          std::vector<SsgNode>& nodes, std::vector<int32_t>& roots) {
  if (r.type == "interp") {
    desc.kind = SSG_KIND_INTERP;
    internal_check(r.axes.size() == static_cast<std::size_t>(desc.nf),
                   "interp predict: feature count mismatch");
    for (int f = 0; f < desc.nf; ++f) {
      desc.axis_len[f] = static_cast<int32_t>(r.axes[f].size());
      desc.axis_off[f] = static_cast<int64_t>(dpool.size());
      dpool.insert(dpool.end(), r.axes[f].begin(), r.axes[f].end());
    }
    desc.values_off = static_cast<int64_t>(dpool.size());
    dpool.insert(dpool.end(), r.values.begin(), r.values.end());
  } else {
    desc.kind = SSG_KIND_FOREST;
    internal_check(r.num_features == static_cast<std::size_t>(desc.nf),
                   "forest predict: feature count mismatch");
    desc.ntrees = static_cast<int32_t>(r.trees.size());
    desc.roots_off = static_cast<int64_t>(roots.size());
    desc.y_lo = r.y_lo;
    desc.y_hi = r.y_hi;
    for (const auto& t : r.trees) roots.push_back(append_tree(t, r.num_features, nodes));
  }
  int64_t qb = 8 * desc.nf + 8;
  if (desc.kind == SSG_KIND_INTERP) {
    qb += 8 * (int64_t(1) << desc.nf);
    for (int f = 0; f < desc.nf; ++f)
      qb += 8 * static_cast<int64_t>(std::ceil(std::log2(std::max(1, desc.axis_len[f]))));
  } else {
    for (const auto& t : r.trees) {
      // mean internal-node depth of the tree's leaves
      std::vector<std::pair<int, int>> st{{0, 0}};
      double sum = 0.0;
      int leaves = 0;
      while (!st.empty()) {
        auto [node, depth] = st.back();
        st.pop_back();
        if (t.feature[node] >= 0) {
          st.push_back({t.left[node], depth + 1});
          st.push_back({t.right[node], depth + 1});
        } else {
          sum += depth;
          ++leaves;
        }
      }
      qb += static_cast<int64_t>(std::llround(20.0 * sum / std::max(1, leaves))) + 8 * (desc.nf + 1);
    }
  }
  return qb;
}

// Uploads the pools (each kept non-empty so the view never carries null pointers).
void upload_pools(DeviceEstimator& d, std::vector<double>& dpool, std::vector<SsgNode>& nodes,
                  std::vector<int32_t>& roots) {
  auto& ctx = ssg::context();
  internal_check(nodes.size() < (1u << 31), "forest: node pool exceeds int32 addressing");
  if (dpool.empty()) dpool.push_back(0.0);
  if (nodes.empty()) nodes.push_back(SsgNode{});
  if (roots.empty()) roots.push_back(0);
  d.models.upload(d.host_models, ctx.stream);
  d.dpool.upload(dpool, ctx.stream);
  d.nodes.upload(nodes, ctx.stream);
  d.roots.upload(roots, ctx.stream);
  ssg::cuda_check(cudaStreamSynchronize(ctx.stream), "estimator upload");
  d.bytes = d.host_models.size() * sizeof(SsgModelDesc) + dpool.size() * 8 +
            nodes.size() * sizeof(SsgNode) + roots.size() * 4;
  d.view.models = d.models.ptr;
  d.view.dpool = d.dpool.ptr;
  d.view.nodes = d.nodes.ptr;
#if SSG_FOREST_SOA
  {
    std::vector<double> a(nodes.size());
    std::vector<int2> fr(nodes.size());
    for (std::size_t i = 0; i < nodes.size(); ++i) {
      a[i] = nodes[i].a;
      fr[i] = make_int2(nodes[i].feat, nodes[i].right);
    }
    d.node_a.upload(a, ctx.stream);
    d.node_fr.upload(fr, ctx.stream);
    ssg::cuda_check(cudaStreamSynchronize(ctx.stream), "SoA upload");
    d.view.node_a = d.node_a.ptr;
    d.view.node_fr = d.node_fr.ptr;
  }
#endif
  d.view.roots = d.roots.ptr;
  d.view.nmodels = static_cast<int32_t>(d.host_models.size());
  d.view.math_fma = ctx.math_fma;
}

// Regressor::predict: the raw regressor output over already-transformed
// features (no guard, no exp), by the same device code as the predictor.
__global__ void k_regress(SsgEstView E, const double* x, double* out) {
  const SsgModelDesc& m = E.models[0];
  const double x1 = m.nf > 1 ? x[1] : 0.0;
  out[0] = m.kind == SSG_KIND_FOREST ? ssg_forest(E, m, x[0], x1) : ssg_interp(E, m, x[0], x1);
}

}  // namespace

struct DeviceRegressor {
  DeviceEstimator est;
};

double Regressor::predict(std::span<const double> x) const {
  auto& ctx = ssg::context();
  static std::mutex upload_mu;  // the first call uploads; predict is const and callable concurrently
  std::unique_lock<std::mutex> up(upload_mu);
  if (!dev_) {
    auto d = std::make_shared<DeviceRegressor>();
    SsgModelDesc desc{};
    desc.nf = static_cast<int32_t>(data_.type == "forest" ? data_.num_features : data_.axes.size());
    internal_check(desc.nf >= 1 && desc.nf <= 2, "regressor upload: models take 1 or 2 features");
    std::vector<double> dpool;
    std::vector<SsgNode> nodes;
    std::vector<int32_t> roots;
    d->est.qbytes.push_back(flatten_regressor(data_, desc, dpool, nodes, roots));
    d->est.host_models.push_back(desc);
    upload_pools(d->est, dpool, nodes, roots);
    dev_ = std::move(d);
  }
  std::shared_ptr<DeviceRegressor> dr = dev_;
  up.unlock();
  const int nf = dr->est.host_models[0].nf;
  internal_check(x.size() >= static_cast<std::size_t>(nf), "regressor predict: feature count mismatch");
  DeviceEstimator& de = dr->est;
  std::lock_guard<std::mutex> lk(de.one_mu);
  if (!de.one_host) {
    ssg::cuda_check(cudaMallocHost(reinterpret_cast<void**>(&de.one_host), 4 * sizeof(double)), "pinned");
    de.one_dev.resize(4);
  }
  double* h = de.one_host;
  h[0] = x[0];
  h[1] = nf > 1 ? x[1] : 0.0;
  ssg::cuda_check(cudaMemcpyAsync(de.one_dev.ptr, h, 2 * sizeof(double), cudaMemcpyHostToDevice, ctx.stream), "H2D");
  k_regress<<<1, 1, 0, ctx.stream>>>(de.view, de.one_dev.ptr, de.one_dev.ptr + 2);
  ssg::cuda_check(cudaGetLastError(), "k_regress launch");
  ssg::cuda_check(cudaMemcpyAsync(h + 2, de.one_dev.ptr + 2, sizeof(double), cudaMemcpyDeviceToHost, ctx.stream), "D2H");
  ssg::cuda_check(cudaStreamSynchronize(ctx.stream), "regressor predict");
  return h[2];
}

const DeviceEstimator& EstimatorModel::device() const {
  if (dev_) return *dev_;
  auto d = std::make_unique<DeviceEstimator>();
  std::vector<double> dpool;
  std::vector<SsgNode> nodes;
  std::vector<int32_t> roots;
  for (const auto& [key, m] : models_) {
    SsgModelDesc desc{};
    desc.op = static_cast<int32_t>(key.op);
    desc.tp = static_cast<int32_t>(key.tp_degree);
    desc.nf = static_cast<int32_t>(m.schema.size());
    internal_check(desc.nf >= 1 && desc.nf <= 2, "estimator upload: models take 1 or 2 features");
    for (int f = 0; f < desc.nf; ++f) {
      const double extent = m.bbox_hi[f] - m.bbox_lo[f];
      const double margin = kExtrapolationMargin * extent;
      desc.lower[f] = m.bbox_lo[f] - margin;
      desc.upper[f] = m.bbox_hi[f] + margin;
    }
    internal_check(m.regressor != nullptr, "estimator upload: model without a regressor");
    const int64_t qb = flatten_regressor(m.regressor->data(), desc, dpool, nodes, roots);
    if (desc.kind == SSG_KIND_FOREST) d->has_forest = true;
    d->qbytes.push_back(qb);
    d->index[key] = static_cast<int32_t>(d->host_models.size());
    d->host_models.push_back(desc);
  }
  upload_pools(*d, dpool, nodes, roots);
  dev_ = std::move(d);
  return *dev_;
}

}  // namespace servesim

namespace ssg {

using namespace servesim;

// Launch on device pointers (no synchronisation).  `first_error` must hold
// SSG_NO_ERROR on entry.
void launch_predict(const DeviceEstimator& de, int64_t n, const int32_t* slots, int32_t uniform,
                    const double* f0, const double* f1, double* out,
                    unsigned long long* first_error, cudaStream_t s, unsigned long long* invalid,
                    unsigned long long* flag_f1) {
  if (n <= 0) return;
  auto& ctx = context();
  const int threads = 256;
  int64_t blocks = (n + threads - 1) / threads;
  const int64_t cap = static_cast<int64_t>(ctx.num_sms) * 8;  // 8 x 256 threads resident per SM
  if (blocks > cap) blocks = cap;
  const int nb = de.view.nmodels * kCells + 1;
  constexpr size_t kSmemMax = 200 * 1024;  // per-block bucket histograms (opt-in above 48 KB)
  const bool group = slots && n >= (1 << 16) && n < INT32_MAX &&
                     nb * sizeof(unsigned) <= kSmemMax && std::getenv("SSG_NO_GROUPING") == nullptr;
  static const bool smem_attr = [] {
    cuda_check(cudaFuncSetAttribute(k_bucket_hist, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    static_cast<int>(kSmemMax)), "smem attr");
    cuda_check(cudaFuncSetAttribute(k_bucket_scatter, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    static_cast<int>(kSmemMax)), "smem attr");
    return true;
  }();
  (void)smem_attr;
  if (group) {
    // scratch on the launch stream (stream-ordered pool: freed behind the kernels)
    StreamScope scope(s);
    DeviceBuffer<unsigned> hist(nb), cursor(nb);
    DeviceBuffer<int32_t> perm(n), sslot(n);
    DeviceBuffer<double> sf0(n), sf1(f1 ? n : 1);
    cuda_check(cudaMemsetAsync(hist.ptr, 0, nb * sizeof(unsigned), s), "memset");
    const unsigned tiles = static_cast<unsigned>((n + kTile - 1) / kTile);
    const size_t smem = nb * sizeof(unsigned);
    k_bucket_hist<<<tiles, 256, smem, s>>>(de.view, n, slots, f0, f1, nb, hist.ptr);
    k_bucket_scan<<<1, 1024, 0, s>>>(nb, hist.ptr, cursor.ptr);
    k_bucket_scatter<<<tiles, 256, smem, s>>>(de.view, n, slots, f0, f1, nb, cursor.ptr, perm.ptr,
                                              sslot.ptr, sf0.ptr, f1 ? sf1.ptr : nullptr);
    k_predict<<<static_cast<unsigned>(blocks), threads, 0, s>>>(
        de.view, n, sslot.ptr, uniform, sf0.ptr, f1 ? sf1.ptr : nullptr, out, first_error, invalid,
        flag_f1, perm.ptr);
    cuda_check(cudaGetLastError(), "k_predict launch");
    stats().launches_setup += 3;
  } else {
    k_predict<<<static_cast<unsigned>(blocks), threads, 0, s>>>(de.view, n, slots, uniform, f0, f1,
                                                                out, first_error, invalid, flag_f1,
                                                                nullptr);
    cuda_check(cudaGetLastError(), "k_predict launch");
  }
  stats().launches_predict += 1;
  stats().queries += n;
}

// Turns the packed first-error word into the reference's exception.
[[noreturn]] void raise_predict_error(const EstimatorModel& est, unsigned long long word,
                                      const int32_t* slots_host, int32_t uniform,
                                      const double* f0_host, const double* f1_host) {
  const auto& de = est.device();
  const int64_t i = static_cast<int64_t>(word >> 8);
  const int code = static_cast<int>(word & 0xff);
  const int32_t slot = slots_host ? slots_host[i] : uniform;
  const SsgModelDesc& d = de.host_models.at(slot);
  const OpModelKey key{static_cast<OpName>(d.op), d.tp};
  if (code == SSG_ERR_BBOX) {
    const auto& m = est.find(key.op, key.tp_degree);
    const double v0 = f0_host[i];
    const bool first_bad = !(v0 >= d.lower[0] && v0 <= d.upper[0]);
    const int f = first_bad ? 0 : 1;
    throw Error(bbox_error_message(m, key, f, f == 0 ? v0 : f1_host[i]));
  }
  throw InternalError("predict: regressor output outside exp range for " + to_string(key));
}

}  // namespace ssg

namespace servesim {

namespace {
// One EstimatorModel::predict query: {v0, v1} in, {runtime, status code} out.
__global__ void k_predict_one(SsgEstView E, int32_t slot, const double* in, double* out) {
  double r = 0.0;
  int bad = 0;
  const int code = ssg_predict_one(E, slot, in[0], in[1], &r, &bad);
  out[0] = r;
  out[1] = (double)code;
}
}  // namespace

DeviceEstimator::~DeviceEstimator() {
  if (one_host) cudaFreeHost(one_host);
}

double EstimatorModel::predict(OpName op, std::int64_t tp, const FeatureMap& features) const {
  const PerOpModel& m = find(op, tp);
  double v[2] = {0.0, 0.0};
  for (std::size_t f = 0; f < m.schema.size(); ++f) {
    auto it = features.find(m.schema[f]);
    require(it != features.end(), "estimator: query for " + to_string(OpModelKey{op, tp}) +
                                      " missing feature " + m.schema[f]);
    v[f] = it->second;
  }
  auto& de = const_cast<DeviceEstimator&>(device());
  auto& ctx = ssg::context();
  const int32_t slot = de.slot(op, tp);
  // a single query is latency: one 16 B copy in, one launch, one 16 B copy out,
  // through buffers the estimator keeps (pinned host + HBM), one caller at a time
  std::lock_guard<std::mutex> lk(de.one_mu);
  if (!de.one_host) {
    ssg::cuda_check(cudaMallocHost(reinterpret_cast<void**>(&de.one_host), 4 * sizeof(double)), "pinned");
    de.one_dev.resize(4);
  }
  double* h = de.one_host;
  h[0] = v[0];
  h[1] = v[1];
  ssg::cuda_check(cudaMemcpyAsync(de.one_dev.ptr, h, 2 * sizeof(double), cudaMemcpyHostToDevice, ctx.stream), "H2D");
  k_predict_one<<<1, 1, 0, ctx.stream>>>(de.view, slot, de.one_dev.ptr, de.one_dev.ptr + 2);
  ssg::cuda_check(cudaGetLastError(), "k_predict_one launch");
  ssg::cuda_check(cudaMemcpyAsync(h + 2, de.one_dev.ptr + 2, 2 * sizeof(double), cudaMemcpyDeviceToHost, ctx.stream), "D2H");
  ssg::cuda_check(cudaStreamSynchronize(ctx.stream), "predict");
  ssg::stats().launches_predict += 1;
  ssg::stats().queries += 1;
  const int code = static_cast<int>(h[3]);
  if (code != SSG_OK) ssg::raise_predict_error(*this, static_cast<unsigned long long>(code), nullptr, slot, v, v + 1);
  return h[2];
}

}  // namespace servesim
