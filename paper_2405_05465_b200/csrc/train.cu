// train.cu -- K6: random-forest estimator build on sm_100a, one warp per tree.
//
// reference: regressor.hpp:82-101 (train), 158-191 (build_node), 193-232
//            (find_random_split), 234-254 (fit_leaf), 42-67 (solve_linear)
//
// The forest of every (op, tp) model of a training call -- and the hold-out
// probe forests -- grow in one launch: 48 trees per forest, each tree one warp.
// Bit-identical to the reference because every order-dependent step keeps the
// reference's order:
//   * the tree's mt19937_64 stream (seed * 0x9e3779b97f4a7c15 + t + 1) is
//     consumed by lane 0 in the reference's order -- nodes in preorder, then
//     feature, then draw -- through libstdc++'s generate_canonical<double, 53>
//     (one 64-bit draw, round-to-nearest to double, / 2^64);
//   * fp64 sums (node total, each candidate's left sum, each normal-equation
//     entry, the fallback mean) run sequentially over the node's samples in
//     their reference order, one lane per independent sum;
//   * the best split is chosen in (feature, draw) order with the reference's
//     `score > best + 1e-15` rule; the plane solve is the reference's
//     elimination with partial pivoting, on lane 0;
//   * the node's samples are split by a stable (ballot-ranked) partition, so
//     child sample orders equal the reference's push_back order.
// Order-free steps run across the warp: per-feature min / max of the node's
// samples, the candidate evaluations (one lane per candidate), the partition.
// Device code is built with --fmad=false, so a*b+c is never contracted.
#include <cmath>

#include "runtime.h"
#include "train.h"

namespace ssgk {

struct FJob {
  int64_t x0, x1, y;  // offsets into the double pool (x1 < 0: one feature)
  int32_t n, nf, max_depth, min_leaf, draws, pad;
  uint64_t seed;
};
struct TJob {
  int32_t job, tree, node_cap, leaf_cap;
  int64_t idx_off, node_off, leaf_off;
};
struct TOut {
  int32_t nnodes, nleaves, status, pad;
};

constexpr int kMaxDepthStack = 70;  // max_depth <= 64 (host check): stack <= depth + 2
constexpr int kMaxCand = 32;        // nf * threshold_draws <= 32 (host check)

struct TreeSmem {
  uint64_t mt[312];
  int32_t mti, sp;
  int32_t st_off[kMaxDepthStack], st_len[kMaxDepthStack], st_depth[kMaxDepthStack];
  int32_t st_parent[kMaxDepthStack], st_side[kMaxDepthStack];
  double cand_th[kMaxCand];
  int32_t cand_f[kMaxCand];
};

// std::mt19937_64 (libstdc++ mersenne_twister_engine parameters)
__device__ __forceinline__ void mt_seed(TreeSmem& g, uint64_t s) {
  g.mt[0] = s;
  for (int i = 1; i < 312; ++i) g.mt[i] = 6364136223846793005ULL * (g.mt[i - 1] ^ (g.mt[i - 1] >> 62)) + (uint64_t)i;
  g.mti = 312;
}
__device__ __forceinline__ uint64_t mt_next(TreeSmem& g) {
  if (g.mti >= 312) {
    const uint64_t up = ~0ULL << 31, low = ~up, a = 0xb5026f5aa96619e9ULL;
    for (int k = 0; k < 312; ++k) {
      const uint64_t y = (g.mt[k] & up) | (g.mt[(k + 1) % 312] & low);
      g.mt[k] = g.mt[(k + 156) % 312] ^ (y >> 1) ^ ((y & 1ULL) ? a : 0ULL);
    }
    g.mti = 0;
  }
  uint64_t z = g.mt[g.mti++];
  z ^= (z >> 29) & 0x5555555555555555ULL;
  z ^= (z << 17) & 0x71d67fffeda60000ULL;
  z ^= (z << 37) & 0xfff7eee000000000ULL;
  z ^= (z >> 43);
  return z;
}
// uniform_real_distribution<double>(0, 1) = generate_canonical<double, 53>
__device__ __forceinline__ double mt_canonical(TreeSmem& g) {
  const double s = __ull2double_rn(mt_next(g));
  double r = s / 18446744073709551616.0;  // exact: a power of two
  if (r >= 1.0) r = nextafter(1.0, 0.0);
  return r;
}

__device__ __forceinline__ double xval(const double* x0, const double* x1, int f, int32_t i) {
  return f ? x1[i] : x0[i];
}

__global__ void __launch_bounds__(32) k_grow_trees(const FJob* __restrict__ jobs,
                                                   const TJob* __restrict__ trees, int ntrees,
                                                   const double* __restrict__ pool,
                                                   int32_t* __restrict__ idxbuf, int32_t* __restrict__ tmpbuf,
                                                   int32_t* __restrict__ feat, double* __restrict__ thr,
                                                   int32_t* __restrict__ left, int32_t* __restrict__ right,
                                                   double* __restrict__ leafw, TOut* __restrict__ out) {
  __shared__ TreeSmem S;
  const int g = blockIdx.x;
  if (g >= ntrees) return;
  const int lane = threadIdx.x;
  const TJob T = trees[g];
  const FJob J = jobs[T.job];
  const double* x0 = pool + J.x0;
  const double* x1 = J.nf > 1 ? pool + J.x1 : x0;
  const double* y = pool + J.y;
  int32_t* idx = idxbuf + T.idx_off;
  int32_t* tmp = tmpbuf + T.idx_off;
  int32_t* F = feat + T.node_off;
  double* TH = thr + T.node_off;
  int32_t* Lc = left + T.node_off;
  int32_t* Rc = right + T.node_off;
  double* W = leafw + T.leaf_off;
  const int dim = J.nf + 1;
#pragma unroll 1
  for (int32_t k = lane; k < J.n; k += 32) idx[k] = k;
  if (lane == 0) {
    mt_seed(S, J.seed * 0x9e3779b97f4a7c15ULL + (uint64_t)T.tree + 1ULL);
    S.sp = 1;
    S.st_off[0] = 0;
    S.st_len[0] = J.n;
    S.st_depth[0] = 0;
    S.st_parent[0] = -1;
    S.st_side[0] = 0;
  }
  __syncwarp();
  int nn = 0, nleaves = 0, status = 0;
  while (true) {
    __syncwarp();
    const int sp = S.sp;
    if (sp == 0) break;
    const int32_t off = S.st_off[sp - 1], len = S.st_len[sp - 1], depth = S.st_depth[sp - 1];
    const int32_t parent = S.st_parent[sp - 1], side = S.st_side[sp - 1];
    __syncwarp();
    if (lane == 0) S.sp = sp - 1;
    const int node = nn++;  // preorder numbering (build_node's t.feature.size())
    if (node >= T.node_cap) {
      status = 1;
      break;
    }
    if (lane == 0) {
      F[node] = 0;
      TH[node] = 0.0;
      Lc[node] = -1;
      Rc[node] = -1;
      if (parent >= 0) (side ? Rc : Lc)[parent] = node;
    }
    int split_f = -1, split_nl = 0;
    double split_th = 0.0;
    if (depth < J.max_depth && len >= 2 * J.min_leaf) {
      // ---- find_random_split
      double total = 0.0;
      if (lane == 0)
#pragma unroll 1
        for (int32_t k = 0; k < len; ++k) total = __dadd_rn(total, y[idx[off + k]]);
      total = __shfl_sync(0xffffffffu, total, 0);
      int nc = 0;
      for (int f = 0; f < J.nf; ++f) {
        double lo = xval(x0, x1, f, idx[off]), hi = lo;
#pragma unroll 1
        for (int32_t k = lane; k < len; k += 32) {
          const double v = xval(x0, x1, f, idx[off + k]);
          lo = v < lo ? v : lo;
          hi = hi < v ? v : hi;
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          const double a = __shfl_xor_sync(0xffffffffu, lo, o), b = __shfl_xor_sync(0xffffffffu, hi, o);
          lo = a < lo ? a : lo;
          hi = hi < b ? b : hi;
        }
        if (lo == hi) continue;  // no draws consumed for a constant feature
        if (lane == 0)
          for (int d = 0; d < J.draws; ++d) {
            const double c = mt_canonical(S);
            S.cand_th[nc + d] = __dadd_rn(lo, __dmul_rn(__dsub_rn(hi, lo), c));
            S.cand_f[nc + d] = f;
          }
        nc += J.draws;
      }
      __syncwarp();
      // each candidate's left count and left sum, one lane per candidate
      int32_t cnl = 0;
      double cls = 0.0;
      if (lane < nc) {
        const int f = S.cand_f[lane];
        const double th = S.cand_th[lane];
#pragma unroll 1
        for (int32_t k = 0; k < len; ++k) {
          const int32_t i = idx[off + k];
          if (xval(x0, x1, f, i) <= th) {
            ++cnl;
            cls = __dadd_rn(cls, y[i]);
          }
        }
      }
      // best valid candidate in (feature, draw) order (warp-uniform)
      double best = -1.0;
      for (int c = 0; c < nc; ++c) {
        const int32_t nl = __shfl_sync(0xffffffffu, cnl, c);
        const double ls = __shfl_sync(0xffffffffu, cls, c);
        const int32_t nr = len - nl;
        if (nl < J.min_leaf || nr < J.min_leaf) continue;
        const double rs = __dsub_rn(total, ls);
        const double score = __dadd_rn(__ddiv_rn(__dmul_rn(ls, ls), (double)nl),
                                       __ddiv_rn(__dmul_rn(rs, rs), (double)nr));
        if (score > __dadd_rn(best, 1e-15)) {
          best = score;
          split_f = S.cand_f[c];
          split_th = S.cand_th[c];
          split_nl = nl;
        }
      }
    }
    if (split_f < 0) {
      // ---- leaf: least-squares plane (normal equations, one lane per entry)
      const int leaf = nleaves++;
      if (leaf >= T.leaf_cap) {
        status = 2;
        break;
      }
      const int na = dim * dim;
      double acc = 0.0;
      if (lane < na + dim) {
        const int r = lane < na ? lane / dim : lane - na;
        const int c = lane < na ? lane % dim : -1;
#pragma unroll 1
        for (int32_t k = 0; k < len; ++k) {
          const int32_t i = idx[off + k];
          const double rr = r == 0 ? 1.0 : xval(x0, x1, r - 1, i);
          const double cc = c < 0 ? y[i] : (c == 0 ? 1.0 : xval(x0, x1, c - 1, i));
          acc = __dadd_rn(acc, __dmul_rn(rr, cc));
        }
      }
      double a[9], b[3];
      for (int q = 0; q < na; ++q) a[q] = __shfl_sync(0xffffffffu, acc, q);
      for (int q = 0; q < dim; ++q) b[q] = __shfl_sync(0xffffffffu, acc, na + q);
      if (lane == 0) {
        const int n = dim;
        for (int i = 0; i < n; ++i) a[i * n + i] = __dadd_rn(a[i * n + i], 1e-9);
        bool ok = true;
        for (int col = 0; col < n && ok; ++col) {
          int piv = col;
          for (int r = col + 1; r < n; ++r)
            if (fabs(a[r * n + col]) > fabs(a[piv * n + col])) piv = r;
          if (fabs(a[piv * n + col]) < 1e-30) {
            ok = false;
            break;
          }
          if (piv != col) {
            for (int c = 0; c < n; ++c) {
              const double t = a[piv * n + c];
              a[piv * n + c] = a[col * n + c];
              a[col * n + c] = t;
            }
            const double t = b[piv];
            b[piv] = b[col];
            b[col] = t;
          }
          for (int r = col + 1; r < n; ++r) {
            const double m = __ddiv_rn(a[r * n + col], a[col * n + col]);
            for (int c = col; c < n; ++c) a[r * n + c] = __dsub_rn(a[r * n + c], __dmul_rn(m, a[col * n + c]));
            b[r] = __dsub_rn(b[r], __dmul_rn(m, b[col]));
          }
        }
        double w[3] = {0.0, 0.0, 0.0};
        if (ok) {
          for (int i = n - 1; i >= 0; --i) {
            double s = b[i];
            for (int c = i + 1; c < n; ++c) s = __dsub_rn(s, __dmul_rn(a[i * n + c], w[c]));
            w[i] = __ddiv_rn(s, a[i * n + i]);
          }
        } else {
          double m = 0.0;
          for (int32_t k = 0; k < len; ++k) m = __dadd_rn(m, y[idx[off + k]]);
          w[0] = __ddiv_rn(m, (double)len);
        }
        for (int q = 0; q < n; ++q) W[(int64_t)leaf * n + q] = w[q];
        F[node] = -leaf - 1;
      }
      continue;
    }
    // ---- stable partition of the node's samples: [x <= th | x > th]
    int32_t seen_l = 0, seen_r = 0;
#pragma unroll 1
    for (int32_t base = 0; base < len; base += 32) {
      const int32_t k = base + lane;
      const bool valid = k < len;
      const int32_t i = valid ? idx[off + k] : 0;
      const bool goes_left = valid && xval(x0, x1, split_f, i) <= split_th;
      const unsigned lm = __ballot_sync(0xffffffffu, goes_left);
      const unsigned vm = __ballot_sync(0xffffffffu, valid);
      const unsigned below = (1u << lane) - 1u;
      if (valid) {
        if (goes_left)
          tmp[off + seen_l + __popc(lm & below)] = i;
        else
          tmp[off + split_nl + seen_r + __popc(vm & ~lm & below)] = i;
      }
      seen_l += __popc(lm);
      seen_r += __popc(vm & ~lm);
    }
    __syncwarp();
#pragma unroll 1
    for (int32_t k = lane; k < len; k += 32) idx[off + k] = tmp[off + k];
    if (lane == 0) {
      F[node] = split_f;
      TH[node] = split_th;
      // right child below the left one: the left subtree is built first
      int s = S.sp;
      S.st_off[s] = off + split_nl;
      S.st_len[s] = len - split_nl;
      S.st_depth[s] = depth + 1;
      S.st_parent[s] = node;
      S.st_side[s] = 1;
      ++s;
      S.st_off[s] = off;
      S.st_len[s] = split_nl;
      S.st_depth[s] = depth + 1;
      S.st_parent[s] = node;
      S.st_side[s] = 0;
      S.sp = s + 1;
    }
    __syncwarp();
  }
  if (lane == 0) out[g] = TOut{nn, nleaves, status, 0};
}

}  // namespace ssgk

namespace ssg {

using namespace servesim;

std::vector<RegressorData> grow_forests(const std::vector<ForestFit>& fits) {
  PhaseTimer timer("train: grow_forests (device)");
  auto& ctx = context();
  cudaStream_t s = ctx.stream;
  std::vector<ssgk::FJob> jobs;
  std::vector<ssgk::TJob> trees;
  std::vector<double> pool;
  std::vector<RegressorData> out(fits.size());
  int64_t idx_words = 0, node_words = 0, leaf_words = 0;
  for (std::size_t j = 0; j < fits.size(); ++j) {
    const auto& x = *fits[j].x;
    const auto& y = *fits[j].y;
    const ForestConfig& cfg = fits[j].cfg;
    require(!x.empty() && x.size() == y.size(), "forest train: empty or mismatched data");
    const std::size_t nf = x.front().size();
    internal_check(nf >= 1 && nf <= 2, "forest train: models take 1 or 2 features");
    internal_check(x.size() < (std::size_t(1) << 30), "forest train: too many samples");
    require(cfg.max_depth <= 64, "ssg: forest max_depth above the device trainer limit (64)");
    require(cfg.threshold_draws >= 0 && cfg.threshold_draws * static_cast<int>(nf) <= ssgk::kMaxCand,
            "ssg: forest threshold_draws above the device trainer limit");
    RegressorData& f = out[j];
    f.type = "forest";
    f.num_features = nf;
    f.y_lo = *std::min_element(y.begin(), y.end());
    f.y_hi = *std::max_element(y.begin(), y.end());
    const double pad = 0.1 * (f.y_hi - f.y_lo);
    f.y_lo -= pad;
    f.y_hi += pad;
    ssgk::FJob J{};
    J.n = static_cast<int32_t>(x.size());
    J.nf = static_cast<int32_t>(nf);
    J.max_depth = cfg.max_depth;
    J.min_leaf = cfg.min_samples_leaf > 0 ? cfg.min_samples_leaf : (nf <= 1 ? 2 : static_cast<int>(nf) + 2);
    J.draws = cfg.threshold_draws;
    J.seed = cfg.seed;
    J.x0 = static_cast<int64_t>(pool.size());
    for (const auto& row : x) pool.push_back(row[0]);
    J.x1 = -1;
    if (nf > 1) {
      J.x1 = static_cast<int64_t>(pool.size());
      for (const auto& row : x) pool.push_back(row[1]);
    }
    J.y = static_cast<int64_t>(pool.size());
    pool.insert(pool.end(), y.begin(), y.end());
    // every leaf of a split holds >= min_leaf samples: leaves <= n / min_leaf
    const int32_t leaves = std::max<int32_t>(1, J.n / std::max(1, J.min_leaf)) + 1;
    for (int t = 0; t < cfg.num_trees; ++t) {
      ssgk::TJob T{};
      T.job = static_cast<int32_t>(jobs.size());
      T.tree = t;
      T.node_cap = 2 * leaves + 1;
      T.leaf_cap = leaves;
      T.idx_off = idx_words;
      idx_words += J.n;
      T.node_off = node_words;
      node_words += T.node_cap;
      T.leaf_off = leaf_words;
      leaf_words += static_cast<int64_t>(T.leaf_cap) * (J.nf + 1);
      trees.push_back(T);
    }
    jobs.push_back(J);
  }
  const int ntrees = static_cast<int>(trees.size());
  if (ntrees == 0) return out;
  DeviceBuffer<ssgk::FJob> d_jobs;
  DeviceBuffer<ssgk::TJob> d_trees;
  DeviceBuffer<double> d_pool, d_thr(node_words), d_leaf(std::max<int64_t>(1, leaf_words));
  DeviceBuffer<int32_t> d_idx(idx_words), d_tmp(idx_words), d_feat(node_words), d_left(node_words),
      d_right(node_words);
  DeviceBuffer<ssgk::TOut> d_out(ntrees);
  d_jobs.upload(jobs, s);
  d_trees.upload(trees, s);
  d_pool.upload(pool, s);
  ssgk::k_grow_trees<<<ntrees, 32, 0, s>>>(d_jobs.ptr, d_trees.ptr, ntrees, d_pool.ptr, d_idx.ptr, d_tmp.ptr,
                                           d_feat.ptr, d_thr.ptr, d_left.ptr, d_right.ptr, d_leaf.ptr,
                                           d_out.ptr);
  cuda_check(cudaGetLastError(), "k_grow_trees launch");
  stats().launches_setup += 1;
  std::vector<ssgk::TOut> res(ntrees);
  std::vector<int32_t> feat(node_words), lft(node_words), rgt(node_words);
  std::vector<double> thr(node_words), leaf(std::max<int64_t>(1, leaf_words));
  d_out.download(res.data(), ntrees, s);
  d_feat.download(feat.data(), node_words, s);
  d_left.download(lft.data(), node_words, s);
  d_right.download(rgt.data(), node_words, s);
  d_thr.download(thr.data(), node_words, s);
  d_leaf.download(leaf.data(), leaf.size(), s);
  cuda_check(cudaStreamSynchronize(s), "grow forests");
  for (int g = 0; g < ntrees; ++g) {
    const ssgk::TJob& T = trees[g];
    const ssgk::FJob& J = jobs[T.job];
    internal_check(res[g].status == 0, "forest train: device tree buffer overflow");
    ForestTree t;
    const int32_t nn = res[g].nnodes, nl = res[g].nleaves;
    t.feature.assign(feat.begin() + T.node_off, feat.begin() + T.node_off + nn);
    t.threshold.assign(thr.begin() + T.node_off, thr.begin() + T.node_off + nn);
    t.left.assign(lft.begin() + T.node_off, lft.begin() + T.node_off + nn);
    t.right.assign(rgt.begin() + T.node_off, rgt.begin() + T.node_off + nn);
    for (int32_t l = 0; l < nl; ++l) {
      const double* w = leaf.data() + T.leaf_off + static_cast<int64_t>(l) * (J.nf + 1);
      t.leaf_weights.emplace_back(w, w + J.nf + 1);
    }
    out[T.job].trees.push_back(std::move(t));
  }
  return out;
}

}  // namespace ssg
