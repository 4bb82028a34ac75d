// predictor.cuh -- device evaluation of one trained operator predictor.
//
//   t = exp( regressor( log1p(v_0), log1p(v_1) ) )     after the bbox guard
//
// reference: estimator.hpp:105-123 (guard, log1p, exp),
//            regressor.hpp:103-108,256-264 (forest), 308-341 (interp)
//
// One thread evaluates one query.  The forest walks FOREST_ILP trees at once
// so a thread keeps several independent 16-byte node loads in flight; the
// clamped leaf values are still added in tree order, which is what makes the
// fp64 sum bit-identical to the reference's sequential loop.
#pragma once
#include "glibc_math.h"
#include "ssg_device.h"

#ifndef FOREST_ILP
#define FOREST_ILP 4
#endif

__device__ __forceinline__ double ssg_clamp(double v, double lo, double hi) {
  // std::clamp(v, lo, hi): (v < lo) ? lo : (hi < v) ? hi : v
  return (v < lo) ? lo : ((hi < v) ? hi : v);
}

__device__ __forceinline__ double2 ssg_ld_node(const SsgNode* nodes, int32_t i) {
  return __ldg(reinterpret_cast<const double2*>(nodes) + i);
}
__device__ __forceinline__ int32_t ssg_node_feat(double2 n) {
  return (int32_t)(uint32_t)(unsigned long long)__double_as_longlong(n.y);
}
__device__ __forceinline__ int32_t ssg_node_right(double2 n) {
  return (int32_t)((unsigned long long)__double_as_longlong(n.y) >> 32);
}

#ifndef SSG_FOREST_SOA
#define SSG_FOREST_SOA 0  // 1: walk SoA node arrays (two 8 B loads per node) -- A/B build only
#endif
// One node (or a leaf's weight tail) of the forest pool.
__device__ __forceinline__ double2 ssg_ld_node_v(const SsgEstView& E, int32_t i) {
#if SSG_FOREST_SOA
  const double a = __ldg(E.node_a + i);
  const int2 fr = __ldg(E.node_fr + i);
  return make_double2(a, __longlong_as_double((long long)(((unsigned long long)(unsigned)fr.y << 32) |
                                                          (unsigned)fr.x)));
#else
  return ssg_ld_node(E.nodes, i);
#endif
}

// Cell of one axis: lo index and clamped fraction (regressor.hpp:314-325).
__device__ __forceinline__ void ssg_axis_cell(const double* __restrict__ ax, int32_t n, double x,
                                              int32_t* lo, double* frac) {
  if (n == 1) {
    *lo = 0;
    *frac = 0.0;
    return;
  }
  // std::upper_bound: first level strictly greater than x
  int32_t first = 0, count = n;
  while (count > 0) {
    const int32_t step = count >> 1;
    if (!(x < __ldg(ax + first + step))) {
      first += step + 1;
      count -= step + 1;
    } else {
      count = step;
    }
  }
  const int32_t hi = first < 1 ? 1 : (first > n - 1 ? n - 1 : first);
  *lo = hi - 1;
  const double a = __ldg(ax + hi - 1), b = __ldg(ax + hi);
  *frac = ssg_clamp((x - a) / (b - a), 0.0, 1.0);
}

// ssg_axis_cell starting from a guess: the bracket test holds exactly when
// std::upper_bound(x) - 1, clamped to [0, n - 2], equals the guess
//   (h == 0 || ax[h] <= x) && (h == n - 2 || x < ax[h + 1])
// so the cell and fraction are ssg_axis_cell's; otherwise the full search runs.
// *hint receives the cell (simulations query neighbouring cells iteration
// after iteration: the context sum grows by one token per decode).
__device__ __forceinline__ void ssg_axis_cell_hint(const double* __restrict__ ax, int32_t n, double x,
                                                   int32_t* hint, int32_t* lo, double* frac) {
  if (n == 1) {
    *lo = 0;
    *frac = 0.0;
    return;
  }
  const int32_t h = *hint < 0 ? 0 : (*hint > n - 2 ? n - 2 : *hint);
  const double a = __ldg(ax + h), b = __ldg(ax + h + 1);
  if ((h == 0 || !(x < a)) && (h == n - 2 || x < b)) {
    *lo = h;
    *frac = ssg_clamp((x - a) / (b - a), 0.0, 1.0);
  } else {
    ssg_axis_cell(ax, n, x, lo, frac);
  }
  *hint = *lo;
}

// Multilinear interpolation (regressor.hpp:308-341), unrolled for the one- and
// two-feature models the estimator trains.  Corner order (mask 0..2^nf-1),
// weight product order (feature nf-1 down to 0, from 1.0) and the fp64
// accumulation are the reference's, including its duplicated corner when an
// axis has a single level.
__device__ __forceinline__ double ssg_interp(const SsgEstView& E, const SsgModelDesc& m,
                                             double x0, double x1) {
  const double* vals = E.dpool + m.values_off;
  int32_t lo0;
  double f0;
  const int32_t n0 = m.axis_len[0];
  ssg_axis_cell(E.dpool + m.axis_off[0], n0, x0, &lo0, &f0);
  const int32_t h0 = n0 == 1 ? 0 : 1;  // high corner offset along axis 0
  const double g0 = __dsub_rn(1.0, f0);
  if (m.nf == 1) {
    // mask 0: w = 1 * (1 - f0); mask 1: w = 1 * f0
    double acc = __dmul_rn(g0, __ldg(vals + lo0));
    acc = __dadd_rn(acc, __dmul_rn(h0 ? f0 : g0, __ldg(vals + lo0 + h0)));
    return acc;
  }
  int32_t lo1;
  double f1;
  const int32_t n1 = m.axis_len[1];
  ssg_axis_cell(E.dpool + m.axis_off[1], n1, x1, &lo1, &f1);
  const int32_t h1 = n1 == 1 ? 0 : 1;
  const double g1 = __dsub_rn(1.0, f1);
  // flat = (lo0 + high0) * n1 + (lo1 + high1); weight = (1 * w1) * w0
  const int64_t r0 = (int64_t)lo0 * n1, r1 = (int64_t)(lo0 + h0) * n1;
  const double w1lo = g1, w1hi = h1 ? f1 : g1;
  const double w0lo = g0, w0hi = h0 ? f0 : g0;
  double acc = __dmul_rn(__dmul_rn(w1lo, w0lo), __ldg(vals + r0 + lo1));        // mask 0
  acc = __dadd_rn(acc, __dmul_rn(__dmul_rn(w1lo, w0hi), __ldg(vals + r1 + lo1)));  // mask 1
  acc = __dadd_rn(acc, __dmul_rn(__dmul_rn(w1hi, w0lo), __ldg(vals + r0 + lo1 + h1)));  // mask 2
  acc = __dadd_rn(acc, __dmul_rn(__dmul_rn(w1hi, w0hi), __ldg(vals + r1 + lo1 + h1)));  // mask 3
  return acc;
}

// Mean of clamped linear-leaf trees (regressor.hpp:103-108, 256-264).
__device__ __forceinline__ double ssg_forest(const SsgEstView& E, const SsgModelDesc& m,
                                             double x0, double x1) {
  const int32_t* roots = E.roots + m.roots_off;
  const int nt = m.ntrees;
  double sum = 0.0;
  for (int t0 = 0; t0 < nt; t0 += FOREST_ILP) {
    int32_t idx[FOREST_ILP];
    double2 nd[FOREST_ILP];
#pragma unroll
    for (int g = 0; g < FOREST_ILP; ++g) {
      idx[g] = (t0 + g < nt) ? __ldg(roots + t0 + g) : -1;
      nd[g] = idx[g] >= 0 ? ssg_ld_node_v(E, idx[g]) : make_double2(0.0, __longlong_as_double(-1ll));
    }
    bool walking = true;
    while (walking) {
      walking = false;
#pragma unroll
      for (int g = 0; g < FOREST_ILP; ++g) {
        const int32_t feat = ssg_node_feat(nd[g]);
        if (feat >= 0) {
          const double xf = feat ? x1 : x0;
          idx[g] = (xf <= nd[g].x) ? idx[g] + 1 : ssg_node_right(nd[g]);
          nd[g] = ssg_ld_node_v(E, idx[g]);
          walking = true;
        }
      }
    }
#pragma unroll
    for (int g = 0; g < FOREST_ILP; ++g) {
      if (t0 + g < nt) {
        const double2 w12 = ssg_ld_node_v(E, idx[g] + 1);
        double v = __dadd_rn(nd[g].x, __dmul_rn(w12.x, x0));
        if (m.nf > 1) v = __dadd_rn(v, __dmul_rn(w12.y, x1));
        sum = __dadd_rn(sum, ssg_clamp(v, m.y_lo, m.y_hi));
      }
    }
  }
  return sum / (double)nt;
}

// Full EstimatorModel::predict for one query.  Returns SSG_OK and the
// runtime in *out, or an SSG_ERR_* code (*bad_feature = schema index).
// FMA selects the glibc contraction variant at compile time (the host's);
// FOREST = 0 compiles the interpolator only (the search default), keeping the
// simulation kernels' instruction footprint small.
template <int FMA, int FOREST>
__device__ __forceinline__ int ssg_predict_t(const SsgEstView& E, int32_t model, double v0,
                                             double v1, double* out, int* bad_feature) {
  const SsgModelDesc& m = E.models[model];
  if (!(v0 >= m.lower[0] && v0 <= m.upper[0])) {
    *bad_feature = 0;
    return SSG_ERR_BBOX;
  }
  const double x0 = ssg_log1p(v0, FMA);
  double x1 = 0.0;
  if (m.nf > 1) {
    if (!(v1 >= m.lower[1] && v1 <= m.upper[1])) {
      *bad_feature = 1;
      return SSG_ERR_BBOX;
    }
    x1 = ssg_log1p(v1, FMA);
  }
  double r;
  if (FOREST && m.kind == SSG_KIND_FOREST)
    r = ssg_forest(E, m, x0, x1);
  else
    r = ssg_interp(E, m, x0, x1);
  if (!ssg_exp_in_range(r)) return SSG_ERR_EXP_RANGE;
  *out = ssg_exp(r, FMA);
  return SSG_OK;
}

// Runtime-dispatched form for the batched predictor kernel (one call site).
__device__ __forceinline__ int ssg_predict_one(const SsgEstView& E, int32_t model, double v0,
                                               double v1, double* out, int* bad_feature) {
  return E.math_fma ? ssg_predict_t<1, 1>(E, model, v0, v1, out, bad_feature)
                    : ssg_predict_t<0, 1>(E, model, v0, v1, out, bad_feature);
}
