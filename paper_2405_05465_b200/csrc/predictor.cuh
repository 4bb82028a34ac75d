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

// Multilinear interpolation, corner order and product order as regressor.hpp:326-340.
__device__ __forceinline__ double ssg_interp(const SsgEstView& E, const SsgModelDesc& m,
                                             double x0, double x1) {
  int32_t lo[2] = {0, 0};
  double frac[2] = {0.0, 0.0};
  const int nf = m.nf;
#pragma unroll
  for (int f = 0; f < 2; ++f) {
    if (f >= nf) break;
    const int32_t n = m.axis_len[f];
    if (n == 1) continue;
    const double x = f ? x1 : x0;
    const double* ax = E.dpool + m.axis_off[f];
    // std::upper_bound: first level strictly greater than x
    int32_t first = 0, count = n;
    while (count > 0) {
      int32_t step = count >> 1;
      if (!(x < __ldg(ax + first + step))) {
        first += step + 1;
        count -= step + 1;
      } else {
        count = step;
      }
    }
    int32_t hi = first < 1 ? 1 : (first > n - 1 ? n - 1 : first);
    lo[f] = hi - 1;
    const double a = __ldg(ax + lo[f]), b = __ldg(ax + hi);
    frac[f] = ssg_clamp((x - a) / (b - a), 0.0, 1.0);
  }
  const double* vals = E.dpool + m.values_off;
  double acc = 0.0;
  const int corners = 1 << nf;
  for (int mask = 0; mask < corners; ++mask) {
    double w = 1.0;
    int64_t flat = 0, stride = 1;
    for (int f = nf - 1; f >= 0; --f) {
      const int32_t n = m.axis_len[f];
      int high = (mask >> f) & 1;
      if (n == 1) high = 0;
      w = __dmul_rn(w, high ? frac[f] : __dsub_rn(1.0, frac[f]));
      flat += (int64_t)(lo[f] + high) * stride;
      stride *= n;
    }
    acc = __dadd_rn(acc, __dmul_rn(w, __ldg(vals + flat)));
  }
  return acc;
}

// Mean of clamped linear-leaf trees (regressor.hpp:103-108, 256-264).
__device__ __forceinline__ double ssg_forest(const SsgEstView& E, const SsgModelDesc& m,
                                             double x0, double x1) {
  const int32_t* roots = E.roots + m.roots_off;
  const SsgNode* nodes = E.nodes;
  const int nt = m.ntrees;
  double sum = 0.0;
  for (int t0 = 0; t0 < nt; t0 += FOREST_ILP) {
    int32_t idx[FOREST_ILP];
    double2 nd[FOREST_ILP];
#pragma unroll
    for (int g = 0; g < FOREST_ILP; ++g) {
      idx[g] = (t0 + g < nt) ? __ldg(roots + t0 + g) : -1;
      nd[g] = idx[g] >= 0 ? ssg_ld_node(nodes, idx[g]) : make_double2(0.0, __longlong_as_double(-1ll));
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
          nd[g] = ssg_ld_node(nodes, idx[g]);
          walking = true;
        }
      }
    }
#pragma unroll
    for (int g = 0; g < FOREST_ILP; ++g) {
      if (t0 + g < nt) {
        const double2 w12 = ssg_ld_node(nodes, idx[g] + 1);
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
__device__ __forceinline__ int ssg_predict_one(const SsgEstView& E, int32_t model, double v0,
                                               double v1, double* out, int* bad_feature) {
  const SsgModelDesc& m = E.models[model];
  if (!(v0 >= m.lower[0] && v0 <= m.upper[0])) {
    *bad_feature = 0;
    return SSG_ERR_BBOX;
  }
  const double x0 = ssg_log1p(v0, E.math_fma);
  double x1 = 0.0;
  if (m.nf > 1) {
    if (!(v1 >= m.lower[1] && v1 <= m.upper[1])) {
      *bad_feature = 1;
      return SSG_ERR_BBOX;
    }
    x1 = ssg_log1p(v1, E.math_fma);
  }
  const double r = (m.kind == SSG_KIND_FOREST) ? ssg_forest(E, m, x0, x1) : ssg_interp(E, m, x0, x1);
  if (!ssg_exp_in_range(r)) return SSG_ERR_EXP_RANGE;
  *out = ssg_exp(r, E.math_fma);
  return SSG_OK;
}
