// ssg_device.h -- plain-old-data layouts shared by host C++ and sm_100a kernels.
//
// Everything the kernels read lives in a handful of flat HBM arrays; no host
// pointers, no C++ containers.  Offsets are element offsets into the pools.
#pragma once
#include <stdint.h>
#include <vector_types.h>

#define SSG_KIND_INTERP 0
#define SSG_KIND_FOREST 1

// Error codes written by kernels (host turns them into the reference's
// exception messages, see predictor.cu / engine.cu).
#define SSG_OK 0
#define SSG_ERR_BBOX 1           // feature outside extrapolation margin (estimator.hpp:115-119)
#define SSG_ERR_EXP_RANGE 2      // regressor output outside exp fast path (internal)
#define SSG_ERR_ENQUEUE 3        // request needs more KV units than the replica has (scheduler.hpp:149)
#define SSG_ERR_INTERNAL 4       // violated invariant (internal_check)
#define SSG_ERR_CAPACITY 5       // a per-sim device buffer was too small (host sizing bug)

// One trained per-(op, tp) predictor.
struct SsgModelDesc {
  int32_t kind;  // SSG_KIND_*
  int32_t nf;    // 1 or 2 features
  int32_t op;    // OpName, for error reporting
  int32_t tp;
  double lower[2], upper[2];  // bbox_lo - margin, bbox_hi + margin (estimator.hpp:113-115)
  // interp: axis levels and row-major values in dpool
  int32_t axis_len[2];
  int64_t axis_off[2];
  int64_t values_off;
  // forest: ntrees roots (absolute node indices) in roots[], nodes in nodes[]
  int32_t ntrees;
  int32_t pad0;
  int64_t roots_off;
  double y_lo, y_hi;
};

// 16-byte tree node, preorder layout so the left child is always node + 1.
//   internal: a = threshold, feat >= 0, right = absolute index of right child
//   leaf:     a = w0, feat = -1; the next slot holds {w1, w2} as two doubles
struct __attribute__((aligned(16))) SsgNode {
  double a;
  int32_t feat;
  int32_t right;
};

struct SsgEstView {
  const SsgModelDesc* models;
  const double* dpool;
  const SsgNode* nodes;
  const int32_t* roots;
  const double* node_a;    // SoA mirror of nodes (SSG_FOREST_SOA builds only): threshold / w
  const int2* node_fr;     //   and (feature, right) -- A/B of the north-star layout
  int32_t nmodels;
  int32_t math_fma;  // SSG_MATH_FMA / SSG_MATH_PLAIN: which glibc contraction the host uses
};

// First failing query of a batched predict: atomicMin over (index << 8 | code),
// so the lowest failing index wins together with its code; the host then
// re-derives the operands of that one query to format the reference message.
#define SSG_NO_ERROR 0xffffffffffffffffull
