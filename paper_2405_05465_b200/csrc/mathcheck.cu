// mathcheck.cu -- the device libm restatement (glibc_math.h) evaluated over a
// whole arithmetic progression of inputs, for the exhaustive self-check of the
// predictor's numerics against the host's glibc.
//
// The predictor applies log1p to integer-valued features (token counts,
// context tokens x KV bytes per token, tokens x payload bytes per token) and
// exp to the regressor's output (estimator.hpp:120-122).  The feature domain
// is finite -- multiples of one quantum up to the trained box + 10 % -- so the
// check walks it completely: x_k = base + k * step, k in [0, n).
#include "glibc_math.h"
#include "runtime.h"

namespace ssgk {

__global__ void k_math_eval(int fn, int fma_variant, double base, double step, int64_t k0, int64_t n,
                            double* __restrict__ out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double x = __dadd_rn(base, __dmul_rn((double)(k0 + i), step));
  double y;
  if (fn == 0)
    y = ssg_log1p(x, fma_variant);
  else
    y = ssg_exp_in_range(x) ? ssg_exp(x, fma_variant) : __longlong_as_double(0x7ff8dead00000000ll);
  out[i] = y;
}

}  // namespace ssgk

namespace ssg {

void launch_math_eval(int fn, int fma_variant, double base, double step, int64_t k0, int64_t n,
                      double* d_out, cudaStream_t s) {
  if (n <= 0) return;
  ssgk::k_math_eval<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(fn, fma_variant, base, step, k0, n,
                                                                 d_out);
  cuda_check(cudaGetLastError(), "k_math_eval launch");
  stats().launches_setup += 1;
}

}  // namespace ssg
