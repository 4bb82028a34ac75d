// select.h -- K5 launch interface (segmented nearest-rank selection).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <vector>

struct SelectTask {
  int64_t segment;
  int64_t rank;  // 0-based order statistic
};

namespace ssg {
int64_t nearest_rank_index(int64_t n, double q);
void launch_select(const double* d_samples, const int64_t* d_seg_off, const SelectTask* d_tasks,
                   int64_t ntasks, double* d_out, cudaStream_t s);
std::vector<double> device_percentiles(const std::vector<double>& samples,
                                       const std::vector<double>& qs);
}  // namespace ssg
