// train.h -- device random-forest build (train.cu): the estimator's forest
// regressors grown on the GPU, one warp per tree, bit-identical to the
// reference's ForestRegressor::train (regressor.hpp:82-254).
#pragma once
#include <cstdint>
#include <vector>

#include "servesim_b200.hpp"

namespace ssg {

// One forest to grow: rows x (n x nf, nf <= 2, already log1p-transformed),
// targets y (log runtimes), and the forest configuration with its seed.
struct ForestFit {
  const std::vector<std::vector<double>>* x;
  const std::vector<double>* y;
  servesim::ForestConfig cfg;
};

// Grows every forest of `fits` in one launch (trees of all forests in
// parallel); returns the forests in the reference's serialized layout.
std::vector<servesim::RegressorData> grow_forests(const std::vector<ForestFit>& fits);

}  // namespace ssg
