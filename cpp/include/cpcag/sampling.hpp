// sampling.hpp -- sampling plan and subsample (proj/core/include/cpcag/sampling.hpp:13-43).
#pragma once

#include <cstdint>

#include "cpcag/types.hpp"

namespace cpcag {

struct SamplingPlan {
  IndexList omega_r;
  IndexList omega_c;
  Index p = 0;
  Index n = 0;
  double delta = 0.0;
  double epsilon = 0.0;
  std::uint64_t seed = 0;
  Index rho_r() const { return static_cast<Index>(omega_r.size()); }
  Index rho_c() const { return static_cast<Index>(omega_c.size()); }
  double norm_const() const;
};

SamplingPlan draw_plan(Index p, Index n, Index rho_r, Index rho_c, double delta, double epsilon, std::uint64_t seed);
Matrix subsample(const Matrix& Y, const SamplingPlan& plan);

}  // namespace cpcag
