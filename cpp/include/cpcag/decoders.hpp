// decoders.hpp -- the alternate decoder (proj/core/include/cpcag/decoders.hpp:11-62).
#pragma once

#include "cpcag/graph.hpp"
#include "cpcag/sampling.hpp"

namespace cpcag {

enum class DecoderVariant { ideal, alternate, approx, approx2, approx3 };

struct DecoderConfig {
  DecoderVariant variant = DecoderVariant::approx;
  double gamma = 1.0;
  double gammap_r = 0.0;
  double gammap_c = 0.0;
  double delta_for_scaling = 0.0;
  double rank_threshold = 0.1;
  double pcg_tol = 1e-10;
  Index pcg_max_iter = 5000;
};

struct AlternateDecodeResult {
  Matrix X;
  bool converged = false;
  Index iterations = 0;
};

AlternateDecodeResult alternate_decode(const Matrix& Xt, const SamplingPlan& plan, const SparseMatrix& Lr,
                                       const SparseMatrix& Lc, const SpectralGap& gap_r, const SpectralGap& gap_c,
                                       const DecoderConfig& cfg);

}  // namespace cpcag
