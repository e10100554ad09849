// solvers.hpp -- PCG and the power-iteration norm (proj/core/include/cpcag/solvers.hpp:13-22,82-91).
#pragma once

#include "cpcag/sparse.hpp"

namespace cpcag {

struct PcgOptions {
  double tol = 1e-10;
  Index max_iter = 1000;
};

struct PcgResult {
  Index iterations = 0;
  bool converged = false;
  double relative_residual = 0.0;
};

// x: start iterate in, solution out.  jacobi: diagonal preconditioner (0 -> 1).
PcgResult pcg_solve(const SparseMatrix& A, const Vector& b, Vector& x, const PcgOptions& opt = {},
                    bool jacobi = true);
double power_iteration_norm(const SparseMatrix& A, double tol = 1e-9, std::uint64_t seed = 0,
                            Index max_iter = 50000);

}  // namespace cpcag
