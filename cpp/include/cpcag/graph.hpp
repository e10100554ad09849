// graph.hpp -- graph construction and Kron reduction
// (proj/core/include/cpcag/graph.hpp:10-58).
#pragma once

#include "cpcag/sparse.hpp"

namespace cpcag {

enum class LaplacianKind { combinatorial, normalized };
enum class Axis { rows, cols };

struct GraphModel {
  Index n_nodes = 0;
  Index K = 0;
  double sigma2 = 0.0;
  SparseMatrix adjacency;
  Vector degrees;
  SparseMatrix laplacian;
  LaplacianKind kind = LaplacianKind::combinatorial;
};

GraphModel build_knn_graph(const Matrix& X, Axis axis, Index K, LaplacianKind kind = LaplacianKind::combinatorial,
                           double sigma2_override = 0.0);
GraphModel graph_from_adjacency(const SparseMatrix& W, LaplacianKind kind = LaplacianKind::combinatorial);
SparseMatrix kron_reduce(const SparseMatrix& L, const IndexList& keep, double pcg_tol = 1e-12,
                         double prune_tol = 1e-12);

struct SpectralGap {
  Index k = 0;
  double lambda_k = 0.0;
  double lambda_k1 = 0.0;
  double ratio = 0.0;
};

}  // namespace cpcag
