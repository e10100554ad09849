// cpcag_b200.cpp -- the reference's cpcag:: API (proj/core/include/cpcag/*.hpp)
// over the C-ABI of libcpcag_cuda.so.  Host types mirror the reference's;
// every hot function is one call into the library, which stages host arrays
// through HBM.  Status codes become the reference's exception types with the
// library's (= the reference's) messages.
#include <algorithm>
#include <cmath>
#include <stdexcept>
#include <string>
#include <utility>

#include "cpcag/decoders.hpp"
#include "cpcag/frpcag.hpp"
#include "cpcag/graph.hpp"
#include "cpcag/sampling.hpp"
#include "cpcag/solvers.hpp"
#include "cpcag/sparse.hpp"
#include "cpcag_cuda.h"

namespace cpcag {
namespace {

void check(int rc) {
  if (rc == CPCAG_OK) return;
  const std::string m = cpcag_cuda_last_error();
  if (rc == CPCAG_ERR_INVALID_ARGUMENT) throw std::invalid_argument(m);
  if (rc == CPCAG_ERR_OUT_OF_RANGE) throw std::out_of_range(m);
  throw std::runtime_error(m);
}

// One library context per thread (the library is re-entrant per context).
cpcag_ctx ctx() {
  thread_local struct Holder {
    cpcag_ctx h = nullptr;
    Holder() { check(cpcag_ctx_create(-1, &h)); }
    ~Holder() {
      if (h) cpcag_ctx_destroy(h);
    }
  } holder;
  return holder.h;
}

// RAII device copy of a host SparseMatrix.
struct DevCsr {
  cpcag_csr h = nullptr;
  explicit DevCsr(const SparseMatrix& A) {
    check(cpcag_csr_create(ctx(), A.rows(), A.cols(), A.nonzeros(), A.row_ptr().data(), A.col_idx().data(),
                           A.values().data(), &h));
  }
  explicit DevCsr(cpcag_csr adopt) : h(adopt) {}
  ~DevCsr() {
    if (h) cpcag_csr_destroy(h);
  }
  DevCsr(const DevCsr&) = delete;
  DevCsr& operator=(const DevCsr&) = delete;
};

SparseMatrix to_host(cpcag_csr h) {
  DevCsr own(h);
  int64_t r = 0, c = 0, z = 0;
  check(cpcag_csr_info(h, &r, &c, &z));
  std::vector<Index> rp(static_cast<size_t>(r) + 1), ci(static_cast<size_t>(z));
  std::vector<double> v(static_cast<size_t>(z));
  check(cpcag_csr_export(ctx(), h, rp.data(), ci.data(), v.data()));
  return SparseMatrix::from_csr(r, c, std::move(rp), std::move(ci), std::move(v));
}

cpcag_frpcag_config cfg_c(const FrpcagConfig& c) {
  return cpcag_frpcag_config{c.gamma_r, c.gamma_c, c.loss == Loss::l2 ? CPCAG_LOSS_L2 : CPCAG_LOSS_L1, c.tol,
                             c.max_iter, c.step};
}

}  // namespace

// ------------------------------------------------------------------ SparseMatrix (host)
SparseMatrix SparseMatrix::from_triplets(Index rows, Index cols, std::vector<Triplet> entries, double drop_below) {
  if (rows < 0 || cols < 0) throw std::invalid_argument("sparse: negative dimension");
  for (const auto& t : entries) {
    if (t.row < 0 || t.row >= rows || t.col < 0 || t.col >= cols)
      throw std::invalid_argument("sparse: triplet index out of range");
    if (!std::isfinite(t.value)) throw std::invalid_argument("sparse: non-finite triplet value");
  }
  std::stable_sort(entries.begin(), entries.end(),
                   [](const Triplet& a, const Triplet& b) { return a.row != b.row ? a.row < b.row : a.col < b.col; });
  SparseMatrix m;
  m.rows_ = rows;
  m.cols_ = cols;
  m.row_ptr_.assign(static_cast<size_t>(rows) + 1, 0);
  for (size_t k = 0; k < entries.size();) {
    size_t e = k;
    double sum = 0.0;
    while (e < entries.size() && entries[e].row == entries[k].row && entries[e].col == entries[k].col)
      sum += entries[e++].value;
    if (sum != 0.0 && std::fabs(sum) > drop_below) {
      m.col_idx_.push_back(entries[k].col);
      m.values_.push_back(sum);
      m.row_ptr_[static_cast<size_t>(entries[k].row) + 1]++;
    }
    k = e;
  }
  for (Index r = 0; r < rows; ++r) m.row_ptr_[r + 1] += m.row_ptr_[r];
  return m;
}

SparseMatrix SparseMatrix::from_dense(const Matrix& d, double drop_below) {
  std::vector<Triplet> t;
  for (Index i = 0; i < d.rows(); ++i)
    for (Index j = 0; j < d.cols(); ++j)
      if (d(i, j) != 0.0) t.push_back({i, j, d(i, j)});
  return from_triplets(d.rows(), d.cols(), std::move(t), drop_below);
}

SparseMatrix SparseMatrix::identity(Index n) {
  std::vector<Triplet> t;
  for (Index i = 0; i < n; ++i) t.push_back({i, i, 1.0});
  return from_triplets(n, n, std::move(t));
}

SparseMatrix SparseMatrix::from_csr(Index rows, Index cols, std::vector<Index> rp, std::vector<Index> ci,
                                    std::vector<double> v) {
  if (static_cast<Index>(rp.size()) != rows + 1 || rp.front() != 0 || rp.back() != static_cast<Index>(ci.size()) ||
      ci.size() != v.size())
    throw std::invalid_argument("sparse: malformed CSR arrays");
  for (Index r = 0; r < rows; ++r) {
    if (rp[r + 1] < rp[r]) throw std::invalid_argument("sparse: row pointers must be monotone");
    for (Index k = rp[r]; k < rp[r + 1]; ++k) {
      if (ci[k] < 0 || ci[k] >= cols || (k > rp[r] && ci[k] <= ci[k - 1]) || v[k] == 0.0)
        throw std::invalid_argument("sparse: CSR invariants violated");
    }
  }
  SparseMatrix m;
  m.rows_ = rows;
  m.cols_ = cols;
  m.row_ptr_ = std::move(rp);
  m.col_idx_ = std::move(ci);
  m.values_ = std::move(v);
  return m;
}

double SparseMatrix::coeff(Index i, Index j) const {
  if (i < 0 || i >= rows_ || j < 0 || j >= cols_) throw std::out_of_range("sparse: coeff index out of range");
  const auto b = col_idx_.begin() + row_ptr_[i], e = col_idx_.begin() + row_ptr_[i + 1];
  const auto it = std::lower_bound(b, e, j);
  return (it != e && *it == j) ? values_[static_cast<size_t>(it - col_idx_.begin())] : 0.0;
}

Vector SparseMatrix::multiply(const Vector& x) const {
  Vector y(rows_);
  DevCsr A(*this);
  check(cpcag_cuda_spmv(ctx(), A.h, CPCAG_F64, x.size(), x.data(), y.data()));
  return y;
}

Matrix SparseMatrix::multiply(const Matrix& X) const {
  Matrix Y(rows_, X.cols());
  DevCsr A(*this);
  check(cpcag_cuda_spmm(ctx(), A.h, CPCAG_LEFT, CPCAG_F64, X.rows(), X.cols(), X.data(), Y.data()));
  return Y;
}

Matrix SparseMatrix::right_multiply(const Matrix& X) const {
  Matrix Y(X.rows(), cols_);
  DevCsr A(*this);
  check(cpcag_cuda_spmm(ctx(), A.h, CPCAG_RIGHT, CPCAG_F64, X.rows(), X.cols(), X.data(), Y.data()));
  return Y;
}

Matrix SparseMatrix::to_dense() const {
  Matrix d(rows_, cols_);
  for (Index r = 0; r < rows_; ++r)
    for (Index k = row_ptr_[r]; k < row_ptr_[r + 1]; ++k) d(r, col_idx_[k]) = values_[k];
  return d;
}

Vector SparseMatrix::diagonal() const {
  Vector d(std::min(rows_, cols_));
  for (Index r = 0; r < d.size(); ++r) d(r) = coeff(r, r);
  return d;
}

Vector SparseMatrix::row_sums() const {
  Vector s(rows_);
  for (Index r = 0; r < rows_; ++r)
    for (Index k = row_ptr_[r]; k < row_ptr_[r + 1]; ++k) s(r) += values_[k];
  return s;
}

// ------------------------------------------------------------------ solvers
PcgResult pcg_solve(const SparseMatrix& A, const Vector& b, Vector& x, const PcgOptions& opt, bool jacobi) {
  if (A.rows() != A.cols() || b.size() != A.rows()) throw std::invalid_argument("pcg: dimension mismatch");
  if (x.size() != b.size()) x = Vector(b.size());
  DevCsr d(A);
  PcgResult r;
  int64_t it = 0;
  int conv = 0;
  check(cpcag_cuda_pcg_solve(ctx(), d.h, b.data(), x.data(), b.size(), opt.tol, opt.max_iter, jacobi ? 1 : 0, &it,
                             &conv, &r.relative_residual));
  r.iterations = it;
  r.converged = conv != 0;
  return r;
}

double power_iteration_norm(const SparseMatrix& A, double tol, std::uint64_t seed, Index max_iter) {
  DevCsr d(A);
  double out = 0.0;
  check(cpcag_cuda_power_norm(ctx(), d.h, tol, seed, max_iter, &out));
  return out;
}

// ------------------------------------------------------------------ graphs
GraphModel build_knn_graph(const Matrix& X, Axis axis, Index K, LaplacianKind kind, double sigma2_override) {
  GraphModel g;
  const Index n = axis == Axis::rows ? X.rows() : X.cols();
  g.degrees = Vector(n);
  cpcag_csr W = nullptr, L = nullptr;
  check(cpcag_cuda_knn_graph(ctx(), CPCAG_F64, X.data(), X.rows(), X.cols(),
                             axis == Axis::rows ? CPCAG_AXIS_ROWS : CPCAG_AXIS_COLS, K,
                             kind == LaplacianKind::normalized ? CPCAG_NORMALIZED : CPCAG_COMBINATORIAL,
                             sigma2_override, &W, &L, g.degrees.data(), &g.sigma2));
  g.n_nodes = n;
  g.K = K;
  g.kind = kind;
  g.adjacency = to_host(W);
  g.laplacian = to_host(L);
  return g;
}

GraphModel graph_from_adjacency(const SparseMatrix& W, LaplacianKind kind) {
  GraphModel g;
  g.degrees = Vector(W.rows());
  DevCsr d(W);
  cpcag_csr L = nullptr;
  check(cpcag_cuda_graph_from_adjacency(ctx(), d.h, kind == LaplacianKind::normalized ? CPCAG_NORMALIZED
                                                                                       : CPCAG_COMBINATORIAL,
                                        &L, g.degrees.data()));
  g.n_nodes = W.rows();
  g.kind = kind;
  g.adjacency = W;
  g.laplacian = to_host(L);
  return g;
}

SparseMatrix kron_reduce(const SparseMatrix& L, const IndexList& keep, double pcg_tol, double prune_tol) {
  DevCsr d(L);
  cpcag_csr out = nullptr;
  check(cpcag_cuda_kron_reduce(ctx(), d.h, keep.data(), static_cast<int64_t>(keep.size()), pcg_tol, prune_tol, &out));
  return to_host(out);
}

// ------------------------------------------------------------------ sampling
double SamplingPlan::norm_const() const {
  return static_cast<double>(p) * static_cast<double>(n) / (static_cast<double>(rho_r()) * static_cast<double>(rho_c()));
}

SamplingPlan draw_plan(Index p, Index n, Index rho_r, Index rho_c, double delta, double epsilon, std::uint64_t seed) {
  SamplingPlan plan;
  plan.omega_r.resize(static_cast<size_t>(std::max<Index>(rho_r, 0)));
  plan.omega_c.resize(static_cast<size_t>(std::max<Index>(rho_c, 0)));
  check(cpcag_cuda_draw_plan(p, n, rho_r, rho_c, seed, plan.omega_r.data(), plan.omega_c.data()));
  plan.p = p;
  plan.n = n;
  plan.delta = delta;
  plan.epsilon = epsilon;
  plan.seed = seed;
  return plan;
}

Matrix subsample(const Matrix& Y, const SamplingPlan& plan) {
  Matrix out(plan.rho_r(), plan.rho_c());
  check(cpcag_cuda_subsample(ctx(), CPCAG_F64, Y.data(), Y.rows(), Y.cols(), plan.omega_r.data(), plan.rho_r(),
                             plan.omega_c.data(), plan.rho_c(), out.data()));
  return out;
}

// ------------------------------------------------------------------ FRPCAG
double objective(const Matrix& X, const Matrix& Y, const SparseMatrix& Lr, const SparseMatrix& Lc,
                 const FrpcagConfig& cfg) {
  if (X.rows() != Y.rows() || X.cols() != Y.cols()) throw std::invalid_argument("objective: dimension mismatch");
  DevCsr r(Lr), c(Lc);
  const cpcag_frpcag_config cc = cfg_c(cfg);
  double out = 0.0;
  check(cpcag_cuda_objective(ctx(), CPCAG_F64, X.data(), Y.data(), X.rows(), X.cols(), r.h, c.h, &cc, &out));
  return out;
}

static Matrix prox(int loss, const Matrix& Z, const Matrix& Y, double lam) {
  if (Z.rows() != Y.rows() || Z.cols() != Y.cols()) throw std::invalid_argument("prox: dimension mismatch");
  Matrix out(Z.rows(), Z.cols());
  check(cpcag_cuda_prox(ctx(), CPCAG_F64, loss, Z.data(), Y.data(), Z.size(), lam, out.data()));
  return out;
}
Matrix prox_l1(const Matrix& Z, const Matrix& Y, double lam) { return prox(CPCAG_LOSS_L1, Z, Y, lam); }
Matrix prox_l2(const Matrix& Z, const Matrix& Y, double lam) { return prox(CPCAG_LOSS_L2, Z, Y, lam); }

Matrix grad_g(const Matrix& Z, const SparseMatrix& Lr, const SparseMatrix& Lc, const FrpcagConfig& cfg) {
  DevCsr r(Lr), c(Lc);
  const cpcag_frpcag_config cc = cfg_c(cfg);
  Matrix G(Z.rows(), Z.cols());
  check(cpcag_cuda_grad_g(ctx(), CPCAG_F64, Z.data(), Z.rows(), Z.cols(), r.h, c.h, &cc, G.data()));
  return G;
}

std::pair<Matrix, SolveTrace> fista_solve(const Matrix& Y, const SparseMatrix& Lr, const SparseMatrix& Lc,
                                          const FrpcagConfig& cfg) {
  DevCsr r(Lr), c(Lc);
  const cpcag_frpcag_config cc = cfg_c(cfg);
  Matrix X(Y.rows(), Y.cols());
  SolveTrace tr;
  tr.objective.resize(static_cast<size_t>(std::max<Index>(cfg.max_iter, 1)));
  cpcag_solve_trace t{};
  check(cpcag_cuda_fista(ctx(), CPCAG_F64, Y.data(), Y.rows(), Y.cols(), r.h, c.h, &cc, X.data(),
                         tr.objective.data(), &t));
  tr.objective.resize(static_cast<size_t>(t.iterations));
  tr.iterations = t.iterations;
  tr.converged = t.converged != 0;
  tr.final_rel_change = t.final_rel_change;
  tr.step = t.step;
  return {std::move(X), std::move(tr)};
}

// ------------------------------------------------------------------ decoder
AlternateDecodeResult alternate_decode(const Matrix& Xt, const SamplingPlan& plan, const SparseMatrix& Lr,
                                       const SparseMatrix& Lc, const SpectralGap& gap_r, const SpectralGap& gap_c,
                                       const DecoderConfig& cfg) {
  if (Xt.rows() != plan.rho_r() || Xt.cols() != plan.rho_c())
    throw std::invalid_argument("alternate decoder: Xt does not match plan");
  DevCsr r(Lr), c(Lc);
  const cpcag_decoder_config dc{cfg.gamma, cfg.pcg_tol, cfg.pcg_max_iter, 0};
  AlternateDecodeResult res;
  res.X = Matrix(plan.p, plan.n);
  int conv = 0;
  int64_t it = 0;
  check(cpcag_cuda_alternate_decode(ctx(), CPCAG_F64, Xt.data(), Xt.rows(), Xt.cols(), plan.omega_r.data(),
                                    plan.omega_c.data(), plan.p, plan.n, r.h, c.h, gap_r.lambda_k1, gap_c.lambda_k1,
                                    &dc, res.X.data(), &conv, &it));
  res.converged = conv != 0;
  res.iterations = it;
  return res;
}

}  // namespace cpcag
