// test_dropin.cpp -- the cpcag:: drop-in layer (cpp/include/cpcag) against
// the reference's own known answers (proj/tests/test_numeric.cpp,
// proj/tests/test_graph.cpp, SPEC.md examples), exception types and message
// substrings.  A self-contained harness (doctest is absent here); exits
// non-zero on the first failed file of checks.  Needs a GPU.
#include <cmath>
#include <cstdio>
#include <functional>
#include <stdexcept>
#include <string>
#include <vector>

#include "cpcag/decoders.hpp"
#include "cpcag/frpcag.hpp"
#include "cpcag/graph.hpp"
#include "cpcag/sampling.hpp"
#include "cpcag/solvers.hpp"

using namespace cpcag;

static int g_fail = 0, g_checks = 0;
#define CHECK(cond)                                                              \
  do {                                                                           \
    ++g_checks;                                                                  \
    if (!(cond)) {                                                               \
      ++g_fail;                                                                  \
      std::fprintf(stderr, "FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond);       \
    }                                                                            \
  } while (0)

template <class E>
static void check_throws(const std::function<void()>& f, const std::string& sub, int line) {
  ++g_checks;
  try {
    f();
  } catch (const E& e) {
    if (std::string(e.what()).find(sub) == std::string::npos) {
      ++g_fail;
      std::fprintf(stderr, "FAIL line %d: message '%s' lacks '%s'\n", line, e.what(), sub.c_str());
    }
    return;
  } catch (const std::exception& e) {
    ++g_fail;
    std::fprintf(stderr, "FAIL line %d: wrong exception type: %s\n", line, e.what());
    return;
  }
  ++g_fail;
  std::fprintf(stderr, "FAIL line %d: no exception\n", line);
}
#define CHECK_THROWS(E, expr, sub) check_throws<E>([&] { expr; }, sub, __LINE__)

static bool near(double a, double b, double tol) { return std::fabs(a - b) <= tol; }

// test_numeric.cpp:16-25
static SparseMatrix path3() {
  return SparseMatrix::from_triplets(
      3, 3, {{0, 0, 1}, {0, 1, -1}, {1, 0, -1}, {1, 1, 2}, {1, 2, -1}, {2, 1, -1}, {2, 2, 1}});
}
// test_numeric.cpp:27-35
static SparseMatrix complete4() {
  std::vector<Triplet> t;
  for (Index i = 0; i < 4; ++i)
    for (Index j = 0; j < 4; ++j) t.push_back({i, j, i == j ? 3.0 : -1.0});
  return SparseMatrix::from_triplets(4, 4, t);
}

static void test_sparse() {
  // sparse.cpp:10-46: duplicates summed, zeros dropped, columns sorted
  const auto A = SparseMatrix::from_triplets(2, 3, {{1, 2, 1.0}, {0, 1, 2.0}, {1, 2, 2.0}, {0, 0, 0.0}});
  CHECK(A.nonzeros() == 2 && A.coeff(1, 2) == 3.0 && A.coeff(0, 1) == 2.0 && A.coeff(0, 0) == 0.0);
  CHECK_THROWS(std::out_of_range, A.coeff(2, 0), "out of range");
  // SpMV / SpMM against the dense product (test_numeric.cpp:76-85)
  const auto L = path3();
  const Vector x{1.0, 2.0, 4.0};
  const Vector y = L.multiply(x);
  CHECK(y(0) == -1.0 && y(1) == -1.0 && y(2) == 2.0);
  Matrix X = Matrix::from_rows({{1, 0}, {2, 1}, {4, -1}});
  const Matrix Y = L.multiply(X);
  const Matrix Yr = L.right_multiply(Matrix::from_rows({{1, 2, 4}}));
  CHECK(Y(0, 0) == -1.0 && Y(1, 0) == -1.0 && Y(2, 0) == 2.0 && Y(0, 1) == -1.0 && Y(1, 1) == 3.0 && Y(2, 1) == -2.0);
  CHECK(Yr(0, 0) == -1.0 && Yr(0, 1) == -1.0 && Yr(0, 2) == 2.0);
  CHECK_THROWS(std::invalid_argument, L.multiply(Matrix(2, 1)), "dimension mismatch");
}

static void test_solvers() {
  // test_numeric.cpp:110-118: the identity converges in one iteration
  const auto I = SparseMatrix::identity(4);
  Vector b{1.0, -2.0, 0.5, 3.0}, x(4);
  auto r = pcg_solve(I, b, x);
  CHECK(r.converged && r.iterations == 1 && near(x(1), -2.0, 1e-12));
  // diag(1, 2, 4) x = (1, 2, 4) -> x = 1
  const auto D = SparseMatrix::from_triplets(3, 3, {{0, 0, 1}, {1, 1, 2}, {2, 2, 4}});
  Vector bd{1.0, 2.0, 4.0}, xd(3);
  r = pcg_solve(D, bd, xd);
  CHECK(r.converged && near(xd(0), 1, 1e-12) && near(xd(1), 1, 1e-12) && near(xd(2), 1, 1e-12));
  // test_numeric.cpp:162-169: breakdown names the iteration
  const auto Z = SparseMatrix::from_triplets(2, 2, {});
  Vector b2{1.0, 1.0}, x2(2);
  CHECK_THROWS(std::runtime_error, pcg_solve(Z, b2, x2, {}, false), "pcg: breakdown (nonpositive curvature) at iteration 0");
  // test_numeric.cpp:171-177: zero right-hand side
  Vector b0(3), x0(3);
  r = pcg_solve(SparseMatrix::identity(3), b0, x0);
  CHECK(r.converged && r.iterations == 0);
  // test_numeric.cpp:179-193 / SPEC.md:60-61
  CHECK(near(power_iteration_norm(D, 1e-12, 3), 4.0, 4e-9));
  CHECK(near(power_iteration_norm(complete4(), 1e-12, 5), 4.0, 4e-9));
  CHECK(power_iteration_norm(SparseMatrix::from_triplets(4, 4, {}), 1e-10, 9) == 0.0);
}

static void test_graphs() {
  // test_graph.cpp:51-58: coincident points get weight 1
  auto g = build_knn_graph(Matrix::from_rows({{1, 1}, {2, 2}}), Axis::cols, 1);
  CHECK(g.adjacency.coeff(0, 1) == 1.0 && g.adjacency.coeff(1, 0) == 1.0);
  // test_graph.cpp:60-75: collinear points 0, 1, 10 with K = 1
  g = build_knn_graph(Matrix::from_rows({{0, 1, 10}}), Axis::cols, 1);
  const double s2 = (1.0 + 1.0 + 81.0) / 3.0;
  CHECK(near(g.sigma2, s2, 1e-15 * s2));
  CHECK(near(g.adjacency.coeff(0, 1), std::exp(-1.0 / s2), 1e-15));
  CHECK(near(g.adjacency.coeff(1, 2), std::exp(-81.0 / s2), 1e-15));
  CHECK(g.adjacency.coeff(0, 2) == 0.0 && g.adjacency.nonzeros() == 4);
  const Vector rs = g.laplacian.row_sums();
  CHECK(near(rs(0), 0, 1e-15) && near(rs(1), 0, 1e-15) && near(rs(2), 0, 1e-15));
  // test_graph.cpp:77-86: ties break toward the lower index
  g = build_knn_graph(Matrix::from_rows({{0, 1, 0, 5}, {0, 0, 1, 5}}), Axis::cols, 1);
  CHECK(g.adjacency.coeff(1, 3) > 0.0 && g.adjacency.coeff(2, 3) == 0.0);
  // test_graph.cpp:95-103
  CHECK_THROWS(std::invalid_argument, build_knn_graph(Matrix::from_rows({{0, 1, 2}}), Axis::cols, 3), "K");
  CHECK_THROWS(std::invalid_argument, build_knn_graph(Matrix::from_rows({{2, 2, 2, 2}}), Axis::cols, 2),
               "fewer distinct points");
  CHECK_THROWS(std::invalid_argument, build_knn_graph(Matrix::from_rows({{0, 1, 2}}), Axis::cols, 0), "K must be");
  // graph_from_adjacency validation (graph.cpp:137-154)
  CHECK_THROWS(std::invalid_argument,
               graph_from_adjacency(SparseMatrix::from_triplets(2, 2, {{0, 1, 1.0}})), "symmetric");
  // test_graph.cpp:171-192 / SPEC.md:149-151: Kron reduction
  const auto L = path3();
  const auto R = kron_reduce(L, {0, 1, 2});
  CHECK(R.nonzeros() == L.nonzeros() && R.coeff(1, 1) == 2.0);
  const auto E = kron_reduce(L, {0, 2});
  CHECK(near(E.coeff(0, 0), 0.5, 1e-12) && near(E.coeff(0, 1), -0.5, 1e-12) && near(E.coeff(1, 1), 0.5, 1e-12));
  const auto two = SparseMatrix::from_triplets(
      4, 4, {{0, 0, 1}, {0, 1, -1}, {1, 0, -1}, {1, 1, 1}, {2, 2, 2}, {2, 3, -2}, {3, 2, -2}, {3, 3, 2}});
  CHECK(kron_reduce(two, {0, 2}).nonzeros() == 0);
  CHECK_THROWS(std::runtime_error, kron_reduce(two, {0, 1}),
               "kron reduction: connected component containing node 2 has no kept node");
}

static void test_sampling_and_frpcag() {
  // sampling.cpp:35-75: draw order kept, deterministic, a selection
  const auto a = draw_plan(9, 7, 9, 7, 0.1, 0.1, 77), b = draw_plan(9, 7, 9, 7, 0.1, 0.1, 77);
  CHECK(a.omega_r == b.omega_r && a.omega_c == b.omega_c);
  std::vector<int> seen(9, 0);
  for (Index i : a.omega_r) seen[static_cast<size_t>(i)]++;
  CHECK(std::all_of(seen.begin(), seen.end(), [](int s) { return s == 1; }));
  const auto plan = draw_plan(5, 4, 2, 3, 0.0, 0.0, 5);
  Matrix Y(5, 4);
  for (Index i = 0; i < 5; ++i)
    for (Index j = 0; j < 4; ++j) Y(i, j) = 10.0 * i + j;
  const Matrix S = subsample(Y, plan);
  CHECK(S.rows() == 2 && S.cols() == 3 && S(1, 2) == Y(plan.omega_r[1], plan.omega_c[2]));
  // prox_l1 examples
  CHECK(prox_l1(Matrix::from_rows({{3}}), Matrix::from_rows({{0}}), 1.0)(0, 0) == 2.0);
  CHECK(prox_l1(Matrix::from_rows({{-0.5}}), Matrix::from_rows({{0}}), 1.0)(0, 0) == 0.0);
  CHECK_THROWS(std::invalid_argument, prox_l1(Matrix(1, 1), Matrix(1, 1), -1.0), "prox: negative threshold");
  // constants are in the graphs' null spaces
  const auto Lr = path3(), Lc = complete4();
  Matrix ones(3, 4);
  for (Index i = 0; i < 3; ++i)
    for (Index j = 0; j < 4; ++j) ones(i, j) = 1.0;
  FrpcagConfig cfg;
  cfg.gamma_r = 2.0;
  cfg.gamma_c = 3.0;
  CHECK(near(objective(ones, ones, Lr, Lc, cfg), 0.0, 1e-12));
  const Matrix G = grad_g(ones, Lr, Lc, cfg);
  CHECK(near(G(1, 2), 0.0, 1e-12));
  // frpcag.cpp:62-112: FISTA decreases the objective and reports its trace
  Matrix Yn(3, 4);
  for (Index i = 0; i < 3; ++i)
    for (Index j = 0; j < 4; ++j) Yn(i, j) = std::sin(1.0 + i * 4 + j);
  cfg.max_iter = 50;
  cfg.tol = 1e-300;
  const auto [X, tr] = fista_solve(Yn, Lr, Lc, cfg);
  CHECK(tr.iterations == 50 && static_cast<Index>(tr.objective.size()) == 50 && tr.step > 0.0);
  CHECK(tr.objective.back() <= tr.objective.front());
  CHECK(near(objective(X, Yn, Lr, Lc, cfg), tr.objective.back(), 1e-9 * std::fabs(tr.objective.back())));
  FrpcagConfig bad = cfg;
  bad.step = 10.0;
  Matrix big = Yn;
  for (Index i = 0; i < 3; ++i)
    for (Index j = 0; j < 4; ++j) big(i, j) *= 1e300;
  CHECK_THROWS(std::runtime_error, fista_solve(big, Lr, Lc, bad), "fista: diverged (non-finite objective at iteration");
  bad = cfg;
  bad.tol = 0.0;
  CHECK_THROWS(std::invalid_argument, fista_solve(Yn, Lr, Lc, bad), "fista: stopping tolerance must be positive");
}

static void test_decoder() {
  // decoders.cpp:145-186 on a 3 x 4 problem: the CG solution satisfies the
  // normal equations M o X + gc X Lc + gr Lr X = scatter(Xt)
  const auto Lr = path3(), Lc = complete4();
  const auto plan = draw_plan(3, 4, 2, 2, 0.0, 0.0, 11);
  const Matrix Xt = Matrix::from_rows({{1.0, -2.0}, {0.5, 3.0}});
  SpectralGap gr, gc;
  gr.lambda_k1 = 0.5;
  gc.lambda_k1 = 2.0;
  DecoderConfig cfg;
  cfg.variant = DecoderVariant::alternate;
  cfg.pcg_tol = 1e-14;
  const auto res = alternate_decode(Xt, plan, Lr, Lc, gr, gc, cfg);
  CHECK(res.converged && res.iterations > 0);
  const Matrix XL = Lc.right_multiply(res.X), LX = Lr.multiply(res.X);
  double worst = 0.0;
  for (Index i = 0; i < 3; ++i)
    for (Index j = 0; j < 4; ++j) {
      double b = 0.0, m = 0.0;
      for (Index a = 0; a < 2; ++a)
        for (Index c = 0; c < 2; ++c)
          if (plan.omega_r[a] == i && plan.omega_c[c] == j) {
            b = Xt(a, c);
            m = 1.0;
          }
      const double ax = m * res.X(i, j) + (1.0 / 2.0) * XL(i, j) + (1.0 / 0.5) * LX(i, j);
      worst = std::max(worst, std::fabs(ax - b));
    }
  CHECK(worst <= 1e-10);
  // zero right-hand side: x = 0 converged at iteration 0 (solvers.hpp:38-42)
  const auto z = alternate_decode(Matrix(2, 2), plan, Lr, Lc, gr, gc, cfg);
  CHECK(z.converged && z.iterations == 0);
  cfg.gamma = 0.0;
  CHECK_THROWS(std::invalid_argument, alternate_decode(Xt, plan, Lr, Lc, gr, gc, cfg), "gamma must be positive");
  cfg.gamma = 1.0;
  CHECK_THROWS(std::invalid_argument, alternate_decode(Xt, plan, Lc, Lc, gr, gc, cfg), "Laplacians do not match");
  CHECK_THROWS(std::invalid_argument, alternate_decode(Matrix(1, 2), plan, Lr, Lc, gr, gc, cfg), "Xt does not match");
}

int main() {
  test_sparse();
  test_solvers();
  test_graphs();
  test_sampling_and_frpcag();
  test_decoder();
  std::printf("cpcag drop-in: %d checks, %d failed\n", g_checks, g_fail);
  return g_fail == 0 ? 0 : 1;
}
