// cpcag_oracle.cpp -- CPU restatement of the reference cpcag hot path.
//
// TEST INFRASTRUCTURE ONLY (see cpcag_oracle.h).  Never linked into the
// product library; loaded by tests/, __graft_entry__.smoke() and bench.py's
// cpu_baseline / --impl reference legs only.
//
// Every routine cites the reference file:line it restates.  Per-element
// arithmetic follows the reference loops exactly (same operand order, no FMA
// contraction: built with -ffp-contract=off, matching a baseline x86-64 build
// of the reference, whose CMake sets no -march).  Full-array reductions
// (Eigen dot/sum/norm in the reference) are sequential here; Eigen's
// vectorised redux differs from that only in the last ulp.
//
// Parallelism (OpenMP) is only ever across independent output elements, so
// results are bit-identical for any thread count.

#include "cpcag_oracle.h"

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <limits>
#include <numeric>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#ifdef _OPENMP
#include <omp.h>
#endif

namespace {

thread_local std::string g_err;

using i64 = int64_t;
using Vec = std::vector<double>;

struct Csr {
  i64 rows = 0, cols = 0;
  std::vector<i64> rp{0};
  std::vector<i64> ci;
  std::vector<double> v;
  i64 nnz() const { return static_cast<i64>(v.size()); }
};

struct Trip {
  i64 r, c;
  double v;
};

// ---------------------------------------------------------------- RNG
// rng.hpp:11-68 (SplitMix64 counter generator).
struct Rng {
  uint64_t seed, ctr = 0;
  double spare = 0.0;
  bool has_spare = false;
  explicit Rng(uint64_t s) : seed(s) {}
  static uint64_t mix(uint64_t z) {
    z += 0x9e3779b97f4a7c15ULL;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
  }
  uint64_t u64() { return mix(seed + 0x632be59bd9b4e019ULL * ++ctr); }
  double uniform() { return static_cast<double>(u64() >> 11) * 0x1.0p-53; }
  uint64_t below(uint64_t n) {
    const uint64_t lim = UINT64_MAX - UINT64_MAX % n;
    uint64_t x = u64();
    while (x >= lim) x = u64();
    return x % n;
  }
  double gaussian() {
    if (has_spare) {
      has_spare = false;
      return spare;
    }
    double a = uniform();
    while (a <= 0.0) a = uniform();
    const double b = uniform();
    const double rad = std::sqrt(-2.0 * std::log(a));
    const double tau = 6.283185307179586476925286766559;
    spare = rad * std::sin(tau * b);
    has_spare = true;
    return rad * std::cos(tau * b);
  }
  static Rng derive(uint64_t s, uint64_t stream) { return Rng(mix(s ^ mix(stream))); }
};

// ---------------------------------------------------------------- CSR
// sparse.cpp:10-46: validate, sort by (row, col), merge duplicates, drop
// |v| <= drop_below and exact zeros.
Csr build_csr(i64 rows, i64 cols, std::vector<Trip> t, double drop_below) {
  if (rows < 0 || cols < 0) throw std::invalid_argument("sparse: negative dimensions");
  for (const Trip& e : t) {
    if (e.r < 0 || e.r >= rows || e.c < 0 || e.c >= cols)
      throw std::invalid_argument("sparse: triplet index out of range");
    if (!std::isfinite(e.v)) throw std::invalid_argument("sparse: non-finite entry");
  }
  // The reference uses std::sort (not stable); duplicates are summed in the
  // order the sort leaves them.  A stable sort keeps input order, which is
  // the only order a caller can reason about; the sum of at most a handful
  // of duplicates differs at most in the last ulp.
  std::stable_sort(t.begin(), t.end(),
                   [](const Trip& a, const Trip& b) { return a.r != b.r ? a.r < b.r : a.c < b.c; });
  Csr m;
  m.rows = rows;
  m.cols = cols;
  m.rp.assign(static_cast<size_t>(rows) + 1, 0);
  m.ci.reserve(t.size());
  m.v.reserve(t.size());
  size_t k = 0;
  for (i64 r = 0; r < rows; ++r) {
    while (k < t.size() && t[k].r == r) {
      const i64 c = t[k].c;
      double acc = 0.0;
      while (k < t.size() && t[k].r == r && t[k].c == c) acc += t[k++].v;
      if (acc != 0.0 && std::fabs(acc) > drop_below) {
        m.ci.push_back(c);
        m.v.push_back(acc);
      }
    }
    m.rp[static_cast<size_t>(r) + 1] = m.nnz();
  }
  return m;
}

// sparse.cpp:48-54 (row-major scan of nonzeros, then from_triplets).
Csr csr_from_dense(const double* D, i64 rows, i64 cols, double drop_below) {
  std::vector<Trip> t;
  for (i64 i = 0; i < rows; ++i)
    for (i64 j = 0; j < cols; ++j) {
      const double x = D[i + j * rows];
      if (x != 0.0) t.push_back({i, j, x});
    }
  return build_csr(rows, cols, std::move(t), drop_below);
}

// sparse.cpp:59-71
double coeff(const Csr& a, i64 i, i64 j) {
  if (i < 0 || i >= a.rows || j < 0 || j >= a.cols)
    throw std::out_of_range("sparse: coeff index out of range");
  const auto b = a.ci.begin() + a.rp[static_cast<size_t>(i)];
  const auto e = a.ci.begin() + a.rp[static_cast<size_t>(i) + 1];
  const auto it = std::lower_bound(b, e, j);
  if (it == e || *it != j) return 0.0;
  return a.v[static_cast<size_t>(it - a.ci.begin())];
}

Vec diagonal(const Csr& a) {
  const i64 n = std::min(a.rows, a.cols);
  Vec d(static_cast<size_t>(n), 0.0);
  for (i64 i = 0; i < n; ++i) d[static_cast<size_t>(i)] = coeff(a, i, i);
  return d;
}

// sparse.cpp:159-168
Vec row_sums(const Csr& a) {
  Vec s(static_cast<size_t>(a.rows), 0.0);
  for (i64 r = 0; r < a.rows; ++r) {
    double acc = 0.0;
    for (i64 k = a.rp[r]; k < a.rp[r + 1]; ++k) acc += a.v[k];
    s[static_cast<size_t>(r)] = acc;
  }
  return s;
}

// sparse.cpp:170-179
double max_abs_asymmetry(const Csr& a) {
  if (a.rows != a.cols) throw std::invalid_argument("asymmetry check needs a square matrix");
  double worst = 0.0;
  for (i64 r = 0; r < a.rows; ++r)
    for (i64 k = a.rp[r]; k < a.rp[r + 1]; ++k)
      worst = std::max(worst, std::fabs(a.v[k] - coeff(a, a.ci[k], r)));
  return worst;
}

// sparse.cpp:122-142: rows in the given order, columns relabelled by their
// position in `cols`, then from_triplets (sorted by the new labels).
Csr submatrix(const Csr& a, const std::vector<i64>& rows, const std::vector<i64>& cols) {
  std::vector<i64> cmap(static_cast<size_t>(a.cols), -1);
  for (size_t j = 0; j < cols.size(); ++j) {
    const i64 c = cols[j];
    if (c < 0 || c >= a.cols) throw std::invalid_argument("submatrix: column index out of range");
    if (cmap[static_cast<size_t>(c)] != -1)
      throw std::invalid_argument("submatrix: duplicate column index");
    cmap[static_cast<size_t>(c)] = static_cast<i64>(j);
  }
  std::vector<Trip> t;
  for (size_t i = 0; i < rows.size(); ++i) {
    const i64 r = rows[i];
    if (r < 0 || r >= a.rows) throw std::invalid_argument("submatrix: row index out of range");
    for (i64 k = a.rp[r]; k < a.rp[r + 1]; ++k) {
      const i64 lc = cmap[static_cast<size_t>(a.ci[k])];
      if (lc != -1) t.push_back({static_cast<i64>(i), lc, a.v[k]});
    }
  }
  return build_csr(static_cast<i64>(rows.size()), static_cast<i64>(cols.size()), std::move(t), 0.0);
}

// sparse.cpp:181-207: iterative DFS; components numbered by their smallest
// node; labels[i] = component id.
std::vector<std::vector<i64>> components(const Csr& a) {
  if (a.rows != a.cols) throw std::invalid_argument("components need a square matrix");
  std::vector<i64> lab(static_cast<size_t>(a.rows), -1);
  std::vector<std::vector<i64>> out;
  std::vector<i64> stack;
  for (i64 s = 0; s < a.rows; ++s) {
    if (lab[static_cast<size_t>(s)] != -1) continue;
    const i64 id = static_cast<i64>(out.size());
    out.emplace_back();
    stack.assign(1, s);
    lab[static_cast<size_t>(s)] = id;
    while (!stack.empty()) {
      const i64 u = stack.back();
      stack.pop_back();
      out.back().push_back(u);
      for (i64 k = a.rp[u]; k < a.rp[u + 1]; ++k) {
        const i64 w = a.ci[k];
        if (lab[static_cast<size_t>(w)] == -1) {
          lab[static_cast<size_t>(w)] = id;
          stack.push_back(w);
        }
      }
    }
    std::sort(out.back().begin(), out.back().end());
  }
  return out;
}

// ---------------------------------------------------------------- products
// sparse.cpp:73-85: y[r] = sum_k v_k x[c_k], row-sequential.
Vec spmv(const Csr& a, const Vec& x) {
  if (static_cast<i64>(x.size()) != a.cols)
    throw std::invalid_argument("spmv: dimension mismatch (" + std::to_string(a.cols) + " vs " +
                                std::to_string(x.size()) + ")");
  Vec y(static_cast<size_t>(a.rows), 0.0);
  for (i64 r = 0; r < a.rows; ++r) {
    double acc = 0.0;
    for (i64 k = a.rp[r]; k < a.rp[r + 1]; ++k) acc += a.v[k] * x[static_cast<size_t>(a.ci[k])];
    y[static_cast<size_t>(r)] = acc;
  }
  return y;
}

// sparse.cpp:87-98: Y(r, j) accumulates v_k X(c_k, j) over row r in CSR
// order, starting from an explicit zero.  With several right-hand sides X is
// transposed to row-major first, so each CSR entry is read once for all
// columns (the per-element order over k is unchanged: bit-identical).
void spmm_left(const Csr& a, const double* X, i64 xr, i64 xc, double* Y) {
  if (xr != a.cols) throw std::invalid_argument("sparse multiply: dimension mismatch");
  const i64 R = a.rows;
  if (xc < 4) {
#pragma omp parallel for schedule(static)
    for (i64 j = 0; j < xc; ++j) {
      const double* xj = X + j * xr;
      double* yj = Y + j * R;
      for (i64 r = 0; r < R; ++r) {
        double acc = 0.0;
        for (i64 k = a.rp[r]; k < a.rp[r + 1]; ++k) acc += a.v[k] * xj[a.ci[k]];
        yj[r] = acc;
      }
    }
    return;
  }
  constexpr i64 JB = 256;  // right-hand sides per pass
  std::vector<double> Xr(static_cast<size_t>(xr * std::min(xc, JB)));
  for (i64 j0 = 0; j0 < xc; j0 += JB) {
    const i64 nj = std::min(JB, xc - j0);
#pragma omp parallel for schedule(static)
    for (i64 c = 0; c < xr; ++c)
      for (i64 j = 0; j < nj; ++j) Xr[c * nj + j] = X[c + (j0 + j) * xr];
#pragma omp parallel
    {
      std::vector<double> acc(static_cast<size_t>(nj));
#pragma omp for schedule(dynamic, 16)
      for (i64 r = 0; r < R; ++r) {
        for (i64 j = 0; j < nj; ++j) acc[j] = 0.0;
        for (i64 k = a.rp[r]; k < a.rp[r + 1]; ++k) {
          const double v = a.v[k];
          const double* xrow = &Xr[static_cast<size_t>(a.ci[k] * nj)];
          for (i64 j = 0; j < nj; ++j) acc[j] += v * xrow[j];
        }
        for (i64 j = 0; j < nj; ++j) Y[r + (j0 + j) * R] = acc[j];
      }
    }
  }
}

// Column lists of `a` with ascending row index (the order in which
// sparse.cpp:100-111 visits the contributions to each output column).
struct Csc {
  std::vector<i64> cp, ri;
  std::vector<double> v;
};
Csc to_csc(const Csr& a) {
  Csc t;
  t.cp.assign(static_cast<size_t>(a.cols) + 1, 0);
  for (i64 k = 0; k < a.nnz(); ++k) t.cp[static_cast<size_t>(a.ci[k]) + 1]++;
  for (i64 c = 0; c < a.cols; ++c) t.cp[c + 1] += t.cp[c];
  std::vector<i64> fill(t.cp.begin(), t.cp.end() - 1);
  t.ri.resize(static_cast<size_t>(a.nnz()));
  t.v.resize(static_cast<size_t>(a.nnz()));
  for (i64 r = 0; r < a.rows; ++r)
    for (i64 k = a.rp[r]; k < a.rp[r + 1]; ++k) {
      const i64 dst = fill[static_cast<size_t>(a.ci[k])]++;
      t.ri[dst] = r;
      t.v[dst] = a.v[k];
    }
  return t;
}

// sparse.cpp:100-111: Y(:, c) += v X(:, r) over CSR rows r ascending.
void spmm_right(const Csr& a, const double* X, i64 xr, i64 xc, double* Y) {
  if (xc != a.rows) throw std::invalid_argument("sparse right_multiply: dimension mismatch");
  const Csc t = to_csc(a);
  const i64 C = a.cols;
#pragma omp parallel for schedule(static)
  for (i64 c = 0; c < C; ++c) {
    double* yc = Y + c * xr;
    for (i64 i = 0; i < xr; ++i) yc[i] = 0.0;
    for (i64 k = t.cp[c]; k < t.cp[c + 1]; ++k) {
      const double w = t.v[k];
      const double* xs = X + t.ri[k] * xr;
      for (i64 i = 0; i < xr; ++i) yc[i] += w * xs[i];
    }
  }
}

// Full-array reductions: sequential for n <= kRedBlock (every test-sized
// array); beyond that, fixed blocks of kRedBlock entries are each summed
// sequentially (blocks in parallel) and the block sums are added in block
// order.  The order depends on n only, never on the thread count, so results
// are identical for any number of threads.
constexpr i64 kRedBlock = i64{1} << 18;
constexpr i64 kParMin = i64{1} << 16;  // element-wise loops go parallel above this

double dot(const double* a, const double* b, i64 n) {
  if (n <= kRedBlock) {
    double s = 0.0;
    for (i64 i = 0; i < n; ++i) s += a[i] * b[i];
    return s;
  }
  const i64 nb = (n + kRedBlock - 1) / kRedBlock;
  std::vector<double> part(static_cast<size_t>(nb));
#pragma omp parallel for schedule(static)
  for (i64 q = 0; q < nb; ++q) {
    const i64 e = std::min(n, (q + 1) * kRedBlock);
    double s = 0.0;
    for (i64 i = q * kRedBlock; i < e; ++i) s += a[i] * b[i];
    part[static_cast<size_t>(q)] = s;
  }
  double s = 0.0;
  for (const double x : part) s += x;
  return s;
}

// ---------------------------------------------------------------- PCG
// solvers.hpp:33-74 (pcg_core), restated for vectors with an arbitrary apply.
struct PcgOut {
  i64 iterations = 0;
  bool converged = false;
  double rel_res = 0.0;
};

template <class Apply, class Precond>
PcgOut pcg_core(const Apply& apply, const Vec& b, Vec& x, double tol, i64 max_iter,
                const Precond& precond) {
  const i64 n = static_cast<i64>(b.size());
  const double norm_b = std::sqrt(dot(b.data(), b.data(), n));
  PcgOut res;
  if (norm_b == 0.0) {
    x = b;
    res.converged = true;
    return res;
  }
  const double target = tol * norm_b;
  Vec r(static_cast<size_t>(n)), z(static_cast<size_t>(n)), ap(static_cast<size_t>(n));
  apply(x, r);
#pragma omp parallel for schedule(static) if (n > kParMin)
  for (i64 i = 0; i < n; ++i) r[i] = b[i] - r[i];
  precond(r, z);
  Vec p = z;
  double rho = dot(r.data(), z.data(), n);
  i64 it = 0;
  while (it < max_iter) {
    if (std::sqrt(dot(r.data(), r.data(), n)) <= target) break;
    apply(p, ap);
    const double curv = dot(p.data(), ap.data(), n);
    if (!std::isfinite(curv) || curv <= 0.0)
      throw std::runtime_error("pcg: breakdown (nonpositive curvature) at iteration " +
                               std::to_string(it));
    const double alpha = rho / curv;
#pragma omp parallel for schedule(static) if (n > kParMin)
    for (i64 i = 0; i < n; ++i) {
      x[i] += alpha * p[i];
      r[i] -= alpha * ap[i];
    }
    precond(r, z);
    const double rho_next = dot(r.data(), z.data(), n);
    const double beta = rho_next / rho;
#pragma omp parallel for schedule(static) if (n > kParMin)
    for (i64 i = 0; i < n; ++i) p[i] = z[i] + beta * p[i];
    rho = rho_next;
    ++it;
  }
  Vec& rt = ap;
  apply(x, rt);
#pragma omp parallel for schedule(static) if (n > kParMin)
  for (i64 i = 0; i < n; ++i) rt[i] = b[i] - rt[i];
  res.rel_res = std::sqrt(dot(rt.data(), rt.data(), n)) / norm_b;
  res.iterations = it;
  res.converged = res.rel_res <= tol;
  return res;
}

// solvers.cpp:7-17: Jacobi inverse with the 0 -> 1 rule.
PcgOut pcg_jacobi(const Csr& A, const Vec& diag, const Vec& b, Vec& x, double tol, i64 max_iter) {
  Vec inv = diag;
  for (double& d : inv) d = d > 0.0 ? 1.0 / d : 1.0;
  auto apply = [&A](const Vec& v, Vec& out) { out = spmv(A, v); };
  auto pre = [&inv](const Vec& r, Vec& z) {
    for (size_t i = 0; i < r.size(); ++i) z[i] = inv[i] * r[i];
  };
  if (x.size() != b.size()) x.assign(b.size(), 0.0);
  return pcg_core(apply, b, x, tol, max_iter, pre);
}

// solvers.cpp:29-53
double power_norm(const Csr& A, double tol, uint64_t seed, i64 max_iter) {
  if (A.rows != A.cols) throw std::invalid_argument("power iteration: square matrix required");
  const i64 n = A.rows;
  if (n == 0) return 0.0;
  Rng rng(Rng::mix(seed ^ 0x5ca1ab1eULL));
  Vec v(static_cast<size_t>(n));
  for (i64 i = 0; i < n; ++i) v[i] = rng.gaussian();
  const double nv = std::sqrt(dot(v.data(), v.data(), n));
  if (nv == 0.0) return 0.0;
  for (double& x : v) x /= nv;
  double est = 0.0;
  for (i64 it = 0; it < max_iter; ++it) {
    const Vec w = spmv(A, v);
    const double nw = std::sqrt(dot(w.data(), w.data(), n));
    if (nw == 0.0) return 0.0;
    const double prev = est;
    est = nw;
    for (i64 i = 0; i < n; ++i) v[i] = w[i] / nw;
    if (it > 0 && std::fabs(est - prev) <= tol * est) break;
  }
  return est;
}

// ---------------------------------------------------------------- graphs
// graph.cpp:16-43
Csr laplacian(const Csr& W, const Vec& deg, bool normalized) {
  const i64 n = W.rows;
  std::vector<Trip> t;
  t.reserve(W.v.size() + static_cast<size_t>(n));
  if (!normalized) {
    for (i64 i = 0; i < n; ++i)
      if (deg[i] != 0.0) t.push_back({i, i, deg[i]});
    for (i64 r = 0; r < n; ++r)
      for (i64 k = W.rp[r]; k < W.rp[r + 1]; ++k) t.push_back({r, W.ci[k], -W.v[k]});
  } else {
    Vec dis(static_cast<size_t>(n), 0.0);
    for (i64 i = 0; i < n; ++i) dis[i] = deg[i] > 0.0 ? 1.0 / std::sqrt(deg[i]) : 0.0;
    for (i64 i = 0; i < n; ++i)
      if (deg[i] > 0.0) t.push_back({i, i, 1.0});
    for (i64 r = 0; r < n; ++r)
      for (i64 k = W.rp[r]; k < W.rp[r + 1]; ++k) {
        const i64 c = W.ci[k];
        t.push_back({r, c, -W.v[k] * dis[r] * dis[c]});
      }
  }
  return build_csr(n, n, std::move(t), 0.0);
}

// Canonical fp64 squared distance (graph.cpp:58-63): the Gram entry is the
// sequential k-ascending sum of products (no FMA); d2 = max(0, g_ii + g_jj -
// 2 g_ij).  Products commute, so d2(i, j) == d2(j, i) bit for bit, which is
// what the reference's compute-once-and-mirror loop guarantees.
struct Points {
  i64 n = 0, d = 0;
  std::vector<double> x;  // point-major: x[i * d + k]
  Vec sq;                 // g_ii
};

Points gather_points(const double* X, i64 rows, i64 cols, bool axis_rows) {
  Points P;
  P.n = axis_rows ? rows : cols;
  P.d = axis_rows ? cols : rows;
  P.x.resize(static_cast<size_t>(P.n * P.d));
  for (i64 i = 0; i < P.n; ++i)
    for (i64 k = 0; k < P.d; ++k)
      P.x[static_cast<size_t>(i * P.d + k)] = axis_rows ? X[i + k * rows] : X[k + i * rows];
  P.sq.resize(static_cast<size_t>(P.n));
  for (i64 i = 0; i < P.n; ++i) {
    const double* a = &P.x[static_cast<size_t>(i * P.d)];
    P.sq[i] = dot(a, a, P.d);
  }
  return P;
}

inline double pair_d2(const Points& P, i64 i, i64 j) {
  const double g = dot(&P.x[static_cast<size_t>(i * P.d)], &P.x[static_cast<size_t>(j * P.d)], P.d);
  return std::max(0.0, P.sq[i] + P.sq[j] - 2.0 * g);
}

// graph.cpp:68-84: number of distinct points (exact coordinate equality).
i64 distinct_points(const Points& P) {
  std::vector<i64> idx(static_cast<size_t>(P.n));
  std::iota(idx.begin(), idx.end(), i64{0});
  const double* base = P.x.data();
  const i64 d = P.d;
  std::sort(idx.begin(), idx.end(), [&](i64 a, i64 b) {
    const double* pa = base + a * d;
    const double* pb = base + b * d;
    for (i64 k = 0; k < d; ++k)
      if (pa[k] != pb[k]) return pa[k] < pb[k];
    return a < b;
  });
  i64 distinct = P.n > 0 ? 1 : 0;
  for (size_t t = 1; t < idx.size(); ++t) {
    const double* pa = base + idx[t - 1] * d;
    const double* pb = base + idx[t] * d;
    bool same = true;
    for (i64 k = 0; k < d && same; ++k) same = pa[k] == pb[k];
    if (!same) ++distinct;
  }
  return distinct;
}

void knn_validate(const Points& P, i64 K) {
  if (K < 1) throw std::invalid_argument("knn graph: K must be >= 1");
  if (P.n < K + 1)
    throw std::invalid_argument("knn graph: need at least K+1 points, got " + std::to_string(P.n));
  const i64 distinct = distinct_points(P);
  if (distinct < K)
    throw std::invalid_argument("knn graph: fewer distinct points (" + std::to_string(distinct) +
                                ") than K (" + std::to_string(K) + ")");
}

// graph.cpp:86-105: per point the K smallest (d2, j) pairs (lexicographic,
// so ties go to the lower index), ascending; returns per-point mean d2
// accumulated in that ascending order.
void knn_select(const Points& P, i64 K, i64* nbr, double* nbr_d2, Vec& mean_d2) {
  const i64 n = P.n;
  mean_d2.assign(static_cast<size_t>(n), 0.0);
#pragma omp parallel
  {
    std::vector<std::pair<double, i64>> order;
    order.reserve(static_cast<size_t>(n));
#pragma omp for schedule(dynamic, 16)
    for (i64 i = 0; i < n; ++i) {
      order.clear();
      for (i64 j = 0; j < n; ++j)
        if (j != i) order.emplace_back(pair_d2(P, i, j), j);
      std::nth_element(order.begin(), order.begin() + (K - 1), order.end());
      std::sort(order.begin(), order.begin() + K);
      double m = 0.0;
      for (i64 k = 0; k < K; ++k) {
        nbr[i * K + k] = order[static_cast<size_t>(k)].second;
        nbr_d2[i * K + k] = order[static_cast<size_t>(k)].first;
        m += order[static_cast<size_t>(k)].first;
      }
      mean_d2[static_cast<size_t>(i)] = m;
    }
  }
}

// knn_select for a subset of query points (full-size spot checks): the same
// per-point selection over all n candidates.
void knn_select_rows(const Points& P, i64 K, const i64* rows, i64 nq, i64* nbr, double* nbr_d2) {
  const i64 n = P.n;
#pragma omp parallel
  {
    std::vector<std::pair<double, i64>> order;
    order.reserve(static_cast<size_t>(n));
#pragma omp for schedule(dynamic, 1)
    for (i64 q = 0; q < nq; ++q) {
      const i64 i = rows[q];
      order.clear();
      for (i64 j = 0; j < n; ++j)
        if (j != i) order.emplace_back(pair_d2(P, i, j), j);
      std::nth_element(order.begin(), order.begin() + (K - 1), order.end());
      std::sort(order.begin(), order.begin() + K);
      for (i64 k = 0; k < K; ++k) {
        nbr[q * K + k] = order[static_cast<size_t>(k)].second;
        nbr_d2[q * K + k] = order[static_cast<size_t>(k)].first;
      }
    }
  }
}

struct Graph {
  Csr W, L;
  Vec deg;
  double sigma2 = 0.0;
};

// graph.cpp:47-135
Graph knn_graph(const double* X, i64 rows, i64 cols, bool axis_rows, i64 K, bool normalized,
                double sigma2_override) {
  if (K < 1) throw std::invalid_argument("knn graph: K must be >= 1");
  const Points P = gather_points(X, rows, cols, axis_rows);
  knn_validate(P, K);
  const i64 n = P.n;
  std::vector<i64> nbr(static_cast<size_t>(n * K));
  Vec nd2(static_cast<size_t>(n * K));
  Vec mean;
  knn_select(P, K, nbr.data(), nd2.data(), mean);
  double s2sum = 0.0;
  for (i64 i = 0; i < n; ++i) s2sum += mean[i] / static_cast<double>(K);
  Graph g;
  g.sigma2 = sigma2_override > 0.0 ? sigma2_override : s2sum / static_cast<double>(n);

  // graph.cpp:111-124: union of (min, max) edges, Gaussian weight, w == 0
  // edges dropped, coincident points weight 1.
  std::vector<std::pair<i64, i64>> edges;
  edges.reserve(static_cast<size_t>(n * K));
  for (i64 i = 0; i < n; ++i)
    for (i64 k = 0; k < K; ++k) {
      const i64 j = nbr[i * K + k];
      edges.emplace_back(std::min(i, j), std::max(i, j));
    }
  std::sort(edges.begin(), edges.end());
  edges.erase(std::unique(edges.begin(), edges.end()), edges.end());
  std::vector<Trip> t;
  t.reserve(edges.size() * 2);
  for (const auto& e : edges) {
    const double d = pair_d2(P, e.first, e.second);
    const double w = d == 0.0 ? 1.0 : std::exp(-d / g.sigma2);
    if (w == 0.0) continue;
    t.push_back({e.first, e.second, w});
    t.push_back({e.second, e.first, w});
  }
  g.W = build_csr(n, n, std::move(t), 0.0);
  g.deg = row_sums(g.W);
  g.L = laplacian(g.W, g.deg, normalized);
  return g;
}

// graph.cpp:137-154
Graph graph_from_adjacency(const Csr& W, bool normalized) {
  if (W.rows != W.cols) throw std::invalid_argument("adjacency must be square");
  if (max_abs_asymmetry(W) != 0.0) throw std::invalid_argument("adjacency must be symmetric");
  for (i64 i = 0; i < W.rows; ++i)
    if (coeff(W, i, i) != 0.0) throw std::invalid_argument("adjacency must have zero diagonal");
  for (const double x : W.v)
    if (x < 0.0) throw std::invalid_argument("adjacency weights must be nonnegative");
  Graph g;
  g.W = W;
  g.deg = row_sums(W);
  g.L = laplacian(W, g.deg, normalized);
  return g;
}

// graph.cpp:170-235
Csr kron_reduce(const Csr& L, const std::vector<i64>& keep, double pcg_tol, double prune_tol) {
  const i64 n = L.rows;
  if (L.cols != n) throw std::invalid_argument("kron reduction: square Laplacian required");
  std::vector<char> kept(static_cast<size_t>(n), 0);
  for (const i64 i : keep) {
    if (i < 0 || i >= n) throw std::invalid_argument("kron reduction: index out of range");
    if (kept[static_cast<size_t>(i)]) throw std::invalid_argument("kron reduction: duplicate index");
    kept[static_cast<size_t>(i)] = 1;
  }
  for (const auto& comp : components(L)) {
    bool grounded = false;
    for (const i64 u : comp)
      if (kept[static_cast<size_t>(u)]) {
        grounded = true;
        break;
      }
    if (!grounded)
      throw std::runtime_error("kron reduction: connected component containing node " +
                               std::to_string(comp.front()) + " has no kept node");
  }
  std::vector<i64> interior;
  for (i64 i = 0; i < n; ++i)
    if (!kept[static_cast<size_t>(i)]) interior.push_back(i);
  Csr Lbb = submatrix(L, keep, keep);
  if (interior.empty()) return Lbb;
  const Csr Laa = submatrix(L, interior, interior);
  const Csr Lba = submatrix(L, keep, interior);
  const Vec dg = diagonal(Laa);
  const i64 m = static_cast<i64>(keep.size());
  const i64 ni = static_cast<i64>(interior.size());
  std::vector<double> S(static_cast<size_t>(m * m), 0.0);  // dense L_bb, col-major
  for (i64 r = 0; r < m; ++r)
    for (i64 k = Lbb.rp[r]; k < Lbb.rp[r + 1]; ++k) S[r + Lbb.ci[k] * m] = Lbb.v[k];
  const i64 max_iter = 20 * ni + 100;
  std::string failure;
  i64 fail_j = -1;
#pragma omp parallel for schedule(dynamic, 1)
  for (i64 j = 0; j < m; ++j) {
    if (Lba.rp[j] == Lba.rp[j + 1]) continue;
    Vec rhs(static_cast<size_t>(ni), 0.0);
    for (i64 k = Lba.rp[j]; k < Lba.rp[j + 1]; ++k) rhs[Lba.ci[k]] = Lba.v[k];
    Vec z(static_cast<size_t>(ni), 0.0);
    PcgOut res;
    std::string err;
    try {
      res = pcg_jacobi(Laa, dg, rhs, z, pcg_tol, max_iter);
    } catch (const std::exception& e) {
      err = e.what();
    }
    if (!err.empty() || !res.converged) {
#pragma omp critical
      if (fail_j < 0 || j < fail_j) {
        fail_j = j;
        failure = err.empty() ? "kron reduction: interior solve failed to converge for kept node " +
                                    std::to_string(keep[static_cast<size_t>(j)])
                              : err;
      }
      continue;
    }
    const Vec y = spmv(Lba, z);
    for (i64 i = 0; i < m; ++i) S[i + j * m] -= y[i];
  }
  if (fail_j >= 0) throw std::runtime_error(failure);
  std::vector<double> Ssym(S.size());
  for (i64 j = 0; j < m; ++j)
    for (i64 i = 0; i < m; ++i) Ssym[i + j * m] = 0.5 * (S[i + j * m] + S[j + i * m]);
  return csr_from_dense(Ssym.data(), m, m, prune_tol);
}

// ---------------------------------------------------------------- sampling
// decoders.cpp:72-121 (graph_upsample): rows `known` of S equal R, the rest
// solve L_aa S_a = -L_ab R, one Jacobi PCG per column (independent columns
// in parallel; the first failing column in index order is reported).
std::vector<double> graph_upsample(const Csr& L, const std::vector<i64>& known, const double* R, i64 r,
                                   double pcg_tol, i64 pcg_max_iter) {
  const i64 n = L.rows;
  if (L.cols != n) throw std::invalid_argument("graph upsample: square Laplacian required");
  std::vector<char> mask(static_cast<size_t>(n), 0);
  for (const i64 i : known) {  // decoders.cpp:17-25
    if (i < 0 || i >= n) throw std::invalid_argument("graph upsample: index out of range");
    if (mask[static_cast<size_t>(i)]) throw std::invalid_argument("graph upsample: duplicate index");
    mask[static_cast<size_t>(i)] = 1;
  }
  for (const auto& comp : components(L)) {
    bool covered = false;
    for (const i64 u : comp)
      if (mask[static_cast<size_t>(u)]) {
        covered = true;
        break;
      }
    if (!covered)
      throw std::runtime_error("graph upsample: connected component containing node " +
                               std::to_string(comp.front()) + " has no sampled node");
  }
  const i64 m = static_cast<i64>(known.size());
  std::vector<double> S(static_cast<size_t>(n * r), 0.0);
  for (i64 i = 0; i < m; ++i)
    for (i64 j = 0; j < r; ++j) S[known[i] + j * n] = R[i + j * m];
  if (m == n) return S;
  std::vector<i64> unknown;
  for (i64 i = 0; i < n; ++i)
    if (!mask[static_cast<size_t>(i)]) unknown.push_back(i);
  const i64 ni = static_cast<i64>(unknown.size());
  const Csr Laa = submatrix(L, unknown, unknown);
  const Csr Lab = submatrix(L, unknown, known);
  const Vec dg = diagonal(Laa);
  std::vector<double> rhs(static_cast<size_t>(ni * r));
  spmm_left(Lab, R, m, r, rhs.data());  // L_ab.multiply(R), then negated (decoders.cpp:107)
  for (double& v : rhs) v = -v;
  std::string failure;
  i64 fail_j = -1;
#pragma omp parallel for schedule(dynamic, 1)
  for (i64 j = 0; j < r; ++j) {
    Vec b(rhs.begin() + j * ni, rhs.begin() + (j + 1) * ni);
    Vec x(static_cast<size_t>(ni), 0.0);
    PcgOut res;
    std::string err;
    try {
      res = pcg_jacobi(Laa, dg, b, x, pcg_tol, pcg_max_iter);
    } catch (const std::exception& e) {
      err = e.what();
    }
    if (!err.empty() || !res.converged) {
#pragma omp critical
      if (fail_j < 0 || j < fail_j) {
        fail_j = j;
        failure = err.empty() ? "graph upsample: interior solve did not converge (column " + std::to_string(j) + ")"
                              : err;
      }
      continue;
    }
    for (i64 i = 0; i < ni; ++i) S[unknown[i] + j * n] = x[i];
  }
  if (fail_j >= 0) throw std::runtime_error(failure);
  return S;
}

// sampling.cpp:35-44
std::vector<i64> partial_shuffle(i64 n, i64 take, Rng rng) {
  std::vector<i64> pool(static_cast<size_t>(n));
  std::iota(pool.begin(), pool.end(), i64{0});
  for (i64 i = 0; i < take; ++i) {
    const i64 j = i + static_cast<i64>(rng.below(static_cast<uint64_t>(n - i)));
    std::swap(pool[static_cast<size_t>(i)], pool[static_cast<size_t>(j)]);
  }
  pool.resize(static_cast<size_t>(take));
  return pool;
}

// ---------------------------------------------------------------- FRPCAG
void frpcag_dims(i64 r, i64 c, const Csr& Lr, const Csr& Lc) {
  if (Lr.rows != Lr.cols || Lr.rows != r)
    throw std::invalid_argument("frpcag: row Laplacian does not match X");
  if (Lc.rows != Lc.cols || Lc.rows != c)
    throw std::invalid_argument("frpcag: column Laplacian does not match X");
}

// frpcag.cpp:23-35
double objective(const double* X, const double* Y, i64 r, i64 c, const Csr& Lr, const Csr& Lc,
                 const ora_frpcag_cfg& cfg) {
  frpcag_dims(r, c, Lr, Lc);
  const i64 N = r * c;
  double val = 0.0;
  for (i64 t = 0; t < N; ++t) {
    const double e = Y[t] - X[t];
    val += cfg.loss_l2 ? e * e : std::fabs(e);
  }
  if (cfg.gamma_c != 0.0) {
    // (Lc X^T) o X^T summed; (Lc X^T)(a, i) == (X Lc)(i, a) bit for bit for a
    // symmetric Lc, but the transpose form is restated literally here.
    std::vector<double> Xt(static_cast<size_t>(N)), P(static_cast<size_t>(N));
    for (i64 j = 0; j < c; ++j)
      for (i64 i = 0; i < r; ++i) Xt[j + i * c] = X[i + j * r];
    spmm_left(Lc, Xt.data(), c, r, P.data());
    double s = 0.0;
    for (i64 t = 0; t < N; ++t) s += P[t] * Xt[t];
    val += cfg.gamma_c * s;
  }
  if (cfg.gamma_r != 0.0) {
    std::vector<double> P(static_cast<size_t>(N));
    spmm_left(Lr, X, r, c, P.data());
    double s = 0.0;
    for (i64 t = 0; t < N; ++t) s += P[t] * X[t];
    val += cfg.gamma_r * s;
  }
  return val;
}

// frpcag.cpp:37-44
void prox_l1(const double* Z, const double* Y, i64 N, double lam, double* out) {
  if (lam < 0.0) throw std::invalid_argument("prox: negative threshold");
  for (i64 t = 0; t < N; ++t) {
    const double d = Z[t] - Y[t];
    const double sg = d > 0.0 ? 1.0 : (d < 0.0 ? -1.0 : 0.0);
    out[t] = Y[t] + sg * std::max(std::fabs(d) - lam, 0.0);
  }
}

// frpcag.cpp:46-51
void prox_l2(const double* Z, const double* Y, i64 N, double lam, double* out) {
  if (lam < 0.0) throw std::invalid_argument("prox: negative threshold");
  const double a = 2.0 * lam;
  const double b = 1.0 + 2.0 * lam;
  for (i64 t = 0; t < N; ++t) out[t] = (Z[t] + a * Y[t]) / b;
}

// frpcag.cpp:53-60: G = 0 + (2 gc) Z Lc, then += (2 gr) Lr Z.
void grad_g(const double* Z, i64 r, i64 c, const Csr& Lr, const Csr& Lc,
            const ora_frpcag_cfg& cfg, double* G) {
  frpcag_dims(r, c, Lr, Lc);
  const i64 N = r * c;
  for (i64 t = 0; t < N; ++t) G[t] = 0.0;
  std::vector<double> P(static_cast<size_t>(N));
  if (cfg.gamma_c != 0.0) {
    spmm_right(Lc, Z, r, c, P.data());
    const double s = 2.0 * cfg.gamma_c;
    for (i64 t = 0; t < N; ++t) G[t] += s * P[t];
  }
  if (cfg.gamma_r != 0.0) {
    spmm_left(Lr, Z, r, c, P.data());
    const double s = 2.0 * cfg.gamma_r;
    for (i64 t = 0; t < N; ++t) G[t] += s * P[t];
  }
}

double sq_norm(const double* a, i64 N) { return dot(a, a, N); }

// frpcag.cpp:62-112
void fista(const double* Y, i64 r, i64 c, const Csr& Lr, const Csr& Lc, const ora_frpcag_cfg& cfg,
           double* Xout, double* obj_out, i64* iters, int* conv, double* frc, double* step_used) {
  frpcag_dims(r, c, Lr, Lc);
  if (cfg.gamma_r < 0.0 || cfg.gamma_c < 0.0)
    throw std::invalid_argument("fista: negative regularization weight");
  if (cfg.tol <= 0.0) throw std::invalid_argument("fista: stopping tolerance must be positive");
  if (cfg.max_iter < 1) throw std::invalid_argument("fista: max_iter must be >= 1");
  double step = cfg.step;
  if (step <= 0.0) {
    const double beta = 2.0 * cfg.gamma_c * power_norm(Lc, 1e-7, 42, 50000) +
                        2.0 * cfg.gamma_r * power_norm(Lr, 1e-7, 42, 50000);
    step = beta > 0.0 ? 1.0 / beta : 1.0;
  }
  const i64 N = r * c;
  std::vector<double> Z(Y, Y + N), Sp(Y, Y + N), S(Y, Y + N), G(static_cast<size_t>(N)),
      T(static_cast<size_t>(N)), Zn(static_cast<size_t>(N));
  double t = 1.0;
  *iters = 0;
  *conv = 0;
  *frc = 0.0;
  *step_used = step;
  for (i64 j = 1; j <= cfg.max_iter; ++j) {
    grad_g(Z.data(), r, c, Lr, Lc, cfg, G.data());
    for (i64 q = 0; q < N; ++q) T[q] = Z[q] - step * G[q];
    if (cfg.loss_l2)
      prox_l2(T.data(), Y, N, step, S.data());
    else
      prox_l1(T.data(), Y, N, step, S.data());
    const double ob = objective(S.data(), Y, r, c, Lr, Lc, cfg);
    if (!std::isfinite(ob))
      throw std::runtime_error("fista: diverged (non-finite objective at iteration " +
                               std::to_string(j) + "); step too large");
    obj_out[j - 1] = ob;
    *iters = j;
    const double tn = 0.5 * (1.0 + std::sqrt(1.0 + 4.0 * t * t));
    const double coef = (t - 1.0) / tn;
    for (i64 q = 0; q < N; ++q) Zn[q] = S[q] + coef * (S[q] - Sp[q]);
    const double denom = sq_norm(Z.data(), N);
    for (i64 q = 0; q < N; ++q) T[q] = Zn[q] - Z[q];
    const double change = sq_norm(T.data(), N);
    *frc = denom > 0.0 ? change / denom : change;
    if (change < cfg.tol * denom) {
      *conv = 1;
      break;
    }
    Sp = S;
    Z.swap(Zn);
    t = tn;
  }
  std::copy(S.begin(), S.end(), Xout);
}

// ---------------------------------------------------------------- decoder
// decoders.cpp:160-170: out = gbar_c X Lc + gbar_r Lr X, then the mask adds
// X on the sampled grid.
struct DecoderOp {
  const Csr& Lr;
  const Csr& Lc;
  Csc Lct;
  const std::vector<i64>& omr;
  const std::vector<i64>& omc;
  double gr, gc;
  i64 p, n;
  // Row tiles of RT rows: the X L_c sums of a tile read only that tile of
  // every column (cache resident), then L_r X of the tile's rows; each
  // output keeps the reference's per-element order (the X Lc sum over the
  // rows of Lc ascending, the Lr X sum in CSR order, then gc * a + gr * s).
  void apply(const double* X, double* out) const {
    const i64 P = p;
    constexpr i64 RT = 128;
    const i64 tiles = (P + RT - 1) / RT;
#pragma omp parallel for schedule(dynamic, 1)
    for (i64 t = 0; t < tiles; ++t) {
      const i64 i0 = t * RT, i1 = std::min(P, i0 + RT), m = i1 - i0;
      double acc[RT];
      for (i64 c = 0; c < n; ++c) {
        for (i64 i = 0; i < m; ++i) acc[i] = 0.0;
        for (i64 k = Lct.cp[c]; k < Lct.cp[c + 1]; ++k) {
          const double w = Lct.v[k];
          const double* xs = X + Lct.ri[k] * P + i0;
          for (i64 i = 0; i < m; ++i) acc[i] += w * xs[i];
        }
        const double* xc = X + c * P;
        double* oc = out + c * P;
        for (i64 i = i0; i < i1; ++i) {
          double s = 0.0;
          for (i64 k = Lr.rp[i]; k < Lr.rp[i + 1]; ++k) s += Lr.v[k] * xc[Lr.ci[k]];
          oc[i] = gc * acc[i - i0] + gr * s;
        }
      }
    }
    for (size_t j = 0; j < omc.size(); ++j) {
      const i64 cj = omc[j];
      for (size_t i = 0; i < omr.size(); ++i) {
        const i64 ri = omr[i];
        out[ri + cj * P] += X[ri + cj * P];
      }
    }
  }
};

void alternate_decode(const double* Xt, i64 rho_r, i64 rho_c, const std::vector<i64>& omr,
                      const std::vector<i64>& omc, i64 p, i64 n, const Csr& Lr, const Csr& Lc,
                      double lk1_r, double lk1_c, double gamma, double tol, i64 max_iter,
                      double* Xout, int* conv, i64* iters) {
  if (static_cast<i64>(omr.size()) != rho_r || static_cast<i64>(omc.size()) != rho_c)
    throw std::invalid_argument("alternate decoder: Xt does not match plan");
  if (Lr.rows != p || Lc.rows != n)
    throw std::invalid_argument("alternate decoder: Laplacians do not match plan");
  if (gamma <= 0.0) throw std::invalid_argument("alternate decoder: gamma must be positive");
  const double gbar_r = gamma / lk1_r;
  const double gbar_c = gamma / lk1_c;
  DecoderOp op{Lr, Lc, to_csc(Lc), omr, omc, gbar_r, gbar_c, p, n};
  const i64 N = p * n;
  Vec b(static_cast<size_t>(N), 0.0);
  for (i64 j = 0; j < rho_c; ++j)
    for (i64 i = 0; i < rho_r; ++i) b[omr[i] + omc[j] * p] = Xt[i + j * rho_r];
  Vec x(static_cast<size_t>(N), 0.0);
  auto apply = [&op](const Vec& v, Vec& o) { op.apply(v.data(), o.data()); };
  auto identity = [N](const Vec& r, Vec& z) {
#pragma omp parallel for schedule(static) if (N > kParMin)
    for (i64 i = 0; i < N; ++i) z[i] = r[i];
  };
  const PcgOut res = pcg_core(apply, b, x, tol, max_iter, identity);
  std::copy(x.begin(), x.end(), Xout);
  *conv = res.converged ? 1 : 0;
  *iters = res.iterations;
}

template <class F>
int guard(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return 1;
  } catch (const std::out_of_range& e) {
    g_err = e.what();
    return 3;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 2;
  }
}

std::vector<i64> to_list(const int64_t* p, int64_t n) { return std::vector<i64>(p, p + n); }

}  // namespace

// ---------------------------------------------------------------- clustering
// clustering.cpp:40-137: Lloyd iterations with k-means++ seeding on the
// columns of X (rows x n, column-major); squared norms are sequential sums
// over the rows (Eigen's squaredNorm order is unspecified: the device
// kernels use this same order, so they are compared bit for bit).
namespace {

double col_d2(const double* X, i64 rows, i64 j, const double* c) {
  double s = 0.0;
  const double* x = X + j * rows;
  for (i64 i = 0; i < rows; ++i) {
    const double d = x[i] - c[i];
    s += d * d;
  }
  return s;
}

struct LloydRun {
  std::vector<int> a;
  double wcss = std::numeric_limits<double>::infinity();
};

LloydRun lloyd_once(const double* X, i64 rows, i64 n, i64 k, i64 max_iter, Rng rng) {
  std::vector<double> cent(static_cast<size_t>(rows * k));
  auto col = [&](i64 c) { return cent.data() + c * rows; };
  auto set_col = [&](i64 c, i64 j) { std::copy(X + j * rows, X + (j + 1) * rows, col(c)); };
  set_col(0, static_cast<i64>(rng.below(static_cast<uint64_t>(n))));  // :44
  std::vector<double> min_d2(static_cast<size_t>(n), std::numeric_limits<double>::infinity());
  for (i64 c = 1; c < k; ++c) {  // :46-66
    for (i64 j = 0; j < n; ++j) min_d2[j] = std::min(min_d2[j], col_d2(X, rows, j, col(c - 1)));
    double total = 0.0;
    for (i64 j = 0; j < n; ++j) total += min_d2[j];
    i64 pick = 0;
    if (total > 0.0) {
      double target = rng.uniform() * total;
      for (i64 j = 0; j < n; ++j) {
        target -= min_d2[j];
        if (target <= 0.0) {
          pick = j;
          break;
        }
        pick = j;
      }
    } else {
      pick = static_cast<i64>(rng.below(static_cast<uint64_t>(n)));
    }
    set_col(c, pick);
  }
  LloydRun run;
  run.a.assign(static_cast<size_t>(n), 0);
  std::vector<i64> counts(static_cast<size_t>(k));
  std::vector<double> sums(static_cast<size_t>(rows * k));
  for (i64 it = 0; it < max_iter; ++it) {  // :71-107
    bool changed = false;
    for (i64 j = 0; j < n; ++j) {
      i64 best = 0;
      double bd = std::numeric_limits<double>::infinity();
      for (i64 c = 0; c < k; ++c) {
        const double d = col_d2(X, rows, j, col(c));
        if (d < bd) {
          bd = d;
          best = c;
        }
      }
      if (static_cast<int>(best) != run.a[j]) {
        run.a[j] = static_cast<int>(best);
        changed = true;
      }
    }
    if (!changed && it > 0) break;
    std::fill(sums.begin(), sums.end(), 0.0);
    std::fill(counts.begin(), counts.end(), i64{0});
    for (i64 j = 0; j < n; ++j) {
      double* sc = sums.data() + static_cast<i64>(run.a[j]) * rows;
      const double* x = X + j * rows;
      for (i64 i = 0; i < rows; ++i) sc[i] += x[i];
      ++counts[run.a[j]];
    }
    for (i64 c = 0; c < k; ++c) {
      if (counts[c] > 0) {
        const double cn = static_cast<double>(counts[c]);
        for (i64 i = 0; i < rows; ++i) col(c)[i] = sums[c * rows + i] / cn;
      } else {
        i64 far = 0;
        double fd = -1.0;
        for (i64 j = 0; j < n; ++j) {
          const double d = col_d2(X, rows, j, col(run.a[j]));
          if (d > fd) {
            fd = d;
            far = j;
          }
        }
        set_col(c, far);
        run.a[far] = static_cast<int>(c);
      }
    }
  }
  run.wcss = 0.0;
  for (i64 j = 0; j < n; ++j) run.wcss += col_d2(X, rows, j, col(run.a[j]));
  return run;
}

// clustering.cpp:165-218 (Hungarian method on cost = -score).
std::vector<i64> max_assignment(const std::vector<double>& score, i64 n) {
  std::vector<double> u(static_cast<size_t>(n) + 1, 0.0), v(static_cast<size_t>(n) + 1, 0.0);
  std::vector<i64> match(static_cast<size_t>(n) + 1, 0), way(static_cast<size_t>(n) + 1, 0);
  const double inf = std::numeric_limits<double>::infinity();
  for (i64 i = 1; i <= n; ++i) {
    match[0] = i;
    i64 j0 = 0;
    std::vector<double> minv(static_cast<size_t>(n) + 1, inf);
    std::vector<char> used(static_cast<size_t>(n) + 1, 0);
    do {
      used[j0] = 1;
      const i64 i0 = match[j0];
      double delta = inf;
      i64 j1 = 0;
      for (i64 j = 1; j <= n; ++j) {
        if (used[j]) continue;
        const double cur = -score[(i0 - 1) + (j - 1) * n] - u[i0] - v[j];
        if (cur < minv[j]) {
          minv[j] = cur;
          way[j] = j0;
        }
        if (minv[j] < delta) {
          delta = minv[j];
          j1 = j;
        }
      }
      for (i64 j = 0; j <= n; ++j) {
        if (used[j]) {
          u[match[j]] += delta;
          v[j] -= delta;
        } else {
          minv[j] -= delta;
        }
      }
      j0 = j1;
    } while (match[j0] != 0);
    do {
      const i64 j1 = way[j0];
      match[j0] = match[j1];
      j0 = j1;
    } while (j0 != 0);
  }
  std::vector<i64> r2c(static_cast<size_t>(n), 0);
  for (i64 j = 1; j <= n; ++j) r2c[match[j] - 1] = j - 1;
  return r2c;
}

}  // namespace

struct ora_csr : Csr {
  explicit ora_csr(Csr&& m) : Csr(std::move(m)) {}
};

static ora_csr* box(Csr&& m) { return new ora_csr(std::move(m)); }

extern "C" {

const char* ora_last_error(void) { return g_err.c_str(); }

void ora_set_threads(int n) {
#ifdef _OPENMP
  omp_set_num_threads(n > 0 ? n : 1);
#else
  (void)n;
#endif
}

int ora_get_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

int ora_csr_from_triplets(int64_t rows, int64_t cols, int64_t n, const int64_t* ti,
                          const int64_t* tj, const double* tv, double drop_below, ora_csr** out) {
  return guard([&] {
    std::vector<Trip> t(static_cast<size_t>(n));
    for (int64_t k = 0; k < n; ++k) t[k] = {ti[k], tj[k], tv[k]};
    *out = box(build_csr(rows, cols, std::move(t), drop_below));
  });
}

int ora_csr_from_csr(int64_t rows, int64_t cols, const int64_t* row_ptr, const int64_t* col_idx,
                     const double* values, ora_csr** out) {
  return guard([&] {
    Csr m;
    m.rows = rows;
    m.cols = cols;
    m.rp.assign(row_ptr, row_ptr + rows + 1);
    const int64_t nnz = row_ptr[rows];
    m.ci.assign(col_idx, col_idx + nnz);
    m.v.assign(values, values + nnz);
    *out = box(std::move(m));
  });
}

int ora_csr_from_dense(const double* D, int64_t rows, int64_t cols, double drop_below,
                       ora_csr** out) {
  return guard([&] { *out = box(csr_from_dense(D, rows, cols, drop_below)); });
}

void ora_csr_free(ora_csr* a) { delete a; }
int64_t ora_csr_rows(const ora_csr* a) { return a->rows; }
int64_t ora_csr_cols(const ora_csr* a) { return a->cols; }
int64_t ora_csr_nnz(const ora_csr* a) { return a->nnz(); }

void ora_csr_export(const ora_csr* a, int64_t* row_ptr, int64_t* col_idx, double* values) {
  if (row_ptr) std::copy(a->rp.begin(), a->rp.end(), row_ptr);
  if (col_idx) std::copy(a->ci.begin(), a->ci.end(), col_idx);
  if (values) std::copy(a->v.begin(), a->v.end(), values);
}

int ora_csr_submatrix(const ora_csr* a, const int64_t* rows, int64_t nr, const int64_t* cols,
                      int64_t nc, ora_csr** out) {
  return guard([&] { *out = box(submatrix(*a, to_list(rows, nr), to_list(cols, nc))); });
}

void ora_csr_row_sums(const ora_csr* a, double* out) {
  const Vec s = row_sums(*a);
  std::copy(s.begin(), s.end(), out);
}

int ora_csr_components(const ora_csr* a, int64_t* labels, int64_t* n_comp) {
  return guard([&] {
    const auto comps = components(*a);
    for (size_t c = 0; c < comps.size(); ++c)
      for (const i64 u : comps[c]) labels[u] = static_cast<int64_t>(c);
    *n_comp = static_cast<int64_t>(comps.size());
  });
}

int ora_spmv(const ora_csr* a, const double* x, int64_t n, double* y) {
  return guard([&] {
    const Vec out = spmv(*a, Vec(x, x + n));
    std::copy(out.begin(), out.end(), y);
  });
}

int ora_spmm_left(const ora_csr* a, const double* X, int64_t xr, int64_t xc, double* Y) {
  return guard([&] { spmm_left(*a, X, xr, xc, Y); });
}

int ora_spmm_right(const ora_csr* a, const double* X, int64_t xr, int64_t xc, double* Y) {
  return guard([&] { spmm_right(*a, X, xr, xc, Y); });
}

uint64_t ora_rng_mix(uint64_t z) { return Rng::mix(z); }

void ora_rng_u64(uint64_t seed, int64_t count, uint64_t* out) {
  Rng r(seed);
  for (int64_t i = 0; i < count; ++i) out[i] = r.u64();
}

void ora_rng_gaussian(uint64_t seed, int64_t count, double* out) {
  Rng r(seed);
  for (int64_t i = 0; i < count; ++i) out[i] = r.gaussian();
}

uint64_t ora_rng_derive_seed(uint64_t seed, uint64_t stream) { return Rng::derive(seed, stream).seed; }

int ora_pcg_solve(const ora_csr* A, const double* b, double* x, int64_t n, double tol,
                  int64_t max_iter, int jacobi, int64_t* iterations, int* converged,
                  double* rel_res) {
  return guard([&] {
    if (A->rows != A->cols || A->cols != n) throw std::invalid_argument("pcg: dimension mismatch");
    const Vec bv(b, b + n);
    Vec xv(x, x + n);
    PcgOut r;
    if (jacobi) {
      r = pcg_jacobi(*A, diagonal(*A), bv, xv, tol, max_iter);
    } else {
      auto apply = [A](const Vec& v, Vec& out) { out = spmv(*A, v); };
      r = pcg_core(apply, bv, xv, tol, max_iter, [](const Vec& q, Vec& z) { z = q; });
    }
    std::copy(xv.begin(), xv.end(), x);
    *iterations = r.iterations;
    *converged = r.converged ? 1 : 0;
    *rel_res = r.rel_res;
  });
}

int ora_power_iteration_norm(const ora_csr* A, double tol, uint64_t seed, int64_t max_iter,
                             double* out) {
  return guard([&] { *out = power_norm(*A, tol, seed, max_iter); });
}

int ora_knn_graph(const double* X, int64_t rows, int64_t cols, int axis_rows, int64_t K,
                  int normalized, double sigma2_override, ora_csr** adjacency,
                  ora_csr** laplacian_out, double* degrees, double* sigma2) {
  return guard([&] {
    Graph g = knn_graph(X, rows, cols, axis_rows != 0, K, normalized != 0, sigma2_override);
    std::copy(g.deg.begin(), g.deg.end(), degrees);
    *sigma2 = g.sigma2;
    *adjacency = box(std::move(g.W));
    *laplacian_out = box(std::move(g.L));
  });
}

int ora_knn_neighbors(const double* X, int64_t rows, int64_t cols, int axis_rows, int64_t K,
                      int64_t* nbr, double* nbr_d2) {
  return guard([&] {
    const Points P = gather_points(X, rows, cols, axis_rows != 0);
    if (K < 1) throw std::invalid_argument("knn graph: K must be >= 1");
    if (P.n < K + 1)
      throw std::invalid_argument("knn graph: need at least K+1 points, got " + std::to_string(P.n));
    Vec mean;
    knn_select(P, K, nbr, nbr_d2, mean);
  });
}

int ora_knn_rows(const double* X, int64_t rows, int64_t cols, int axis_rows, int64_t K, const int64_t* query,
                 int64_t nq, int64_t* nbr, double* nbr_d2) {
  return guard([&] {
    const Points P = gather_points(X, rows, cols, axis_rows != 0);
    if (K < 1 || P.n < K + 1) throw std::invalid_argument("knn rows: bad K");
    for (int64_t q = 0; q < nq; ++q)
      if (query[q] < 0 || query[q] >= P.n) throw std::invalid_argument("knn rows: query out of range");
    knn_select_rows(P, K, query, nq, nbr, nbr_d2);
  });
}

int ora_graph_from_adjacency(const ora_csr* W, int normalized, ora_csr** laplacian_out,
                             double* degrees) {
  return guard([&] {
    Graph g = graph_from_adjacency(*W, normalized != 0);
    std::copy(g.deg.begin(), g.deg.end(), degrees);
    *laplacian_out = box(std::move(g.L));
  });
}

int ora_kron_reduce(const ora_csr* L, const int64_t* keep, int64_t nkeep, double pcg_tol,
                    double prune_tol, ora_csr** out) {
  return guard([&] { *out = box(kron_reduce(*L, to_list(keep, nkeep), pcg_tol, prune_tol)); });
}

int ora_graph_upsample(const ora_csr* L, const int64_t* known, int64_t n_known, const double* R, int64_t r,
                       double pcg_tol, int64_t pcg_max_iter, double* S) {
  return guard([&] {
    const auto out = graph_upsample(*L, to_list(known, n_known), R, r, pcg_tol, pcg_max_iter);
    std::copy(out.begin(), out.end(), S);
  });
}

int ora_draw_plan(int64_t p, int64_t n, int64_t rho_r, int64_t rho_c, uint64_t seed,
                  int64_t* omega_r, int64_t* omega_c) {
  return guard([&] {
    if (rho_r < 1 || rho_r > p)
      throw std::invalid_argument("draw_plan: rho_r out of range [1, " + std::to_string(p) + "]");
    if (rho_c < 1 || rho_c > n)
      throw std::invalid_argument("draw_plan: rho_c out of range [1, " + std::to_string(n) + "]");
    const auto r = partial_shuffle(p, rho_r, Rng::derive(seed, 0x726f7773ULL));
    const auto c = partial_shuffle(n, rho_c, Rng::derive(seed, 0x636f6c73ULL));
    std::copy(r.begin(), r.end(), omega_r);
    std::copy(c.begin(), c.end(), omega_c);
  });
}

int ora_subsample(const double* Y, int64_t p, int64_t n, const int64_t* omega_r, int64_t rho_r,
                  const int64_t* omega_c, int64_t rho_c, double* out) {
  return guard([&] {
    for (int64_t j = 0; j < rho_c; ++j)
      for (int64_t i = 0; i < rho_r; ++i) {
        const int64_t r = omega_r[i], c = omega_c[j];
        if (r < 0 || r >= p || c < 0 || c >= n)
          throw std::invalid_argument("subsample: plan does not match matrix dimensions");
        out[i + j * rho_r] = Y[r + c * p];
      }
  });
}

int ora_objective(const double* X, const double* Y, int64_t r, int64_t c, const ora_csr* Lr,
                  const ora_csr* Lc, const ora_frpcag_cfg* cfg, double* out) {
  return guard([&] { *out = objective(X, Y, r, c, *Lr, *Lc, *cfg); });
}

int ora_prox_l1(const double* Z, const double* Y, int64_t count, double lam, double* out) {
  return guard([&] { prox_l1(Z, Y, count, lam, out); });
}

int ora_prox_l2(const double* Z, const double* Y, int64_t count, double lam, double* out) {
  return guard([&] { prox_l2(Z, Y, count, lam, out); });
}

int ora_grad_g(const double* Z, int64_t r, int64_t c, const ora_csr* Lr, const ora_csr* Lc,
               const ora_frpcag_cfg* cfg, double* G) {
  return guard([&] { grad_g(Z, r, c, *Lr, *Lc, *cfg, G); });
}

int ora_fista_solve(const double* Y, int64_t r, int64_t c, const ora_csr* Lr, const ora_csr* Lc,
                    const ora_frpcag_cfg* cfg, double* X_out, double* objective_out,
                    int64_t* iterations, int* converged, double* final_rel_change,
                    double* step_used) {
  return guard([&] {
    fista(Y, r, c, *Lr, *Lc, *cfg, X_out, objective_out, iterations, converged, final_rel_change,
          step_used);
  });
}

int ora_alternate_decode(const double* Xt, int64_t rho_r, int64_t rho_c, const int64_t* omega_r,
                         const int64_t* omega_c, int64_t p, int64_t n, const ora_csr* Lr,
                         const ora_csr* Lc, double lambda_k1_r, double lambda_k1_c, double gamma,
                         double pcg_tol, int64_t pcg_max_iter, double* X_out, int* converged,
                         int64_t* iterations) {
  return guard([&] {
    alternate_decode(Xt, rho_r, rho_c, to_list(omega_r, rho_r), to_list(omega_c, rho_c), p, n, *Lr,
                     *Lc, lambda_k1_r, lambda_k1_c, gamma, pcg_tol, pcg_max_iter, X_out, converged,
                     iterations);
  });
}

int ora_decoder_apply(const double* X, int64_t p, int64_t n, const int64_t* omega_r,
                      int64_t rho_r, const int64_t* omega_c, int64_t rho_c, const ora_csr* Lr,
                      const ora_csr* Lc, double gbar_r, double gbar_c, double* out) {
  return guard([&] {
    const auto omr = to_list(omega_r, rho_r);
    const auto omc = to_list(omega_c, rho_c);
    DecoderOp op{*Lr, *Lc, to_csc(*Lc), omr, omc, gbar_r, gbar_c, p, n};
    op.apply(X, out);
  });
}

int ora_kmeans(const double* X, int64_t rows, int64_t n, int64_t k, int64_t restarts, uint64_t seed,
               int64_t max_iter, int* assignments, double* wcss) {
  return guard([&] {
    if (k < 1) throw std::invalid_argument("kmeans: k must be >= 1");
    if (k > n) throw std::invalid_argument("kmeans: more clusters than points");
    if (restarts < 1) throw std::invalid_argument("kmeans: restarts must be >= 1");
    LloydRun best;
    for (int64_t r = 0; r < restarts; ++r) {  // clustering.cpp:131-134
      LloydRun run = lloyd_once(X, rows, n, k, max_iter, Rng::derive(seed, static_cast<uint64_t>(r)));
      if (run.wcss < best.wcss) best = std::move(run);
    }
    std::copy(best.a.begin(), best.a.end(), assignments);
    if (wcss) *wcss = best.wcss;
  });
}

int ora_clustering_error(const int* pred, const int* truth, int64_t n, int64_t k, double* out) {
  return guard([&] {
    if (n == 0) throw std::invalid_argument("clustering error: empty labels");
    std::vector<double> cont(static_cast<size_t>(k * k), 0.0);
    for (int64_t i = 0; i < n; ++i) cont[pred[i] + static_cast<int64_t>(truth[i]) * k] += 1.0;
    const std::vector<i64> perm = max_assignment(cont, k);
    double agree = 0.0;
    for (int64_t c = 0; c < k; ++c) agree += cont[c + perm[c] * k];
    *out = 1.0 - agree / static_cast<double>(n);
  });
}

}  // extern "C"
