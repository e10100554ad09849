// fista.cu -- FRPCAG solved by FISTA on the sampled matrix
// (frpcag.cpp:62-112, Algorithm 1 of the paper).
//
// One iteration j is three kernels; all scalar bookkeeping (t, momentum
// coefficient, objective trace, stopping test, divergence check) stays on
// the device and is done by the last block of the kernel that completes the
// reduction, so the host only polls a done flag once per chunk of
// iterations:
//   K1 grad+prox  S_j = prox(Z_j - step * grad_g(Z_j), Y, step)
//   K2 objective  phi(Y - S_j) + gc sum (S Lc) o S + gr sum (Lr S) o S,
//                 finite check, trace[j-1], t_{j+1}, (t_j - 1) / t_{j+1}
//   K3 momentum   Z_{j+1} = S_j + coef (S_j - S_{j-1}), ||Z_j||^2,
//                 ||Z_{j+1} - Z_j||^2, stop test
// Buffers rotate by parity of j (S_j in S[j&1], Z_j in Z[j&1]).
#include <cstdlib>
#include <string>
#include <algorithm>

#include "common.cuh"
#include "frpcag.cuh"
#include "fista_persist.cuh"
#include "fista_dense.cuh"

namespace cpcag_cuda {

struct FistaState {
  double t, t_next, coef;
  double frc;
  i64 j;           // iteration about to run (1-based)
  i64 iterations;  // completed objective evaluations
  int done, converged, err, pad;
  i64 err_j;
  unsigned cnt[4];
};

template <typename T>
__global__ void fista_grad_prox_k(i64 rows, i64 cols, Pull<T> Lr, Pull<T> Lc, T s_r, T s_c,
                                  int use_r, int use_c, int loss, T step,
                                  const T* __restrict__ Z, const T* __restrict__ Y,
                                  T* __restrict__ S, const FistaState* st) {
  if (st->done) return;
  const i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x;
  if (i >= rows) return;
  for (i64 c = blockIdx.y; c < cols; c += gridDim.y) {
    const i64 at = i + c * rows;
    const T g = grad_elem(Lr, Lc, s_r, s_c, use_r, use_c, Z, rows, i, c);
    const T arg = sub_rn(Z[at], mul_rn(step, g));
    S[at] = loss == CPCAG_LOSS_L2 ? prox_l2_elem(arg, Y[at], step) : prox_l1_elem(arg, Y[at], step);
  }
}

template <typename T>
__global__ void fista_objective_k(i64 rows, i64 cols, Pull<T> Lr, Pull<T> Lc, double gamma_r,
                                  double gamma_c, int loss, const T* __restrict__ S,
                                  const T* __restrict__ Y, double* partials, double* trace,
                                  FistaState* st) {
  if (st->done) return;
  double s[3] = {0.0, 0.0, 0.0};
  const i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x;
  const int use_r = gamma_r != 0.0, use_c = gamma_c != 0.0;
  if (i < rows) {
    for (i64 c = blockIdx.y; c < cols; c += gridDim.y) {
      const i64 at = i + c * rows;
      const double x = static_cast<double>(S[at]);
      const double e = static_cast<double>(Y[at]) - x;
      s[0] += loss == CPCAG_LOSS_L2 ? e * e : fabs(e);
      if (use_c) s[1] += static_cast<double>(pull_right(Lc.rp[c], Lc.rp[c + 1], Lc.ci, Lc.v, S, rows, i)) * x;
      if (use_r) s[2] += static_cast<double>(pull_left(Lr.rp[i], Lr.rp[i + 1], Lr.ci, Lr.v, S + c * rows)) * x;
    }
  }
  double tot[3];
  if (grid_sum_last<3>(s, partials, &st->cnt[0], tot) && threadIdx.x == 0) {
    double val = tot[0];
    if (use_c) val += gamma_c * tot[1];
    if (use_r) val += gamma_r * tot[2];
    const i64 j = st->j;
    if (!isfinite(val)) {
      st->err = 1;
      st->err_j = j;
      st->done = 1;
      return;
    }
    trace[j - 1] = val;
    st->iterations = j;
    const double t = st->t;
    const double tn = 0.5 * (1.0 + sqrt(1.0 + 4.0 * t * t));
    st->t_next = tn;
    st->coef = (t - 1.0) / tn;
  }
}

template <typename T>
__global__ void fista_momentum_k(i64 N, const T* __restrict__ S, const T* __restrict__ Sp,
                                 const T* __restrict__ Z, T* __restrict__ Zn, double tol,
                                 i64 max_iter, double* partials, FistaState* st) {
  if (st->done) return;
  const T coef = static_cast<T>(st->coef);
  double s[2] = {0.0, 0.0};
  for (i64 q = blockIdx.x * (i64)blockDim.x + threadIdx.x; q < N; q += (i64)gridDim.x * blockDim.x) {
    const T sv = S[q];
    const T zn = add_rn(sv, mul_rn(coef, sub_rn(sv, Sp[q])));
    const T z = Z[q];
    Zn[q] = zn;
    const double zd = static_cast<double>(z);
    const double dd = static_cast<double>(sub_rn(zn, z));
    s[0] += zd * zd;
    s[1] += dd * dd;
  }
  double tot[2];
  if (grid_sum_last<2>(s, partials, &st->cnt[1], tot) && threadIdx.x == 0) {
    const double denom = tot[0], change = tot[1];
    st->frc = denom > 0.0 ? change / denom : change;
    if (change < tol * denom) {
      st->converged = 1;
      st->done = 1;
      return;
    }
    st->t = st->t_next;
    st->j += 1;
    if (st->j > max_iter) st->done = 1;
  }
}

// ------------------------------------------------------------------ dense-operator path
// The Kron-reduced Laplacians are near dense (config 0: 82 % / 65 % fill,
// config 1: 55 % / 71 %).  Above 25 % fill both products run as tiled dense
// GEMMs (32 x 32 output tile per CTA, k staged through shared memory in
// chunks of 32).  Every output accumulates over k in ascending order; for
// fp64 each step is an explicit mul then add, which over the dense row equals
// the reference's CSR-order sum (added zeros do not change a sum), so fp64
// stays bit-exact; fp32 uses FMA.
template <typename T>
__global__ void __launch_bounds__(256) fista_dense_grad_prox_k(i64 rr, i64 rc, const T* __restrict__ Lr,
                                                               const T* __restrict__ Lc, T s_r, T s_c, int use_r,
                                                               int use_c, int loss, T step, const T* __restrict__ Z,
                                                               const T* __restrict__ Y, T* __restrict__ S,
                                                               const FistaState* st) {
  if (st->done) return;
  const i64 i0 = static_cast<i64>(blockIdx.x) * kDT, c0 = static_cast<i64>(blockIdx.y) * kDT;
  T acc1[2][2], acc2[2][2];
  dual_gemm_tile(Lr, Lc, Z, rr, rc, use_r, use_c, i0, c0, acc1, acc2);
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int b = 0; b < 2; ++b) {
      const i64 i = i0 + ty + 16 * a, c = c0 + tx + 16 * b;
      if (i >= rr || c >= rc) continue;
      const i64 at = i + c * rr;
      // grad_elem order: 0 + (2 gc)(Z Lc), then + (2 gr)(Lr Z)
      T g = T(0);
      if (use_c) g = add_rn(g, mul_rn(s_c, acc2[a][b]));
      if (use_r) g = add_rn(g, mul_rn(s_r, acc1[a][b]));
      const T arg = sub_rn(Z[at], mul_rn(step, g));
      S[at] = loss == CPCAG_LOSS_L2 ? prox_l2_elem(arg, Y[at], step) : prox_l1_elem(arg, Y[at], step);
    }
}

template <typename T>
__global__ void __launch_bounds__(256) fista_dense_objective_k(i64 rr, i64 rc, const T* __restrict__ Lr,
                                                               const T* __restrict__ Lc, double gamma_r,
                                                               double gamma_c, int loss, const T* __restrict__ S,
                                                               const T* __restrict__ Y, double* partials,
                                                               double* trace, FistaState* st) {
  if (st->done) return;
  const int use_r = gamma_r != 0.0, use_c = gamma_c != 0.0;
  const i64 i0 = static_cast<i64>(blockIdx.x) * kDT, c0 = static_cast<i64>(blockIdx.y) * kDT;
  T acc1[2][2], acc2[2][2];
  dual_gemm_tile(Lr, Lc, S, rr, rc, use_r, use_c, i0, c0, acc1, acc2);
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  double s[3] = {0.0, 0.0, 0.0};
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int b = 0; b < 2; ++b) {
      const i64 i = i0 + ty + 16 * a, c = c0 + tx + 16 * b;
      if (i >= rr || c >= rc) continue;
      const i64 at = i + c * rr;
      const double x = static_cast<double>(S[at]);
      const double e = static_cast<double>(Y[at]) - x;
      s[0] += loss == CPCAG_LOSS_L2 ? e * e : fabs(e);
      s[1] += static_cast<double>(acc2[a][b]) * x;
      s[2] += static_cast<double>(acc1[a][b]) * x;
    }
  double tot[3];
  if (grid_sum_last<3>(s, partials, &st->cnt[0], tot) && threadIdx.x == 0) {
    double val = tot[0];
    if (use_c) val += gamma_c * tot[1];
    if (use_r) val += gamma_r * tot[2];
    const i64 j = st->j;
    if (!isfinite(val)) {
      st->err = 1;
      st->err_j = j;
      st->done = 1;
      return;
    }
    trace[j - 1] = val;
    st->iterations = j;
    const double t = st->t;
    const double tn = 0.5 * (1.0 + sqrt(1.0 + 4.0 * t * t));
    st->t_next = tn;
    st->coef = (t - 1.0) / tn;
  }
}

// ---- fp32 split-K: the concatenated k-space [0, rr) u [rr, rr + rc) of the
// two products is cut into S ranges; CTA (tile, s) writes its partial tile,
// and the last CTA of the tile (per-tile arrival counter) sums the S partials
// in s order (deterministic) and runs the epilogue.
struct SplitWs {
  double* part1;       // S x m partial (Lr Z), fp64 (see splitk_gemm)
  double* part2;       // S x m partial (Z Lc)
  unsigned* tile_cnt;  // tiles
  unsigned* done_cnt;  // 1
  double* tile_sums;   // 3 x tiles (objective)
};

constexpr int kST = 64;  // split-K output tile side
constexpr int kSK = 16;  // k chunk

// 64 x 64 output tile per CTA, 4 x 4 outputs per thread (rows ty + 16 a,
// columns tx + 16 b), k staged through shared memory 16 at a time.
template <bool kLeft>
__device__ __forceinline__ void splitk_gemm(const float* __restrict__ A, i64 lda, i64 arows,
                                            const float* __restrict__ B, i64 ldb, i64 bcols, i64 ka, i64 kb,
                                            i64 i0, i64 c0, double (&acc)[4][4]) {
  // kLeft:  acc += Lr[i, k] * Z[k, c]   (A = Lr dense col-major rr x rr, B = Z)
  // !kLeft: acc += Z[i, k] * Lc[k, c]   (A = Z, B = Lc dense col-major)
  __shared__ float As[kSK][kST + 1];
  __shared__ float Bs[kSK][kST + 1];
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  for (i64 k0 = ka; k0 < kb; k0 += kSK) {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int ii = tid & 63, kk = (tid >> 6) + 4 * q;
      const i64 gi = i0 + ii, gk = k0 + kk;
      As[kk][ii] = (gi < arows && gk < kb) ? A[gk * lda + gi] : 0.f;
      const int kk2 = tid & 15, cc = (tid >> 4) + 16 * q;
      const i64 gk2 = k0 + kk2, gc = c0 + cc;
      Bs[kk2][cc] = (gk2 < kb && gc < bcols) ? B[gc * ldb + gk2] : 0.f;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < kSK; ++kk) {
      float av[4], bv[4];
#pragma unroll
      for (int a = 0; a < 4; ++a) av[a] = As[kk][ty + 16 * a];
#pragma unroll
      for (int b = 0; b < 4; ++b) bv[b] = Bs[kk][tx + 16 * b];
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b)
          acc[a][b] = fma(static_cast<double>(av[a]), static_cast<double>(bv[b]), acc[a][b]);
    }
    __syncthreads();
  }
}

__device__ __forceinline__ void splitk_partial(const float* __restrict__ Lr, const float* __restrict__ Lc,
                                               const float* __restrict__ Z, i64 rr, i64 rc, int use_r,
                                               int use_c, i64 i0, i64 c0, i64 ka, i64 kb, double (&acc1)[4][4],
                                               double (&acc2)[4][4]) {
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc1[a][b] = acc2[a][b] = 0.0;
  if (use_r && ka < rr) splitk_gemm<true>(Lr, rr, rr, Z, rr, rc, ka, min(kb, rr), i0, c0, acc1);
  if (use_c && kb > rr) splitk_gemm<false>(Z, rr, rr, Lc, rc, rc, max(ka, rr) - rr, kb - rr, i0, c0, acc2);
}

// Partial products of split s into ws.part1/part2[s] (no reduction here).
__global__ void __launch_bounds__(256) fista_splitk_partial_k(i64 rr, i64 rc, const float* __restrict__ Lr,
                                                              const float* __restrict__ Lc, int use_r, int use_c,
                                                              const float* __restrict__ Z, SplitWs ws,
                                                              const FistaState* st) {
  if (st->done) return;
  const int Sn = gridDim.z;
  const i64 ktot = rr + rc, ka = (ktot * blockIdx.z) / Sn, kb = (ktot * (blockIdx.z + 1)) / Sn;
  const i64 i0 = static_cast<i64>(blockIdx.x) * kST, c0 = static_cast<i64>(blockIdx.y) * kST;
  double acc1[4][4], acc2[4][4];
  splitk_partial(Lr, Lc, Z, rr, rc, use_r, use_c, i0, c0, ka, kb, acc1, acc2);
  const i64 m = rr * rc;
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  double* p1 = ws.part1 + static_cast<i64>(blockIdx.z) * m;
  double* p2 = ws.part2 + static_cast<i64>(blockIdx.z) * m;
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const i64 i = i0 + ty + 16 * a, c = c0 + tx + 16 * b;
      if (i < rr && c < rc) {
        p1[i + c * rr] = acc1[a][b];
        p2[i + c * rr] = acc2[a][b];
      }
    }
}

// Sum of the split partials in split order, in fp64, rounded once to fp32.
__device__ __forceinline__ void splitk_sum(const SplitWs& ws, i64 m, int S, i64 e, float& x1, float& x2) {
  double s1 = 0.0, s2 = 0.0;
  for (int q = 0; q < S; ++q) {
    s1 += ws.part1[static_cast<i64>(q) * m + e];
    s2 += ws.part2[static_cast<i64>(q) * m + e];
  }
  x1 = static_cast<float>(s1);
  x2 = static_cast<float>(s2);
}

__global__ void fista_splitk_grad_prox_k(i64 rr, i64 rc, int S, float s_r, float s_c, int use_r, int use_c, int loss,
                                         float step, const float* __restrict__ Z, const float* __restrict__ Y,
                                         float* __restrict__ Sout, SplitWs ws, const FistaState* st) {
  if (st->done) return;
  const i64 m = rr * rc;
  for (i64 e = blockIdx.x * (i64)blockDim.x + threadIdx.x; e < m; e += (i64)gridDim.x * blockDim.x) {
    float x1, x2;
    splitk_sum(ws, m, S, e, x1, x2);
    float g = 0.f;
    if (use_c) g = __fadd_rn(g, __fmul_rn(s_c, x2));
    if (use_r) g = __fadd_rn(g, __fmul_rn(s_r, x1));
    const float arg = __fsub_rn(Z[e], __fmul_rn(step, g));
    Sout[e] = loss == CPCAG_LOSS_L2 ? prox_l2_elem(arg, Y[e], step) : prox_l1_elem(arg, Y[e], step);
  }
}

__global__ void fista_splitk_objective_k(i64 rr, i64 rc, int S, double gamma_r, double gamma_c, int loss,
                                         const float* __restrict__ Sv, const float* __restrict__ Y, SplitWs ws,
                                         double* partials, double* trace, FistaState* st) {
  if (st->done) return;
  const int use_r = gamma_r != 0.0, use_c = gamma_c != 0.0;
  const i64 m = rr * rc;
  double sm3[3] = {0.0, 0.0, 0.0};
  for (i64 e = blockIdx.x * (i64)blockDim.x + threadIdx.x; e < m; e += (i64)gridDim.x * blockDim.x) {
    float x1, x2;
    splitk_sum(ws, m, S, e, x1, x2);
    const double x = static_cast<double>(Sv[e]);
    const double d = static_cast<double>(Y[e]) - x;
    sm3[0] += loss == CPCAG_LOSS_L2 ? d * d : fabs(d);
    sm3[1] += static_cast<double>(x2) * x;
    sm3[2] += static_cast<double>(x1) * x;
  }
  double tot[3];
  if (grid_sum_last<3>(sm3, partials, &st->cnt[0], tot) && threadIdx.x == 0) {
    double val = tot[0];
    if (use_c) val += gamma_c * tot[1];
    if (use_r) val += gamma_r * tot[2];
    const i64 j = st->j;
    if (!isfinite(val)) {
      st->err = 1;
      st->err_j = j;
      st->done = 1;
      return;
    }
    trace[j - 1] = val;
    st->iterations = j;
    const double t = st->t;
    const double tn = 0.5 * (1.0 + sqrt(1.0 + 4.0 * t * t));
    st->t_next = tn;
    st->coef = (t - 1.0) / tn;
  }
}

// ---- linearity variant of the fp32 split-K path.  The
// objective already computes L_r S_j and S_j L_c; by linearity
//   L Z_{j+1} = L (S_j + coef (S_j - S_{j-1})) = LS_j + coef (LS_j - LS_{j-1}),
// so the gradient of the next iteration needs no GEMM: one GEMM pair per
// iteration instead of two.  LS is recomputed from S every iteration, so
// rounding does not accumulate; the result stays within the fp32 tolerance
// (the fp64 paths keep the reference's direct products).
struct LinBufs {
  float *LZr, *LZc;      // L_r Z_j, Z_j L_c
  float *LSr[2], *LSc[2];  // L_r S_j, S_j L_c for j and j - 1 (index j & 1)
};

__global__ void fista_lin_init_k(i64 rr, i64 rc, int S, SplitWs ws, LinBufs lb) {
  const i64 m = rr * rc;
  for (i64 e = blockIdx.x * (i64)blockDim.x + threadIdx.x; e < m; e += (i64)gridDim.x * blockDim.x) {
    float x1, x2;
    splitk_sum(ws, m, S, e, x1, x2);
    lb.LZr[e] = x1;
    lb.LZc[e] = x2;
    lb.LSr[0][e] = x1;  // S_0 = Y = Z_1
    lb.LSc[0][e] = x2;
  }
}

__global__ void fista_lin_grad_prox_k(i64 rr, i64 rc, float s_r, float s_c, int use_r, int use_c, int loss,
                                      float step, const float* __restrict__ Z, const float* __restrict__ Y,
                                      float* __restrict__ Sout, LinBufs lb, const FistaState* st) {
  if (st->done) return;
  const i64 m = rr * rc;
  for (i64 e = blockIdx.x * (i64)blockDim.x + threadIdx.x; e < m; e += (i64)gridDim.x * blockDim.x) {
    float g = 0.f;
    if (use_c) g = __fadd_rn(g, __fmul_rn(s_c, lb.LZc[e]));
    if (use_r) g = __fadd_rn(g, __fmul_rn(s_r, lb.LZr[e]));
    const float arg = __fsub_rn(Z[e], __fmul_rn(step, g));
    Sout[e] = loss == CPCAG_LOSS_L2 ? prox_l2_elem(arg, Y[e], step) : prox_l1_elem(arg, Y[e], step);
  }
}

__global__ void fista_lin_objective_k(i64 rr, i64 rc, int S, double gamma_r, double gamma_c, int loss,
                                      const float* __restrict__ Sv, const float* __restrict__ Y, SplitWs ws,
                                      float* __restrict__ LSr, float* __restrict__ LSc, double* partials,
                                      double* trace, FistaState* st) {
  if (st->done) return;
  const int use_r = gamma_r != 0.0, use_c = gamma_c != 0.0;
  const i64 m = rr * rc;
  double sm3[3] = {0.0, 0.0, 0.0};
  for (i64 e = blockIdx.x * (i64)blockDim.x + threadIdx.x; e < m; e += (i64)gridDim.x * blockDim.x) {
    float x1, x2;
    splitk_sum(ws, m, S, e, x1, x2);
    LSr[e] = x1;
    LSc[e] = x2;
    const double x = static_cast<double>(Sv[e]);
    const double d = static_cast<double>(Y[e]) - x;
    sm3[0] += loss == CPCAG_LOSS_L2 ? d * d : fabs(d);
    sm3[1] += static_cast<double>(x2) * x;
    sm3[2] += static_cast<double>(x1) * x;
  }
  double tot[3];
  if (grid_sum_last<3>(sm3, partials, &st->cnt[0], tot) && threadIdx.x == 0) {
    double val = tot[0];
    if (use_c) val += gamma_c * tot[1];
    if (use_r) val += gamma_r * tot[2];
    const i64 j = st->j;
    if (!isfinite(val)) {
      st->err = 1;
      st->err_j = j;
      st->done = 1;
      return;
    }
    trace[j - 1] = val;
    st->iterations = j;
    const double t = st->t;
    const double tn = 0.5 * (1.0 + sqrt(1.0 + 4.0 * t * t));
    st->t_next = tn;
    st->coef = (t - 1.0) / tn;
  }
}

__global__ void fista_lin_momentum_k(i64 N, const float* __restrict__ S, const float* __restrict__ Sp,
                                     const float* __restrict__ Z, float* __restrict__ Zn,
                                     const float* __restrict__ LSr, const float* __restrict__ LSrp,
                                     const float* __restrict__ LSc, const float* __restrict__ LScp, LinBufs lb,
                                     double tol, i64 max_iter, double* partials, FistaState* st) {
  if (st->done) return;
  const float coef = static_cast<float>(st->coef);
  double s[2] = {0.0, 0.0};
  for (i64 q = blockIdx.x * (i64)blockDim.x + threadIdx.x; q < N; q += (i64)gridDim.x * blockDim.x) {
    const float sv = S[q];
    const float zn = add_rn(sv, mul_rn(coef, sub_rn(sv, Sp[q])));
    const float z = Z[q];
    Zn[q] = zn;
    const float a = LSr[q], b = LSc[q];
    lb.LZr[q] = add_rn(a, mul_rn(coef, sub_rn(a, LSrp[q])));
    lb.LZc[q] = add_rn(b, mul_rn(coef, sub_rn(b, LScp[q])));
    const double zd = static_cast<double>(z);
    const double dd = static_cast<double>(sub_rn(zn, z));
    s[0] += zd * zd;
    s[1] += dd * dd;
  }
  double tot[2];
  if (grid_sum_last<2>(s, partials, &st->cnt[1], tot) && threadIdx.x == 0) {
    const double denom = tot[0], change = tot[1];
    st->frc = denom > 0.0 ? change / denom : change;
    if (change < tol * denom) {
      st->converged = 1;
      st->done = 1;
      return;
    }
    st->t = st->t_next;
    st->j += 1;
    if (st->j > max_iter) st->done = 1;
  }
}

template <typename T>
struct SplitLauncher {
  static void grad(Ctx*, dim3, unsigned, i64, i64, const T*, const T*, T, T, int, int, int, T, const T*, const T*, T*,
                   const SplitWs&, FistaState*) {}
  static void obj(Ctx*, dim3, unsigned, i64, i64, const T*, const T*, double, double, int, const T*, const T*,
                  const SplitWs&, double*, double*, FistaState*) {}
};
template <>
struct SplitLauncher<float> {
  static void grad(Ctx* c, dim3 g, unsigned eb, i64 rr, i64 rc, const float* Lr, const float* Lc, float s_r,
                   float s_c, int use_r, int use_c, int loss, float step, const float* Z, const float* Y, float* S,
                   const SplitWs& ws, FistaState* st) {
    fista_splitk_partial_k<<<g, 256, 0, c->stream>>>(rr, rc, Lr, Lc, use_r, use_c, Z, ws, st);
    launched(c);
    fista_splitk_grad_prox_k<<<eb, 256, 0, c->stream>>>(rr, rc, static_cast<int>(g.z), s_r, s_c, use_r, use_c, loss,
                                                        step, Z, Y, S, ws, st);
    launched(c);
  }
  static void obj(Ctx* c, dim3 g, unsigned eb, i64 rr, i64 rc, const float* Lr, const float* Lc, double gr, double gc,
                  int loss, const float* S, const float* Y, const SplitWs& ws, double* partials, double* trace,
                  FistaState* st) {
    fista_splitk_partial_k<<<g, 256, 0, c->stream>>>(rr, rc, Lr, Lc, gr != 0.0, gc != 0.0, S, ws, st);
    launched(c);
    fista_splitk_objective_k<<<eb, 256, 0, c->stream>>>(rr, rc, static_cast<int>(g.z), gr, gc, loss, S, Y, ws,
                                                        partials, trace, st);
    launched(c);
  }
};

template <typename T>
struct LinLauncher {  // fp32 only; other precisions never take the linearity path
  static void init(Ctx*, dim3, unsigned, i64, i64, const T*, const T*, int, int, const T*, const SplitWs&,
                   const LinBufs&, FistaState*) {}
  static void step(Ctx*, dim3, unsigned, i64, i64, const T*, const T*, T, T, int, int, const cpcag_frpcag_config&, T,
                   const T*, const T*, T*, const T*, T*, const SplitWs&, const LinBufs&, i64, double*, double*,
                   FistaState*) {}
};
template <>
struct LinLauncher<float> {
  static void init(Ctx* c, dim3 g, unsigned eb, i64 rr, i64 rc, const float* Lr, const float* Lc, int use_r, int use_c,
                   const float* Y, const SplitWs& ws, const LinBufs& lb, FistaState* st) {
    fista_splitk_partial_k<<<g, 256, 0, c->stream>>>(rr, rc, Lr, Lc, use_r, use_c, Y, ws, st);
    launched(c);
    fista_lin_init_k<<<eb, 256, 0, c->stream>>>(rr, rc, static_cast<int>(g.z), ws, lb);
    launched(c);
  }
  // One FISTA iteration: prox from L Z (no GEMM), one GEMM pair on S_j for
  // the objective, momentum carrying L Z_{j+1} forward.
  static void step(Ctx* c, dim3 g, unsigned eb, i64 rr, i64 rc, const float* Lr, const float* Lc, float s_r, float s_c,
                   int use_r, int use_c, const cpcag_frpcag_config& cfg, float stepT, const float* Z, const float* Y,
                   float* S, const float* Sp, float* Zn, const SplitWs& ws, const LinBufs& lb, i64 j, double* partials,
                   double* trace, FistaState* st) {
    const i64 m = rr * rc;
    {
      KScope ks_(c, "fista_grad_prox");
      fista_lin_grad_prox_k<<<eb, 256, 0, c->stream>>>(rr, rc, s_r, s_c, use_r, use_c, cfg.loss, stepT, Z, Y, S, lb,
                                                       st);
      launched(c);
    }
    {
      KScope ks_(c, "fista_objective");
      fista_splitk_partial_k<<<g, 256, 0, c->stream>>>(rr, rc, Lr, Lc, cfg.gamma_r != 0.0, cfg.gamma_c != 0.0, S, ws,
                                                       st);
      launched(c);
      fista_lin_objective_k<<<eb, 256, 0, c->stream>>>(rr, rc, static_cast<int>(g.z), cfg.gamma_r, cfg.gamma_c,
                                                       cfg.loss, S, Y, ws, lb.LSr[j & 1], lb.LSc[j & 1], partials,
                                                       trace, st);
      launched(c);
    }
    {
      KScope ks_(c, "fista_momentum");
      fista_lin_momentum_k<<<eb, 256, 0, c->stream>>>(m, S, Sp, Z, Zn, lb.LSr[j & 1], lb.LSr[(j - 1) & 1],
                                                      lb.LSc[j & 1], lb.LSc[(j - 1) & 1], lb, cfg.tol, cfg.max_iter,
                                                      partials, st);
      launched(c);
    }
  }
};

template <typename T>
void fista_device(Ctx* c, const T* Y, i64 rows, i64 cols, Csr* Lr, Csr* Lc,
                  const cpcag_frpcag_config& cfg, T* X, double* objective_host,
                  cpcag_solve_trace* trace) {
  frpcag_check_dims(rows, cols, Lr, Lc);
  if (cfg.gamma_r < 0.0 || cfg.gamma_c < 0.0) invalid("fista: negative regularization weight");
  if (cfg.tol <= 0.0) invalid("fista: stopping tolerance must be positive");
  if (cfg.max_iter < 1) invalid("fista: max_iter must be >= 1");
  double step = cfg.step;
  if (step <= 0.0) {
    // frpcag.cpp:70-75 (both norms with tol 1e-7, seed 42).
    double nc = 0.0, nr = 0.0;
    if (cfg.gamma_c != 0.0 && cfg.gamma_r != 0.0)
      power_norm_pair(c, Lc, Lr, 1e-7, 42, 50000, &nc, &nr);
    else if (cfg.gamma_c != 0.0)
      nc = power_norm(c, Lc, 1e-7, 42, 50000);
    else if (cfg.gamma_r != 0.0)
      nr = power_norm(c, Lr, 1e-7, 42, 50000);
    const double beta = 2.0 * cfg.gamma_c * nc + 2.0 * cfg.gamma_r * nr;
    step = beta > 0.0 ? 1.0 / beta : 1.0;
  }
  const i64 N = rows * cols;
  DevBuf<T> Sb[2] = {DevBuf<T>(c, N), DevBuf<T>(c, N)};
  DevBuf<T> Zb[2] = {DevBuf<T>(c, N), DevBuf<T>(c, N)};
  if (N) {
    CUDA_OK(cudaMemcpyAsync(Sb[0].p, Y, sizeof(T) * N, cudaMemcpyDeviceToDevice, c->stream));
    CUDA_OK(cudaMemcpyAsync(Zb[1].p, Y, sizeof(T) * N, cudaMemcpyDeviceToDevice, c->stream));
  }
  DevBuf<double> tr(c, cfg.max_iter);
  FistaState init{};
  init.t = 1.0;
  init.j = 1;
  DevBuf<FistaState> st(c, 1);
  CUDA_OK(cudaMemcpyAsync(st.p, &init, sizeof(init), cudaMemcpyHostToDevice, c->stream));

  const Pull<T> pr = make_pull<T>(c, Lr, false), pc = make_pull<T>(c, Lc, true);
  const int use_r = cfg.gamma_r != 0.0, use_c = cfg.gamma_c != 0.0;
  const unsigned gx = blocks_for(std::max<i64>(rows, 1));
  const i64 ycap = std::max<i64>(1, (static_cast<i64>(c->num_sms) * 16) / gx);
  dim3 g2(gx, static_cast<unsigned>(std::max<i64>(1, std::min<i64>({cols, ycap, 65535}))));
  const unsigned nb2 = g2.x * g2.y;
  const unsigned nb1 = stride_blocks(c, N);
  DevBuf<double> part(c, 3 * static_cast<size_t>(std::max(nb2, nb1)));
  const T s_r = static_cast<T>(2.0 * cfg.gamma_r), s_c = static_cast<T>(2.0 * cfg.gamma_c);
  const T stepT = static_cast<T>(step);

  // Dense path when both reduced Laplacians are >= 25 % full and exactly
  // symmetric (Kron outputs always are).
  const bool dense = dense_worthwhile(Lr) && dense_worthwhile(Lc) && csr_symmetric(c, Lr) && csr_symmetric(c, Lc);
  DevBuf<T> Dr, Dc;
  if (dense) {
    densify<T>(c, Lr, Dr);
    densify<T>(c, Lc, Dc);
  }
  dim3 gd(static_cast<unsigned>((rows + kDT - 1) / kDT), static_cast<unsigned>((cols + kDT - 1) / kDT));
  if (dense) part.alloc(c, 3 * static_cast<size_t>(std::max<unsigned>(gd.x * gd.y, nb1)));
  // dense: the whole solve as one cooperative kernel (fista_persist.cu) when
  // the tiling fits; otherwise the per-kernel paths below.
  {
    FistaPersistOut pres{};
    if (dense && fista_persist_enabled() &&
        fista_persist_run(c, Y, rows, cols, Dr.p, Dc.p, cfg, step, X, tr.p, &pres)) {
      if (pres.err)
        runtime("fista: diverged (non-finite objective at iteration " + std::to_string(pres.iterations) +
                "); step too large");
      const i64 J = pres.iterations;
      if (objective_host && J > 0)
        CUDA_OK(cudaMemcpyAsync(objective_host, tr.p, sizeof(double) * J, cudaMemcpyDefault, c->stream));
      sync(c);
      trace->iterations = J;
      trace->converged = pres.converged;
      trace->final_rel_change = pres.frc;
      trace->step = step;
      return;
    }
  }
  // fp32: split the k-space so the grid covers ~6 CTAs per SM.
  const bool splitk = dense && sizeof(T) == 4;
  DevBuf<double> sp1, sp2;
  DevBuf<unsigned> scnt;
  DevBuf<double> ssum;
  SplitWs ws{};
  dim3 gk(static_cast<unsigned>((rows + kST - 1) / kST), static_cast<unsigned>((cols + kST - 1) / kST));
  if (splitk) {
    const unsigned tiles = gk.x * gk.y;
    unsigned S = static_cast<unsigned>(std::max<i64>(1, (2 * static_cast<i64>(c->num_sms)) / tiles));  // measured: ~8 splits best at cfg1
    S = static_cast<unsigned>(std::min<i64>({static_cast<i64>(S), (rows + cols) / (4 * kSK) + 1, 32}));
    gk.z = S;
    sp1.alloc(c, static_cast<size_t>(S) * N);
    sp2.alloc(c, static_cast<size_t>(S) * N);
    scnt.alloc(c, tiles + 1);
    scnt.zero(c);
    ssum.alloc(c, 3 * static_cast<size_t>(tiles));
    ws = SplitWs{sp1.p, sp2.p, scnt.p, scnt.p + tiles, ssum.p};
  }
  // Linearity variant (fp32 split-K): one GEMM pair per iteration.
  const bool lin = splitk;
  DevBuf<T> lbuf;
  LinBufs lb{};
  if (lin) {
    lbuf.alloc(c, 6 * static_cast<size_t>(N));
    float* b = reinterpret_cast<float*>(lbuf.p);
    lb = LinBufs{b, b + N, {b + 2 * N, b + 3 * N}, {b + 4 * N, b + 5 * N}};
    LinLauncher<T>::init(c, gk, nb1, rows, cols, Dr.p, Dc.p, use_r, use_c, Y, ws, lb, st.p);
  }
  i64 j = 1;
  FistaState host{};
  const i64 chunk = 32;
  while (j <= cfg.max_iter && N > 0) {
    const i64 jend = std::min<i64>(cfg.max_iter, j + chunk - 1);
    for (; j <= jend; ++j) {
      const T* Zj = Zb[j & 1].p;
      T* Sj = Sb[j & 1].p;
      const T* Sprev = Sb[(j - 1) & 1].p;
      T* Znext = Zb[(j + 1) & 1].p;
      if (lin) {
        LinLauncher<T>::step(c, gk, nb1, rows, cols, Dr.p, Dc.p, s_r, s_c, use_r, use_c, cfg, stepT, Zj, Y, Sj, Sprev,
                             Znext, ws, lb, j, part.p, tr.p, st.p);
        continue;
      }
      if (splitk) {
        {
          KScope ks_(c, "fista_grad_prox");
          SplitLauncher<T>::grad(c, gk, nb1, rows, cols, Dr.p, Dc.p, s_r, s_c, use_r, use_c, cfg.loss, stepT, Zj, Y,
                                 Sj, ws, st.p);
        }
        {
          KScope ks_(c, "fista_objective");
          SplitLauncher<T>::obj(c, gk, nb1, rows, cols, Dr.p, Dc.p, cfg.gamma_r, cfg.gamma_c, cfg.loss, Sj, Y, ws,
                                part.p, tr.p, st.p);
        }
      } else if (dense) {
        {
          KScope ks_(c, "fista_grad_prox");
          fista_dense_grad_prox_k<T><<<gd, 256, 0, c->stream>>>(rows, cols, Dr.p, Dc.p, s_r, s_c, use_r, use_c,
                                                                cfg.loss, stepT, Zj, Y, Sj, st.p);
          launched(c);
        }
        {
          KScope ks_(c, "fista_objective");
          fista_dense_objective_k<T><<<gd, 256, 0, c->stream>>>(rows, cols, Dr.p, Dc.p, cfg.gamma_r, cfg.gamma_c,
                                                                cfg.loss, Sj, Y, part.p, tr.p, st.p);
          launched(c);
        }
      } else {
        {
          KScope ks_(c, "fista_grad_prox");
          fista_grad_prox_k<T><<<g2, kBlock, 0, c->stream>>>(rows, cols, pr, pc, s_r, s_c, use_r, use_c,
                                                             cfg.loss, stepT, Zj, Y, Sj, st.p);
          launched(c);
        }
        {
          KScope ks_(c, "fista_objective");
          fista_objective_k<T><<<g2, kBlock, 0, c->stream>>>(rows, cols, pr, pc, cfg.gamma_r, cfg.gamma_c,
                                                             cfg.loss, Sj, Y, part.p, tr.p, st.p);
          launched(c);
        }
      }
      {
        KScope ks_(c, "fista_momentum");
        fista_momentum_k<T><<<nb1, kBlock, 0, c->stream>>>(N, Sj, Sprev, Zj, Znext, cfg.tol,
                                                           cfg.max_iter, part.p, st.p);
        launched(c);
      }
    }
    host = read_back(c, st.p);
    if (host.done) break;
  }
  if (N == 0) {
    // Empty problem: the reference loop still runs; every norm is zero and
    // change < tol * denom is false (0 < 0), so it runs to max_iter with a
    // zero objective.
    host.iterations = cfg.max_iter;
    host.frc = 0.0;
    std::vector<double> z(static_cast<size_t>(cfg.max_iter), 0.0);
    if (objective_host) std::copy(z.begin(), z.end(), objective_host);
    trace->iterations = cfg.max_iter;
    trace->converged = 0;
    trace->final_rel_change = 0.0;
    trace->step = step;
    return;
  }
  if (host.err)
    runtime("fista: diverged (non-finite objective at iteration " + std::to_string(host.err_j) +
            "); step too large");
  const i64 J = host.iterations;
  CUDA_OK(cudaMemcpyAsync(X, Sb[J & 1].p, sizeof(T) * N, cudaMemcpyDeviceToDevice, c->stream));
  if (objective_host && J > 0)
    CUDA_OK(cudaMemcpyAsync(objective_host, tr.p, sizeof(double) * J, cudaMemcpyDefault, c->stream));
  sync(c);
  trace->iterations = J;
  trace->converged = host.converged;
  trace->final_rel_change = host.frc;
  trace->step = step;
}

template void fista_device<double>(Ctx*, const double*, i64, i64, Csr*, Csr*, const cpcag_frpcag_config&,
                                   double*, double*, cpcag_solve_trace*);
template void fista_device<float>(Ctx*, const float*, i64, i64, Csr*, Csr*, const cpcag_frpcag_config&,
                                  float*, double*, cpcag_solve_trace*);

}  // namespace cpcag_cuda

using namespace cpcag_cuda;

extern "C" int cpcag_cuda_fista(cpcag_ctx ctx, int precision, const void* Y, int64_t rows, int64_t cols,
                                cpcag_csr Lr, cpcag_csr Lc, const cpcag_frpcag_config* cfg, void* X,
                                double* objective, cpcag_solve_trace* trace) {
  auto run = [&](auto tag) {
    using T = decltype(tag);
    return guard([&] {
      Ctx* c = as_ctx(ctx);
      if (!cfg || !trace) invalid("null argument");
      InView<T> y(c, static_cast<const T*>(Y), static_cast<size_t>(rows * cols));
      OutView<T> x(c, static_cast<T*>(X), static_cast<size_t>(rows * cols));
      std::vector<double> obj_host;
      double* obj_dst = objective;
      if (objective && is_device_ptr(objective)) {
        obj_host.resize(static_cast<size_t>(std::max<int64_t>(cfg->max_iter, 1)));
        obj_dst = obj_host.data();
      }
      fista_device<T>(c, y.d, rows, cols, as_csr(Lr), as_csr(Lc), *cfg, x.d, obj_dst, trace);
      x.flush(c);
      if (!obj_host.empty() && trace->iterations > 0)
        CUDA_OK(cudaMemcpyAsync(objective, obj_host.data(), sizeof(double) * trace->iterations,
                                cudaMemcpyHostToDevice, c->stream));
      sync(c);
    });
  };
  if (precision == CPCAG_F64) return run(double{});
  if (precision == CPCAG_F32) return run(float{});
  set_last_error("unknown precision flag");
  return CPCAG_ERR_INVALID_ARGUMENT;
}
