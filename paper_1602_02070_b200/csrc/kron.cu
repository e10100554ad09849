// kron.cu -- Kron reduction of a Laplacian onto the kept node set
// (graph.cpp:170-235) and the Jacobi-preconditioned CG it runs per kept node
// (solvers.cpp:7-27, solvers.hpp:33-74).
//
// Device plan:
//   1. connected components of the pattern by lock-free union-find (roots =
//      smallest node, the node the reference's error message names);
//   2. interior / kept index maps, L_aa and L_ba gathered as device CSR,
//      L_bb scattered into the dense Schur matrix S (keep order);
//   3. every kept node j with a nonempty row of L_ba is one column of a
//      batched, per-column-independent Jacobi PCG on L_aa (each column runs
//      the reference recurrence with its own alpha/beta and its own stop
//      test; finished columns freeze);
//   4. S(:, j) -= L_ba z_j, S <- (S + S^T)/2, prune |v| <= prune_tol,
//      CSR in keep order.
// RHS blocks are sized to the free HBM so 50 000-column reductions run in
// slices.
#include <algorithm>
#include <string>
#include <cstdio>
#include <cstdlib>
#include <cub/cub.cuh>
#include <memory>
#include <numeric>

#include <cuda_fp16.h>

#include "common.cuh"
#include "frpcag.cuh"

namespace cpcag_cuda {

// ------------------------------------------------------------------ components
// Find with path halving.  Roots only ever link under smaller roots, so
// every parent pointer points to a smaller index and replacing parent[x] by
// its grandparent (a plain store racing with other finds) keeps the forest
// valid.
__device__ __forceinline__ int uf_root(volatile int* parent, int x) {
  while (true) {
    const int p = parent[x];
    if (p == x) return x;
    const int gp = parent[p];
    if (gp != p) parent[x] = gp;
    x = gp;
  }
}

__global__ void uf_init_k(i64 n, int* parent) {
  const i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x;
  if (i < n) parent[i] = static_cast<int>(i);
}

__global__ void uf_hook_k(i64 n, const i64* __restrict__ rp, const int* __restrict__ ci, int* parent) {
  const i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x;
  if (i >= n) return;
  for (i64 k = rp[i]; k < rp[i + 1]; ++k) {
    int a = static_cast<int>(i), b = ci[k];
    while (true) {
      a = uf_root(parent, a);
      b = uf_root(parent, b);
      if (a == b) break;
      if (a < b) {
        const int t = a;
        a = b;
        b = t;
      }
      // link the larger root under the smaller one: the surviving root of a
      // component is its smallest node.
      const int old = atomicCAS(parent + a, a, b);
      if (old == a) break;
      a = old;
    }
  }
}

__global__ void uf_flatten_k(i64 n, int* parent) {
  const i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x;
  if (i < n) parent[i] = uf_root(parent, static_cast<int>(i));
}

__global__ void ground_k(i64 m, const i64* __restrict__ keep, const int* __restrict__ parent, int* grounded) {
  const i64 j = blockIdx.x * (i64)blockDim.x + threadIdx.x;
  if (j < m) grounded[parent[keep[j]]] = 1;
}

__global__ void ungrounded_k(i64 n, const int* __restrict__ parent, const int* __restrict__ grounded, int* first) {
  const i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x;
  if (i < n && parent[i] == i && !grounded[i]) atomicMin(first, static_cast<int>(i));
}

// ------------------------------------------------------------------ gathers
// Count / fill of a row-gathered, column-filtered submatrix: rows rsrc[r],
// columns kept when cmap[col] >= 0 (cmap monotone, so columns stay sorted).
__global__ void sub_count_k(i64 nr, const i64* __restrict__ rsrc, const i64* __restrict__ rp,
                            const int* __restrict__ ci, const int* __restrict__ cmap, i64* __restrict__ cnt) {
  const i64 r = blockIdx.x * (i64)blockDim.x + threadIdx.x;
  if (r >= nr) return;
  const i64 u = rsrc[r];
  i64 c = 0;
  for (i64 k = rp[u]; k < rp[u + 1]; ++k) c += cmap[ci[k]] >= 0;
  cnt[r] = c;
}

__global__ void sub_fill_k(i64 nr, const i64* __restrict__ rsrc, const i64* __restrict__ rp,
                           const int* __restrict__ ci, const double* __restrict__ v,
                           const int* __restrict__ cmap, const i64* __restrict__ orp,
                           int* __restrict__ oci, double* __restrict__ ov) {
  const i64 r = blockIdx.x * (i64)blockDim.x + threadIdx.x;
  if (r >= nr) return;
  const i64 u = rsrc[r];
  i64 o = orp[r];
  for (i64 k = rp[u]; k < rp[u + 1]; ++k) {
    const int m = cmap[ci[k]];
    if (m >= 0) {
      oci[o] = m;
      ov[o] = v[k];
      ++o;
    }
  }
}

// S(j, kpos[col]) = L(keep[j], col) for kept columns (dense m x m, col-major).
__global__ void scatter_bb_k(i64 m, const i64* __restrict__ keep, const i64* __restrict__ rp,
                             const int* __restrict__ ci, const double* __restrict__ v,
                             const int* __restrict__ kpos, double* __restrict__ S) {
  const i64 j = blockIdx.x * (i64)blockDim.x + threadIdx.x;
  if (j >= m) return;
  const i64 u = keep[j];
  for (i64 k = rp[u]; k < rp[u + 1]; ++k) {
    const int q = kpos[ci[k]];
    if (q >= 0) S[j + static_cast<i64>(q) * m] = v[k];
  }
}

// Jacobi inverse of the diagonal (solvers.cpp:14-15: d > 0 ? 1/d : 1).
__global__ void jacobi_inv_k(i64 n, const i64* __restrict__ rp, const int* __restrict__ ci,
                             const double* __restrict__ v, double* __restrict__ inv) {
  const i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x;
  if (i >= n) return;
  double d = 0.0;
  for (i64 k = rp[i]; k < rp[i + 1]; ++k)
    if (ci[k] == i) d = v[k];
  inv[i] = d > 0.0 ? 1.0 / d : 1.0;
}

__global__ void ones_k(i64 n, double* a) {
  const i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x;
  if (i < n) a[i] = 1.0;
}

// ------------------------------------------------------------------ batched PCG
// Column c of the batch is one independent PCG (solvers.hpp:33-74).  Per
// column scalars live in ColState; per-column reductions go through
// partials[c][rb] and the last row-block of the column (per-column arrival
// counter) finalises them in a fixed order.
struct ColState {
  double rho, rho_next, rr, curv, alpha, beta, norm_b, target, rel_res;
  i64 it;
  int done, err;  // err: 1 breakdown
  unsigned cnt;
  int pad;
};

constexpr int kPcgBlock = 256;

__device__ __forceinline__ bool col_last_block(ColState* s, unsigned nrb) {
  __shared__ bool last;
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    last = atomicAdd(&s->cnt, 1u) == nrb - 1;
  }
  __syncthreads();
  if (last) __threadfence();
  return last;
}

template <int NV>
__device__ __forceinline__ void col_partial(double (&v)[NV], double* partials, i64 c, unsigned rb, unsigned nrb) {
  block_sum<NV>(v);
  if (threadIdx.x == 0) {
#pragma unroll
    for (int q = 0; q < NV; ++q) partials[(c * NV + q) * nrb + rb] = v[q];
  }
}

template <int NV>
__device__ __forceinline__ void col_total(double (&t)[NV], const double* partials, i64 c, unsigned nrb) {
#pragma unroll
  for (int q = 0; q < NV; ++q) {
    double s = 0.0;
    for (unsigned i = threadIdx.x; i < nrb; i += blockDim.x) s += __ldcg(partials + (c * NV + q) * nrb + i);
    t[q] = s;
  }
  block_sum<NV>(t);
}

// r = b - A x, z = inv o r, p = z; rho = <r, z>, ||b||^2, ||r||^2.
__global__ void pcg_init_k(i64 n, i64 nb, const i64* __restrict__ rp, const int* __restrict__ ci,
                           const double* __restrict__ v, const double* __restrict__ inv,
                           const double* __restrict__ B, const double* __restrict__ X, double* __restrict__ R,
                           double* __restrict__ Z, double* __restrict__ P, double tol, i64 max_iter,
                           double* partials, ColState* st, unsigned* ndone) {
  const unsigned rb = blockIdx.x, nrb = gridDim.x;
  for (i64 c = blockIdx.y; c < nb; c += gridDim.y) {
    double s[3] = {0.0, 0.0, 0.0};
    const i64 i = rb * (i64)blockDim.x + threadIdx.x;
    if (i < n) {
      const i64 at = i + c * n;
      const double ax = pull_left(rp[i], rp[i + 1], ci, v, X + c * n);
      const double b = B[at];
      const double r = __dsub_rn(b, ax);
      const double z = __dmul_rn(inv[i], r);
      R[at] = r;
      Z[at] = z;
      P[at] = z;
      s[0] = b * b;
      s[1] = r * z;
      s[2] = r * r;
    }
    col_partial<3>(s, partials, c, rb, nrb);
    if (col_last_block(st + c, nrb)) {
      double t[3];
      col_total<3>(t, partials, c, nrb);
      if (threadIdx.x == 0) {
        ColState& S = st[c];
        S.cnt = 0u;
        S.norm_b = sqrt(t[0]);
        S.rho = t[1];
        S.rr = t[2];
        S.it = 0;
        S.target = tol * S.norm_b;
        if (S.norm_b == 0.0) {
          S.done = 2;  // zero rhs: x = b, converged, no true-residual pass
          atomicAdd(ndone, 1u);
        } else if (sqrt(S.rr) <= S.target || max_iter <= 0) {
          S.done = 1;
          atomicAdd(ndone, 1u);
        }
      }
    }
  }
}

__global__ void pcg_apply_k(i64 n, i64 nb, const i64* __restrict__ rp, const int* __restrict__ ci,
                            const double* __restrict__ v, const double* __restrict__ P,
                            double* __restrict__ AP, double* partials, ColState* st) {
  const unsigned rb = blockIdx.x, nrb = gridDim.x;
  for (i64 c = blockIdx.y; c < nb; c += gridDim.y) {
    if (st[c].done) continue;
    double s[1] = {0.0};
    const i64 i = rb * (i64)blockDim.x + threadIdx.x;
    if (i < n) {
      const double ap = pull_left(rp[i], rp[i + 1], ci, v, P + c * n);
      AP[i + c * n] = ap;
      s[0] = P[i + c * n] * ap;
    }
    col_partial<1>(s, partials, c, rb, nrb);
  }
}

__global__ void pcg_update_k(i64 n, i64 nb, const double* __restrict__ inv, double* __restrict__ X,
                             double* __restrict__ R, double* __restrict__ Z, const double* __restrict__ P,
                             const double* __restrict__ AP, double* partials, double* partials2,
                             ColState* st, unsigned* ndone) {
  const unsigned rb = blockIdx.x, nrb = gridDim.x;
  for (i64 c = blockIdx.y; c < nb; c += gridDim.y) {
    if (st[c].done) continue;
    double t[1];
    col_total<1>(t, partials, c, nrb);
    const double curv = t[0];
    const bool bad = !isfinite(curv) || curv <= 0.0;
    double s[2] = {0.0, 0.0};
    if (!bad) {
      const double alpha = st[c].rho / curv;
      const i64 i = rb * (i64)blockDim.x + threadIdx.x;
      if (i < n) {
        const i64 at = i + c * n;
        X[at] = __dadd_rn(X[at], __dmul_rn(alpha, P[at]));
        const double r = __dsub_rn(R[at], __dmul_rn(alpha, AP[at]));
        const double z = __dmul_rn(inv[i], r);
        R[at] = r;
        Z[at] = z;
        s[0] = r * z;
        s[1] = r * r;
      }
    }
    col_partial<2>(s, partials2, c, rb, nrb);
    if (col_last_block(st + c, nrb) && threadIdx.x == 0) {
      ColState& S = st[c];
      S.cnt = 0u;
      S.curv = curv;
      if (bad) {
        S.err = 1;
        S.done = 1;
        atomicAdd(ndone, 1u);
      } else {
        S.alpha = S.rho / curv;
      }
    }
  }
}

__global__ void pcg_direction_k(i64 n, i64 nb, i64 max_iter, const double* __restrict__ Z,
                                double* __restrict__ P, const double* partials2, ColState* st,
                                unsigned* ndone) {
  const unsigned rb = blockIdx.x, nrb = gridDim.x;
  for (i64 c = blockIdx.y; c < nb; c += gridDim.y) {
    if (st[c].done) continue;
    double t[2];
    col_total<2>(t, partials2, c, nrb);
    const double beta = t[0] / st[c].rho;
    const i64 i = rb * (i64)blockDim.x + threadIdx.x;
    if (i < n) {
      const i64 at = i + c * n;
      P[at] = __dadd_rn(Z[at], __dmul_rn(beta, P[at]));
    }
    if (col_last_block(st + c, nrb) && threadIdx.x == 0) {
      ColState& S = st[c];
      S.cnt = 0u;
      S.rho = t[0];
      S.rr = t[1];
      S.it += 1;
      if (sqrt(S.rr) <= S.target || S.it >= max_iter) {
        S.done = 1;
        atomicAdd(ndone, 1u);
      }
    }
  }
}

// True residual ||b - A x|| / ||b|| per column (solvers.hpp:69-72).
__global__ void pcg_true_k(i64 n, i64 nb, const i64* __restrict__ rp, const int* __restrict__ ci,
                           const double* __restrict__ v, const double* __restrict__ B,
                           const double* __restrict__ X, double* partials, ColState* st) {
  const unsigned rb = blockIdx.x, nrb = gridDim.x;
  for (i64 c = blockIdx.y; c < nb; c += gridDim.y) {
    if (st[c].done == 2) continue;
    double s[1] = {0.0};
    const i64 i = rb * (i64)blockDim.x + threadIdx.x;
    if (i < n) {
      const double e = __dsub_rn(B[i + c * n], pull_left(rp[i], rp[i + 1], ci, v, X + c * n));
      s[0] = e * e;
    }
    col_partial<1>(s, partials, c, rb, nrb);
    if (col_last_block(st + c, nrb)) {
      double t[1];
      col_total<1>(t, partials, c, nrb);
      if (threadIdx.x == 0) {
        st[c].cnt = 0u;
        st[c].rel_res = sqrt(t[0]) / st[c].norm_b;
      }
    }
  }
}

// ------------------------------------------------------------------ persistent batched PCG
// Each CTA owns kCpb complete RHS columns, stored as a row-interleaved slab
// (element (i, c) at ((c / kCpb) * n + i) * kCpb + c % kCpb), so one
// 32-byte load fetches a row of all its columns and every per-column dot
// product is a block reduction.  The CTA runs its columns' PCG iterations to
// completion in one launch (columns are independent; no grid-wide sync), in
// the reference recurrence with z = inv o r recomputed instead of stored.
constexpr int kCpb = 4;

__device__ __forceinline__ i64 slab_at(i64 n, i64 i, i64 c) { return ((c / kCpb) * n + i) * kCpb + (c % kCpb); }

// One slab row (kCpb = 4 columns, 32 bytes, 32-byte aligned) per access:
// two 16-byte loads/stores instead of four 8-byte ones (the kernel is
// L1/LSU-throughput bound on the scalar form).
static_assert(kCpb == 4, "slab records are 4 doubles");
__device__ __forceinline__ void ld4(const double* __restrict__ p, double (&o)[4]) {
  const double2 x = *reinterpret_cast<const double2*>(p);
  const double2 y = *reinterpret_cast<const double2*>(p + 2);
  o[0] = x.x;
  o[1] = x.y;
  o[2] = y.x;
  o[3] = y.y;
}
__device__ __forceinline__ void st4(double* __restrict__ p, const double (&v)[4]) {
  *reinterpret_cast<double2*>(p) = make_double2(v[0], v[1]);
  *reinterpret_cast<double2*>(p + 2) = make_double2(v[2], v[3]);
}

template <int NT, int MINB>
__global__ void __launch_bounds__(NT, MINB) pcg_persistent_k(i64 n, i64 nb, const i64* __restrict__ rp,
                                                        const int* __restrict__ ci, const double* __restrict__ v,
                                                        const double* __restrict__ inv, const double* __restrict__ B,
                                                        double* __restrict__ X, double* __restrict__ R,
                                                        double* __restrict__ P, double* __restrict__ AP, double tol,
                                                        i64 max_iter, ColState* st, i64 gbase) {
  const i64 grp = gbase + blockIdx.x;  // column group of this CTA
  const i64 c0 = grp * kCpb;
  const i64 base = grp * n * kCpb;
  __shared__ int done_s[kCpb];
  __shared__ double rho_s[kCpb], target_s[kCpb];
  __shared__ i64 it_s[kCpb];
  // r = b - A x, z = inv o r, p = z
  double s3[3 * kCpb];
#pragma unroll
  for (int q = 0; q < 3 * kCpb; ++q) s3[q] = 0.0;
  for (i64 i = threadIdx.x; i < n; i += blockDim.x) {
    double ax[kCpb];
#pragma unroll
    for (int q = 0; q < kCpb; ++q) ax[q] = 0.0;
    for (i64 k = rp[i]; k < rp[i + 1]; ++k) {
      const double a = v[k];
      double xr[4];
      ld4(X + base + static_cast<i64>(ci[k]) * kCpb, xr);
#pragma unroll
      for (int q = 0; q < kCpb; ++q) ax[q] = __dadd_rn(ax[q], __dmul_rn(a, xr[q]));
    }
    const double iv = inv[i];
    const i64 at = base + i * kCpb;
    double bv[4], rv[4], zv[4];
    ld4(B + at, bv);
#pragma unroll
    for (int q = 0; q < kCpb; ++q) {
      const double b = bv[q];
      const double r = __dsub_rn(b, ax[q]);
      const double z = __dmul_rn(iv, r);
      rv[q] = r;
      zv[q] = z;
      s3[q] += b * b;
      s3[kCpb + q] += r * z;
      s3[2 * kCpb + q] += r * r;
    }
    st4(R + at, rv);
    st4(P + at, zv);
  }
  block_sum<3 * kCpb>(s3);
  if (threadIdx.x == 0) {
    for (int q = 0; q < kCpb; ++q) {
      const i64 c = c0 + q;
      it_s[q] = 0;
      if (c >= nb) {
        done_s[q] = 3;
        continue;
      }
      ColState& S = st[c];
      S.norm_b = sqrt(s3[q]);
      S.target = tol * S.norm_b;
      rho_s[q] = s3[kCpb + q];
      target_s[q] = S.target;
      S.it = 0;
      if (S.norm_b == 0.0)
        done_s[q] = 2;
      else if (sqrt(s3[2 * kCpb + q]) <= S.target || max_iter <= 0)
        done_s[q] = 1;
      else
        done_s[q] = 0;
      S.done = done_s[q];
    }
  }
  __syncthreads();
  while (true) {
    bool any = false;
#pragma unroll
    for (int q = 0; q < kCpb; ++q) any |= done_s[q] == 0;
    if (!any) break;
    // ap = A p, curvature
    double cv[kCpb];
#pragma unroll
    for (int q = 0; q < kCpb; ++q) cv[q] = 0.0;
    for (i64 i = threadIdx.x; i < n; i += blockDim.x) {
      double ap[kCpb];
#pragma unroll
      for (int q = 0; q < kCpb; ++q) ap[q] = 0.0;
      for (i64 k = rp[i]; k < rp[i + 1]; ++k) {
        const double a = v[k];
        double pr[4];
        ld4(P + base + static_cast<i64>(ci[k]) * kCpb, pr);
#pragma unroll
        for (int q = 0; q < kCpb; ++q) ap[q] = __dadd_rn(ap[q], __dmul_rn(a, pr[q]));
      }
      const i64 at = base + i * kCpb;
      double pv[4];
      ld4(P + at, pv);
      st4(AP + at, ap);
#pragma unroll
      for (int q = 0; q < kCpb; ++q) cv[q] += pv[q] * ap[q];
    }
    block_sum<kCpb>(cv);
    // alpha, breakdown
    double alpha[kCpb];
    bool live[kCpb];
#pragma unroll
    for (int q = 0; q < kCpb; ++q) {
      live[q] = done_s[q] == 0;
      const bool bad = !isfinite(cv[q]) || cv[q] <= 0.0;
      alpha[q] = rho_s[q] / cv[q];
      if (live[q] && bad) live[q] = false;
    }
    __syncthreads();
    if (threadIdx.x == 0)
      for (int q = 0; q < kCpb; ++q)
        if (done_s[q] == 0 && (!isfinite(cv[q]) || cv[q] <= 0.0)) {
          st[c0 + q].err = 1;
          st[c0 + q].curv = cv[q];
          done_s[q] = 1;
        }
    // x += alpha p, r -= alpha ap, <r, z>, <r, r>
    double s2[2 * kCpb];
#pragma unroll
    for (int q = 0; q < 2 * kCpb; ++q) s2[q] = 0.0;
    for (i64 i = threadIdx.x; i < n; i += blockDim.x) {
      const double iv = inv[i];
      const i64 at = base + i * kCpb;
      double xv[4], pv[4], rv[4], av[4];
      ld4(X + at, xv);
      ld4(P + at, pv);
      ld4(R + at, rv);
      ld4(AP + at, av);
#pragma unroll
      for (int q = 0; q < kCpb; ++q) {
        if (!live[q]) continue;
        xv[q] = __dadd_rn(xv[q], __dmul_rn(alpha[q], pv[q]));
        const double r = __dsub_rn(rv[q], __dmul_rn(alpha[q], av[q]));
        rv[q] = r;
        const double z = __dmul_rn(iv, r);
        s2[q] += r * z;
        s2[kCpb + q] += r * r;
      }
      st4(X + at, xv);
      st4(R + at, rv);
    }
    block_sum<2 * kCpb>(s2);
    // p = z + beta p
    double beta[kCpb];
#pragma unroll
    for (int q = 0; q < kCpb; ++q) beta[q] = s2[q] / rho_s[q];
    for (i64 i = threadIdx.x; i < n; i += blockDim.x) {
      const double iv = inv[i];
      const i64 at = base + i * kCpb;
      double pv[4], rv[4];
      ld4(P + at, pv);
      ld4(R + at, rv);
#pragma unroll
      for (int q = 0; q < kCpb; ++q)
        if (live[q]) pv[q] = __dadd_rn(__dmul_rn(iv, rv[q]), __dmul_rn(beta[q], pv[q]));
      st4(P + at, pv);
    }
    __syncthreads();
    if (threadIdx.x == 0)
      for (int q = 0; q < kCpb; ++q) {
        if (!live[q]) continue;
        rho_s[q] = s2[q];
        it_s[q] += 1;
        if (sqrt(s2[kCpb + q]) <= target_s[q] || it_s[q] >= max_iter) done_s[q] = 1;
      }
    __syncthreads();
  }
  // true residual
  double sr[kCpb];
#pragma unroll
  for (int q = 0; q < kCpb; ++q) sr[q] = 0.0;
  for (i64 i = threadIdx.x; i < n; i += blockDim.x) {
    double ax[kCpb];
#pragma unroll
    for (int q = 0; q < kCpb; ++q) ax[q] = 0.0;
    for (i64 k = rp[i]; k < rp[i + 1]; ++k) {
      const double a = v[k];
      double xr[4];
      ld4(X + base + static_cast<i64>(ci[k]) * kCpb, xr);
#pragma unroll
      for (int q = 0; q < kCpb; ++q) ax[q] = __dadd_rn(ax[q], __dmul_rn(a, xr[q]));
    }
    double bv[4];
    ld4(B + base + i * kCpb, bv);
#pragma unroll
    for (int q = 0; q < kCpb; ++q) {
      const double e = __dsub_rn(bv[q], ax[q]);
      sr[q] += e * e;
    }
  }
  block_sum<kCpb>(sr);
  if (threadIdx.x == 0)
    for (int q = 0; q < kCpb; ++q) {
      const i64 c = c0 + q;
      if (c >= nb) continue;
      ColState& S = st[c];
      S.it = it_s[q];
      S.done = done_s[q] == 2 ? 2 : 1;
      S.rel_res = sqrt(sr[q]) / S.norm_b;
    }
}

// ------------------------------------------------------------------ shared-memory resident PCG
// One CTA per right-hand side, for interiors whose p, x and the Jacobi
// inverse (3 n fp64) fit in one CTA's shared memory (config 1 rows: n = 9 273,
// 222 KB).  Thread t owns rows t + r NT (r < RPT) and keeps their r and A p in
// registers; the SpMV gathers p from shared memory; the matrix is read as ELL
// (entry k of row i at k n + i, zero padded with the row's own column, CSR
// order kept) from L2, shared by every CTA.  Per iteration three CTA barriers
// (two reductions, the p update); every CTA runs its column to completion and
// the hardware schedules the next column on the freed SM.  Same recurrence
// and per-entry arithmetic as pcg_persistent_k (solvers.hpp:33-74).
template <int NV, int NW>
__device__ __forceinline__ void cta_sum(double (&v)[NV], double* red, int& par) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
  for (int q = 0; q < NV; ++q) v[q] = warp_sum(v[q]);
  double* b = red + par * NV * NW;
  if (lane == 0)
#pragma unroll
    for (int q = 0; q < NV; ++q) b[q * NW + wid] = v[q];
  __syncthreads();
#pragma unroll
  for (int q = 0; q < NV; ++q) {
    double t = 0.0;
#pragma unroll
    for (int w = 0; w < NW; ++w) t += b[q * NW + w];
    v[q] = t;
  }
  par ^= 1;
}

__global__ void csr_to_ell_k(i64 n, int E, const i64* __restrict__ rp, const int* __restrict__ ci,
                             const double* __restrict__ v, double* __restrict__ ev, int* __restrict__ ec) {
  const i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const i64 k0 = rp[i], d = rp[i + 1] - k0;
  for (int k = 0; k < E; ++k) {
    ev[k * n + i] = k < d ? v[k0 + k] : 0.0;
    ec[k * n + i] = k < d ? ci[k0 + k] : static_cast<int>(i);
  }
}

// Packed ELL when every value is exact in fp32: one 8-byte word per entry
// (fp32 value bits, column), two thirds of the bytes of (fp64, int32); the
// flag reports a value that fp32 cannot hold.
__global__ void csr_to_ell_packed_k(i64 n, int E, const i64* __restrict__ rp, const int* __restrict__ ci,
                                    const double* __restrict__ v, uint2* __restrict__ ep, int* flag) {
  const i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const i64 k0 = rp[i], d = rp[i + 1] - k0;
  // flag[1]: the half bandwidth max |column - row| (the reach of one product)
  int bw = 0;
  for (i64 k = 0; k < d; ++k) bw = max(bw, abs(ci[k0 + k] - static_cast<int>(i)));
  if (bw > 0) atomicMax(flag + 1, bw);
  for (int k = 0; k < E; ++k) {
    const double x = k < d ? v[k0 + k] : 0.0;
    const float f = static_cast<float>(x);
    if (static_cast<double>(f) != x) atomicOr(flag, 1);
    if (static_cast<double>(__half2float(__float2half_rn(f))) != x) atomicOr(flag, 2);
    ep[k * n + i] = make_uint2(__float_as_uint(f), static_cast<unsigned>(k < d ? ci[k0 + k] : static_cast<int>(i)));
  }
}

// Narrowest packing: (fp16 value, u16 column) in one 4-byte word, when every
// value is exact in fp16 (unit-weight grids: small integers) and n < 65536.
__global__ void ell_pack16_k(i64 n, int E, const uint2* __restrict__ ep, unsigned* __restrict__ eh) {
  const i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x;
  if (i >= n) return;
  for (int k = 0; k < E; ++k) {
    const uint2 w = ep[k * n + i];
    const unsigned short h = __half_as_ushort(__float2half_rn(__uint_as_float(w.x)));
    eh[k * n + i] = static_cast<unsigned>(h) | (w.y << 16);
  }
}

constexpr int kPcgSmemThreads = 512;

// E > 0: the matrix as ELL with E entries a row, read from global memory;
// E == 0: the CSR (rp, ci, v of nnz entries) staged in shared memory after
// the three vectors (small interiors, e.g. config 1's 900-node column graph).
// PK: the ELL packed as (fp32 value, column) 8-byte words (ev is then a uint2
// array, PK == 1) or (fp16 value, u16 column) 4-byte words (PK == 2).
template <int RPT, int E, int PK = 0>
__global__ void __launch_bounds__(kPcgSmemThreads, 1) pcg_smem_k(int n, i64 nb, const double* __restrict__ ev,
                                                                 const int* __restrict__ ec,
                                                                 const i64* __restrict__ crp,
                                                                 const double* __restrict__ inv,
                                                                 const double* __restrict__ B, double* __restrict__ X,
                                                                 double tol, i64 max_iter, ColState* st,
                                                                 const int* __restrict__ bwp) {
  constexpr int NT = kPcgSmemThreads, NW = NT / 32;
  // Support window.  With half bandwidth bw = max |column - row|, one product
  // widens the rows where p, r and A p can be nonzero by bw on each side; a
  // Kron right-hand side (one kept node's few interior neighbours) starts
  // narrow, so most rows are exact zeros for the first n / (2 bw) iterations.
  // Rows outside the window are skipped -- they would compute 0 = 0 + v * 0
  // and x += alpha * 0, so every value is bit-identical to the full sweep.
  const int bw = bwp ? *bwp : n;
  __shared__ int s_lo, s_hi;
  if (threadIdx.x == 0) {
    s_lo = n;
    s_hi = -1;
  }
  extern __shared__ __align__(16) double smd[];
  double* Ps = smd;
  double* Xs = smd + n;
  double* Is = smd + 2 * n;
  // E == 0: CSR in shared memory (values, row pointers as int, columns)
  const int nnz = E == 0 ? static_cast<int>(crp[n]) : 0;
  double* Sv = smd + 3 * n;
  int* Srp = reinterpret_cast<int*>(Sv + nnz);
  int* Sci = Srp + n + 1;
  __shared__ double red[2 * 3 * NW];
  const i64 col = blockIdx.x;
  const int t = threadIdx.x;
  for (int i = t; i < n; i += NT) {
    Is[i] = inv[i];
    Xs[i] = X[slab_at(n, i, col)];
  }
  if constexpr (E == 0) {
    for (int k = t; k < nnz; k += NT) {
      Sv[k] = ev[k];
      Sci[k] = ec[k];
    }
    for (int i = t; i <= n; i += NT) Srp[i] = static_cast<int>(crp[i]);
  }
  __syncthreads();
  int par = 0;
  auto spmv = [&](const double* src, int i) {
    double a = 0.0;
    if constexpr (E == 0) {
      for (int k = Srp[i]; k < Srp[i + 1]; ++k) a = __dadd_rn(a, __dmul_rn(Sv[k], src[Sci[k]]));
    } else if constexpr (PK == 2) {
      const unsigned* eh = reinterpret_cast<const unsigned*>(ev);
#pragma unroll
      for (int k = 0; k < E; ++k) {
        const unsigned w = eh[static_cast<i64>(k) * n + i];
        a = __dadd_rn(a, __dmul_rn(static_cast<double>(__half2float(__ushort_as_half(static_cast<unsigned short>(w & 0xffffu)))),
                                   src[w >> 16]));
      }
    } else if constexpr (PK == 1) {
      const uint2* ep = reinterpret_cast<const uint2*>(ev);
#pragma unroll
      for (int k = 0; k < E; ++k) {
        const uint2 w = ep[static_cast<i64>(k) * n + i];
        a = __dadd_rn(a, __dmul_rn(static_cast<double>(__uint_as_float(w.x)), src[w.y]));
      }
    } else {
#pragma unroll
      for (int k = 0; k < E; ++k)
        a = __dadd_rn(a, __dmul_rn(ev[static_cast<i64>(k) * n + i], src[ec[static_cast<i64>(k) * n + i]]));
    }
    return a;
  };
  double R[RPT], AP[RPT];
  // r = b - A x, z = inv o r, p = z
  double s3[3] = {0.0, 0.0, 0.0};
  int my_lo = n, my_hi = -1;
#pragma unroll
  for (int r = 0; r < RPT; ++r) {
    const int i = t + r * NT;
    R[r] = 0.0;
    if (i < n) {
      const double b = B[slab_at(n, i, col)];
      const double rr = __dsub_rn(b, spmv(Xs, i));
      const double z = __dmul_rn(Is[i], rr);
      R[r] = rr;
      Ps[i] = z;
      s3[0] += b * b;
      s3[1] += rr * z;
      s3[2] += rr * rr;
      if (rr != 0.0 || z != 0.0) {
        my_lo = min(my_lo, i);
        my_hi = max(my_hi, i);
      }
    }
  }
  if (my_hi >= 0) {
    atomicMin(&s_lo, my_lo);
    atomicMax(&s_hi, my_hi);
  }
  cta_sum<3, NW>(s3, red, par);
  const double norm_b = sqrt(s3[0]), target = tol * norm_b;
  double rho = s3[1];
  int done = norm_b == 0.0 ? 2 : ((sqrt(s3[2]) <= target || max_iter <= 0) ? 1 : 0);
  int err = 0;
  double curv = 0.0;
  i64 it = 0;
  __syncthreads();  // p and the support window complete
  int lo = s_lo, hi = s_hi + 1;  // rows [lo, hi) hold every nonzero of p and r
  while (done == 0) {
    const int alo = max(0, lo - bw), ahi = static_cast<int>(min(static_cast<i64>(n), static_cast<i64>(hi) + bw));
    double cv[1] = {0.0};
#pragma unroll
    for (int r = 0; r < RPT; ++r) {
      const int i = t + r * NT;
      AP[r] = 0.0;
      if (i >= alo && i < ahi) {
        AP[r] = spmv(Ps, i);
        cv[0] += Ps[i] * AP[r];
      }
    }
    cta_sum<1, NW>(cv, red, par);
    if (!isfinite(cv[0]) || cv[0] <= 0.0) {
      err = 1;
      curv = cv[0];
      done = 1;
      break;
    }
    const double alpha = rho / cv[0];
    double s2[2] = {0.0, 0.0};
#pragma unroll
    for (int r = 0; r < RPT; ++r) {
      const int i = t + r * NT;
      if (i >= alo && i < ahi) {
        Xs[i] = __dadd_rn(Xs[i], __dmul_rn(alpha, Ps[i]));
        const double rr = __dsub_rn(R[r], __dmul_rn(alpha, AP[r]));
        R[r] = rr;
        const double z = __dmul_rn(Is[i], rr);
        s2[0] += rr * z;
        s2[1] += rr * rr;
      }
    }
    cta_sum<2, NW>(s2, red, par);
    const double beta = s2[0] / rho;
#pragma unroll
    for (int r = 0; r < RPT; ++r) {
      const int i = t + r * NT;
      if (i >= alo && i < ahi) Ps[i] = __dadd_rn(__dmul_rn(Is[i], R[r]), __dmul_rn(beta, Ps[i]));
    }
    lo = alo;
    hi = ahi;
    rho = s2[0];
    it += 1;
    if (sqrt(s2[1]) <= target || it >= max_iter) done = 1;
    __syncthreads();  // p and x complete
  }
  __syncthreads();
  // true residual; x back to the slab layout
  double sr[1] = {0.0};
#pragma unroll
  for (int r = 0; r < RPT; ++r) {
    const int i = t + r * NT;
    if (i < n) {
      const double e = __dsub_rn(B[slab_at(n, i, col)], spmv(Xs, i));
      sr[0] += e * e;
      X[slab_at(n, i, col)] = Xs[i];
    }
  }
  cta_sum<1, NW>(sr, red, par);
  if (t == 0 && col < nb) {
    ColState& S = st[col];
    S.norm_b = norm_b;
    S.target = target;
    S.it = it;
    S.err = err;
    S.curv = curv;
    S.done = done == 2 ? 2 : 1;
    S.rel_res = sqrt(sr[0]) / norm_b;
  }
}

// Runs pcg_smem_k when it applies: 3 n fp64 within a CTA's shared memory,
// n <= 20 x 512, and the matrix either staged in shared memory too (CSR) or
// read as ELL (rows of <= 16 entries).  Returns false otherwise.
template <int RPT>
void pcg_smem_rpt(Ctx* c, int E, int packed, size_t smem, const double* ev, const int* ec, const i64* crp,
                  const double* inv, const double* B, double* X, i64 n, i64 nb, double tol, i64 max_iter,
                  ColState* st, const int* bwp) {
  auto launch = [&](auto k) {
    ensure_smem(k, smem);
    KScope ks_(c, "pcg_persistent");
    k<<<static_cast<unsigned>(nb), kPcgSmemThreads, smem, c->stream>>>(static_cast<int>(n), nb, ev, ec, crp, inv, B, X,
                                                                      tol, max_iter, st, bwp);
    launched(c);
  };
  if (E == 0)
    launch(pcg_smem_k<RPT, 0>);
  else if (E <= 9)
    packed == 2 ? launch(pcg_smem_k<RPT, 9, 2>) : packed == 1 ? launch(pcg_smem_k<RPT, 9, 1>) : launch(pcg_smem_k<RPT, 9>);
  else
    packed == 2 ? launch(pcg_smem_k<RPT, 16, 2>)
                : packed == 1 ? launch(pcg_smem_k<RPT, 16, 1>) : launch(pcg_smem_k<RPT, 16>);
}

bool pcg_smem(Ctx* c, Csr* A, const double* inv, const double* B, double* X, i64 n, i64 nb, double tol,
              i64 max_iter, ColState* st) {
  constexpr size_t kMax = 227 * 1024 - 2 * 3 * 16 * sizeof(double);
  const size_t vec = static_cast<size_t>(3 * n) * sizeof(double);
  if (n <= 0 || n > 20 * kPcgSmemThreads || vec > kMax || A->nnz == 0) return false;
  const size_t csr = static_cast<size_t>(A->nnz) * 12 + static_cast<size_t>(n + 1) * 4 + 16;
  const i64 rpt = (n + kPcgSmemThreads - 1) / kPcgSmemThreads;
  const int* bwp = nullptr;  // device half bandwidth (ELL paths); null: no window
  auto run = [&](int E, int pk, size_t smem, const double* ev, const int* ec, const i64* crp) {
    if (rpt <= 4) return pcg_smem_rpt<4>(c, E, pk, smem, ev, ec, crp, inv, B, X, n, nb, tol, max_iter, st, bwp);
    if (rpt <= 8) return pcg_smem_rpt<8>(c, E, pk, smem, ev, ec, crp, inv, B, X, n, nb, tol, max_iter, st, bwp);
    if (rpt <= 12) return pcg_smem_rpt<12>(c, E, pk, smem, ev, ec, crp, inv, B, X, n, nb, tol, max_iter, st, bwp);
    if (rpt <= 16) return pcg_smem_rpt<16>(c, E, pk, smem, ev, ec, crp, inv, B, X, n, nb, tol, max_iter, st, bwp);
    return pcg_smem_rpt<20>(c, E, pk, smem, ev, ec, crp, inv, B, X, n, nb, tol, max_iter, st, bwp);
  };
  if (vec + csr <= kMax && A->nnz < (i64{1} << 30)) {  // the whole operator in shared memory
    run(0, 0, vec + csr, A->v, A->ci, A->rp);
    return true;
  }
  // longest row (E): one small reduction on the host copy of the row pointers
  std::vector<i64> rp(static_cast<size_t>(n) + 1);
  CUDA_OK(cudaMemcpyAsync(rp.data(), A->rp, sizeof(i64) * (n + 1), cudaMemcpyDeviceToHost, c->stream));
  sync(c);
  i64 E = 0;
  for (i64 i = 0; i < n; ++i) E = std::max(E, rp[i + 1] - rp[i]);
  if (E > 16) return false;
  const int Ep = E <= 9 ? 9 : 16;
  // packed (fp32 value, column) words when every value is exact in fp32
  // (unit-weight grids: the interior's values are small integers)
  DevBuf<uint2> ep(c, static_cast<size_t>(Ep) * n);
  DevBuf<int> flag(c, 2);  // [0] packing flags, [1] half bandwidth
  flag.zero(c);
  csr_to_ell_packed_k<<<blocks_for(n), kBlock, 0, c->stream>>>(n, Ep, A->rp, A->ci, A->v, ep.p, flag.p);
  launched(c);
  const int fl = read_back(c, flag.p);
  bwp = flag.p + 1;
  if (!(fl & 2) && n < 65536) {
    DevBuf<unsigned> eh(c, static_cast<size_t>(Ep) * n);
    ell_pack16_k<<<blocks_for(n), kBlock, 0, c->stream>>>(n, Ep, ep.p, eh.p);
    launched(c);
    run(Ep, 2, vec, reinterpret_cast<const double*>(eh.p), nullptr, nullptr);
    return true;
  }
  if (!(fl & 1)) {
    run(Ep, 1, vec, reinterpret_cast<const double*>(ep.p), nullptr, nullptr);
    return true;
  }
  DevBuf<double> ev(c, static_cast<size_t>(Ep) * n);
  DevBuf<int> ec(c, static_cast<size_t>(Ep) * n);
  csr_to_ell_k<<<blocks_for(n), kBlock, 0, c->stream>>>(n, Ep, A->rp, A->ci, A->v, ev.p, ec.p);
  launched(c);
  run(Ep, 0, vec, ev.p, ec.p, nullptr);
  return true;
}

struct PcgBatchOut {
  std::vector<ColState> cols;
};

// Solves A X(:,c) = B(:,c) for every column c (A square device CSR, inv the
// Jacobi inverse or all ones).  X holds the start iterates and receives the
// solutions.
void pcg_batched(Ctx* c, Csr* A, const double* inv, const double* B, double* X, i64 n, i64 nb,
                 double tol, i64 max_iter, PcgBatchOut* out) {
  out->cols.assign(static_cast<size_t>(nb), ColState{});
  if (nb == 0) return;
  DevBuf<double> R(c, n * nb), Z(c, n * nb), P(c, n * nb), AP(c, n * nb);
  const unsigned nrb = blocks_for(std::max<i64>(n, 1), kPcgBlock);
  const i64 ycap = std::max<i64>(1, (static_cast<i64>(c->num_sms) * 32) / nrb);
  dim3 g(nrb, static_cast<unsigned>(std::max<i64>(1, std::min<i64>({nb, ycap, 65535}))));
  DevBuf<double> part(c, 3 * nb * nrb), part2(c, 2 * nb * nrb);
  DevBuf<ColState> st(c, nb);
  st.zero(c);
  DevBuf<unsigned> ndone(c, 1);
  ndone.zero(c);
  pcg_init_k<<<g, kPcgBlock, 0, c->stream>>>(n, nb, A->rp, A->ci, A->v, inv, B, X, R.p, Z.p, P.p, tol, max_iter,
                                             part.p, st.p, ndone.p);
  launched(c);
  unsigned done = read_back(c, ndone.p);
  const i64 chunk = 16;
  while (done < nb) {
    for (i64 k = 0; k < chunk; ++k) {
      {
        KScope ks_(c, "pcg_apply");
        pcg_apply_k<<<g, kPcgBlock, 0, c->stream>>>(n, nb, A->rp, A->ci, A->v, P.p, AP.p, part.p, st.p);
        launched(c);
      }
      {
        KScope ks_(c, "pcg_update");
        pcg_update_k<<<g, kPcgBlock, 0, c->stream>>>(n, nb, inv, X, R.p, Z.p, P.p, AP.p, part.p, part2.p, st.p,
                                                     ndone.p);
        launched(c);
      }
      {
        KScope ks_(c, "pcg_direction");
        pcg_direction_k<<<g, kPcgBlock, 0, c->stream>>>(n, nb, max_iter, Z.p, P.p, part2.p, st.p, ndone.p);
        launched(c);
      }
    }
    done = read_back(c, ndone.p);
  }
  pcg_true_k<<<g, kPcgBlock, 0, c->stream>>>(n, nb, A->rp, A->ci, A->v, B, X, part.p, st.p);
  launched(c);
  CUDA_OK(cudaMemcpyAsync(out->cols.data(), st.p, sizeof(ColState) * nb, cudaMemcpyDeviceToHost, c->stream));
  sync(c);
}

// Slab-layout batched PCG (B, X in slab layout with nb padded to kCpb).
void pcg_slab(Ctx* c, Csr* A, const double* inv, const double* B, double* X, i64 n, i64 nb, double tol,
              i64 max_iter, PcgBatchOut* out) {
  out->cols.assign(static_cast<size_t>(nb), ColState{});
  if (nb == 0) return;
  const i64 nbp = (nb + kCpb - 1) / kCpb * kCpb;
  DevBuf<ColState> st(c, nb);
  st.zero(c);
  if (pcg_smem(c, A, inv, B, X, n, nb, tol, max_iter, st.p)) {
    CUDA_OK(cudaMemcpyAsync(out->cols.data(), st.p, sizeof(ColState) * nb, cudaMemcpyDeviceToHost, c->stream));
    sync(c);
    return;
  }
  DevBuf<double> R(c, n * nbp), P(c, n * nbp), AP(c, n * nbp);
  {
    // One CTA per kCpb columns: 1024 threads while the CTAs fit in one wave,
    // else 512 threads at 2 CTAs per SM (cfg1 rows: 258 CTAs, one wave).
    const i64 ctas = nbp / kCpb;
    const std::string cfg = ctas > c->num_sms ? "512x2" : "1024x1";
    KScope ks_(c, "pcg_persistent");
    const i64 batches = 1;  // one launch for all column groups (sequential batches measured slower)
    const i64 per = (ctas + batches - 1) / batches;
    for (i64 g0 = 0; g0 < ctas; g0 += per) {
      const unsigned g = static_cast<unsigned>(std::min(per, ctas - g0));
      if (cfg == "512x2")
        pcg_persistent_k<512, 2><<<g, 512, 0, c->stream>>>(n, nb, A->rp, A->ci, A->v, inv, B, X, R.p, P.p, AP.p, tol,
                                                          max_iter, st.p, g0);
      else if (cfg == "512x1")
        pcg_persistent_k<512, 1><<<g, 512, 0, c->stream>>>(n, nb, A->rp, A->ci, A->v, inv, B, X, R.p, P.p, AP.p, tol,
                                                          max_iter, st.p, g0);
      else
        pcg_persistent_k<1024, 1><<<g, 1024, 0, c->stream>>>(n, nb, A->rp, A->ci, A->v, inv, B, X, R.p, P.p, AP.p, tol,
                                                            max_iter, st.p, g0);
      launched(c);
    }
  }
  CUDA_OK(cudaMemcpyAsync(out->cols.data(), st.p, sizeof(ColState) * nb, cudaMemcpyDeviceToHost, c->stream));
  sync(c);
}

// ------------------------------------------------------------------ Schur assembly
__global__ void rhs_fill_slab_k(i64 ni, i64 nb, const i64* __restrict__ rows, const i64* __restrict__ rp,
                                const int* __restrict__ ci, const double* __restrict__ v, double* __restrict__ B) {
  const i64 c = blockIdx.x * (i64)blockDim.x + threadIdx.x;
  if (c >= nb) return;
  const i64 j = rows[c];
  for (i64 k = rp[j]; k < rp[j + 1]; ++k) B[slab_at(ni, ci[k], c)] = v[k];
}

__global__ void schur_update_slab_k(i64 m, i64 ni, i64 nb, const i64* __restrict__ cols, const i64* __restrict__ rp,
                                    const int* __restrict__ ci, const double* __restrict__ v,
                                    const double* __restrict__ Zs, double* __restrict__ S) {
  const i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x;
  if (i >= m) return;
  for (i64 c = blockIdx.y; c < nb; c += gridDim.y) {
    double y = 0.0;
    for (i64 k = rp[i]; k < rp[i + 1]; ++k) y = __dadd_rn(y, __dmul_rn(v[k], Zs[slab_at(ni, ci[k], c)]));
    const i64 at = i + cols[c] * m;
    S[at] = __dsub_rn(S[at], y);
  }
}

__global__ void rhs_fill_k(i64 ni, i64 nb, const i64* __restrict__ rows, const i64* __restrict__ rp,
                           const int* __restrict__ ci, const double* __restrict__ v, double* __restrict__ B) {
  const i64 c = blockIdx.x * (i64)blockDim.x + threadIdx.x;
  if (c >= nb) return;
  const i64 j = rows[c];
  for (i64 k = rp[j]; k < rp[j + 1]; ++k) B[ci[k] + c * ni] = v[k];
}

// S(i, j_c) -= (L_ba z_c)(i), CSR order per row (graph.cpp:230).
__global__ void schur_update_k(i64 m, i64 ni, i64 nb, const i64* __restrict__ cols, const i64* __restrict__ rp,
                               const int* __restrict__ ci, const double* __restrict__ v,
                               const double* __restrict__ Zs, double* __restrict__ S) {
  const i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x;
  if (i >= m) return;
  for (i64 c = blockIdx.y; c < nb; c += gridDim.y) {
    const double y = pull_left(rp[i], rp[i + 1], ci, v, Zs + c * ni);
    const i64 at = i + cols[c] * m;
    S[at] = __dsub_rn(S[at], y);
  }
}

// Symmetrise (0.5 (S + S^T)) and prune (v != 0 and |v| > tol) row by row.
// Row-contiguous copy of the dense result: T[j + i m] = x(i, j), x = 0.5 (S(i, j) +
// S(j, i)) (symmetrize; commutative, so T is exactly symmetric) or S(i, j),
// through 32 x 32 shared-memory tiles so both reads and the write coalesce.
// Rows [r0, r1) only (T row-local), so large m works in blocks.
__global__ void row_major_k(i64 m, i64 r0, i64 r1, const double* __restrict__ S, bool symmetrize,
                            double* __restrict__ T) {
  __shared__ double a[32][33], b[32][33];
  const i64 bi = r0 + static_cast<i64>(blockIdx.x) * 32, bj = static_cast<i64>(blockIdx.y) * 32;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 32 x 8 threads
  for (int r = ty; r < 32; r += 8) {
    const i64 i = bi + tx, j = bj + r;  // S(i, j), i contiguous
    a[r][tx] = (i < r1 && j < m) ? S[i + j * m] : 0.0;
    const i64 i2 = bj + tx, j2 = bi + r;  // S(j, i) as (row bj + tx, column bi + r)
    b[r][tx] = (i2 < m && j2 < r1) ? S[i2 + j2 * m] : 0.0;
  }
  __syncthreads();
  // write T[j + i m] for i = bi + r, j = bj + tx: x(i, j) = S(i, j) [= a[tx][r]] (+ S(j, i) [= b[r][tx]])
  for (int r = ty; r < 32; r += 8) {
    const i64 i = bi + r, j = bj + tx;
    if (i < r1 && j < m) T[j + (i - r0) * m] = symmetrize ? __dmul_rn(0.5, __dadd_rn(a[tx][r], b[r][tx])) : a[tx][r];
  }
}

// Warp per row over the row-contiguous copy: counts, then compacted (column,
// value) pairs in increasing column order (ballot prefix).
__global__ void row_count_k(i64 m, i64 r0, i64 r1, const double* __restrict__ T, double prune, i64* cnt) {
  const i64 il = (blockIdx.x * (i64)blockDim.x + threadIdx.x) >> 5, i = r0 + il;
  const int lane = threadIdx.x & 31;
  if (i >= r1) return;
  i64 k = 0;
  for (i64 j0 = 0; j0 < m; j0 += 32) {
    const i64 j = j0 + lane;
    const double x = j < m ? T[j + il * m] : 0.0;
    k += __popc(__ballot_sync(0xffffffffu, x != 0.0 && fabs(x) > prune));
  }
  if (lane == 0) cnt[i] = k;
}

__global__ void row_fill_k(i64 m, i64 r0, i64 r1, const double* __restrict__ T, double prune,
                           const i64* __restrict__ rp, int* __restrict__ ci, double* __restrict__ v) {
  const i64 il = (blockIdx.x * (i64)blockDim.x + threadIdx.x) >> 5, i = r0 + il;
  const int lane = threadIdx.x & 31;
  if (i >= r1) return;
  i64 o = rp[i];
  for (i64 j0 = 0; j0 < m; j0 += 32) {
    const i64 j = j0 + lane;
    const double x = j < m ? T[j + il * m] : 0.0;
    const bool keep = x != 0.0 && fabs(x) > prune;
    const unsigned bal = __ballot_sync(0xffffffffu, keep);
    if (keep) {
      const i64 at = o + __popc(bal & ((1u << lane) - 1u));
      ci[at] = static_cast<int>(j);
      v[at] = x;
    }
    o += __popc(bal);
  }
}

// Exclusive scan of per-row counts into row pointers (rp[0] = 0); returns nnz.
i64 scan_counts(Ctx* c, const i64* cnt, i64 rows, i64* rp) {
  CUDA_OK(cudaMemsetAsync(rp, 0, sizeof(i64), c->stream));
  if (rows == 0) return 0;
  size_t tmp = 0;
  CUDA_OK(cub::DeviceScan::InclusiveSum(nullptr, tmp, cnt, rp + 1, static_cast<int>(rows), c->stream));
  DevBuf<char> ws(c, tmp);
  CUDA_OK(cub::DeviceScan::InclusiveSum(ws.p, tmp, cnt, rp + 1, static_cast<int>(rows), c->stream));
  launched(c);
  i64 nnz = 0;
  CUDA_OK(cudaMemcpyAsync(&nnz, rp + rows, sizeof(i64), cudaMemcpyDeviceToHost, c->stream));
  sync(c);
  return nnz;
}

// Dense (m x m, col-major) to CSR with the from_dense / prune rules.
Csr* dense_to_csr(Ctx* c, const double* S, i64 m, double prune, bool symmetrize) {
  DevBuf<i64> cnt(c, std::max<i64>(m, 1));
  Csr* out = csr_alloc(c, m, m, 0);
  // row blocks of the row-contiguous copy, <= 256 MB each
  const i64 rb = std::max<i64>(32, std::min<i64>(m, ((i64{32} << 20) / std::max<i64>(m, 1)) / 32 * 32));
  DevBuf<double> T(c, std::max<i64>(std::min(rb, m) * m, 1));
  auto to_rows = [&](i64 r0, i64 r1) {
    row_major_k<<<dim3(static_cast<unsigned>((r1 - r0 + 31) / 32), static_cast<unsigned>((m + 31) / 32)), 256, 0,
                  c->stream>>>(m, r0, r1, S, symmetrize, T.p);
    launched(c);
  };
  for (i64 r0 = 0; r0 < m; r0 += rb) {
    const i64 r1 = std::min(m, r0 + rb);
    to_rows(r0, r1);
    row_count_k<<<static_cast<unsigned>(((r1 - r0) * 32 + 255) / 256), 256, 0, c->stream>>>(m, r0, r1, T.p, prune,
                                                                                           cnt.p);
    launched(c);
  }
  const i64 nnz = scan_counts(c, cnt.p, m, out->rp);
  out->nnz = nnz;
  if (nnz) {
    out->ci = static_cast<int*>(csr_malloc(c, sizeof(int) * nnz));
    out->v = static_cast<double*>(csr_malloc(c, sizeof(double) * nnz));
    for (i64 r0 = 0; r0 < m; r0 += rb) {
      const i64 r1 = std::min(m, r0 + rb);
      if (rb < m) to_rows(r0, r1);  // one block: the copy from the counting pass is still there
      row_fill_k<<<static_cast<unsigned>(((r1 - r0) * 32 + 255) / 256), 256, 0, c->stream>>>(m, r0, r1, T.p, prune,
                                                                                            out->rp, out->ci, out->v);
      launched(c);
    }
  }
  return out;
}

// Row-gathered, column-filtered submatrix as a new device CSR.
Csr* gather_sub(Ctx* c, Csr* L, const i64* rsrc_dev, i64 nr, const int* cmap_dev, i64 ncols) {
  Csr* out = csr_alloc(c, nr, ncols, 0);
  DevBuf<i64> cnt(c, std::max<i64>(nr, 1));
  if (nr) {
    sub_count_k<<<blocks_for(nr), kBlock, 0, c->stream>>>(nr, rsrc_dev, L->rp, L->ci, cmap_dev, cnt.p);
    launched(c);
  }
  const i64 nnz = scan_counts(c, cnt.p, nr, out->rp);
  out->nnz = nnz;
  if (nnz) {
    out->ci = static_cast<int*>(csr_malloc(c, sizeof(int) * nnz));
    out->v = static_cast<double*>(csr_malloc(c, sizeof(double) * nnz));
    sub_fill_k<<<blocks_for(nr), kBlock, 0, c->stream>>>(nr, rsrc_dev, L->rp, L->ci, L->v, cmap_dev, out->rp,
                                                         out->ci, out->v);
    launched(c);
  }
  return out;
}

// Every connected component of L must hold a node of keep (graph.cpp:183-193,
// decoders.cpp:84-94); throws "<what>: connected component containing node X
// has no <noun> node" naming the smallest node of the first such component.
void check_components(Ctx* c, Csr* L, const i64* keep_d, i64 m, const char* what, const char* noun) {
  const i64 n = L->rows;
  if (!n) return;
  DevBuf<int> parent(c, n), grounded(c, n), first(c, 1);
  grounded.zero(c);
  const int big = INT32_MAX;
  CUDA_OK(cudaMemcpyAsync(first.p, &big, sizeof(int), cudaMemcpyHostToDevice, c->stream));
  uf_init_k<<<blocks_for(n), kBlock, 0, c->stream>>>(n, parent.p);
  launched(c);
  uf_hook_k<<<blocks_for(n), kBlock, 0, c->stream>>>(n, L->rp, L->ci, parent.p);
  launched(c);
  uf_flatten_k<<<blocks_for(n), kBlock, 0, c->stream>>>(n, parent.p);
  launched(c);
  if (m) {
    ground_k<<<blocks_for(m), kBlock, 0, c->stream>>>(m, keep_d, parent.p, grounded.p);
    launched(c);
  }
  ungrounded_k<<<blocks_for(n), kBlock, 0, c->stream>>>(n, parent.p, grounded.p, first.p);
  launched(c);
  const int bad = read_back(c, first.p);
  if (bad != INT32_MAX)
    runtime(std::string(what) + ": connected component containing node " + std::to_string(bad) + " has no " + noun +
            " node");
}

Csr* kron_reduce_device(Ctx* c, Csr* L, const std::vector<i64>& keep, double pcg_tol, double prune_tol) {
  const i64 n = L->rows;
  if (L->cols != n) invalid("kron reduction: square Laplacian required");
  if (n > INT32_MAX) invalid("kron reduction: graphs above 2^31 nodes are not supported");
  std::vector<int> kpos(static_cast<size_t>(n), -1);
  for (size_t j = 0; j < keep.size(); ++j) {
    const i64 u = keep[j];
    if (u < 0 || u >= n) invalid("kron reduction: index out of range");
    if (kpos[u] != -1) invalid("kron reduction: duplicate index");
    kpos[u] = static_cast<int>(j);
  }
  const i64 m = static_cast<i64>(keep.size());
  trace_mark(c, "kron: enter");

  // graph.cpp:183-193: every component must hold a kept node.
  DevBuf<i64> keep_d(c, std::max<i64>(m, 1));
  if (m) CUDA_OK(cudaMemcpyAsync(keep_d.p, keep.data(), sizeof(i64) * m, cudaMemcpyHostToDevice, c->stream));
  check_components(c, L, keep_d.p, m, "kron reduction", "kept");

  trace_mark(c, "kron: components");
  std::vector<i64> interior;
  interior.reserve(static_cast<size_t>(n - m));
  std::vector<int> ipos(static_cast<size_t>(n), -1);
  for (i64 u = 0; u < n; ++u)
    if (kpos[u] < 0) {
      ipos[u] = static_cast<int>(interior.size());
      interior.push_back(u);
    }
  const i64 ni = static_cast<i64>(interior.size());

  DevBuf<int> kpos_d(c, std::max<i64>(n, 1)), ipos_d(c, std::max<i64>(n, 1));
  if (n) {
    CUDA_OK(cudaMemcpyAsync(kpos_d.p, kpos.data(), sizeof(int) * n, cudaMemcpyHostToDevice, c->stream));
    CUDA_OK(cudaMemcpyAsync(ipos_d.p, ipos.data(), sizeof(int) * n, cudaMemcpyHostToDevice, c->stream));
  }
  // Dense Schur matrix initialised with L_bb (graph.cpp:208).
  DevBuf<double> S(c, std::max<i64>(m * m, 1));
  S.zero(c);
  if (m) {
    scatter_bb_k<<<blocks_for(m), kBlock, 0, c->stream>>>(m, keep_d.p, L->rp, L->ci, L->v, kpos_d.p, S.p);
    launched(c);
  }
  if (ni == 0) return dense_to_csr(c, S.p, m, 0.0, false);  // graph.cpp:201: L_bb as is

  DevBuf<i64> int_d(c, ni);
  CUDA_OK(cudaMemcpyAsync(int_d.p, interior.data(), sizeof(i64) * ni, cudaMemcpyHostToDevice, c->stream));
  trace_mark(c, "kron: maps+Lbb");
  Csr* Laa = gather_sub(c, L, int_d.p, ni, ipos_d.p, ni);
  Csr* Lba = gather_sub(c, L, keep_d.p, m, ipos_d.p, ni);
  std::unique_ptr<Csr> own_aa(Laa), own_ba(Lba);
  DevBuf<double> inv(c, ni);
  jacobi_inv_k<<<blocks_for(ni), kBlock, 0, c->stream>>>(ni, Laa->rp, Laa->ci, Laa->v, inv.p);
  launched(c);

  trace_mark(c, "kron: gathers");
  // Kept nodes with a nonempty row of L_ba get a solve (graph.cpp:213-220).
  std::vector<i64> rp_ba(static_cast<size_t>(m) + 1);
  CUDA_OK(cudaMemcpyAsync(rp_ba.data(), Lba->rp, sizeof(i64) * (m + 1), cudaMemcpyDeviceToHost, c->stream));
  sync(c);
  std::vector<i64> active;
  for (i64 j = 0; j < m; ++j)
    if (rp_ba[j + 1] > rp_ba[j]) active.push_back(j);

  // Columns per slice: 6 dense |int| x b fp64 vectors within ~40% of free HBM
  // (cudaMemGetInfo only for reductions above 1 GB: the query itself was
  // measured stalling the stream by up to tens of ms).
  const double per_col = 6.0 * 8.0 * static_cast<double>(ni) + 64.0;
  i64 slice = static_cast<i64>(active.size());
  if (per_col * static_cast<double>(active.size()) > 1e9) {
    size_t free_b = 0, total_b = 0;
    CUDA_OK(cudaMemGetInfo(&free_b, &total_b));
    slice = static_cast<i64>(0.4 * static_cast<double>(free_b) / per_col);
  }
  slice = std::max<i64>(1, std::min<i64>(slice, static_cast<i64>(active.size())));
  const i64 max_iter = 20 * ni + 100;

  i64 fail_j = -1;
  std::string fail_msg;
  for (size_t s0 = 0; s0 < active.size(); s0 += static_cast<size_t>(slice)) {
    const i64 nb = std::min<i64>(slice, static_cast<i64>(active.size() - s0));
    std::vector<i64> cols(active.begin() + s0, active.begin() + s0 + nb);
    DevBuf<i64> cols_d(c, nb);
    CUDA_OK(cudaMemcpyAsync(cols_d.p, cols.data(), sizeof(i64) * nb, cudaMemcpyHostToDevice, c->stream));
    const i64 nbp = (nb + kCpb - 1) / kCpb * kCpb;
    DevBuf<double> B(c, ni * nbp), X(c, ni * nbp);
    B.zero(c);
    X.zero(c);
    rhs_fill_slab_k<<<blocks_for(nb), kBlock, 0, c->stream>>>(ni, nb, cols_d.p, Lba->rp, Lba->ci, Lba->v, B.p);
    launched(c);
    trace_mark(c, "kron: slice setup");
    PcgBatchOut res;
    pcg_slab(c, Laa, inv.p, B.p, X.p, ni, nb, pcg_tol, max_iter, &res);
    if (std::getenv("CPCAG_TRACE")) {
      i64 mx = 0, sum = 0;
      for (const ColState& cs : res.cols) {
        mx = std::max<i64>(mx, cs.it);
        sum += cs.it;
      }
      std::fprintf(stderr, "[kron] interior %lld, %lld solves, PCG iterations mean %.1f max %lld\n",
                   static_cast<long long>(ni), static_cast<long long>(nb),
                   nb ? static_cast<double>(sum) / nb : 0.0, static_cast<long long>(mx));
    }
    for (i64 q = 0; q < nb; ++q) {
      const ColState& cs = res.cols[q];
      const i64 j = cols[q];
      std::string msg;
      if (cs.err)
        msg = "pcg: breakdown (nonpositive curvature) at iteration " + std::to_string(cs.it);
      else if (cs.done != 2 && !(cs.rel_res <= pcg_tol))
        msg = "kron reduction: interior solve failed to converge for kept node " + std::to_string(keep[j]);
      if (!msg.empty() && (fail_j < 0 || j < fail_j)) {
        fail_j = j;
        fail_msg = msg;
      }
    }
    if (fail_j >= 0) break;
    dim3 g(blocks_for(m), static_cast<unsigned>(std::min<i64>(nb, 65535)));
    schur_update_slab_k<<<g, kBlock, 0, c->stream>>>(m, ni, nb, cols_d.p, Lba->rp, Lba->ci, Lba->v, X.p, S.p);
    launched(c);
  }
  if (fail_j >= 0) runtime(fail_msg);
  trace_mark(c, "kron: solves+schur");
  Csr* out = dense_to_csr(c, S.p, m, prune_tol, true);
  trace_mark(c, "kron: to csr");
  return out;
}

// ------------------------------------------------------------------ graph upsampling
// Rows of a gathered submatrix re-sorted by (new) column: submatrix() goes
// through from_triplets (sparse.cpp:122-141), so when the column map is not
// monotone (known = Omega in draw order) the entries come out in map order.
__global__ void sort_rows_k(i64 nr, const i64* __restrict__ rp, int* __restrict__ ci, double* __restrict__ v) {
  const i64 r = blockIdx.x * (i64)blockDim.x + threadIdx.x;
  if (r >= nr) return;
  for (i64 a = rp[r] + 1; a < rp[r + 1]; ++a) {
    const int kc = ci[a];
    const double kv = v[a];
    i64 b = a - 1;
    while (b >= rp[r] && ci[b] > kc) {
      ci[b + 1] = ci[b];
      v[b + 1] = v[b];
      --b;
    }
    ci[b + 1] = kc;
    v[b + 1] = kv;
  }
}

// B(:, j) = -(L_ab R)(:, j) in slab layout (decoders.cpp:107, CSR order).
__global__ void upsample_rhs_slab_k(i64 ni, i64 r, const i64* __restrict__ rp, const int* __restrict__ ci,
                                    const double* __restrict__ v, const double* __restrict__ R, i64 ldr,
                                    double* __restrict__ B) {
  const i64 a = blockIdx.x * (i64)blockDim.x + threadIdx.x;
  if (a >= ni) return;
  for (i64 j = blockIdx.y; j < r; j += gridDim.y) {
    const double y = pull_left(rp[a], rp[a + 1], ci, v, R + j * ldr);
    B[slab_at(ni, a, j)] = -y;
  }
}

// S(i, :) = R(kpos[i], :) on known rows, the interior solution elsewhere.
__global__ void upsample_scatter_k(i64 n, i64 r, const int* __restrict__ kpos, const int* __restrict__ ipos,
                                   const double* __restrict__ R, i64 ldr, const double* __restrict__ Xs, i64 ni,
                                   double* __restrict__ S) {
  const i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x;
  if (i >= n) return;
  for (i64 j = blockIdx.y; j < r; j += gridDim.y)
    S[i + j * n] = kpos[i] >= 0 ? R[kpos[i] + j * ldr] : Xs[slab_at(ni, ipos[i], j)];
}

void graph_upsample_device(Ctx* c, Csr* L, const std::vector<i64>& known, const double* R, i64 r, double pcg_tol,
                           i64 pcg_max_iter, double* S) {
  const i64 n = L->rows;
  if (L->cols != n) invalid("graph upsample: square Laplacian required");
  if (n > INT32_MAX) invalid("graph upsample: graphs above 2^31 nodes are not supported");
  const i64 m = static_cast<i64>(known.size());
  std::vector<int> kpos(static_cast<size_t>(n), -1);
  for (i64 j = 0; j < m; ++j) {  // decoders.cpp:17-25
    const i64 u = known[j];
    if (u < 0 || u >= n) invalid("graph upsample: index out of range");
    if (kpos[u] != -1) invalid("graph upsample: duplicate index");
    kpos[u] = static_cast<int>(j);
  }
  DevBuf<i64> known_d(c, std::max<i64>(m, 1));
  if (m) CUDA_OK(cudaMemcpyAsync(known_d.p, known.data(), sizeof(i64) * m, cudaMemcpyHostToDevice, c->stream));
  check_components(c, L, known_d.p, m, "graph upsample", "sampled");

  std::vector<i64> interior;
  std::vector<int> ipos(static_cast<size_t>(n), -1);
  for (i64 u = 0; u < n; ++u)
    if (kpos[u] < 0) {
      ipos[u] = static_cast<int>(interior.size());
      interior.push_back(u);
    }
  const i64 ni = static_cast<i64>(interior.size());
  DevBuf<int> kpos_d(c, std::max<i64>(n, 1)), ipos_d(c, std::max<i64>(n, 1));
  if (n) {
    CUDA_OK(cudaMemcpyAsync(kpos_d.p, kpos.data(), sizeof(int) * n, cudaMemcpyHostToDevice, c->stream));
    CUDA_OK(cudaMemcpyAsync(ipos_d.p, ipos.data(), sizeof(int) * n, cudaMemcpyHostToDevice, c->stream));
  }
  const i64 nbp = std::max<i64>((r + kCpb - 1) / kCpb * kCpb, kCpb);
  DevBuf<double> X(c, std::max<i64>(ni, 1) * nbp);
  if (ni > 0 && r > 0) {
    DevBuf<i64> int_d(c, ni);
    CUDA_OK(cudaMemcpyAsync(int_d.p, interior.data(), sizeof(i64) * ni, cudaMemcpyHostToDevice, c->stream));
    Csr* Laa = gather_sub(c, L, int_d.p, ni, ipos_d.p, ni);
    Csr* Lab = gather_sub(c, L, int_d.p, ni, kpos_d.p, m);
    std::unique_ptr<Csr> own_aa(Laa), own_ab(Lab);
    if (Lab->nnz) {
      sort_rows_k<<<blocks_for(ni), kBlock, 0, c->stream>>>(ni, Lab->rp, Lab->ci, Lab->v);
      launched(c);
    }
    DevBuf<double> inv(c, ni), B(c, ni * nbp);
    jacobi_inv_k<<<blocks_for(ni), kBlock, 0, c->stream>>>(ni, Laa->rp, Laa->ci, Laa->v, inv.p);
    launched(c);
    B.zero(c);
    X.zero(c);
    dim3 g(blocks_for(ni), static_cast<unsigned>(std::min<i64>(r, 65535)));
    upsample_rhs_slab_k<<<g, kBlock, 0, c->stream>>>(ni, r, Lab->rp, Lab->ci, Lab->v, R, m, B.p);
    launched(c);
    PcgBatchOut res;
    pcg_slab(c, Laa, inv.p, B.p, X.p, ni, r, pcg_tol, pcg_max_iter, &res);
    for (i64 j = 0; j < r; ++j) {  // first failing column, as the reference's column loop
      const ColState& cs = res.cols[j];
      if (cs.err) runtime("pcg: breakdown (nonpositive curvature) at iteration " + std::to_string(cs.it));
      if (cs.done != 2 && !(cs.rel_res <= pcg_tol))
        runtime("graph upsample: interior solve did not converge (column " + std::to_string(j) + ")");
    }
  }
  if (n && r) {
    dim3 g(blocks_for(n), static_cast<unsigned>(std::min<i64>(r, 65535)));
    upsample_scatter_k<<<g, kBlock, 0, c->stream>>>(n, r, kpos_d.p, ipos_d.p, R, m, X.p, std::max<i64>(ni, 1), S);
    launched(c);
  }
}

}  // namespace cpcag_cuda

using namespace cpcag_cuda;

extern "C" int cpcag_cuda_graph_upsample(cpcag_ctx ctx, cpcag_csr Lh, const int64_t* known, int64_t n_known,
                                         const double* R, int64_t r, double pcg_tol, int64_t pcg_max_iter,
                                         double* S) {
  return guard([&] {
    Ctx* c = as_ctx(ctx);
    Csr* L = as_csr(Lh);
    if (r < 0 || n_known < 0) invalid("graph upsample: negative size");
    if ((n_known * r && !R) || (L->rows * r && !S)) invalid("null argument");
    std::vector<i64> k(static_cast<size_t>(n_known));
    if (!k.empty()) {
      if (!known) invalid("null argument");
      if (is_device_ptr(known))
        CUDA_OK(cudaMemcpy(k.data(), known, sizeof(i64) * k.size(), cudaMemcpyDeviceToHost));
      else
        std::copy(known, known + k.size(), k.begin());
    }
    InView<double> rv(c, R, static_cast<size_t>(n_known * r));
    OutView<double> sv(c, S, static_cast<size_t>(L->rows * r));
    graph_upsample_device(c, L, k, rv.d, r, pcg_tol, pcg_max_iter, sv.d);
    sv.flush(c);
    sync(c);
  });
}

extern "C" int cpcag_cuda_kron_reduce(cpcag_ctx ctx, cpcag_csr Lh, const int64_t* keep, int64_t n_keep,
                                      double pcg_tol, double prune_tol, cpcag_csr* out) {
  return guard([&] {
    Ctx* c = as_ctx(ctx);
    if (!out) invalid("null output pointer");
    std::vector<i64> k(static_cast<size_t>(std::max<int64_t>(n_keep, 0)));
    if (!k.empty()) {
      if (is_device_ptr(keep))
        CUDA_OK(cudaMemcpy(k.data(), keep, sizeof(i64) * k.size(), cudaMemcpyDeviceToHost));
      else
        std::copy(keep, keep + k.size(), k.begin());
    }
    Csr* r = kron_reduce_device(c, as_csr(Lh), k, pcg_tol, prune_tol);
    r->sym = 1;
    *out = reinterpret_cast<cpcag_csr>(r);
  });
}

extern "C" int cpcag_cuda_pcg_solve(cpcag_ctx ctx, cpcag_csr Ah, const double* b, double* x, int64_t n,
                                    double tol, int64_t max_iter, int jacobi, int64_t* iterations,
                                    int* converged, double* relative_residual) {
  return guard([&] {
    Ctx* c = as_ctx(ctx);
    Csr* A = as_csr(Ah);
    if (A->rows != A->cols || A->cols != n) invalid("pcg: dimension mismatch");
    InView<double> bin(c, b, static_cast<size_t>(n));
    DevBuf<double> X(c, std::max<i64>(n, 1)), inv(c, std::max<i64>(n, 1));
    if (n) {
      if (is_device_ptr(x))
        CUDA_OK(cudaMemcpyAsync(X.p, x, sizeof(double) * n, cudaMemcpyDeviceToDevice, c->stream));
      else
        CUDA_OK(cudaMemcpyAsync(X.p, x, sizeof(double) * n, cudaMemcpyHostToDevice, c->stream));
      if (jacobi)
        jacobi_inv_k<<<blocks_for(n), kBlock, 0, c->stream>>>(n, A->rp, A->ci, A->v, inv.p);
      else
        ones_k<<<blocks_for(n), kBlock, 0, c->stream>>>(n, inv.p);
      launched(c);
    }
    PcgBatchOut res;
    pcg_batched(c, A, inv.p, bin.d, X.p, n, n ? 1 : 0, tol, max_iter, &res);
    if (n == 0) {
      *iterations = 0;
      *converged = 1;
      *relative_residual = 0.0;
      return;
    }
    const ColState& cs = res.cols[0];
    if (cs.err) runtime("pcg: breakdown (nonpositive curvature) at iteration " + std::to_string(cs.it));
    if (cs.done == 2) {
      // Zero right-hand side: x = b (solvers.hpp:38-42).
      CUDA_OK(cudaMemcpyAsync(X.p, bin.d, sizeof(double) * n, cudaMemcpyDeviceToDevice, c->stream));
    }
    if (is_device_ptr(x))
      CUDA_OK(cudaMemcpyAsync(x, X.p, sizeof(double) * n, cudaMemcpyDeviceToDevice, c->stream));
    else
      CUDA_OK(cudaMemcpyAsync(x, X.p, sizeof(double) * n, cudaMemcpyDeviceToHost, c->stream));
    sync(c);
    *iterations = cs.it;
    *converged = cs.done == 2 ? 1 : (cs.rel_res <= tol ? 1 : 0);
    *relative_residual = cs.done == 2 ? 0.0 : cs.rel_res;
  });
}
