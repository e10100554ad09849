// fista_dense.cuh -- the dense-operator tile of the FISTA kernels (shared by
// fista.cu and the column-sharded solve in sharded.cu): both products of one
// 32 x 32 output tile, and the densified image of a Kron-reduced Laplacian.
#pragma once

#include "common.cuh"

namespace cpcag_cuda {

constexpr int kDT = 32;   // output tile side
constexpr int kDK = 32;   // k chunk

template <typename T>
__device__ __forceinline__ T madd(T acc, T a, T b) {
  if constexpr (sizeof(T) == 8)
    return __dadd_rn(acc, __dmul_rn(a, b));
  else
    return fmaf(a, b, acc);
}

// acc1 = (Lr Z)(i, c) over k < rr;  acc2 = (Z Lc)(i, c) over k < rc.
// Lr, Lc dense column-major (symmetric), Z rr x rc column-major.
template <typename T>
__device__ __forceinline__ void dual_gemm_tile(const T* __restrict__ Lr, const T* __restrict__ Lc,
                                               const T* __restrict__ Z, i64 rr, i64 rc, int use_r, int use_c,
                                               i64 i0, i64 c0, T (&acc1)[2][2], T (&acc2)[2][2]) {
  __shared__ T As[kDK][kDT + 1];
  __shared__ T Bs[kDK][kDT + 1];
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int b = 0; b < 2; ++b) acc1[a][b] = acc2[a][b] = T(0);
  // The next chunk's eight operands are loaded into registers while the
  // current chunk is multiplied (the k-loop is serial per CTA; the sums keep
  // their ascending-k order).
  const int lo = tid & 31, hi = tid >> 5;
  T ra[4], rb[4];
  if (use_r) {
    auto fetch = [&](i64 k0) {
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const i64 gi = i0 + lo, gk = k0 + hi + 8 * q;
        ra[q] = (gi < rr && gk < rr) ? Lr[gk * rr + gi] : T(0);
        const i64 gk2 = k0 + lo, gc = c0 + hi + 8 * q;
        rb[q] = (gk2 < rr && gc < rc) ? Z[gc * rr + gk2] : T(0);
      }
    };
    fetch(0);
    for (i64 k0 = 0; k0 < rr; k0 += kDK) {
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        As[hi + 8 * q][lo] = ra[q];
        Bs[lo][hi + 8 * q] = rb[q];
      }
      __syncthreads();
      if (k0 + kDK < rr) fetch(k0 + kDK);
#pragma unroll 8
      for (int kk = 0; kk < kDK; ++kk) {
        const T a0 = As[kk][ty], a1 = As[kk][ty + 16];
        const T b0 = Bs[kk][tx], b1 = Bs[kk][tx + 16];
        acc1[0][0] = madd(acc1[0][0], a0, b0);
        acc1[0][1] = madd(acc1[0][1], a0, b1);
        acc1[1][0] = madd(acc1[1][0], a1, b0);
        acc1[1][1] = madd(acc1[1][1], a1, b1);
      }
      __syncthreads();
    }
  }
  if (use_c) {
    auto fetch = [&](i64 k0) {
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const i64 gi = i0 + lo, gk = k0 + hi + 8 * q;
        ra[q] = (gi < rr && gk < rc) ? Z[gk * rr + gi] : T(0);
        const i64 gk2 = k0 + lo, gc = c0 + hi + 8 * q;
        rb[q] = (gk2 < rc && gc < rc) ? Lc[gc * rc + gk2] : T(0);
      }
    };
    fetch(0);
    for (i64 k0 = 0; k0 < rc; k0 += kDK) {
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        As[hi + 8 * q][lo] = ra[q];
        Bs[lo][hi + 8 * q] = rb[q];
      }
      __syncthreads();
      if (k0 + kDK < rc) fetch(k0 + kDK);
#pragma unroll 8
      for (int kk = 0; kk < kDK; ++kk) {
        const T a0 = As[kk][ty], a1 = As[kk][ty + 16];
        const T b0 = Bs[kk][tx], b1 = Bs[kk][tx + 16];
        acc2[0][0] = madd(acc2[0][0], a0, b0);
        acc2[0][1] = madd(acc2[0][1], a0, b1);
        acc2[1][0] = madd(acc2[1][0], a1, b0);
        acc2[1][1] = madd(acc2[1][1], a1, b1);
      }
      __syncthreads();
    }
  }
}

template <typename T>
__global__ void densify_k(i64 n, const i64* __restrict__ rp, const int* __restrict__ ci,
                          const double* __restrict__ v, T* __restrict__ D) {
  const i64 r = blockIdx.x * (i64)blockDim.x + threadIdx.x;
  if (r >= n) return;
  // column-major D(r, c); the operator is exactly symmetric, so this is also
  // its row-major image.
  for (i64 k = rp[r]; k < rp[r + 1]; ++k) D[r + static_cast<i64>(ci[k]) * n] = static_cast<T>(v[k]);
}

template <typename T>
void densify(Ctx* c, Csr* A, DevBuf<T>& D) {
  const i64 n = A->rows;
  D.alloc(c, std::max<i64>(n * n, 1));
  D.zero(c);
  if (n) {
    densify_k<T><<<blocks_for(n), kBlock, 0, c->stream>>>(n, A->rp, A->ci, A->v, D.p);
    launched(c);
  }
}

inline bool dense_worthwhile(Csr* A) {
  const double n = static_cast<double>(A->rows);
  return A->rows > 0 && A->rows <= 16384 && static_cast<double>(A->nnz) >= 0.25 * n * n;
}

}  // namespace cpcag_cuda
