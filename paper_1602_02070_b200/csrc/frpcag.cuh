// frpcag.cuh -- per-element device building blocks shared by the SpMM,
// FISTA and decoder kernels.
//
// Every pull reproduces the reference's accumulation order for one output
// entry with explicit round-to-nearest multiply then add (no FMA), so fp64
// results match sparse.cpp:87-111 bit for bit:
//   pull_left  (Lr X)(i, c) = sum over CSR row i of Lr    (sparse.cpp:90-96)
//   pull_right (X Lc)(i, c) = sum over CSR row c of Lc^T  (sparse.cpp:103-109)
#pragma once

#include "common.cuh"

namespace cpcag_cuda {

template <typename T>
struct Pull {
  const i64* rp;
  const int* ci;
  const T* v;
};

// Accumulation step of the pulls: exact multiply-then-add for fp64 (bit
// parity with the reference loop); fused multiply-add for fp32 (whose
// results are compared to the fp64 oracle with a tolerance anyway).
template <typename T>
__device__ __forceinline__ T acc_step(T acc, T v, T x) {
  if constexpr (sizeof(T) == 8)
    return __dadd_rn(acc, __dmul_rn(v, x));
  else
    return fmaf(v, x, acc);
}

template <typename T>
__device__ __forceinline__ T pull_left(i64 k0, i64 k1, const int* __restrict__ ci,
                                       const T* __restrict__ v, const T* __restrict__ xcol) {
  T acc = T(0);
  for (i64 k = k0; k < k1; ++k) acc = acc_step(acc, v[k], xcol[ci[k]]);
  return acc;
}

template <typename T>
__device__ __forceinline__ T pull_right(i64 k0, i64 k1, const int* __restrict__ ci,
                                        const T* __restrict__ v, const T* __restrict__ X, i64 ld,
                                        i64 i) {
  T acc = T(0);
  for (i64 k = k0; k < k1; ++k) acc = acc_step(acc, v[k], X[i + static_cast<i64>(ci[k]) * ld]);
  return acc;
}

// frpcag.cpp:37-44: Y + sign(D) o max(|D| - lam, 0), D = Z - Y, sign(0) = 0.
template <typename T>
__device__ __forceinline__ T prox_l1_elem(T z, T y, T lam) {
  const T d = sub_rn(z, y);
  const T sg = d > T(0) ? T(1) : (d < T(0) ? T(-1) : T(0));
  T m = sub_rn(fabs(d), lam);
  m = m > T(0) ? m : T(0);
  return add_rn(y, mul_rn(sg, m));
}

// frpcag.cpp:46-51: (Z + (2 lam) Y) / (1 + 2 lam).
template <typename T>
__device__ __forceinline__ T prox_l2_elem(T z, T y, T lam) {
  const T a = mul_rn(T(2), lam);
  const T b = add_rn(T(1), a);
  if constexpr (sizeof(T) == 8)
    return __ddiv_rn(add_rn(z, mul_rn(a, y)), b);
  else
    return __fdiv_rn(add_rn(z, mul_rn(a, y)), b);
}

// frpcag.cpp:53-60: G = (2 gc) (Z Lc) + (2 gr) (Lr Z), terms skipped when
// their weight is zero.
template <typename T>
__device__ __forceinline__ T grad_elem(const Pull<T>& Lr, const Pull<T>& Lc, T s_r, T s_c, int use_r,
                                       int use_c, const T* __restrict__ Z, i64 rows, i64 i, i64 c) {
  T g = T(0);
  if (use_c) g = add_rn(g, mul_rn(s_c, pull_right(Lc.rp[c], Lc.rp[c + 1], Lc.ci, Lc.v, Z, rows, i)));
  if (use_r) g = add_rn(g, mul_rn(s_r, pull_left(Lr.rp[i], Lr.rp[i + 1], Lr.ci, Lr.v, Z + c * rows)));
  return g;
}

template <typename T>
Pull<T> make_pull(Ctx* c, Csr* A, bool right);

void frpcag_check_dims(i64 rows, i64 cols, Csr* Lr, Csr* Lc);

template <typename T>
void subsample_device(Ctx* c, const T* Y, i64 p, const i64* om_r, i64 rho_r, const i64* om_c,
                      i64 rho_c, T* out);

template <typename T>
double objective_device(Ctx* c, const T* X, const T* Y, i64 rows, i64 cols, Csr* Lr, Csr* Lc,
                        const cpcag_frpcag_config& cfg);

}  // namespace cpcag_cuda
