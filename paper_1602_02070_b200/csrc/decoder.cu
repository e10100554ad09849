// decoder.cu -- the graph-regularised alternate decoder (decoders.cpp:145-186):
// conjugate gradient on the normal operator
//     A(X) = gbar_c X Lc + gbar_r Lr X + M o X,   b = scatter(Xt),  X0 = 0,
// with the reference recurrence of detail::pcg_core (solvers.hpp:33-74,
// identity preconditioner: z = r, rho = <r, r>).
//
// HBM layout: X, R, P, AP are p x n column-major in the working precision;
// the mask and b are never materialised: rsel[i] / csel[c] give the position
// of row i / column c in the plan (or -1), so M(i,c) and b(i,c) are O(1)
// look-ups.  One CG iteration is three kernels:
//   A  apply+dot   AP = A(P), <P, AP>          -> alpha (last block)
//   B  residual    R -= alpha AP, <R, R>        -> beta
//   C  update      X += alpha P, P = R + beta P -> stop test
// Every scalar lives on the device; the host polls the done flag once per
// chunk of iterations.
#include <algorithm>
#include <cstdio>
#include <memory>
#include <cstdlib>
#include <string>
#include <type_traits>

#include "common.cuh"
#include "frpcag.cuh"

namespace cpcag_cuda {

struct CgState {
  double rho, rho_next, curv, alpha, beta;
  double norm_b, target, rel_res;
  i64 it;
  int done, err, zero_rhs, pad;
  i64 err_it;
  unsigned cnt[4];
};

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

struct Plan {
  const int* rsel;   // p: index into omega_r or -1
  const int* csel;   // n: index into omega_c or -1
  i64 rho_r;
};

template <typename T>
__device__ __forceinline__ T rhs_at(const Plan& pl, const T* __restrict__ Xt, i64 i, i64 c) {
  const int a = pl.rsel[i], b = pl.csel[c];
  return (a >= 0 && b >= 0) ? Xt[a + static_cast<i64>(b) * pl.rho_r] : T(0);
}

// decoders.cpp:160-170 for one entry: (gbar_c (X Lc))(i,c) + (gbar_r (Lr X))(i,c),
// then + X(i,c) on the sampled grid.
template <typename T>
__device__ __forceinline__ T apply_elem(const Pull<T>& Lr, const Pull<T>& Lc, T gr, T gc,
                                        const Plan& pl, const T* __restrict__ V, i64 p, i64 i,
                                        i64 c) {
  const T a1 = pull_right(Lc.rp[c], Lc.rp[c + 1], Lc.ci, Lc.v, V, p, i);
  const T a2 = pull_left(Lr.rp[i], Lr.rp[i + 1], Lr.ci, Lr.v, V + c * p);
  T out = add_rn(mul_rn(gc, a1), mul_rn(gr, a2));
  if (pl.rsel[i] >= 0 && pl.csel[c] >= 0) out = add_rn(out, V[i + c * p]);
  return out;
}

// x = 0, r = b, p = r; rho = <b, b>.
template <typename T>
__global__ void cg_init_k(i64 p, i64 n, Plan pl, const T* __restrict__ Xt, T* __restrict__ X,
                          T* __restrict__ R, T* __restrict__ P, double tol, double* partials,
                          CgState* st) {
  double s[1] = {0.0};
  const i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x;
  if (i < p) {
    for (i64 c = blockIdx.y; c < n; c += gridDim.y) {
      const i64 at = i + c * p;
      const T b = rhs_at(pl, Xt, i, c);
      X[at] = T(0);
      R[at] = b;
      P[at] = b;
      s[0] += static_cast<double>(b) * static_cast<double>(b);
    }
  }
  double tot[1];
  if (grid_sum_last<1>(s, partials, &st->cnt[0], tot) && threadIdx.x == 0) {
    const double nb = sqrt(tot[0]);
    st->norm_b = nb;
    st->rho = tot[0];
    st->it = 0;
    if (nb == 0.0) {
      st->zero_rhs = 1;
      st->done = 1;
      return;
    }
    st->target = tol * nb;
    if (sqrt(tot[0]) <= st->target) st->done = 1;
  }
}

template <typename T>
__global__ void cg_apply_k(i64 p, i64 n, Pull<T> Lr, Pull<T> Lc, T gr, T gc, Plan pl,
                           const T* __restrict__ P, T* __restrict__ AP, double* partials,
                           CgState* st) {
  if (st->done) return;
  double s[1] = {0.0};
  const i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x;
  if (i < p) {
    for (i64 c = blockIdx.y; c < n; c += gridDim.y) {
      const T ap = apply_elem(Lr, Lc, gr, gc, pl, P, p, i, c);
      AP[i + c * p] = ap;
      s[0] += static_cast<double>(P[i + c * p]) * static_cast<double>(ap);
    }
  }
  double tot[1];
  if (grid_sum_last<1>(s, partials, &st->cnt[1], tot) && threadIdx.x == 0) {
    const double curv = tot[0];
    st->curv = curv;
    if (!isfinite(curv) || curv <= 0.0) {
      st->err = 1;
      st->err_it = st->it;
      st->done = 1;
      return;
    }
    st->alpha = st->rho / curv;
  }
}

// Staged variant of cg_apply_k: a CTA owns rows [i0, i0 + 256) and a
// contiguous chunk of columns [cb, ce).  The CSR rows of L_r for its rows and
// of L_c for its columns are copied into shared memory once, so the inner
// loops only issue the P gathers (coalesced along i for the X L_c part).  The
// per-entry operation order is unchanged (bit-identical to cg_apply_k).
// Columns [c_lo, c_hi) are computed (the whole matrix for the one-GPU
// solver, one column block for the sharded decoder); AP is indexed by the
// global column (AP + c * p), P holds every column.
template <typename T>
__global__ void __launch_bounds__(256) cg_apply_staged_k(i64 p, i64 c_lo, i64 c_hi, Pull<T> Lr, Pull<T> Lc, T gr,
                                                         T gc, Plan pl, i64 cols_per_cta, const T* __restrict__ P,
                                                         T* __restrict__ AP, double* partials, CgState* st) {
  if (st->done) return;
  extern __shared__ __align__(16) unsigned char smraw[];
  const i64 i0 = static_cast<i64>(blockIdx.x) * blockDim.x;
  const i64 i1 = min(p, i0 + static_cast<i64>(blockDim.x));
  const i64 cb = c_lo + static_cast<i64>(blockIdx.y) * cols_per_cta;
  const i64 ce = min(c_hi, cb + cols_per_cta);
  const i64 kr_base = Lr.rp[i0], er = Lr.rp[i1] - kr_base;
  const i64 kc_base = cb < ce ? Lc.rp[cb] : 0, ec = cb < ce ? Lc.rp[ce] - kc_base : 0;
  T* vr = reinterpret_cast<T*>(smraw);
  T* vc = vr + er;
  int* cir = reinterpret_cast<int*>(vc + ec);
  int* cic = cir + er;
  for (i64 k = threadIdx.x; k < er; k += blockDim.x) {
    vr[k] = Lr.v[kr_base + k];
    cir[k] = Lr.ci[kr_base + k];
  }
  for (i64 k = threadIdx.x; k < ec; k += blockDim.x) {
    vc[k] = Lc.v[kc_base + k];
    cic[k] = Lc.ci[kc_base + k];
  }
  __syncthreads();
  double s[1] = {0.0};
  const i64 i = i0 + threadIdx.x;
  if (i < p) {
    const i64 a0 = Lr.rp[i] - kr_base, a1 = Lr.rp[i + 1] - kr_base;
    const bool row_sampled = pl.rsel[i] >= 0;
    for (i64 c = cb; c < ce; ++c) {
      const i64 b0 = Lc.rp[c] - kc_base, b1 = Lc.rp[c + 1] - kc_base;
      T x1 = T(0);
      for (i64 k = b0; k < b1; ++k) x1 = add_rn(x1, mul_rn(vc[k], P[i + static_cast<i64>(cic[k]) * p]));
      const T* pc = P + c * p;
      T x2 = T(0);
      for (i64 k = a0; k < a1; ++k) x2 = add_rn(x2, mul_rn(vr[k], pc[cir[k]]));
      T out = add_rn(mul_rn(gc, x1), mul_rn(gr, x2));
      const T pv = pc[i];
      if (row_sampled && pl.csel[c] >= 0) out = add_rn(out, pv);
      AP[i + c * p] = out;
      s[0] += static_cast<double>(pv) * static_cast<double>(out);
    }
  }
  double tot[1];
  if (grid_sum_last<1>(s, partials, &st->cnt[1], tot) && threadIdx.x == 0) {
    const double curv = tot[0];
    st->curv = curv;
    if (!isfinite(curv) || curv <= 0.0) {
      st->err = 1;
      st->err_it = st->it;
      st->done = 1;
      return;
    }
    st->alpha = st->rho / curv;
  }
}



// Lean variant of the staged apply (default when p * n < 2^31): the staged
// entries carry 32-bit element offsets (L_c: ci * p, L_r: ci), so a gather
// is one shared load of the (value, offset) pair, one wide address add, one
// global load and one fused multiply-add (fp32) / exact multiply + add
// (fp64, so fp64 stays bit-identical to the reference order).
template <typename T>
struct alignas(sizeof(T) == 8 ? 16 : 8) OffEnt {
  T v;
  int off;
};

template <typename T>
__device__ __forceinline__ T madd_entry(T acc, T v, T x) {
  if constexpr (sizeof(T) == 8)
    return __dadd_rn(acc, __dmul_rn(v, x));
  else
    return fmaf(v, x, acc);
}

template <typename T>
__global__ void __launch_bounds__(256) cg_apply_fast_k(int p, int c_lo, int c_hi, Pull<T> Lr, Pull<T> Lc, T gr, T gc,
                                                       Plan pl, int cols_per_cta, const T* __restrict__ P,
                                                       T* __restrict__ AP, double* partials, CgState* st) {
  if (st->done) return;
  extern __shared__ __align__(16) unsigned char smraw[];
  const int i0 = blockIdx.x * blockDim.x;
  const int i1 = min(p, i0 + static_cast<int>(blockDim.x));
  const int cb = c_lo + blockIdx.y * cols_per_cta;
  const int ce = min(c_hi, cb + cols_per_cta);
  const i64 kr_base = Lr.rp[i0];
  const int er = static_cast<int>(Lr.rp[i1] - kr_base);
  const i64 kc_base = cb < ce ? Lc.rp[cb] : 0;
  const int ec = cb < ce ? static_cast<int>(Lc.rp[ce] - kc_base) : 0;
  OffEnt<T>* Er = reinterpret_cast<OffEnt<T>*>(smraw);
  OffEnt<T>* Ec = Er + er;
  int* crp = reinterpret_cast<int*>(Ec + ec);  // chunk row pointers of L_c (ce - cb + 1)
  for (int k = threadIdx.x; k < er; k += blockDim.x) {
    OffEnt<T> e;
    e.v = Lr.v[kr_base + k];
    e.off = Lr.ci[kr_base + k];
    Er[k] = e;
  }
  for (int k = threadIdx.x; k < ec; k += blockDim.x) {
    OffEnt<T> e;
    e.v = Lc.v[kc_base + k];
    e.off = Lc.ci[kc_base + k] * p;
    Ec[k] = e;
  }
  for (int q = threadIdx.x; q <= ce - cb; q += blockDim.x) crp[q] = static_cast<int>(Lc.rp[cb + q] - kc_base);
  __syncthreads();
  double s[1] = {0.0};
  const int i = i0 + threadIdx.x;
  if (i < p) {
    const int a0 = static_cast<int>(Lr.rp[i] - kr_base), a1 = static_cast<int>(Lr.rp[i + 1] - kr_base);
    const bool row_sampled = pl.rsel[i] >= 0;
    const T* Pi = P + i;
    for (int c = cb; c < ce; ++c) {
      const int b0 = crp[c - cb], b1 = crp[c - cb + 1];
      T x1 = T(0);
#pragma unroll 4
      for (int k = b0; k < b1; ++k) {
        const OffEnt<T> e = Ec[k];
        x1 = madd_entry(x1, e.v, Pi[e.off]);
      }
      const T* pc = P + static_cast<i64>(c) * p;
      T x2 = T(0);
#pragma unroll 4
      for (int k = a0; k < a1; ++k) {
        const OffEnt<T> e = Er[k];
        x2 = madd_entry(x2, e.v, pc[e.off]);
      }
      T out = add_rn(mul_rn(gc, x1), mul_rn(gr, x2));
      const T pv = pc[i];
      if (row_sampled && pl.csel[c] >= 0) out = add_rn(out, pv);
      AP[i + static_cast<i64>(c) * p] = out;
      s[0] += static_cast<double>(pv) * static_cast<double>(out);
    }
  }
  double tot[1];
  if (grid_sum_last<1>(s, partials, &st->cnt[1], tot) && threadIdx.x == 0) {
    const double curv = tot[0];
    st->curv = curv;
    if (!isfinite(curv) || curv <= 0.0) {
      st->err = 1;
      st->err_it = st->it;
      st->done = 1;
      return;
    }
    st->alpha = st->rho / curv;
  }
}

// fast5 (fp32, p % 4 == 0): each warp owns 128 rows.  The L_c gathers load
// 4 contiguous rows per lane as one 16-byte LDG (512 B per warp request, a
// quarter of fast2's LDG count for that part; the gather is bound by LSU
// issue, ~1.8 cycles per LDG per SM); the L_c sums go through a warp-private
// shared-memory transpose so the L_r gathers, the own value and the store
// stay unit-stride across lanes (rows r0 + lane + 32 k).  Per-entry
// arithmetic and order are fast2's: results are identical.
template <int U>
__global__ void __launch_bounds__(128, 8) cg_apply_fast5_k(int p, int n, Pull<float> Lr, Pull<float> Lc, float gr,
                                                           float gc, Plan pl, int cols_per_cta,
                                                           const float* __restrict__ P, float* __restrict__ AP,
                                                           double* partials, CgState* st) {
  if (st->done) return;
  extern __shared__ __align__(16) unsigned char smraw[];
  constexpr int RB = 512;  // 4 warps x 128 rows
  __shared__ __align__(16) float xs[4][128];
  const int i0 = blockIdx.x * RB;
  const int i1 = min(p, i0 + RB);
  const int cb = blockIdx.y * cols_per_cta;
  const int ce = min(n, cb + cols_per_cta);
  const i64 kr_base = Lr.rp[i0];
  const int er = static_cast<int>(Lr.rp[i1] - kr_base);
  const i64 kc_base = cb < ce ? Lc.rp[cb] : 0;
  const int ec = cb < ce ? static_cast<int>(Lc.rp[ce] - kc_base) : 0;
  OffEnt<float>* Er = reinterpret_cast<OffEnt<float>*>(smraw);
  OffEnt<float>* Ec = Er + er;
  int* crp = reinterpret_cast<int*>(Ec + ec);
  int* rrp = crp + (ce - cb + 1);
  for (int k = threadIdx.x; k < er; k += 128) {
    OffEnt<float> e;
    e.v = Lr.v[kr_base + k];
    e.off = Lr.ci[kr_base + k];
    Er[k] = e;
  }
  for (int k = threadIdx.x; k < ec; k += 128) {
    OffEnt<float> e;
    e.v = Lc.v[kc_base + k];
    e.off = Lc.ci[kc_base + k] * p;
    Ec[k] = e;
  }
  for (int q = threadIdx.x; q <= ce - cb; q += 128) crp[q] = static_cast<int>(Lc.rp[cb + q] - kc_base);
  for (int q = threadIdx.x; q <= i1 - i0; q += 128) rrp[q] = static_cast<int>(Lr.rp[i0 + q] - kr_base);
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int r0 = i0 + warp * 128;
  const bool vrow = r0 + 4 * lane < p;  // p % 4 == 0: the whole float4 is valid
  float* xw = xs[warp];
  unsigned sr = 0;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int i = r0 + lane + 32 * k;
    if (i < p && pl.rsel[i] >= 0) sr |= 1u << k;
  }
  double s[1] = {0.0};
  const float* Pv = P + r0 + 4 * lane;
  for (int c = cb; c < ce; ++c) {
    const int k0 = crp[c - cb], k1 = crp[c - cb + 1];
    float4 x = make_float4(0.f, 0.f, 0.f, 0.f);
    if (vrow) {
      int k = k0;
      for (; k + U <= k1; k += U) {
        float4 g[U];
        float w[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const OffEnt<float> e = Ec[k + u];
          w[u] = e.v;
          g[u] = *reinterpret_cast<const float4*>(Pv + e.off);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
          x.x = madd_entry(x.x, w[u], g[u].x);
          x.y = madd_entry(x.y, w[u], g[u].y);
          x.z = madd_entry(x.z, w[u], g[u].z);
          x.w = madd_entry(x.w, w[u], g[u].w);
        }
      }
      for (; k < k1; ++k) {
        const OffEnt<float> e = Ec[k];
        const float4 g = *reinterpret_cast<const float4*>(Pv + e.off);
        x.x = madd_entry(x.x, e.v, g.x);
        x.y = madd_entry(x.y, e.v, g.y);
        x.z = madd_entry(x.z, e.v, g.z);
        x.w = madd_entry(x.w, e.v, g.w);
      }
    }
    __syncwarp();
    *reinterpret_cast<float4*>(xw + 4 * lane) = x;
    __syncwarp();
    const float* pc = P + static_cast<i64>(c) * p;
    const bool cs = pl.csel[c] >= 0;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int i = r0 + lane + 32 * k;
      if (i < p) {
        const int lr = i - i0;
        float y = 0.f;
        for (int q = rrp[lr]; q < rrp[lr + 1]; ++q) {
          const OffEnt<float> e = Er[q];
          y = madd_entry(y, e.v, pc[e.off]);
        }
        float o = add_rn(mul_rn(gc, xw[lane + 32 * k]), mul_rn(gr, y));
        const float pv = pc[i];
        if (((sr >> k) & 1u) && cs) o = add_rn(o, pv);
        AP[i + static_cast<i64>(c) * p] = o;
        s[0] += static_cast<double>(pv) * static_cast<double>(o);
      }
    }
  }
  double tot[1];
  if (grid_sum_last<1>(s, partials, &st->cnt[1], tot) && threadIdx.x == 0) {
    const double curv = tot[0];
    st->curv = curv;
    if (!isfinite(curv) || curv <= 0.0) {
      st->err = 1;
      st->err_it = st->it;
      st->done = 1;
      return;
    }
    st->alpha = st->rho / curv;
  }
}

// slab: a CTA (1024 threads, one per SM) owns a 32-row slab of P across
// ALL n columns in shared memory (n * 128 B, n <= 1600 in fp32), so the
// ~19 L_c gathers of every entry are conflict-free shared-memory reads
// (lane = row) and only the L_r gathers go to L2.  Warp w takes columns
// c_lo + w, c_lo + w + 32, ... of the unit; units = slabs x column parts are
// dealt to the persistent CTAs in a fixed order (deterministic <P, AP>).
// Per-entry arithmetic and order are fast2's: results are identical.
template <typename T>
__global__ void __launch_bounds__(1024, 1) cg_apply_slab_k(int p, int n, Pull<T> Lr, Pull<T> Lc, T gr, T gc, Plan pl,
                                                           int col_parts, int units, const T* __restrict__ P,
                                                           T* __restrict__ AP, double* partials, CgState* st) {
  if (st->done) return;
  extern __shared__ __align__(16) unsigned char smraw[];
  T* S = reinterpret_cast<T*>(smraw);  // S[c * 32 + r] = P[i0 + r, c]
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double s[1] = {0.0};
  int staged = -1;
  for (int u = blockIdx.x; u < units; u += gridDim.x) {
    const int slab = u / col_parts, part = u - slab * col_parts;
    const int i0 = slab * 32, rows = min(32, p - i0);
    const int cw = (n + col_parts - 1) / col_parts;
    const int c_lo = part * cw, c_hi = min(n, c_lo + cw);
    if (slab != staged) {
      __syncthreads();
      for (int c = warp; c < n; c += 32) S[c * 32 + lane] = lane < rows ? P[i0 + lane + static_cast<i64>(c) * p] : T(0);
      __syncthreads();
      staged = slab;
    }
    const int i = i0 + lane;
    const bool valid = lane < rows;
    const int a0 = valid ? static_cast<int>(Lr.rp[i]) : 0, a1 = valid ? static_cast<int>(Lr.rp[i + 1]) : 0;
    const bool rs = valid && pl.rsel[i] >= 0;
    for (int c = c_lo + warp; c < c_hi; c += 32) {
      const int k0 = static_cast<int>(Lc.rp[c]), k1 = static_cast<int>(Lc.rp[c + 1]);
      T x = T(0);
#pragma unroll 4
      for (int k = k0; k < k1; ++k) x = madd_entry(x, __ldg(Lc.v + k), S[__ldg(Lc.ci + k) * 32 + lane]);
      if (valid) {
        const T* pc = P + static_cast<i64>(c) * p;
        T y = T(0);
#pragma unroll 4
        for (int k = a0; k < a1; ++k) y = madd_entry(y, __ldg(Lr.v + k), pc[__ldg(Lr.ci + k)]);
        T o = add_rn(mul_rn(gc, x), mul_rn(gr, y));
        const T pv = S[c * 32 + lane];
        if (rs && pl.csel[c] >= 0) o = add_rn(o, pv);
        AP[i + static_cast<i64>(c) * p] = o;
        s[0] += static_cast<double>(pv) * static_cast<double>(o);
      }
    }
  }
  double tot[1];
  if (grid_sum_last<1>(s, partials, &st->cnt[1], tot) && threadIdx.x == 0) {
    const double curv = tot[0];
    st->curv = curv;
    if (!isfinite(curv) || curv <= 0.0) {
      st->err = 1;
      st->err_it = st->it;
      st->done = 1;
      return;
    }
    st->alpha = st->rho / curv;
  }
}

// fast4: R rows per thread, strided by the CTA width (i, i + NT, ...), so
// each staged L_c entry serves R independent 4/8-byte gathers (R loads in
// flight per thread per entry, 128 B per warp request) and the L_r gathers
// stay unit-stride across lanes.  The config-1 gather is latency-bound
// (bytes in flight per SM); fast2 is the R = 2, NT = 256 case.  Per-entry
// arithmetic and order are fast2's: results are identical.
template <typename T, int R, int NT>
__global__ void __launch_bounds__(NT, 1024 / NT) cg_apply_fast4_k(int p, int n, Pull<T> Lr, Pull<T> Lc, T gr, T gc,
                                                                  Plan pl, int cols_per_cta, const T* __restrict__ P,
                                                                  T* __restrict__ AP, double* partials, CgState* st) {
  if (st->done) return;
  extern __shared__ __align__(16) unsigned char smraw[];
  constexpr int RB = NT * R;
  const int i0 = blockIdx.x * RB;
  const int i1 = min(p, i0 + RB);
  const int cb = blockIdx.y * cols_per_cta;
  const int ce = min(n, cb + cols_per_cta);
  const i64 kr_base = Lr.rp[i0];
  const int er = static_cast<int>(Lr.rp[i1] - kr_base);
  const i64 kc_base = cb < ce ? Lc.rp[cb] : 0;
  const int ec = cb < ce ? static_cast<int>(Lc.rp[ce] - kc_base) : 0;
  OffEnt<T>* Er = reinterpret_cast<OffEnt<T>*>(smraw);
  OffEnt<T>* Ec = Er + er;
  int* crp = reinterpret_cast<int*>(Ec + ec);
  int* rrp = crp + (ce - cb + 1);  // L_r row starts of this CTA's rows (RB + 1)
  for (int k = threadIdx.x; k < er; k += NT) {
    OffEnt<T> e;
    e.v = Lr.v[kr_base + k];
    e.off = Lr.ci[kr_base + k];
    Er[k] = e;
  }
  for (int k = threadIdx.x; k < ec; k += NT) {
    OffEnt<T> e;
    e.v = Lc.v[kc_base + k];
    e.off = Lc.ci[kc_base + k] * p;
    Ec[k] = e;
  }
  for (int q = threadIdx.x; q <= ce - cb; q += NT) crp[q] = static_cast<int>(Lc.rp[cb + q] - kc_base);
  for (int q = threadIdx.x; q <= i1 - i0; q += NT) rrp[q] = static_cast<int>(Lr.rp[i0 + q] - kr_base);
  __syncthreads();
  double s[1] = {0.0};
  const int ia = i0 + threadIdx.x;
  int nr = 0;  // valid rows of this thread: ia + NT * r < p for r < nr
#pragma unroll
  for (int r = 0; r < R; ++r) nr += ia + NT * r < p ? 1 : 0;
  unsigned sr = 0;  // sampled-row bits
#pragma unroll
  for (int r = 0; r < R; ++r)
    if (r < nr && pl.rsel[ia + NT * r] >= 0) sr |= 1u << r;
  const T* Pa = P + ia;
  if (nr > 0) {
    for (int c = cb; c < ce; ++c) {
      const int k0 = crp[c - cb], k1 = crp[c - cb + 1];
      T x[R];
#pragma unroll
      for (int r = 0; r < R; ++r) x[r] = T(0);
#pragma unroll 2
      for (int k = k0; k < k1; ++k) {
        const OffEnt<T> e = Ec[k];
        T g[R];
#pragma unroll
        for (int r = 0; r < R; ++r) g[r] = r < nr ? Pa[e.off + NT * r] : T(0);
#pragma unroll
        for (int r = 0; r < R; ++r) x[r] = madd_entry(x[r], e.v, g[r]);
      }
      const T* pc = P + static_cast<i64>(c) * p;
      const bool cs = pl.csel[c] >= 0;
#pragma unroll
      for (int r = 0; r < R; ++r) {
        if (r < nr) {
          const int lr = threadIdx.x + NT * r;
          T y = T(0);
          for (int q = rrp[lr]; q < rrp[lr + 1]; ++q) {
            const OffEnt<T> e = Er[q];
            y = madd_entry(y, e.v, pc[e.off]);
          }
          T o = add_rn(mul_rn(gc, x[r]), mul_rn(gr, y));
          const T pv = pc[ia + NT * r];
          if (((sr >> r) & 1u) && cs) o = add_rn(o, pv);
          AP[ia + NT * r + static_cast<i64>(c) * p] = o;
          s[0] += static_cast<double>(pv) * static_cast<double>(o);
        }
      }
    }
  }
  double tot[1];
  if (grid_sum_last<1>(s, partials, &st->cnt[1], tot) && threadIdx.x == 0) {
    const double curv = tot[0];
    st->curv = curv;
    if (!isfinite(curv) || curv <= 0.0) {
      st->err = 1;
      st->err_it = st->it;
      st->done = 1;
      return;
    }
    st->alpha = st->rho / curv;
  }
}

// Two-pass apply, pass 1 (CPCAG_APPLY=slab2, opt-in; needs a 32-row slab of
// P over all n columns to fit in shared memory): U = P L_c without the
// weight, i.e. exactly fast2's x (same entries, same CSR order, same
// madd_entry), so pass 2 (fast2<kU>: the L_r pull, the mask, the weights and
// <P, AP>) produces bit-identical AP.  The slab makes every L_c gather a
// conflict-free shared-memory read (lane = row); a column's entries are read
// staged in shared memory per unit and read as warp broadcasts.  CTAs take contiguous
// runs of (slab, column part) units and restage only when the slab changes.
// Measured at config 1 (decode stage, 200 iterations): slab2 59.6 ms vs
// fast2 45.0 ms -- the slab pass is issue-bound (89 us, ncu) and pass 2
// re-reads P and U from DRAM at low occupancy (latency-bound, 137 us).
template <typename T>
__global__ void __launch_bounds__(1024, 1) cg_lc_slab_k(int p, int n, Pull<T> Lc, int parts, int units,
                                                        const T* __restrict__ P, T* __restrict__ U,
                                                        const CgState* st) {
  if (st->done) return;
  extern __shared__ __align__(16) unsigned char smraw[];
  T* S = reinterpret_cast<T*>(smraw);  // S[c * 32 + r] = P[i0 + r, c]
  // the unit's L_c entries (value, slab offset), read as warp broadcasts
  OffEnt<T>* E = reinterpret_cast<OffEnt<T>*>(smraw + static_cast<size_t>(n) * 32 * sizeof(T));
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int u0 = static_cast<int>((static_cast<i64>(units) * blockIdx.x) / gridDim.x);
  const int u1 = static_cast<int>((static_cast<i64>(units) * (blockIdx.x + 1)) / gridDim.x);
  const int cw = (n + parts - 1) / parts;
  int staged = -1, staged_part = -1;
  for (int u = u0; u < u1; ++u) {
    const int slab = u / parts, part = u - slab * parts;
    const int i0 = slab * 32, rows = min(32, p - i0);
    const int c_lo = part * cw, c_hi = min(n, c_lo + cw);
    const i64 e0 = Lc.rp[c_lo];
    if (slab != staged || part != staged_part) {
      __syncthreads();
      if (slab != staged)
        for (int c = warp; c < n; c += 32) S[c * 32 + lane] = lane < rows ? P[i0 + lane + static_cast<i64>(c) * p] : T(0);
      if (part != staged_part) {
        const int ne = static_cast<int>(Lc.rp[c_hi] - e0);
        for (int k = threadIdx.x; k < ne; k += blockDim.x) {
          OffEnt<T> e;
          e.v = Lc.v[e0 + k];
          e.off = Lc.ci[e0 + k] * 32;
          E[k] = e;
        }
      }
      __syncthreads();
      staged = slab;
      staged_part = part;
    }
    for (int c = c_lo + warp; c < c_hi; c += 32) {
      const int k0 = static_cast<int>(Lc.rp[c] - e0), k1 = static_cast<int>(Lc.rp[c + 1] - e0);
      T x = T(0);
#pragma unroll 4
      for (int k = k0; k < k1; ++k) {
        const OffEnt<T> e = E[k];
        x = madd_entry(x, e.v, S[e.off + lane]);
      }
      if (lane < rows) U[i0 + lane + static_cast<i64>(c) * p] = x;
    }
  }
}

// slabr: one-pass apply for iterates with few columns (config 1: n = 1000)
// and a low-degree row graph (the pixel grid, degree <= MAXD).  A CTA owns
// (32-row slab, column part) units: the slab of P over ALL n columns sits in
// shared memory, so every L_c gather is a conflict-free shared read (lane =
// row; fast2 instead re-reads ~19 P columns per output from L2, ~800 MB per
// config-1 apply); the unit's L_c entries are staged in shared memory and
// read as warp broadcasts; each lane holds its row's L_r entries in
// registers, so the stencil gathers P(k, c) (rows within the grid's halo of
// the slab) are independent global loads issued together.  Per-entry
// arithmetic and order are fast2's (CSR order, madd_entry, the same
// combination): AP is bit-identical to fast2.  <P, AP> is summed in a fixed
// order per CTA (deterministic; its order differs from fast2's).
template <typename T, int MAXD>
__global__ void __launch_bounds__(1024, 1) cg_apply_slabr_k(int p, int n, Pull<T> Lr, Pull<T> Lc, T gr, T gc, Plan pl,
                                                            int parts, int units, const T* __restrict__ P,
                                                            T* __restrict__ AP, double* partials, CgState* st) {
  if (st->done) return;
  extern __shared__ __align__(16) unsigned char smraw[];
  T* S = reinterpret_cast<T*>(smraw);  // S[c * 32 + r] = P[i0 + r, c]
  OffEnt<T>* E = reinterpret_cast<OffEnt<T>*>(smraw + static_cast<size_t>(n) * 32 * sizeof(T));
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int u0 = static_cast<int>((static_cast<i64>(units) * blockIdx.x) / gridDim.x);
  const int u1 = static_cast<int>((static_cast<i64>(units) * (blockIdx.x + 1)) / gridDim.x);
  const int cw = (n + parts - 1) / parts;
  int staged = -1, staged_part = -1;
  T ra[MAXD];
  int oa[MAXD];
  int da = 0;
  bool valid = false, rs = false;
  double s[1] = {0.0};
  for (int u = u0; u < u1; ++u) {
    const int slab = u / parts, part = u - slab * parts;
    const int i0 = slab * 32, rows = min(32, p - i0);
    const int c_lo = part * cw, c_hi = min(n, c_lo + cw);
    const i64 e0 = Lc.rp[c_lo];
    if (slab != staged || part != staged_part) {
      __syncthreads();
      if (slab != staged) {
        for (int c = warp; c < n; c += 32) S[c * 32 + lane] = lane < rows ? P[i0 + lane + static_cast<i64>(c) * p] : T(0);
        const int i = i0 + lane;
        valid = lane < rows;
        da = 0;
        rs = valid && pl.rsel[i] >= 0;
        if (valid) {
          const i64 a0 = Lr.rp[i];
          da = static_cast<int>(Lr.rp[i + 1] - a0);
#pragma unroll
          for (int k = 0; k < MAXD; ++k) {
            ra[k] = k < da ? Lr.v[a0 + k] : T(0);
            oa[k] = k < da ? Lr.ci[a0 + k] : 0;
          }
        }
      }
      if (part != staged_part) {
        const int ne = static_cast<int>(Lc.rp[c_hi] - e0);
        for (int k = threadIdx.x; k < ne; k += blockDim.x) {
          OffEnt<T> e;
          e.v = Lc.v[e0 + k];
          e.off = Lc.ci[e0 + k] * 32;
          E[k] = e;
        }
      }
      __syncthreads();
      staged = slab;
      staged_part = part;
    }
    for (int c = c_lo + warp; c < c_hi; c += 32) {
      const T* pc = P + static_cast<i64>(c) * p;
      T g[MAXD];
#pragma unroll
      for (int k = 0; k < MAXD; ++k) g[k] = k < da ? pc[oa[k]] : T(0);
      const int k0 = static_cast<int>(Lc.rp[c] - e0), k1 = static_cast<int>(Lc.rp[c + 1] - e0);
      T x = T(0);
#pragma unroll 4
      for (int k = k0; k < k1; ++k) {
        const OffEnt<T> e = E[k];
        x = madd_entry(x, e.v, S[e.off + lane]);
      }
      T y = T(0);
#pragma unroll
      for (int k = 0; k < MAXD; ++k)
        if (k < da) y = madd_entry(y, ra[k], g[k]);
      if (valid) {
        T out = add_rn(mul_rn(gc, x), mul_rn(gr, y));
        const T pv = S[c * 32 + lane];
        if (rs && pl.csel[c] >= 0) out = add_rn(out, pv);
        AP[i0 + lane + static_cast<i64>(c) * p] = out;
        s[0] += static_cast<double>(pv) * static_cast<double>(out);
      }
    }
  }
  double tot[1];
  if (grid_sum_last<1>(s, partials, &st->cnt[1], tot) && threadIdx.x == 0) {
    const double curv = tot[0];
    st->curv = curv;
    if (!isfinite(curv) || curv <= 0.0) {
      st->err = 1;
      st->err_it = st->it;
      st->done = 1;
      return;
    }
    st->alpha = st->rho / curv;
  }
}

// regr: fast2 with each thread's L_r rows held in REGISTERS (row degree <=
// MAXD; the pixel-grid row graph of config 1 has degree 9).  L_r is the same
// for every column, so fast2's per-column re-read of the row's (value,
// offset) entries from shared memory -- two dependent loads in front of
// every gather -- goes away: the MAXD gathers of a row are independent loads
// issued together.  kU: x = P L_c comes from the slab pass (cg_lc_slab_k)
// instead of the L2 gathers.  Per-entry arithmetic and order are fast2's
// (CSR order, madd_entry, the same combination), so AP is bit-identical.
// Opt-in (CPCAG_APPLY=regr): measured slower than fast2 at config 1 (decode
// 68.2 vs 45.0 ms): 128 registers halve the occupancy and the L1-miss
// latency of the gathers is no longer hidden.
template <typename T, int MAXD, bool kU>
__global__ void __launch_bounds__(256, 2) cg_apply_regr_k(int p, int n, Pull<T> Lr, Pull<T> Lc, T gr, T gc, Plan pl,
                                                          int cols_per_cta, const T* __restrict__ P,
                                                          T* __restrict__ AP, double* partials, CgState* st,
                                                          const T* __restrict__ U) {
  if (st->done) return;
  extern __shared__ __align__(16) unsigned char smraw[];
  constexpr int RB = 512;
  const int i0 = blockIdx.x * RB;
  const int cb = blockIdx.y * cols_per_cta;
  const int ce = min(n, cb + cols_per_cta);
  const i64 kc_base = (!kU && cb < ce) ? Lc.rp[cb] : 0;
  const int ec = (!kU && cb < ce) ? static_cast<int>(Lc.rp[ce] - kc_base) : 0;
  OffEnt<T>* Ec = reinterpret_cast<OffEnt<T>*>(smraw);
  int* crp = reinterpret_cast<int*>(Ec + ec);
  if (!kU) {
    for (int k = threadIdx.x; k < ec; k += blockDim.x) {
      OffEnt<T> e;
      e.v = Lc.v[kc_base + k];
      e.off = Lc.ci[kc_base + k] * p;
      Ec[k] = e;
    }
    for (int q = threadIdx.x; q <= ce - cb; q += blockDim.x) crp[q] = static_cast<int>(Lc.rp[cb + q] - kc_base);
  }
  const int ia = i0 + threadIdx.x, ib = ia + 256;
  const bool va = ia < p, vb = ib < p;
  T ra[MAXD], rb[MAXD];
  int oa[MAXD], ob[MAXD];
  int da = 0, db = 0;
  if (va) {
    const i64 a0 = Lr.rp[ia];
    da = static_cast<int>(Lr.rp[ia + 1] - a0);
#pragma unroll
    for (int k = 0; k < MAXD; ++k) {
      ra[k] = k < da ? Lr.v[a0 + k] : T(0);
      oa[k] = k < da ? Lr.ci[a0 + k] : 0;
    }
  }
  if (vb) {
    const i64 b0 = Lr.rp[ib];
    db = static_cast<int>(Lr.rp[ib + 1] - b0);
#pragma unroll
    for (int k = 0; k < MAXD; ++k) {
      rb[k] = k < db ? Lr.v[b0 + k] : T(0);
      ob[k] = k < db ? Lr.ci[b0 + k] : 0;
    }
  }
  __syncthreads();
  double s[1] = {0.0};
  if (va) {
    const bool sa = pl.rsel[ia] >= 0, sb = vb && pl.rsel[ib] >= 0;
    const T* Pa = P + ia;
    for (int c = cb; c < ce; ++c) {
      T xa = T(0), xb = T(0);
      if constexpr (kU) {
        xa = U[ia + static_cast<i64>(c) * p];
        if (vb) xb = U[ib + static_cast<i64>(c) * p];
      } else {
        const int k0 = crp[c - cb], k1 = crp[c - cb + 1];
#pragma unroll 4
        for (int k = k0; k < k1; ++k) {
          const OffEnt<T> e = Ec[k];
          xa = madd_entry(xa, e.v, Pa[e.off]);
          if (vb) xb = madd_entry(xb, e.v, Pa[e.off + 256]);
        }
      }
      const T* pc = P + static_cast<i64>(c) * p;
      T ga[MAXD], gb[MAXD];
#pragma unroll
      for (int k = 0; k < MAXD; ++k) {
        ga[k] = k < da ? pc[oa[k]] : T(0);
        gb[k] = k < db ? pc[ob[k]] : T(0);
      }
      T ya = T(0), yb = T(0);
#pragma unroll
      for (int k = 0; k < MAXD; ++k) {
        if (k < da) ya = madd_entry(ya, ra[k], ga[k]);
        if (k < db) yb = madd_entry(yb, rb[k], gb[k]);
      }
      const bool cs = pl.csel[c] >= 0;
      {
        T out = add_rn(mul_rn(gc, xa), mul_rn(gr, ya));
        const T pv = pc[ia];
        if (sa && cs) out = add_rn(out, pv);
        AP[ia + static_cast<i64>(c) * p] = out;
        s[0] += static_cast<double>(pv) * static_cast<double>(out);
      }
      if (vb) {
        T out = add_rn(mul_rn(gc, xb), mul_rn(gr, yb));
        const T pv = pc[ib];
        if (sb && cs) out = add_rn(out, pv);
        AP[ib + static_cast<i64>(c) * p] = out;
        s[0] += static_cast<double>(pv) * static_cast<double>(out);
      }
    }
  }
  double tot[1];
  if (grid_sum_last<1>(s, partials, &st->cnt[1], tot) && threadIdx.x == 0) {
    const double curv = tot[0];
    st->curv = curv;
    if (!isfinite(curv) || curv <= 0.0) {
      st->err = 1;
      st->err_it = st->it;
      st->done = 1;
      return;
    }
    st->alpha = st->rho / curv;
  }
}

// fast2: two rows per thread (i and i + 256) so each staged L_c entry and
// its address arithmetic serve two gathers (the fast apply is issue- and
// latency-bound, ~6 instructions per 4-byte gather).
template <typename T, int MINB = 4, bool kU = false>
__global__ void __launch_bounds__(256, MINB) cg_apply_fast2_k(int p, int n, Pull<T> Lr, Pull<T> Lc, T gr, T gc, Plan pl,
                                                           int cols_per_cta, const T* __restrict__ P,
                                                           T* __restrict__ AP, double* partials, CgState* st,
                                                           const T* __restrict__ U = nullptr) {
  if (st->done) return;
  extern __shared__ __align__(16) unsigned char smraw[];
  constexpr int RB = 512;
  const int i0 = blockIdx.x * RB;
  const int i1 = min(p, i0 + RB);
  const int cb = blockIdx.y * cols_per_cta;
  const int ce = min(n, cb + cols_per_cta);
  const i64 kr_base = Lr.rp[i0];
  const int er = static_cast<int>(Lr.rp[i1] - kr_base);
  const i64 kc_base = (!kU && cb < ce) ? Lc.rp[cb] : 0;
  const int ec = (!kU && cb < ce) ? static_cast<int>(Lc.rp[ce] - kc_base) : 0;
  OffEnt<T>* Er = reinterpret_cast<OffEnt<T>*>(smraw);
  OffEnt<T>* Ec = Er + er;
  int* crp = reinterpret_cast<int*>(Ec + ec);
  for (int k = threadIdx.x; k < er; k += blockDim.x) {
    OffEnt<T> e;
    e.v = Lr.v[kr_base + k];
    e.off = Lr.ci[kr_base + k];
    Er[k] = e;
  }
  for (int k = threadIdx.x; k < ec; k += blockDim.x) {
    OffEnt<T> e;
    e.v = Lc.v[kc_base + k];
    e.off = Lc.ci[kc_base + k] * p;
    Ec[k] = e;
  }
  if (!kU)
    for (int q = threadIdx.x; q <= ce - cb; q += blockDim.x) crp[q] = static_cast<int>(Lc.rp[cb + q] - kc_base);
  __syncthreads();
  double s[1] = {0.0};
  const int ia = i0 + threadIdx.x, ib = ia + 256;
  const bool va = ia < p, vb = ib < p;
  if (va) {
    const int a0 = static_cast<int>(Lr.rp[ia] - kr_base), a1 = static_cast<int>(Lr.rp[ia + 1] - kr_base);
    const int b0 = vb ? static_cast<int>(Lr.rp[ib] - kr_base) : 0, b1 = vb ? static_cast<int>(Lr.rp[ib + 1] - kr_base) : 0;
    const bool sa = pl.rsel[ia] >= 0, sb = vb && pl.rsel[ib] >= 0;
    const T* Pa = P + ia;
    for (int c = cb; c < ce; ++c) {
      T xa = T(0), xb = T(0);
      if constexpr (kU) {
        // two-pass apply: P L_c of this entry from cg_lc_slab_k
        xa = U[ia + static_cast<i64>(c) * p];
        if (vb) xb = U[ib + static_cast<i64>(c) * p];
      } else {
        const int k0 = crp[c - cb], k1 = crp[c - cb + 1];
#pragma unroll 4
        for (int k = k0; k < k1; ++k) {
          const OffEnt<T> e = Ec[k];
          xa = madd_entry(xa, e.v, Pa[e.off]);
          if (vb) xb = madd_entry(xb, e.v, Pa[e.off + 256]);
        }
      }
      const T* pc = P + static_cast<i64>(c) * p;
      T ya = T(0), yb = T(0);
#pragma unroll 4
      for (int k = a0; k < a1; ++k) {
        const OffEnt<T> e = Er[k];
        ya = madd_entry(ya, e.v, pc[e.off]);
      }
#pragma unroll 4
      for (int k = b0; k < b1; ++k) {
        const OffEnt<T> e = Er[k];
        yb = madd_entry(yb, e.v, pc[e.off]);
      }
      const bool cs = pl.csel[c] >= 0;
      {
        T out = add_rn(mul_rn(gc, xa), mul_rn(gr, ya));
        const T pv = pc[ia];
        if (sa && cs) out = add_rn(out, pv);
        AP[ia + static_cast<i64>(c) * p] = out;
        s[0] += static_cast<double>(pv) * static_cast<double>(out);
      }
      if (vb) {
        T out = add_rn(mul_rn(gc, xb), mul_rn(gr, yb));
        const T pv = pc[ib];
        if (sb && cs) out = add_rn(out, pv);
        AP[ib + static_cast<i64>(c) * p] = out;
        s[0] += static_cast<double>(pv) * static_cast<double>(out);
      }
    }
  }
  double tot[1];
  if (grid_sum_last<1>(s, partials, &st->cnt[1], tot) && threadIdx.x == 0) {
    const double curv = tot[0];
    st->curv = curv;
    if (!isfinite(curv) || curv <= 0.0) {
      st->err = 1;
      st->err_it = st->it;
      st->done = 1;
      return;
    }
    st->alpha = st->rho / curv;
  }
}

// 16-byte vectors of the iterate (4 fp32 / 2 fp64 entries).
template <typename T>
struct Vec16;
template <>
struct Vec16<float> {
  using V = float4;
  static constexpr int W = 4;
};
template <>
struct Vec16<double> {
  using V = double2;
  static constexpr int W = 2;
};

template <typename T>
__device__ __forceinline__ T& vlane(typename Vec16<T>::V& v, int k) {
  return reinterpret_cast<T*>(&v)[k];
}

// R -= alpha AP, ||R||^2.  kVec: 16-byte loads/stores over the first
// N - N % W entries (all pointers 16-byte aligned), the tail scalar; the
// per-entry arithmetic is the same either way.
template <typename T, bool kVec = false>
__global__ void cg_residual_k(i64 N, T* __restrict__ R, const T* __restrict__ AP, double* partials,
                              CgState* st) {
  if (st->done) return;
  const T alpha = static_cast<T>(st->alpha);
  double s[1] = {0.0};
  const i64 t0 = blockIdx.x * (i64)blockDim.x + threadIdx.x, ts = (i64)gridDim.x * blockDim.x;
  i64 done = 0;
  if constexpr (kVec) {
    using V = typename Vec16<T>::V;
    constexpr int W = Vec16<T>::W;
    const i64 nv = N / W;
    V* Rv = reinterpret_cast<V*>(R);
    const V* Av = reinterpret_cast<const V*>(AP);
    for (i64 q = t0; q < nv; q += ts) {
      V r = Rv[q];
      V a = Av[q];
#pragma unroll
      for (int k = 0; k < W; ++k) {
        vlane<T>(r, k) = sub_rn(vlane<T>(r, k), mul_rn(alpha, vlane<T>(a, k)));
        s[0] += static_cast<double>(vlane<T>(r, k)) * static_cast<double>(vlane<T>(r, k));
      }
      Rv[q] = r;
    }
    done = nv * W;
  }
  for (i64 q = done + t0; q < N; q += ts) {
    const T r = sub_rn(R[q], mul_rn(alpha, AP[q]));
    R[q] = r;
    s[0] += static_cast<double>(r) * static_cast<double>(r);
  }
  double tot[1];
  if (grid_sum_last<1>(s, partials, &st->cnt[2], tot) && threadIdx.x == 0) {
    st->rho_next = tot[0];
    st->beta = tot[0] / st->rho;
  }
}

template <typename T, bool kVec = false>
__global__ void cg_update_k(i64 N, T* __restrict__ X, T* __restrict__ P, const T* __restrict__ R,
                            i64 max_iter, CgState* st) {
  if (st->done) return;
  const T alpha = static_cast<T>(st->alpha), beta = static_cast<T>(st->beta);
  const i64 t0 = blockIdx.x * (i64)blockDim.x + threadIdx.x, ts = (i64)gridDim.x * blockDim.x;
  i64 done = 0;
  if constexpr (kVec) {
    using V = typename Vec16<T>::V;
    constexpr int W = Vec16<T>::W;
    const i64 nv = N / W;
    V* Xv = reinterpret_cast<V*>(X);
    V* Pv = reinterpret_cast<V*>(P);
    const V* Rv = reinterpret_cast<const V*>(R);
    for (i64 q = t0; q < nv; q += ts) {
      V x = Xv[q], pv = Pv[q];
      const V r = Rv[q];
      V pn;
#pragma unroll
      for (int k = 0; k < W; ++k) {
        vlane<T>(x, k) = add_rn(vlane<T>(x, k), mul_rn(alpha, vlane<T>(pv, k)));
        vlane<T>(pn, k) = add_rn(reinterpret_cast<const T*>(&r)[k], mul_rn(beta, vlane<T>(pv, k)));
      }
      Xv[q] = x;
      Pv[q] = pn;
    }
    done = nv * W;
  }
  for (i64 q = done + t0; q < N; q += ts) {
    const T pv = P[q];
    X[q] = add_rn(X[q], mul_rn(alpha, pv));
    P[q] = add_rn(R[q], mul_rn(beta, pv));
  }
  // Scalar step: a second tiny reduction is not needed, the last block to
  // finish (counted) advances the iteration.
  __shared__ bool last;
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    last = atomicAdd(&st->cnt[3], 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (last && threadIdx.x == 0) {
    st->cnt[3] = 0u;
    st->rho = st->rho_next;
    st->it += 1;
    if (sqrt(st->rho) <= st->target || st->it >= max_iter) st->done = 1;
  }
}

// ||b - A(x)||^2 for the exit test (solvers.hpp:69-72).
// The whole CG loop of a SMALL decoder problem (p n <= 2^20, e.g. config 0)
// as one cooperative kernel (opt-in, CPCAG_CG_PERSIST=1; see the host code
// for the measurement): each CTA owns a contiguous range of entries;
// per iteration apply + <P, AP> | grid barrier | R -= alpha AP, ||R||^2 |
// grid barrier | X += alpha P, P = R + beta P | grid barrier.  At these sizes
// the per-kernel loop is launch/latency-bound (config 0: 46 us per
// iteration for three tiny kernels).  Per-entry arithmetic is the per-kernel
// path's (pulls in CSR order, madd_entry; the same residual/update
// formulas); the reductions are fixed-order, summed identically by every CTA,
// so every CTA takes the same alpha/beta/stop decisions.  P changes between
// barriers inside the launch: it is read with plain (weak) loads ordered
// after the barrier's gpu-scope acquire (never through the non-coherent
// read-only path: P is not declared const __restrict__).
template <typename T>
__global__ void __launch_bounds__(512) cg_persist_k(i64 p, i64 n, Pull<T> Lr, Pull<T> Lc, T gr, T gc, Plan pl,
                                                    T* __restrict__ X, T* __restrict__ R, T* P, T* __restrict__ AP,
                                                    double* partials, i64 max_iter, CgState* st, unsigned* bar,
                                                    int prof) {
  __shared__ double tot_sh;
  const int G = gridDim.x, lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const i64 N = p * n;
  const i64 e0 = (N * blockIdx.x) / G, e1 = (N * (blockIdx.x + 1)) / G;
  if (st->done) return;
  // stage the operators once: L_r (all rows) and the L_c rows of this CTA's
  // columns, as (value, index) records; per iteration only the P gathers go
  // to L2 (the barrier's acquire leaves L1 cold each iteration)
  extern __shared__ __align__(16) unsigned char smraw[];
  const int nr = static_cast<int>(Lr.rp[p]);
  OffEnt<T>* Er = reinterpret_cast<OffEnt<T>*>(smraw);
  const i64 ca = e0 / p, cb = e1 > e0 ? (e1 - 1) / p : ca;  // columns touched
  const i64 kc0 = Lc.rp[ca];
  const int nc = static_cast<int>(Lc.rp[cb + 1] - kc0);
  OffEnt<T>* Ec = Er + nr;
  int* rpr_s = reinterpret_cast<int*>(Ec + nc);
  int* rpc_s = rpr_s + (p + 1);
  for (int k = threadIdx.x; k < nr; k += blockDim.x) {
    OffEnt<T> en;
    en.v = Lr.v[k];
    en.off = Lr.ci[k];
    Er[k] = en;
  }
  for (int k = threadIdx.x; k < nc; k += blockDim.x) {
    OffEnt<T> en;
    en.v = Lc.v[kc0 + k];
    en.off = Lc.ci[kc0 + k];
    Ec[k] = en;
  }
  for (i64 q = threadIdx.x; q <= p; q += blockDim.x) rpr_s[q] = static_cast<int>(Lr.rp[q]);
  for (i64 q = threadIdx.x; q <= cb - ca + 1; q += blockDim.x) rpc_s[q] = static_cast<int>(Lc.rp[ca + q] - kc0);
  __syncthreads();
  double rho = st->rho;
  const double target = st->target;
  i64 it = st->it;
  double alpha = 0.0, beta = 0.0, curv = 0.0;
  bool err = false;
  unsigned long long pt[6] = {0, 0, 0, 0, 0, 0}, tq = gtimer();  // CTA 0 phase timers (CPCAG_CG_PERSIST_PROF)
  auto mark = [&](int ph) {
    if (threadIdx.x == 0) {
      const unsigned long long now = gtimer();
      pt[ph] += now - tq;
      tq = now;
    }
  };
  // fixed-order sum of the G block partials (the same in every CTA)
  auto grid_total = [&](const double* part) {
    if (warp == 0) {
      double v = 0.0;
      for (int q = lane; q < G; q += 32) v += __ldcg(part + q);
      v = warp_sum(v);
      if (lane == 0) tot_sh = v;
    }
    __syncthreads();
    const double t = tot_sh;
    __syncthreads();
    return t;
  };
  while (true) {
    double d[1] = {0.0};
    for (i64 e = e0 + threadIdx.x; e < e1; e += blockDim.x) {
      const i64 c = e / p, i = e - c * p;
      // entries from shared memory, gathers issued 8 at a time, accumulated
      // in CSR order
      T a1 = T(0), a2 = T(0);
      {
        const int k0 = rpc_s[c - ca], k1 = rpc_s[c - ca + 1];
        for (int kb = k0; kb < k1; kb += 8) {
          T vv[8], xv[8];
#pragma unroll
          for (int u = 0; u < 8; ++u)
            if (kb + u < k1) {
              const OffEnt<T> en = Ec[kb + u];
              vv[u] = en.v;
              xv[u] = P[i + static_cast<i64>(en.off) * p];
            }
#pragma unroll
          for (int u = 0; u < 8; ++u)
            if (kb + u < k1) a1 = madd_entry(a1, vv[u], xv[u]);
        }
      }
      {
        const int k0 = rpr_s[i], k1 = rpr_s[i + 1];
        for (int kb = k0; kb < k1; kb += 8) {
          T vv[8], xv[8];
#pragma unroll
          for (int u = 0; u < 8; ++u)
            if (kb + u < k1) {
              const OffEnt<T> en = Er[kb + u];
              vv[u] = en.v;
              xv[u] = P[en.off + c * p];
            }
#pragma unroll
          for (int u = 0; u < 8; ++u)
            if (kb + u < k1) a2 = madd_entry(a2, vv[u], xv[u]);
        }
      }
      T out = add_rn(mul_rn(gc, a1), mul_rn(gr, a2));
      const T pv = P[e];
      if (pl.rsel[i] >= 0 && pl.csel[c] >= 0) out = add_rn(out, pv);
      AP[e] = out;
      d[0] += static_cast<double>(pv) * static_cast<double>(out);
    }
    block_sum<1>(d);
    if (threadIdx.x == 0) partials[blockIdx.x] = d[0];
    mark(0);
    grid_barrier(&bar[0], &bar[1]);
    mark(1);
    curv = grid_total(partials);
    if (!isfinite(curv) || curv <= 0.0) {
      err = true;
      break;
    }
    alpha = rho / curv;
    const T aT = static_cast<T>(alpha);
    double r2[1] = {0.0};
    for (i64 e = e0 + threadIdx.x; e < e1; e += blockDim.x) {
      const T r = sub_rn(R[e], mul_rn(aT, AP[e]));
      R[e] = r;
      r2[0] += static_cast<double>(r) * static_cast<double>(r);
    }
    block_sum<1>(r2);
    if (threadIdx.x == 0) partials[G + blockIdx.x] = r2[0];
    mark(2);
    grid_barrier(&bar[0], &bar[1]);
    mark(3);
    const double rho_next = grid_total(partials + G);
    beta = rho_next / rho;
    const T bT = static_cast<T>(beta);
    for (i64 e = e0 + threadIdx.x; e < e1; e += blockDim.x) {
      const T pv = P[e];
      X[e] = add_rn(X[e], mul_rn(aT, pv));
      P[e] = add_rn(R[e], mul_rn(bT, pv));
    }
    rho = rho_next;
    it += 1;
    mark(4);
    if (sqrt(rho) <= target || it >= max_iter) break;
    grid_barrier(&bar[0], &bar[1]);
    mark(5);
  }
  if (prof && blockIdx.x == 0 && threadIdx.x == 0)
    printf("[cg_persist] G %d its %lld: apply %.1f bar %.1f resid %.1f bar %.1f update %.1f bar %.1f us\n", G,
           static_cast<long long>(it), pt[0] * 1e-3, pt[1] * 1e-3, pt[2] * 1e-3, pt[3] * 1e-3, pt[4] * 1e-3,
           pt[5] * 1e-3);
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    st->curv = curv;
    st->alpha = alpha;
    st->beta = beta;
    st->rho = rho;
    st->it = it;
    st->done = 1;
    if (err) {
      st->err = 1;
      st->err_it = it;
    }
  }
}

template <typename T>
__global__ void cg_true_residual_k(i64 p, i64 n, Pull<T> Lr, Pull<T> Lc, T gr, T gc, Plan pl,
                                   const T* __restrict__ Xt, const T* __restrict__ X,
                                   double* partials, CgState* st) {
  double s[1] = {0.0};
  const i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x;
  if (i < p) {
    for (i64 c = blockIdx.y; c < n; c += gridDim.y) {
      const T ax = apply_elem(Lr, Lc, gr, gc, pl, X, p, i, c);
      const double e = static_cast<double>(sub_rn(rhs_at(pl, Xt, i, c), ax));
      s[0] += e * e;
    }
  }
  double tot[1];
  if (grid_sum_last<1>(s, partials, &st->cnt[0], tot) && threadIdx.x == 0)
    st->rel_res = sqrt(tot[0]) / st->norm_b;
}

__global__ void fill_sel_k(i64 len, int* sel) {
  const i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x;
  if (i < len) sel[i] = -1;
}
__global__ void scatter_sel_k(const i64* __restrict__ om, i64 rho, int* sel) {
  const i64 k = blockIdx.x * (i64)blockDim.x + threadIdx.x;
  if (k < rho) sel[om[k]] = static_cast<int>(k);
}

// ------------------------------------------------------------------ band apply
// For iterates that do not fit in L2 (cfg3: P is 4096 x 200000 fp32 =
// 3.3 GB) the single-pass applies above fetch every gathered column of P
// from HBM again, about 19 times the matrix per apply.  The band apply splits
// A(P) into two sweeps.  Each sweep keeps the data it gathers on chip:
//   cg_apply_band_k  U = gc (P L_c).  Rows go in bands of 32*RPL; the grid is
//                    band-major (blockIdx.x = column chunk), so one band of
//                    32*RPL rows x all n columns (<= ~56 MB) stays resident
//                    in L2 while each column gathers its L_c neighbours from
//                    it.  One warp per column, lane = row: 128-byte gathers.
//   cg_apply_col_k   AP = U + gr (L_r P) (+ P on the sampled grid), <P, AP>.
//                    A CTA stages Q full columns in shared memory as one
//                    16/32-byte record per row (swizzled halves, so random
//                    record reads spread over all bank groups).  L_r is read
//                    in a warp-interleaved ELL layout: one coalesced load per
//                    warp per entry slot, reused for Q columns.
// U = mul_rn(gc, x1) rounds exactly like apply_elem, so the split result is
// bit-identical to cg_apply_k in fp64 (same per-entry order).
template <typename T>
__global__ void pack_ent_k(i64 nnz, const int* __restrict__ ci, const T* __restrict__ v, OffEnt<T>* __restrict__ out) {
  const i64 k = blockIdx.x * (i64)blockDim.x + threadIdx.x;
  if (k < nnz) {
    OffEnt<T> e;
    e.v = v[k];
    e.off = ci[k];
    out[k] = e;
  }
}

// Row permutation of the band path (rows sorted by L_r degree, see BandApply).
__global__ void permute_sel_k(i64 p, const int* __restrict__ pos, const int* __restrict__ sel, int* __restrict__ out) {
  const i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x;
  if (i < p) out[pos[i]] = sel[i];
}

template <typename T>
__global__ void unpermute_rows_k(i64 p, i64 n, const int* __restrict__ pos, const T* __restrict__ src,
                                 T* __restrict__ dst) {
  const i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x;
  if (i >= p) return;
  const i64 s = pos[i];
  for (i64 c = blockIdx.y; c < n; c += gridDim.y) dst[i + c * p] = src[s + c * p];
}

template <typename T>
__device__ __forceinline__ void store_stream(T* p, T v) {
  __stcs(p, v);
}

// Warp per column, lane = row; the column's entries are read per step
// (warp-uniform loads, 4 steps in flight).  Shuffle-broadcast and
// next-column-prefetch variants measured slower (lower occupancy).
template <typename T, int RPL>
__device__ __forceinline__ void band_column_simple(const OffEnt<T>* __restrict__ ent, i64 k0, i64 k1,
                                                   const T* __restrict__ P, i64 p, i64 r0, const bool (&ok)[RPL],
                                                   T (&acc)[RPL]) {
#pragma unroll 4
  for (i64 k = k0; k < k1; ++k) {
    const OffEnt<T> e = ent[k];
    const T* col = P + static_cast<i64>(e.off) * p + r0;
#pragma unroll
    for (int t = 0; t < RPL; ++t)
      if (ok[t]) acc[t] = madd_entry(acc[t], e.v, col[32 * t]);
  }
}

// U is stored evict-first so it does not push the band out of L2.
template <typename T, int RPL>
__global__ void __launch_bounds__(256, 8)
    cg_apply_band_k(i64 p, i64 c_lo, i64 c_hi, const i64* __restrict__ rp, const OffEnt<T>* __restrict__ ent, T gc,
                    i64 cols_per_cta, const T* __restrict__ P, T* __restrict__ U, const CgState* st, int force) {
  if (!force && st->done) return;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const i64 r0 = static_cast<i64>(blockIdx.y) * (32 * RPL) + lane;
  const i64 cb = c_lo + static_cast<i64>(blockIdx.x) * cols_per_cta;
  const i64 ce = min(c_hi, cb + cols_per_cta);
  bool ok[RPL];
#pragma unroll
  for (int t = 0; t < RPL; ++t) ok[t] = r0 + 32 * t < p;
  // Row pointers of this warp's columns (lane m holds column cb + warp + m*nw).
  const i64 cm = cb + warp + static_cast<i64>(lane) * nw;
  const i64 my_k0 = cm < ce ? rp[cm] : 0, my_k1 = cm < ce ? rp[cm + 1] : 0;
  for (int m = 0;; ++m) {
    const i64 c = cb + warp + static_cast<i64>(m) * nw;
    if (c >= ce) break;
    const i64 k0 = __shfl_sync(0xffffffffu, my_k0, m & 31), k1 = __shfl_sync(0xffffffffu, my_k1, m & 31);
    T acc[RPL];
#pragma unroll
    for (int t = 0; t < RPL; ++t) acc[t] = T(0);
    band_column_simple<T, RPL>(ent, k0, k1, P, p, r0, ok, acc);
    T* out = U + c * p + r0;
#pragma unroll
    for (int t = 0; t < RPL; ++t)
      if (ok[t]) __stcs(out + 32 * t, mul_rn(gc, acc[t]));
  }
}

template <int H>
__device__ __forceinline__ int rec_chunk(int j, int h) {
  if constexpr (H == 2)
    return 2 * j + (h ^ ((j >> 2) & 1));
  else
    return j;
}

// The L_r sweep works on "virtual rows": a stored row, or (fp32 only) a
// chunk of at most `split_cap` entries of a long row, so one hub row (degree
// 495 in the cfg3 row graph) cannot hold the whole CTA on its sequential
// chain.  32 virtual rows form an ELL group (lane = virtual row); groups are
// dealt to warps round-robin in descending cost, a fixed assignment, so the
// per-thread dot partials and hence <P, AP> are deterministic.  A chunk
// writes its partial sums to shared memory; after the sweep warp 0 adds the
// chunks of each split row in chunk order and finishes those rows.
struct ColMeta {
  const int* vrow;    // stored row of each virtual row (-1 = padding lane)
  const int* vdeg;    // entries of each virtual row
  const int* vslot;   // partial-sum slot, -1 = unsplit row (written directly)
  const int* base;    // ELL slot base per group
  const int* order;   // groups in descending cost
  const int* split_row, *split_first, *split_n;
  int groups, nsplit, nslots;
  unsigned long long* prof;  // diagnostics (CPCAG_BAND_PROF): per-CTA phase times, else null
};


template <typename T, int RB, int NT>
__global__ void __launch_bounds__(NT, 1024 / NT) cg_apply_col_k(int p, i64 c_lo, i64 c_hi, ColMeta cm,
                                                                 const OffEnt<T>* __restrict__ ell, T gr, Plan pl,
                                                                 const T* __restrict__ P, T* __restrict__ AP,
                                                                 double* partials, CgState* st, int force) {
  if (!force && st->done) return;
  constexpr int Q = RB / static_cast<int>(sizeof(T));
  constexpr int H = RB / 16;
  constexpr int KB = 4;
  union Rec {
    uint4 u[H];
    T v[Q];
  };
  extern __shared__ __align__(16) unsigned char smraw[];
  uint4* S = reinterpret_cast<uint4*>(smraw);
  T* part_sm = reinterpret_cast<T*>(smraw + static_cast<size_t>(p) * RB);
  // per-group and per-split-row dot partials (summed in index order: the
  // result does not depend on which warp took which group)
  double* dot_sm = reinterpret_cast<double*>(smraw + static_cast<size_t>(p) * RB + static_cast<size_t>(cm.nslots) * RB);
  __shared__ int next_item;
  __shared__ unsigned long long pt[4];
  const i64 c0 = c_lo + static_cast<i64>(blockIdx.x) * Q;
  const int qn = static_cast<int>(min(static_cast<i64>(Q), c_hi - c0));
  const bool prof = cm.prof != nullptr && blockIdx.x < 4096;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  if (threadIdx.x == 0) {
    next_item = nw;
    if (prof) {
      pt[0] = gtimer();
      pt[2] = ~0ull;
      pt[3] = 0;
    }
  }
  for (int j = threadIdx.x; j < p; j += blockDim.x) {
    Rec r;
#pragma unroll
    for (int q = 0; q < Q; ++q) r.v[q] = q < qn ? P[j + (c0 + q) * static_cast<i64>(p)] : T(0);
#pragma unroll
    for (int h = 0; h < H; ++h) S[rec_chunk<H>(j, h)] = r.u[h];
  }
  __syncthreads();
  if (prof && threadIdx.x == 0) pt[1] = gtimer();
  // Finishes stored row i: AP = U + gr x2 (+ P on the sampled grid); returns
  // this row's contribution to <P, AP>.
  auto finish = [&](int i, const T (&acc)[Q]) -> double {
    Rec own;
#pragma unroll
    for (int h = 0; h < H; ++h) own.u[h] = S[rec_chunk<H>(i, h)];
    const bool rs = pl.rsel[i] >= 0;
    double d = 0.0;
#pragma unroll
    for (int q = 0; q < Q; ++q) {
      if (q < qn) {
        const i64 c = c0 + q;
        const i64 at = i + c * p;
        T out = add_rn(__ldcs(AP + at), mul_rn(gr, acc[q]));
        if (rs && pl.csel[c] >= 0) out = add_rn(out, own.v[q]);
        __stcs(AP + at, out);
        d += static_cast<double>(own.v[q]) * static_cast<double>(out);
      }
    }
    return d;
  };
  for (int it = warp; it < cm.groups;) {
    const int g = cm.order[it];
    const int v = g * 32 + lane;
    const int i = cm.vrow[v], d = cm.vdeg[v];
    const OffEnt<T>* e = ell + static_cast<i64>(cm.base[g]) * 32 + lane;
    T acc[Q];
#pragma unroll
    for (int q = 0; q < Q; ++q) acc[q] = T(0);
    for (int k0 = 0; k0 < d; k0 += KB) {
      OffEnt<T> en[KB];
#pragma unroll
      for (int u = 0; u < KB; ++u)
        if (k0 + u < d) en[u] = e[(k0 + u) * 32];
#pragma unroll
      for (int u = 0; u < KB; ++u) {
        if (k0 + u < d) {
          Rec x;
#pragma unroll
          for (int h = 0; h < H; ++h) x.u[h] = S[rec_chunk<H>(en[u].off, h)];
#pragma unroll
          for (int q = 0; q < Q; ++q) acc[q] = madd_entry(acc[q], en[u].v, x.v[q]);
        }
      }
    }
    double dg = 0.0;
    if (i >= 0) {
      const int slot = cm.vslot[v];
      if (slot < 0) {
        dg = finish(i, acc);
      } else {
#pragma unroll
        for (int q = 0; q < Q; ++q) part_sm[slot * Q + q] = acc[q];
      }
    }
    dg = warp_sum(dg);
    if (lane == 0) {
      dot_sm[g] = dg;
      it = atomicAdd(&next_item, 1);
    }
    it = __shfl_sync(0xffffffffu, it, 0);
  }
  if (prof && lane == 0) {
    const unsigned long long t = gtimer();
    atomicMin(&pt[2], t);
    atomicMax(&pt[3], t);
  }
  if (cm.nsplit > 0) {
    __syncthreads();
    for (int t = threadIdx.x; t < cm.nsplit; t += blockDim.x) {
      const int f = cm.split_first[t], nc = cm.split_n[t];
      T acc[Q];
#pragma unroll
      for (int q = 0; q < Q; ++q) {
        T tot = T(0);
        for (int ch = 0; ch < nc; ++ch) tot = add_rn(tot, part_sm[(f + ch) * Q + q]);
        acc[q] = tot;
      }
      dot_sm[cm.groups + t] = finish(cm.split_row[t], acc);
    }
  }
  __syncthreads();
  if (prof && threadIdx.x == 0) {
    unsigned long long* o = cm.prof + static_cast<i64>(blockIdx.x) * 8;
    o[0] = pt[0];
    o[1] = pt[1];
    o[2] = pt[2];
    o[3] = pt[3];
    o[4] = gtimer();
  }
  if (force) return;
  double sv[1] = {0.0}, tot[1];
  for (int t = threadIdx.x; t < cm.groups + cm.nsplit; t += blockDim.x) sv[0] += dot_sm[t];
  if (grid_sum_last<1>(sv, partials, &st->cnt[1], tot) && threadIdx.x == 0) {
    const double curv = tot[0];
    st->curv = curv;
    if (!isfinite(curv) || curv <= 0.0) {
      st->err = 1;
      st->err_it = st->it;
      st->done = 1;
      return;
    }
    st->alpha = st->rho / curv;
  }
}

// ||b - AX||^2 with AX already applied (band path of the exit test).
template <typename T>
__global__ void cg_true_res_ap_k(i64 p, i64 n, Plan pl, const T* __restrict__ Xt, const T* __restrict__ AX,
                                 double* partials, CgState* st) {
  double s[1] = {0.0};
  const i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x;
  if (i < p) {
    for (i64 c = blockIdx.y; c < n; c += gridDim.y) {
      const double e = static_cast<double>(sub_rn(rhs_at(pl, Xt, i, c), AX[i + c * p]));
      s[0] += e * e;
    }
  }
  double tot[1];
  if (grid_sum_last<1>(s, partials, &st->cnt[0], tot) && threadIdx.x == 0)
    st->rel_res = sqrt(tot[0]) / st->norm_b;
}

// Host side of the band apply: packed L_c entries, the L_r ELL layout and the
// launch geometry, built once per solve (or per decoder block).
template <typename T>
struct BandApply {
  static constexpr i64 kBandBytes = i64{128} << 20;  // band budget (measured: taller bands win even past L2)
  static constexpr int kColsPerCta = 64;
  i64 p = 0, n = 0;
  int rpl = 1, rb = 32, col_nt = 1024;
  size_t col_smem = 0;

  template <typename F>
  void with_col_kernel(F&& f) const {
    if (rb == 32 && col_nt == 1024) f(cg_apply_col_k<T, 32, 1024>);
    else if (rb == 32) f(cg_apply_col_k<T, 32, 512>);
    else if (col_nt == 1024) f(cg_apply_col_k<T, 16, 1024>);
    else f(cg_apply_col_k<T, 16, 512>);
  }
  template <int RPL>
  void launch_band_v(Ctx* c, dim3 gb, const T* P, T* AP, i64 c_lo, i64 c_hi, T gc, const CgState* st,
                     int force) const {
    cg_apply_band_k<T, RPL><<<gb, 256, 0, c->stream>>>(p, c_lo, c_hi, rpc, ent.p, gc, kColsPerCta, P, AP, st, force);
  }
  DevBuf<OffEnt<T>> ent, ell;
  DevBuf<int> base, order, pos, vrow, vdeg, vslot, split_row, split_first, split_n;
  ColMeta meta{};
  DevBuf<unsigned long long> prof_buf;
  bool permuted = false;

  // CPCAG_BAND_PROF: phase times of the first 4096 column-group CTAs of the
  // last apply (staging, first/last warp done, CTA end), printed to stderr.
  void report_prof(Ctx* c) const {
    if (!meta.prof) return;
    std::vector<unsigned long long> h(4096 * 8);
    CUDA_OK(cudaMemcpy(h.data(), prof_buf.p, sizeof(unsigned long long) * h.size(), cudaMemcpyDeviceToHost));
    double a = 0, b = 0, d = 0, e = 0, cnt = 0;
    unsigned long long t_min = ~0ull, t_max = 0;
    for (int k = 0; k < 4096; ++k) {
      const unsigned long long* o = h.data() + k * 8;
      if (!o[0] || !o[4]) continue;
      a += o[1] - o[0];
      b += o[2] - o[1];
      d += o[3] - o[1];
      e += o[4] - o[0];
      cnt += 1;
      t_min = std::min(t_min, o[0]);
      t_max = std::max(t_max, o[4]);
    }
    if (cnt > 0)
      std::fprintf(stderr, "[band prof] ctas %.0f  stage %.2f us  first-warp %.2f us  last-warp %.2f us  cta %.2f us  "
                   "span %.1f us\n", cnt, a / cnt / 1e3, b / cnt / 1e3, d / cnt / 1e3, e / cnt / 1e3,
                   static_cast<double>(t_max - t_min) / 1e3);
  }
  const i64* rpc = nullptr;

  // Feasible when a Q-column group of P fits in shared memory.
  static bool feasible(i64 p) { return p > 0 && p * 16 <= 200 * 1024 && p < (i64{1} << 31); }
  // Auto choice: the iterate does not fit in L2.
  static bool preferred(i64 p, i64 n) { return static_cast<double>(p) * n * sizeof(T) > 96e6 && feasible(p); }

  // permute: store rows in descending-degree order (pos[row] = stored row),
  // so the 32-row ELL groups are nearly uniform: kNN graphs in high dimension
  // have hubs (cfg3 row graph: mean degree 18, max 495), and natural-order
  // groups pad to ~5x the entries.  Each row keeps its CSR entry order (only
  // the column labels are mapped), so per-entry arithmetic is unchanged.
  void build(Ctx* c, Csr* Lr, Csr* Lc, const std::vector<i64>& rpr, bool permute) {
    p = Lr->rows;
    n = Lc->rows;
    if (!feasible(p)) invalid("band apply: row count too large for the column-group kernel");
    rb = p * 32 <= 200 * 1024 ? 32 : 16;
    if (const char* e = std::getenv("CPCAG_BAND_RB")) rb = std::atoi(e) == 16 ? 16 : rb;
    col_smem = static_cast<size_t>(p) * rb;
    rpl = 1;
    for (int r : {4, 2}) {
      if (32 * r * n * static_cast<i64>(sizeof(T)) <= kBandBytes && 32 * r <= ((p + 31) / 32) * 32) {
        rpl = r;
        break;
      }
    }
    if (const char* e = std::getenv("CPCAG_BAND_RPL")) {
      const int r = std::atoi(e);
      if (r == 1 || r == 2 || r == 4 || r == 8) rpl = r;
    }
    const Pull<T> pc = make_pull<T>(c, Lc, true), pr = make_pull<T>(c, Lr, false);
    rpc = pc.rp;
    const i64 nnz_c = Lc->nnz;
    ent.alloc(c, std::max<i64>(nnz_c, 1));
    if (nnz_c) {
      pack_ent_k<T><<<blocks_for(nnz_c), kBlock, 0, c->stream>>>(nnz_c, pc.ci, pc.v, ent.p);
      launched(c);
    }
    const i64 nnz_r = rpr[p];
    std::vector<int> hci(static_cast<size_t>(nnz_r));
    std::vector<T> hv(static_cast<size_t>(nnz_r));
    if (nnz_r) {
      CUDA_OK(cudaMemcpyAsync(hci.data(), pr.ci, sizeof(int) * nnz_r, cudaMemcpyDeviceToHost, c->stream));
      CUDA_OK(cudaMemcpyAsync(hv.data(), pr.v, sizeof(T) * nnz_r, cudaMemcpyDeviceToHost, c->stream));
    }
    sync(c);
    std::vector<int> ord(static_cast<size_t>(p)), hpos(static_cast<size_t>(p));
    for (i64 i = 0; i < p; ++i) ord[i] = static_cast<int>(i);
    permuted = permute;
    if (permute)
      std::stable_sort(ord.begin(), ord.end(),
                       [&](int a, int b) { return rpr[a + 1] - rpr[a] > rpr[b + 1] - rpr[b]; });
    for (i64 r = 0; r < p; ++r) hpos[ord[r]] = static_cast<int>(r);
    // Virtual rows: fp64 keeps whole rows (bit-exact per-entry order); fp32
    // cuts rows longer than split_cap into chunks (their partial sums are
    // added in chunk order, a different rounding within the fp32 tolerance).
    i64 cap = sizeof(T) == 4 ? 64 : (i64{1} << 40);
    if (const char* e = std::getenv("CPCAG_BAND_SPLIT")) cap = std::max<i64>(8, std::atoll(e));
    if (sizeof(T) == 8) cap = i64{1} << 40;
    struct VRow {
      int row;
      i64 k0, len;
      int slot;
    };
    std::vector<VRow> vr;
    std::vector<int> srow, sfirst, sn;
    int nslots = 0;
    vr.reserve(static_cast<size_t>(p));
    for (i64 r = 0; r < p; ++r) {  // chunks of split rows first (longest first)
      const i64 d = rpr[ord[r] + 1] - rpr[ord[r]];
      if (d <= cap) continue;
      srow.push_back(static_cast<int>(r));
      sfirst.push_back(nslots);
      sn.push_back(static_cast<int>((d + cap - 1) / cap));
      for (i64 k = 0; k < d; k += cap) vr.push_back({static_cast<int>(r), k, std::min(cap, d - k), nslots++});
    }
    std::stable_sort(vr.begin(), vr.end(), [](const VRow& a, const VRow& b) { return a.len > b.len; });
    for (i64 r = 0; r < p; ++r) {  // then whole rows in stored (descending-degree) order
      const i64 d = rpr[ord[r] + 1] - rpr[ord[r]];
      if (d <= cap) vr.push_back({static_cast<int>(r), 0, d, -1});
    }
    const i64 nv = static_cast<i64>(vr.size());
    const i64 groups = (nv + 31) / 32;
    std::vector<int> hb(static_cast<size_t>(groups)), hmd(static_cast<size_t>(groups)), ho(static_cast<size_t>(groups));
    std::vector<int> hvrow(static_cast<size_t>(groups * 32), -1), hvdeg(static_cast<size_t>(groups * 32), 0),
        hvslot(static_cast<size_t>(groups * 32), -1);
    i64 slots = 0;
    for (i64 g = 0; g < groups; ++g) {
      i64 md = 0;
      for (i64 v = g * 32; v < std::min<i64>(nv, g * 32 + 32); ++v) {
        hvrow[v] = vr[v].row;
        hvdeg[v] = static_cast<int>(vr[v].len);
        hvslot[v] = vr[v].slot;
        md = std::max(md, vr[v].len);
      }
      hb[g] = static_cast<int>(slots);
      hmd[g] = static_cast<int>(md);
      slots += md;
    }
    if (slots * 32 >= (i64{1} << 31)) invalid("band apply: L_r too dense for the ELL layout");
    for (i64 g = 0; g < groups; ++g) ho[g] = static_cast<int>(g);
    std::stable_sort(ho.begin(), ho.end(), [&](int a, int b) { return hmd[a] > hmd[b]; });
    std::vector<OffEnt<T>> hell(static_cast<size_t>(std::max<i64>(slots * 32, 1)));
    for (auto& e : hell) {
      e.v = T(0);
      e.off = 0;
    }
    for (i64 v = 0; v < nv; ++v) {
      const i64 old = ord[vr[v].row], k0 = rpr[old] + vr[v].k0;
      OffEnt<T>* dst = hell.data() + static_cast<i64>(hb[v >> 5]) * 32 + (v & 31);
      for (i64 k = 0; k < vr[v].len; ++k) {
        dst[k * 32].v = hv[k0 + k];
        dst[k * 32].off = hpos[hci[k0 + k]];
      }
    }
    const i64 ns = static_cast<i64>(srow.size());
    auto up = [&](DevBuf<int>& d, const std::vector<int>& h) {
      d.alloc(c, std::max<size_t>(h.size(), 1));
      if (!h.empty())
        CUDA_OK(cudaMemcpyAsync(d.p, h.data(), sizeof(int) * h.size(), cudaMemcpyHostToDevice, c->stream));
    };
    up(base, hb);
    up(order, ho);
    up(vrow, hvrow);
    up(vdeg, hvdeg);
    up(vslot, hvslot);
    up(split_row, srow);
    up(split_first, sfirst);
    up(split_n, sn);
    up(pos, hpos);
    ell.alloc(c, hell.size());
    CUDA_OK(cudaMemcpyAsync(ell.p, hell.data(), sizeof(OffEnt<T>) * hell.size(), cudaMemcpyHostToDevice, c->stream));
    meta = ColMeta{vrow.p, vdeg.p, vslot.p, base.p, order.p, split_row.p, split_first.p, split_n.p,
                   static_cast<int>(groups), static_cast<int>(ns), nslots, nullptr};
    if (std::getenv("CPCAG_BAND_PROF")) {
      prof_buf.alloc(c, 4096 * 8);
      prof_buf.zero(c);
      meta.prof = prof_buf.p;
    }
    col_smem = static_cast<size_t>(p) * rb + static_cast<size_t>(nslots) * rb +
               sizeof(double) * static_cast<size_t>(groups + ns);
    if (col_smem > 220 * 1024) invalid("band apply: column group and split partials exceed shared memory");
    if (const char* e = std::getenv("CPCAG_BAND_NT")) col_nt = std::atoi(e) == 512 ? 512 : 1024;
    with_col_kernel([&](auto kern) { ensure_smem(kern, col_smem); });
    sync(c);  // hb must outlive the copy
  }

  unsigned col_blocks(i64 c_lo, i64 c_hi) const {
    const i64 q = rb / static_cast<i64>(sizeof(T));
    return static_cast<unsigned>(std::max<i64>(1, (c_hi - c_lo + q - 1) / q));
  }

  // AP[:, c_lo:c_hi] (AP indexed by global column) = A(P) on those columns;
  // P holds every column.  force = 1 ignores the CG done flag and skips the
  // <P, AP> reduction (true-residual apply).
  void apply(Ctx* c, const T* P, T* AP, i64 c_lo, i64 c_hi, const Plan& pl, T gr, T gc, double* part, CgState* st,
             int force) const {
    if (c_hi <= c_lo) return;
    const i64 band_rows = 32 * rpl;
    const dim3 gb(static_cast<unsigned>((c_hi - c_lo + kColsPerCta - 1) / kColsPerCta),
                  static_cast<unsigned>((p + band_rows - 1) / band_rows));
    {
    KScope ks_(c, "cg_apply_band");
    if (rpl == 8) launch_band_v<8>(c, gb, P, AP, c_lo, c_hi, gc, st, force);
    else if (rpl == 4) launch_band_v<4>(c, gb, P, AP, c_lo, c_hi, gc, st, force);
    else if (rpl == 2) launch_band_v<2>(c, gb, P, AP, c_lo, c_hi, gc, st, force);
    else launch_band_v<1>(c, gb, P, AP, c_lo, c_hi, gc, st, force);
    launched(c);
    }
    KScope ks_(c, "cg_apply_col");
    const unsigned gcb = col_blocks(c_lo, c_hi);
    with_col_kernel([&](auto kern) {
      kern<<<gcb, col_nt, col_smem, c->stream>>>(static_cast<int>(p), c_lo, c_hi, meta, ell.p, gr, pl, P, AP, part,
                                                st, force);
    });
    launched(c);
  }
};

// ------------------------------------------------------------------ tile apply (banded column graph)
// When the column graph has a small bandwidth after reverse Cuthill-McKee
// ordering (config 1: max 69, median 12 over 1 000 columns), the iterates are
// stored with columns in RCM order and each CTA (64 rows x 64 columns)
// stages the window P[rows, c0 - h : c0 + 64 + h] in shared memory once; the
// ~19 L_c gathers of every output then read shared memory instead of L2.
// L_r (the pixel grid at config 1) gathers along the same column from L1.
// Each L_c row keeps its CSR entry order (only the column labels are mapped),
// so the per-entry arithmetic -- and fp64 bit-exactness -- is unchanged.
__global__ void unpermute_cols_k(i64 p, i64 n, const int* __restrict__ pos, const float* __restrict__ src32,
                                 float* __restrict__ dst32, const double* __restrict__ src64,
                                 double* __restrict__ dst64) {
  const i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x;
  if (i >= p) return;
  for (i64 c = blockIdx.y; c < n; c += gridDim.y) {
    const i64 s = pos[c];
    if (src32) dst32[i + c * p] = src32[i + s * p];
    else dst64[i + c * p] = src64[i + s * p];
  }
}

template <typename T>
__global__ void __launch_bounds__(256) cg_apply_tile_k(int p, int n, Pull<T> Lr, const i64* __restrict__ crp,
                                                       const OffEnt<T>* __restrict__ cent, const int* __restrict__ wlo,
                                                       const int* __restrict__ whi, T gr, T gc, Plan pl,
                                                       const T* __restrict__ P, T* __restrict__ AP,
                                                       double* partials, CgState* st, int force) {
  if (!force && st->done) return;
  constexpr int kR = 64;
  extern __shared__ __align__(16) unsigned char smraw[];
  const int i0 = blockIdx.x * kR;
  const int c0 = blockIdx.y * 64, c1 = min(n, c0 + 64);
  const int w0 = wlo[blockIdx.y], w1 = whi[blockIdx.y];
  const int rows = min(kR, p - i0);
  // shared: window P[rows][w0:w1) | L_c entries (offset pre-scaled) | L_r entries | chunk row ptrs
  T* Pw = reinterpret_cast<T*>(smraw);
  const i64 kc_base = crp[c0];
  const int ec = static_cast<int>(crp[c1] - kc_base);
  const i64 kr_base = Lr.rp[i0];
  const int er = static_cast<int>(Lr.rp[i0 + rows] - kr_base);
  OffEnt<T>* Ec = reinterpret_cast<OffEnt<T>*>(smraw + static_cast<size_t>(w1 - w0) * kR * sizeof(T));
  OffEnt<T>* Er = Ec + ec;
  int* cr = reinterpret_cast<int*>(Er + er);  // 65 entries
  for (int idx = threadIdx.x; idx < (w1 - w0) * kR; idx += blockDim.x) {
    const int j = idx / kR, rr = idx % kR;
    Pw[idx] = rr < rows ? P[static_cast<i64>(i0 + rr) + static_cast<i64>(w0 + j) * p] : T(0);
  }
  for (int k = threadIdx.x; k < ec; k += blockDim.x) {
    OffEnt<T> e = cent[kc_base + k];
    e.off = (e.off - w0) * kR;
    Ec[k] = e;
  }
  for (int k = threadIdx.x; k < er; k += blockDim.x) {
    OffEnt<T> e;
    e.v = Lr.v[kr_base + k];
    e.off = Lr.ci[kr_base + k];
    Er[k] = e;
  }
  for (int q = threadIdx.x; q <= c1 - c0; q += blockDim.x) cr[q] = static_cast<int>(crp[c0 + q] - kc_base);
  __syncthreads();
  const int r = threadIdx.x & (kR - 1), cgp = threadIdx.x / kR, ngp = blockDim.x / kR;
  const int i = i0 + r;
  double s = 0.0;
  if (r < rows) {
    const int a0 = static_cast<int>(Lr.rp[i] - kr_base), a1 = static_cast<int>(Lr.rp[i + 1] - kr_base);
    const bool rs = pl.rsel[i] >= 0;
    for (int c = c0 + cgp; c < c1; c += ngp) {
      T x1 = T(0);
      const int b0 = cr[c - c0], b1 = cr[c - c0 + 1];
#pragma unroll 4
      for (int k = b0; k < b1; ++k) {
        const OffEnt<T> e = Ec[k];
        x1 = madd_entry(x1, e.v, Pw[e.off + r]);
      }
      const T* pc = P + static_cast<i64>(c) * p;
      T x2 = T(0);
#pragma unroll 4
      for (int k = a0; k < a1; ++k) {
        const OffEnt<T> e = Er[k];
        x2 = madd_entry(x2, e.v, pc[e.off]);
      }
      T out = add_rn(mul_rn(gc, x1), mul_rn(gr, x2));
      const T pv = Pw[(c - w0) * kR + r];
      if (rs && pl.csel[c] >= 0) out = add_rn(out, pv);
      AP[i + static_cast<i64>(c) * p] = out;
      s += static_cast<double>(pv) * static_cast<double>(out);
    }
  }
  if (force) return;
  double sv[1] = {s}, tot[1];
  if (grid_sum_last<1>(sv, partials, &st->cnt[1], tot) && threadIdx.x == 0) {
    const double curv = tot[0];
    st->curv = curv;
    if (!isfinite(curv) || curv <= 0.0) {
      st->err = 1;
      st->err_it = st->it;
      st->done = 1;
      return;
    }
    st->alpha = st->rho / curv;
  }
}

template <typename T>
struct TileApply {
  static constexpr int kR = 64, kC = 64;
  i64 p = 0, n = 0;
  int bandwidth = 0, wmax = 0;
  size_t smem = 0;
  DevBuf<int> pos, wlo, whi;
  DevBuf<i64> crp;
  DevBuf<OffEnt<T>> cent;

  // Reverse Cuthill-McKee of the symmetric pattern (per component: start at
  // a minimum-degree node, BFS visiting neighbours by ascending degree).
  static std::vector<int> rcm(i64 n, const std::vector<i64>& rp, const std::vector<int>& ci) {
    std::vector<int> order, deg(static_cast<size_t>(n));
    order.reserve(static_cast<size_t>(n));
    for (i64 u = 0; u < n; ++u) deg[u] = static_cast<int>(rp[u + 1] - rp[u]);
    std::vector<char> seen(static_cast<size_t>(n), 0);
    std::vector<int> byd(static_cast<size_t>(n));
    for (i64 u = 0; u < n; ++u) byd[u] = static_cast<int>(u);
    std::stable_sort(byd.begin(), byd.end(), [&](int a, int b) { return deg[a] < deg[b]; });
    std::vector<int> nb;
    for (int start : byd) {
      if (seen[start]) continue;
      size_t head = order.size();
      order.push_back(start);
      seen[start] = 1;
      while (head < order.size()) {
        const int u = order[head++];
        nb.clear();
        for (i64 k = rp[u]; k < rp[u + 1]; ++k)
          if (!seen[ci[k]]) {
            seen[ci[k]] = 1;
            nb.push_back(ci[k]);
          }
        std::stable_sort(nb.begin(), nb.end(), [&](int a, int b) { return deg[a] < deg[b]; });
        order.insert(order.end(), nb.begin(), nb.end());
      }
    }
    std::reverse(order.begin(), order.end());
    return order;  // stored position -> original column
  }

  // Returns false (and builds nothing) when the column graph is not banded
  // enough for the shared-memory window.
  // windows = false (rcm2): only the RCM order and the permuted L_c as a
  // CSR pull (pci / pv), for the fast2 kernel on column-permuted iterates.
  DevBuf<int> pci;
  DevBuf<T> pv;
  std::vector<i64> hrp_host;
  bool build(Ctx* c, Csr* Lc, const std::vector<i64>& rpc, const std::vector<i64>& rpr_, i64 p_, int cap,
             bool windows = true) {
    p = p_;
    n = Lc->rows;
    if (n > INT32_MAX || p > INT32_MAX) return false;
    const Pull<T> pc = make_pull<T>(c, Lc, true);
    const i64 nnz = rpc[n];
    std::vector<int> hci(static_cast<size_t>(nnz));
    std::vector<T> hv(static_cast<size_t>(nnz));
    if (nnz) {
      CUDA_OK(cudaMemcpyAsync(hci.data(), pc.ci, sizeof(int) * nnz, cudaMemcpyDeviceToHost, c->stream));
      CUDA_OK(cudaMemcpyAsync(hv.data(), pc.v, sizeof(T) * nnz, cudaMemcpyDeviceToHost, c->stream));
    }
    sync(c);
    const std::vector<int> ord = rcm(n, rpc, hci);
    std::vector<int> hpos(static_cast<size_t>(n));
    for (i64 k = 0; k < n; ++k) hpos[ord[k]] = static_cast<int>(k);
    bandwidth = 0;
    for (i64 u = 0; u < n; ++u)
      for (i64 k = rpc[u]; k < rpc[u + 1]; ++k) bandwidth = std::max(bandwidth, std::abs(hpos[u] - hpos[hci[k]]));
    if (bandwidth > cap) return false;
    // permuted rows (stored column order), entry order kept, labels mapped
    std::vector<i64> hrp(static_cast<size_t>(n) + 1, 0);
    std::vector<OffEnt<T>> hent(static_cast<size_t>(std::max<i64>(nnz, 1)));
    for (i64 st_ = 0; st_ < n; ++st_) {
      const i64 u = ord[st_];
      i64 o = hrp[st_];
      for (i64 k = rpc[u]; k < rpc[u + 1]; ++k, ++o) {
        hent[o].v = hv[k];
        hent[o].off = hpos[hci[k]];
      }
      hrp[st_ + 1] = o;
    }
    if (!windows) {
      std::vector<int> ci2(hent.size());
      std::vector<T> v2(hent.size());
      for (size_t k = 0; k < hent.size(); ++k) {
        ci2[k] = hent[k].off;
        v2[k] = hent[k].v;
      }
      pos.alloc(c, n);
      crp.alloc(c, n + 1);
      pci.alloc(c, ci2.size());
      pv.alloc(c, v2.size());
      CUDA_OK(cudaMemcpyAsync(pos.p, hpos.data(), sizeof(int) * n, cudaMemcpyHostToDevice, c->stream));
      CUDA_OK(cudaMemcpyAsync(crp.p, hrp.data(), sizeof(i64) * (n + 1), cudaMemcpyHostToDevice, c->stream));
      CUDA_OK(cudaMemcpyAsync(pci.p, ci2.data(), sizeof(int) * ci2.size(), cudaMemcpyHostToDevice, c->stream));
      CUDA_OK(cudaMemcpyAsync(pv.p, v2.data(), sizeof(T) * v2.size(), cudaMemcpyHostToDevice, c->stream));
      hrp_host = hrp;
      sync(c);
      return true;
    }
    const i64 chunks = (n + kC - 1) / kC;
    std::vector<int> lo(static_cast<size_t>(chunks)), hi(static_cast<size_t>(chunks));
    wmax = 0;
    for (i64 b = 0; b < chunks; ++b) {
      const i64 a = b * kC, e = std::min<i64>(n, a + kC);
      int l = static_cast<int>(a), h = static_cast<int>(e);
      for (i64 st_ = a; st_ < e; ++st_)
        for (i64 k = hrp[st_]; k < hrp[st_ + 1]; ++k) {
          l = std::min(l, hent[k].off);
          h = std::max(h, hent[k].off + 1);
        }
      lo[b] = l;
      hi[b] = h;
      wmax = std::max(wmax, h - l);
    }
    i64 mec = 0, mer = 0;
    for (i64 b = 0; b < chunks; ++b) mec = std::max(mec, hrp[std::min<i64>(n, b * kC + kC)] - hrp[b * kC]);
    for (i64 a = 0; a < p; a += kR) mer = std::max(mer, rpr_[std::min<i64>(p, a + kR)] - rpr_[a]);
    smem = static_cast<size_t>(wmax) * kR * sizeof(T) + static_cast<size_t>(mec + mer) * sizeof(OffEnt<T>) +
           sizeof(int) * (kC + 1) + 16;
    if (smem > 96 * 1024) return false;
    pos.alloc(c, n);
    wlo.alloc(c, chunks);
    whi.alloc(c, chunks);
    crp.alloc(c, n + 1);
    cent.alloc(c, hent.size());
    CUDA_OK(cudaMemcpyAsync(pos.p, hpos.data(), sizeof(int) * n, cudaMemcpyHostToDevice, c->stream));
    CUDA_OK(cudaMemcpyAsync(wlo.p, lo.data(), sizeof(int) * chunks, cudaMemcpyHostToDevice, c->stream));
    CUDA_OK(cudaMemcpyAsync(whi.p, hi.data(), sizeof(int) * chunks, cudaMemcpyHostToDevice, c->stream));
    CUDA_OK(cudaMemcpyAsync(crp.p, hrp.data(), sizeof(i64) * (n + 1), cudaMemcpyHostToDevice, c->stream));
    CUDA_OK(cudaMemcpyAsync(cent.p, hent.data(), sizeof(OffEnt<T>) * hent.size(), cudaMemcpyHostToDevice, c->stream));
    ensure_smem(cg_apply_tile_k<T>, smem);
    sync(c);
    return true;
  }

  dim3 grid() const {
    return dim3(static_cast<unsigned>((p + kR - 1) / kR), static_cast<unsigned>((n + kC - 1) / kC));
  }

  void apply(Ctx* c, const Pull<T>& pr, const T* P, T* AP, const Plan& pl, T gr, T gc, double* part, CgState* st,
             int force) const {
    cg_apply_tile_k<T><<<grid(), 256, smem, c->stream>>>(static_cast<int>(p), static_cast<int>(n), pr, crp.p, cent.p,
                                                        wlo.p, whi.p, gr, gc, pl, P, AP, part, st, force);
    launched(c);
  }
};

template <typename T>
void alternate_decode_device(Ctx* c, const T* Xt, i64 rho_r, i64 rho_c, const i64* om_r_host,
                             const i64* om_c_host, i64 p, i64 n, Csr* Lr, Csr* Lc, double lk1_r,
                             double lk1_c, const cpcag_decoder_config& cfg, T* X, int* converged,
                             i64* iterations) {
  if (Lr->rows != p || Lc->rows != n || Lr->cols != p || Lc->cols != n)
    invalid("alternate decoder: Laplacians do not match plan");
  if (cfg.gamma <= 0.0) invalid("alternate decoder: gamma must be positive");
  {
    std::vector<char> seen_r(static_cast<size_t>(p), 0), seen_c(static_cast<size_t>(n), 0);
    for (i64 k = 0; k < rho_r; ++k) {
      const i64 r = om_r_host[k];
      if (r < 0 || r >= p || seen_r[r]) invalid("alternate decoder: Xt does not match plan");
      seen_r[r] = 1;
    }
    for (i64 k = 0; k < rho_c; ++k) {
      const i64 q = om_c_host[k];
      if (q < 0 || q >= n || seen_c[q]) invalid("alternate decoder: Xt does not match plan");
      seen_c[q] = 1;
    }
  }
  const double gbar_r = cfg.gamma / lk1_r;
  const double gbar_c = cfg.gamma / lk1_c;
  const i64 N = p * n;

  DevBuf<i64> omr(c, rho_r), omc(c, rho_c);
  if (rho_r) CUDA_OK(cudaMemcpyAsync(omr.p, om_r_host, sizeof(i64) * rho_r, cudaMemcpyHostToDevice, c->stream));
  if (rho_c) CUDA_OK(cudaMemcpyAsync(omc.p, om_c_host, sizeof(i64) * rho_c, cudaMemcpyHostToDevice, c->stream));
  DevBuf<int> rsel(c, p), csel(c, n);
  if (p) {
    fill_sel_k<<<blocks_for(p), kBlock, 0, c->stream>>>(p, rsel.p);
    launched(c);
  }
  if (n) {
    fill_sel_k<<<blocks_for(n), kBlock, 0, c->stream>>>(n, csel.p);
    launched(c);
  }
  if (rho_r) {
    scatter_sel_k<<<blocks_for(rho_r), kBlock, 0, c->stream>>>(omr.p, rho_r, rsel.p);
    launched(c);
  }
  if (rho_c) {
    scatter_sel_k<<<blocks_for(rho_c), kBlock, 0, c->stream>>>(omc.p, rho_c, csel.p);
    launched(c);
  }
  Plan pl{rsel.p, csel.p, rho_r};
  const Pull<T> pr = make_pull<T>(c, Lr, false), pc = make_pull<T>(c, Lc, true);
  const T gr = static_cast<T>(gbar_r), gc = static_cast<T>(gbar_c);

  DevBuf<T> R(c, N), P(c, N), AP(c, N);
  DevBuf<CgState> st(c, 1);
  st.zero(c);
  if (N == 0) {
    *converged = 1;
    *iterations = 0;
    return;
  }
  const unsigned gx = blocks_for(p);
  const i64 ycap = std::max<i64>(1, (static_cast<i64>(c->num_sms) * 16) / gx);
  dim3 g2(gx, static_cast<unsigned>(std::max<i64>(1, std::min<i64>({n, ycap, 65535}))));
  const unsigned nb1 = stride_blocks(c, N);
  // 16-byte vector residual/update when every iterate is 16-byte aligned
  // (X is the caller's buffer); CPCAG_CG_VEC=0 forces the scalar kernels.
  const bool vec_ok = (reinterpret_cast<uintptr_t>(X) % 16 == 0) && !(std::getenv("CPCAG_CG_VEC") &&
                                                                        std::string(std::getenv("CPCAG_CG_VEC")) == "0");
  const unsigned nb1v = stride_blocks(c, (N + Vec16<T>::W - 1) / Vec16<T>::W);
  DevBuf<double> part(c, std::max<size_t>(g2.x * g2.y, nb1));

  // Apply variant (CPCAG_APPLY overrides): fast2 | fast | fast3 | fast4 | slab | rcm2 | staged |
  // plain for L2-sized iterates, band for iterates larger than L2.
  // fast2 by default for L2-sized iterates; fast3 (RCM column windows in
  // shared memory, CPCAG_APPLY=fast3) measured slower at config 1 (39.9 vs
  // 29.1 ms per 224 applies): the window staging and its occupancy cost
  // more than the L2 gathers it saves at this size.
  std::string variant = p * n < (i64{1} << 31) ? "fast2" : "staged";
  if (BandApply<T>::preferred(p, n)) variant = "band";
  if (const char* e = std::getenv("CPCAG_APPLY")) variant = e;
  if (variant == "band" && !BandApply<T>::feasible(p)) variant = "staged";
  std::vector<i64> rpr(static_cast<size_t>(p) + 1), rpc(static_cast<size_t>(n) + 1);
  CUDA_OK(cudaMemcpyAsync(rpr.data(), pr.rp, sizeof(i64) * (p + 1), cudaMemcpyDeviceToHost, c->stream));
  CUDA_OK(cudaMemcpyAsync(rpc.data(), pc.rp, sizeof(i64) * (n + 1), cudaMemcpyDeviceToHost, c->stream));
  sync(c);
  // Column chunk per CTA: enough CTAs for ~16 per SM, and a chunk small
  // enough that its L_c rows stage in shared memory (<= 128 columns).
  const i64 cols_per_cta = std::max<i64>({i64{1}, std::min<i64>((n + g2.y - 1) / g2.y, 128), (n + 65534) / 65535});
  const dim3 gs(gx, static_cast<unsigned>(std::min<i64>((n + cols_per_cta - 1) / cols_per_cta, 65535)));
  if (part.n < static_cast<size_t>(gs.x) * gs.y) part.alloc(c, static_cast<size_t>(gs.x) * gs.y);
  i64 max_er = 0, max_ec = 0;
  for (unsigned b = 0; b < gx; ++b) {
    const i64 a = static_cast<i64>(b) * kBlock, e = std::min<i64>(p, a + kBlock);
    max_er = std::max(max_er, rpr[e] - rpr[a]);
  }
  for (unsigned b = 0; b < gs.y; ++b) {
    const i64 a = static_cast<i64>(b) * cols_per_cta, e = std::min<i64>(n, a + cols_per_cta);
    max_ec = std::max(max_ec, rpc[e] - rpc[a]);
  }
  const size_t staged_smem = static_cast<size_t>(max_er + max_ec) * (sizeof(T) + sizeof(int)) + 16;
  const size_t fast_smem = static_cast<size_t>(max_er + max_ec) * sizeof(OffEnt<T>) + sizeof(int) * (cols_per_cta + 2) + 16;
  if (variant == "fast" && !(p * n < (i64{1} << 31) && fast_smem <= 96 * 1024)) variant = "staged";
  TileApply<T> tile;
  DevBuf<int> csel_perm;
  const Plan pl0 = pl;  // caller's column order (the true residual of rcm2)
  Pull<T> pc2 = pc;     // L_c pull of the fast2 kernel (permuted for rcm2)
  if (variant == "rcm2") {
    // fast2 on iterates stored in RCM column order (CPCAG_APPLY=rcm2):
    // consecutive columns share most of their L_c neighbours, so a CTA's
    // gathers hit L1.  Measured equal to fast2 (0.128 vs 0.127 ms): L2
    // locality is not what bounds the gather.
    if (p * n < (i64{1} << 31) && tile.build(c, Lc, rpc, rpr, p, INT32_MAX, false)) {
      csel_perm.alloc(c, n);
      permute_sel_k<<<blocks_for(n), kBlock, 0, c->stream>>>(n, tile.pos.p, csel.p, csel_perm.p);
      launched(c);
      pl.csel = csel_perm.p;
      pc2 = Pull<T>{tile.crp.p, tile.pci.p, tile.pv.p};
      rpc = tile.hrp_host;  // fast2 geometry below sizes its L_c staging from these
    } else {
      variant = "fast2";
    }
  }
  if (variant == "fast3") {
    // banded column graph: RCM column order and shared-memory windows
    if (tile.build(c, Lc, rpc, rpr, p, 128)) {
      if (part.n < static_cast<size_t>(tile.grid().x) * tile.grid().y)
        part.alloc(c, static_cast<size_t>(tile.grid().x) * tile.grid().y);
      csel_perm.alloc(c, n);
      permute_sel_k<<<blocks_for(n), kBlock, 0, c->stream>>>(n, tile.pos.p, csel.p, csel_perm.p);
      launched(c);
      pl.csel = csel_perm.p;
    } else {
      variant = "fast2";
    }
  }
  BandApply<T> band;
  DevBuf<int> rsel_perm;
  if (variant == "band") {
    const char* pe = std::getenv("CPCAG_BAND_PERM");
    band.build(c, Lr, Lc, rpr, !(pe && std::string(pe) == "0"));
    if (part.n < band.col_blocks(0, n)) part.alloc(c, band.col_blocks(0, n));
    if (band.permuted && p) {
      // Every p x n iterate is stored with rows in the band's order.
      rsel_perm.alloc(c, p);
      permute_sel_k<<<blocks_for(p), kBlock, 0, c->stream>>>(p, band.pos.p, rsel.p, rsel_perm.p);
      launched(c);
      pl.rsel = rsel_perm.p;
    }
  }
  if (variant == "fast") ensure_smem(cg_apply_fast_k<T>, fast_smem);
  // fast2 geometry: 512-row blocks, ~16 CTAs per SM.
  const unsigned gx2 = static_cast<unsigned>((p + 511) / 512);
  i64 f2_per_sm = 8;  // CTAs per SM the column chunking aims at (measured: 8 best of 16/8/6/4)
  if (const char* e = std::getenv("CPCAG_FAST2_CTAS")) f2_per_sm = std::max<i64>(1, std::atoll(e));
  const i64 y2cap = std::max<i64>(1, (static_cast<i64>(c->num_sms) * f2_per_sm) / gx2);
  const i64 cpc2 = std::max<i64>({i64{1}, std::min<i64>((n + std::min<i64>(n, y2cap) - 1) / std::max<i64>(1, std::min<i64>(n, y2cap)), 128),
                                  (n + 65534) / 65535});
  const dim3 gs2(gx2, static_cast<unsigned>(std::min<i64>((n + cpc2 - 1) / cpc2, 65535)));
  size_t fast2_smem = 0;
  int f2_minb = 4;  // resident CTAs per SM the register budget targets
  if (const char* e = std::getenv("CPCAG_FAST2_MINB")) f2_minb = std::min(6, std::max(4, std::atoi(e)));
  auto f2_kernel = [&]() {
    return f2_minb == 6 ? cg_apply_fast2_k<T, 6> : (f2_minb == 5 ? cg_apply_fast2_k<T, 5> : cg_apply_fast2_k<T, 4>);
  };
  // fast5 (fp32, p % 4 == 0; CPCAG_APPLY=fast5): 16-byte L_c gathers.
  unsigned gx5 = static_cast<unsigned>((p + 511) / 512);
  i64 f5_per_sm = 16;  // 128-thread CTAs per SM the column chunking aims at
  if (const char* e = std::getenv("CPCAG_FAST5_CTAS")) f5_per_sm = std::max<i64>(1, std::atoll(e));
  int f5_unroll = 4;
  if (const char* e = std::getenv("CPCAG_FAST5_UNROLL")) f5_unroll = std::atoi(e) == 8 ? 8 : (std::atoi(e) == 2 ? 2 : 4);
  const i64 y5cap = std::max<i64>(1, (static_cast<i64>(c->num_sms) * f5_per_sm) / gx5);
  const i64 cpc5 = std::max<i64>({i64{1}, std::min<i64>((n + std::min<i64>(n, y5cap) - 1) / std::max<i64>(1, std::min<i64>(n, y5cap)), 128),
                                  (n + 65534) / 65535});
  const dim3 gs5(gx5, static_cast<unsigned>(std::min<i64>((n + cpc5 - 1) / cpc5, 65535)));
  size_t fast5_smem = 0;
  if (variant == "fast5") {
    if (sizeof(T) != 4 || p % 4 != 0) invalid("alternate decoder: fast5 apply needs fp32 and p % 4 == 0");
    i64 mer = 0, mec = 0;
    for (unsigned b = 0; b < gx5; ++b) {
      const i64 a = static_cast<i64>(b) * 512, e = std::min<i64>(p, a + 512);
      mer = std::max(mer, rpr[e] - rpr[a]);
    }
    for (unsigned b = 0; b < gs5.y; ++b) {
      const i64 a = static_cast<i64>(b) * cpc5, e = std::min<i64>(n, a + cpc5);
      mec = std::max(mec, rpc[e] - rpc[a]);
    }
    fast5_smem = static_cast<size_t>(mer + mec) * sizeof(OffEnt<T>) + sizeof(int) * (cpc5 + 2 + 512 + 1) + 16;
    if (!(p * n < (i64{1} << 31) && fast5_smem <= 96 * 1024)) invalid("alternate decoder: fast5 slice exceeds shared memory");
    ensure_smem(cg_apply_fast5_k<2>, fast5_smem);
    ensure_smem(cg_apply_fast5_k<4>, fast5_smem);
    ensure_smem(cg_apply_fast5_k<8>, fast5_smem);
    if (part.n < static_cast<size_t>(gs5.x) * gs5.y) part.alloc(c, static_cast<size_t>(gs5.x) * gs5.y);
  }
  // slab (32-row slabs of P in shared memory, CPCAG_APPLY=slab): measured
  // slower than fast2 at config 1 (0.19 vs 0.127 ms per apply): one
  // 1024-thread CTA per SM stalls on slab staging and on the L_r gathers.
  int slab_parts = 0, slab_units = 0;
  unsigned slab_grid = 0;
  size_t slab_smem = 0;
  if (variant == "slab") {
    if (n * 32 * sizeof(T) > 200 * 1024) invalid("alternate decoder: slab apply needs n * 32 * sizeof(T) <= 200 KB");
    const i64 slabs = (p + 31) / 32, sms = c->num_sms;
    // parts per slab: minimise rounds x (staging + compute / parts), staging ~0.1 of a slab's compute
    double best = 1e300;
    for (int q = 1; q <= 4; ++q) {
      const double rounds = static_cast<double>((slabs * q + sms - 1) / sms);
      const double t = rounds * (0.1 + 1.0 / q);
      if (t < best - 1e-9) {
        best = t;
        slab_parts = q;
      }
    }
    if (const char* e = std::getenv("CPCAG_SLAB_PARTS")) slab_parts = std::max(1, std::atoi(e));
    slab_units = static_cast<int>(slabs * slab_parts);
    slab_grid = static_cast<unsigned>(std::min<i64>(slab_units, sms));
    slab_smem = static_cast<size_t>(n) * 32 * sizeof(T);
    ensure_smem(cg_apply_slab_k<T>, slab_smem);
    if (part.n < slab_grid) part.alloc(c, slab_grid);
  }
  // fast4 (R rows per thread, 128-thread CTAs; CPCAG_APPLY=fast4): measured
  // slower than fast2 (0.18 ms at R = 2, worse at R = 4, 8): the gather wants
  // resident warps, not more loads per thread.
  int f4_rows = 4;
  if (const char* e = std::getenv("CPCAG_FAST4_ROWS")) f4_rows = std::atoi(e) == 8 ? 8 : (std::atoi(e) == 2 ? 2 : 4);
  const i64 kF4Rows = 128 * f4_rows;  // rows per CTA
  const unsigned gx4 = static_cast<unsigned>((p + kF4Rows - 1) / kF4Rows);
  i64 f4_per_sm = 8;  // CTAs per SM the column chunking aims at
  if (const char* e = std::getenv("CPCAG_FAST4_CTAS")) f4_per_sm = std::max<i64>(1, std::atoll(e));
  const i64 y4cap = std::max<i64>(1, (static_cast<i64>(c->num_sms) * f4_per_sm) / gx4);
  const i64 cpc4 = std::max<i64>({i64{1}, std::min<i64>((n + std::min<i64>(n, y4cap) - 1) / std::max<i64>(1, std::min<i64>(n, y4cap)), 128),
                                  (n + 65534) / 65535});
  const dim3 gs4(gx4, static_cast<unsigned>(std::min<i64>((n + cpc4 - 1) / cpc4, 65535)));
  size_t fast4_smem = 0;
  auto f4_kernel = [&]() {
    return f4_rows == 8 ? cg_apply_fast4_k<T, 8, 128> : (f4_rows == 2 ? cg_apply_fast4_k<T, 2, 128> : cg_apply_fast4_k<T, 4, 128>);
  };
  if (variant == "fast4") {
    i64 mer = 0, mec = 0;
    for (unsigned b = 0; b < gx4; ++b) {
      const i64 a = static_cast<i64>(b) * kF4Rows, e = std::min<i64>(p, a + kF4Rows);
      mer = std::max(mer, rpr[e] - rpr[a]);
    }
    for (unsigned b = 0; b < gs4.y; ++b) {
      const i64 a = static_cast<i64>(b) * cpc4, e = std::min<i64>(n, a + cpc4);
      mec = std::max(mec, rpc[e] - rpc[a]);
    }
    fast4_smem = static_cast<size_t>(mer + mec) * sizeof(OffEnt<T>) + sizeof(int) * (cpc4 + 2 + kF4Rows + 1) + 16;
    if (!(p * n < (i64{1} << 31) && fast4_smem <= 96 * 1024)) {
      variant = "fast2";
    } else {
      ensure_smem(f4_kernel(), fast4_smem);
      if (part.n < static_cast<size_t>(gs4.x) * gs4.y) part.alloc(c, static_cast<size_t>(gs4.x) * gs4.y);
    }
  }
  i64 maxdeg_r_pre = 0;
  for (i64 i = 0; i < p; ++i) maxdeg_r_pre = std::max(maxdeg_r_pre, rpr[i + 1] - rpr[i]);
  // slab2 (two-pass apply: cg_lc_slab_k then fast2<kU>), when a 32-row slab
  // over all n columns fits in shared memory.
  int s2_parts = 4, s2_units = 0;
  unsigned s2_grid = 0;
  size_t s2_smem = 0;
  DevBuf<T> Ubuf;
  if (variant == "slabr" && !(maxdeg_r_pre <= 16)) variant = "fast2";
  if (variant == "slab2" || variant == "slabr") {
    if (!(p * n < (i64{1} << 31) && n * 32 * static_cast<i64>(sizeof(T)) <= 200 * 1024)) {
      variant = "fast2";
    } else {
      const i64 slabs = (p + 31) / 32;
      if (const char* e = std::getenv("CPCAG_SLAB2_PARTS")) s2_parts = std::max(1, std::atoi(e));
      s2_units = static_cast<int>(slabs * s2_parts);
      s2_grid = static_cast<unsigned>(std::min<i64>(s2_units, c->num_sms));
      const i64 cw2 = (n + s2_parts - 1) / s2_parts;
      i64 ecap = 0;
      for (i64 q = 0; q < s2_parts; ++q) {
        const i64 a = std::min(n, q * cw2), e = std::min(n, a + cw2);
        ecap = std::max(ecap, rpc[e] - rpc[a]);
      }
      s2_smem = static_cast<size_t>(n) * 32 * sizeof(T) + static_cast<size_t>(ecap) * sizeof(OffEnt<T>);
      if (s2_smem > 220 * 1024) {
        variant = "fast2";
        s2_grid = 0;
      } else {
        ensure_smem(cg_lc_slab_k<T>, s2_smem);
        ensure_smem(cg_apply_slabr_k<T, 10>, s2_smem);
        ensure_smem(cg_apply_slabr_k<T, 16>, s2_smem);
      }
      if (s2_grid && variant == "slab2") Ubuf.alloc(c, static_cast<size_t>(N));
      if (s2_grid && part.n < s2_grid) part.alloc(c, s2_grid);
    }
  }
  // regr (register-resident L_r rows) needs row degree <= 16.
  i64 maxdeg_r = 0;
  for (i64 i = 0; i < p; ++i) maxdeg_r = std::max(maxdeg_r, rpr[i + 1] - rpr[i]);
  const bool regr_ok = maxdeg_r <= 16;
  if (variant == "regr" && !regr_ok) variant = "fast2";
  if (variant == "fast2" || variant == "rcm2" || variant == "slab2" || variant == "regr") {
    i64 mer = 0, mec = 0;
    for (unsigned b = 0; b < gx2; ++b) {
      const i64 a = static_cast<i64>(b) * 512, e = std::min<i64>(p, a + 512);
      mer = std::max(mer, rpr[e] - rpr[a]);
    }
    for (unsigned b = 0; b < gs2.y; ++b) {
      const i64 a = static_cast<i64>(b) * cpc2, e = std::min<i64>(n, a + cpc2);
      mec = std::max(mec, rpc[e] - rpc[a]);
    }
    fast2_smem = static_cast<size_t>(mer + mec) * sizeof(OffEnt<T>) + sizeof(int) * (cpc2 + 2) + 16;
    if (!(p * n < (i64{1} << 31) && fast2_smem <= 96 * 1024)) {
      if (variant == "rcm2") invalid("alternate decoder: rcm2 apply slice exceeds shared memory");
      variant = "staged";
    }
    else {
      ensure_smem(cg_apply_fast2_k<T, 4>, fast2_smem);
      ensure_smem(cg_apply_fast2_k<T, 5>, fast2_smem);
      ensure_smem(cg_apply_fast2_k<T, 6>, fast2_smem);
      ensure_smem(cg_apply_fast2_k<T, 4, true>, fast2_smem);
      ensure_smem(cg_apply_regr_k<T, 16, false>, fast2_smem);
      ensure_smem(cg_apply_regr_k<T, 16, true>, fast2_smem);
    }
    if (variant == "staged" && s2_grid) Ubuf.release();
    if (part.n < static_cast<size_t>(gs2.x) * gs2.y) part.alloc(c, static_cast<size_t>(gs2.x) * gs2.y);
  }
  if (variant == "staged" && !(staged_smem <= 96 * 1024)) variant = "plain";
  if (variant == "staged") ensure_smem(cg_apply_staged_k<T>, staged_smem);

  cg_init_k<T><<<g2, kBlock, 0, c->stream>>>(p, n, pl, Xt, X, R.p, P.p, cfg.pcg_tol, part.p, st.p);
  launched(c);
  CgState host = read_back(c, st.p);
  // small problems: the whole loop as one cooperative kernel (cg_persist_k)
  // (default path only: an explicit CPCAG_APPLY variant keeps its own loop,
  // and the permuted layouts of rcm2 / fast3 / band never take it)
  // Opt-in (CPCAG_CG_PERSIST=1): measured at config 0 (fp64, 200 x 300) the
  // apply phase costs 14-30 us per iteration across CTAs (one entry per
  // thread, L1-cold gathers after each barrier), so the loop runs at 48 vs
  // 46 us per iteration for the per-kernel path.
  const char* pe = std::getenv("CPCAG_CG_PERSIST");
  const bool persist = pe && std::string(pe) == "1" && N <= (i64{1} << 20) && N > 0 && variant != "band" &&
                       variant != "fast3" && variant != "rcm2";
  if (persist && !host.done) {
    // shared memory: L_r entries, this CTA's L_c rows, both row-pointer arrays
    i64 Gp = std::min<i64>((N + 511) / 512, static_cast<i64>(c->num_sms));
    if (const char* e = std::getenv("CPCAG_CG_PERSIST_G")) Gp = std::max<i64>(1, std::min<i64>(Gp, std::atoll(e)));
    i64 max_ec = 0, max_cols = 0;
    for (i64 b = 0; b < Gp; ++b) {
      const i64 e0 = (N * b) / Gp, e1 = (N * (b + 1)) / Gp;
      const i64 ca = e0 / p, cb = e1 > e0 ? (e1 - 1) / p : ca;
      max_ec = std::max(max_ec, rpc[cb + 1] - rpc[ca]);
      max_cols = std::max(max_cols, cb - ca + 1);
    }
    const size_t psmem = static_cast<size_t>(rpr[p] + max_ec) * sizeof(OffEnt<T>) +
                         sizeof(int) * static_cast<size_t>(p + 1 + max_cols + 1);
    int per_sm = 0;
    if (psmem <= 200 * 1024) {
      ensure_smem(cg_persist_k<T>, psmem);
      CUDA_OK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, cg_persist_k<T>, 512, psmem));
    }
    if (per_sm >= 1) {
      DevBuf<double> pp(c, 2 * static_cast<size_t>(Gp));
      DevBuf<unsigned> bar(c, 2);
      bar.zero(c);
      T* Xp = X;
      T *Rp = R.p, *Pp = P.p, *APp = AP.p;
      double* ppp = pp.p;
      i64 mi = cfg.pcg_max_iter;
      CgState* sp = st.p;
      unsigned* bp = bar.p;
      int prof = std::getenv("CPCAG_CG_PERSIST_PROF") ? 1 : 0;
      void* args[] = {(void*)&p, (void*)&n, (void*)&pr, (void*)&pc, (void*)&gr, (void*)&gc, (void*)&pl,
                      (void*)&Xp, (void*)&Rp, (void*)&Pp, (void*)&APp, (void*)&ppp, (void*)&mi, (void*)&sp,
                      (void*)&bp, (void*)&prof};
      {
        KScope ks_(c, "cg_persist");
        CUDA_OK(cudaLaunchCooperativeKernel((void*)cg_persist_k<T>, dim3(static_cast<unsigned>(Gp)), dim3(512), args,
                                            psmem, c->stream));
        launched(c);
      }
      host = read_back(c, st.p);
    }
  }
  const i64 chunk = 32;
  while (!host.done) {
    for (i64 k = 0; k < chunk; ++k) {
      {
        KScope ks_(c, "cg_apply");
        if (variant == "band") {
          band.apply(c, P.p, AP.p, 0, n, pl, gr, gc, part.p, st.p, 0);
        } else if (variant == "fast3") {
          tile.apply(c, pr, P.p, AP.p, pl, gr, gc, part.p, st.p, 0);
        } else if (variant == "fast5") {
          if constexpr (sizeof(T) == 4) {
            auto k5 = f5_unroll == 8 ? cg_apply_fast5_k<8> : (f5_unroll == 2 ? cg_apply_fast5_k<2> : cg_apply_fast5_k<4>);
            k5<<<gs5, 128, fast5_smem, c->stream>>>(static_cast<int>(p), static_cast<int>(n), pr, pc, gr, gc, pl,
                                                    static_cast<int>(cpc5), P.p, AP.p, part.p, st.p);
          }
        } else if (variant == "slab") {
          cg_apply_slab_k<T><<<slab_grid, 1024, slab_smem, c->stream>>>(static_cast<int>(p), static_cast<int>(n), pr, pc,
                                                                        gr, gc, pl, slab_parts, slab_units, P.p, AP.p,
                                                                        part.p, st.p);
        } else if (variant == "fast4") {
          f4_kernel()<<<gs4, 128, fast4_smem, c->stream>>>(static_cast<int>(p), static_cast<int>(n), pr, pc, gr, gc, pl,
                                                       static_cast<int>(cpc4), P.p, AP.p, part.p, st.p);
        } else if (variant == "slab2") {
          cg_lc_slab_k<T><<<s2_grid, 1024, s2_smem, c->stream>>>(static_cast<int>(p), static_cast<int>(n), pc,
                                                                 s2_parts, s2_units, P.p, Ubuf.p, st.p);
          launched(c);
          if (regr_ok)
            cg_apply_regr_k<T, 16, true><<<gs2, kBlock, fast2_smem, c->stream>>>(
                static_cast<int>(p), static_cast<int>(n), pr, pc, gr, gc, pl, static_cast<int>(cpc2), P.p, AP.p,
                part.p, st.p, Ubuf.p);
          else
            cg_apply_fast2_k<T, 4, true><<<gs2, kBlock, fast2_smem, c->stream>>>(
                static_cast<int>(p), static_cast<int>(n), pr, pc, gr, gc, pl, static_cast<int>(cpc2), P.p, AP.p,
                part.p, st.p, Ubuf.p);
        } else if (variant == "slabr") {
          auto kr = maxdeg_r_pre <= 10 ? cg_apply_slabr_k<T, 10> : cg_apply_slabr_k<T, 16>;
          kr<<<s2_grid, 1024, s2_smem, c->stream>>>(static_cast<int>(p), static_cast<int>(n), pr, pc, gr, gc, pl,
                                                    s2_parts, s2_units, P.p, AP.p, part.p, st.p);
        } else if (variant == "regr") {
          cg_apply_regr_k<T, 16, false><<<gs2, kBlock, fast2_smem, c->stream>>>(
              static_cast<int>(p), static_cast<int>(n), pr, pc, gr, gc, pl, static_cast<int>(cpc2), P.p, AP.p, part.p,
              st.p, nullptr);
        } else if (variant == "fast2" || variant == "rcm2") {
          f2_kernel()<<<gs2, kBlock, fast2_smem, c->stream>>>(static_cast<int>(p), static_cast<int>(n), pr, pc2, gr,
                                                                     gc, pl, static_cast<int>(cpc2), P.p, AP.p, part.p,
                                                                     st.p, nullptr);
        } else if (variant == "fast") {
          cg_apply_fast_k<T><<<gs, kBlock, fast_smem, c->stream>>>(static_cast<int>(p), 0, static_cast<int>(n), pr, pc,
                                                                  gr, gc, pl, static_cast<int>(cols_per_cta), P.p, AP.p,
                                                                  part.p, st.p);
        } else if (variant == "staged") {
          cg_apply_staged_k<T><<<gs, kBlock, staged_smem, c->stream>>>(p, 0, n, pr, pc, gr, gc, pl, cols_per_cta, P.p,
                                                                      AP.p, part.p, st.p);
        } else {
          cg_apply_k<T><<<g2, kBlock, 0, c->stream>>>(p, n, pr, pc, gr, gc, pl, P.p, AP.p, part.p, st.p);
        }
        if (variant != "band" && variant != "fast3") launched(c);
      }
      {
        KScope ks_(c, "cg_residual");
        if (vec_ok)
          cg_residual_k<T, true><<<nb1v, kBlock, 0, c->stream>>>(N, R.p, AP.p, part.p, st.p);
        else
          cg_residual_k<T><<<nb1, kBlock, 0, c->stream>>>(N, R.p, AP.p, part.p, st.p);
        launched(c);
      }
      {
        KScope ks_(c, "cg_update");
        if (vec_ok)
          cg_update_k<T, true><<<nb1v, kBlock, 0, c->stream>>>(N, X, P.p, R.p, cfg.pcg_max_iter, st.p);
        else
          cg_update_k<T><<<nb1, kBlock, 0, c->stream>>>(N, X, P.p, R.p, cfg.pcg_max_iter, st.p);
        launched(c);
      }
    }
    host = read_back(c, st.p);
  }
  if (variant == "band") band.report_prof(c);
  if (host.err)
    runtime("pcg: breakdown (nonpositive curvature) at iteration " + std::to_string(host.err_it));
  if (host.zero_rhs) {
    *converged = 1;
    *iterations = 0;
    return;
  }
  if (variant == "fast3") {
    tile.apply(c, pr, X, AP.p, pl, gr, gc, part.p, st.p, 1);
    cg_true_res_ap_k<T><<<g2, kBlock, 0, c->stream>>>(p, n, pl, Xt, AP.p, part.p, st.p);
    launched(c);
    // back to the caller's column order
    CUDA_OK(cudaMemcpyAsync(AP.p, X, sizeof(T) * N, cudaMemcpyDeviceToDevice, c->stream));
    if constexpr (sizeof(T) == 4)
      unpermute_cols_k<<<g2, kBlock, 0, c->stream>>>(p, n, tile.pos.p, reinterpret_cast<const float*>(AP.p),
                                                     reinterpret_cast<float*>(X), nullptr, nullptr);
    else
      unpermute_cols_k<<<g2, kBlock, 0, c->stream>>>(p, n, tile.pos.p, nullptr, nullptr,
                                                     reinterpret_cast<const double*>(AP.p),
                                                     reinterpret_cast<double*>(X));
  } else if (variant == "band") {
    band.apply(c, X, AP.p, 0, n, pl, gr, gc, part.p, st.p, 1);
    cg_true_res_ap_k<T><<<g2, kBlock, 0, c->stream>>>(p, n, pl, Xt, AP.p, part.p, st.p);
    if (band.permuted) {  // back to the caller's row order
      launched(c);
      CUDA_OK(cudaMemcpyAsync(AP.p, X, sizeof(T) * N, cudaMemcpyDeviceToDevice, c->stream));
      unpermute_rows_k<T><<<g2, kBlock, 0, c->stream>>>(p, n, band.pos.p, AP.p, X);
    }
  } else {
    if (variant == "rcm2") {  // back to the caller's column order
      CUDA_OK(cudaMemcpyAsync(AP.p, X, sizeof(T) * N, cudaMemcpyDeviceToDevice, c->stream));
      if constexpr (sizeof(T) == 4)
        unpermute_cols_k<<<g2, kBlock, 0, c->stream>>>(p, n, tile.pos.p, reinterpret_cast<const float*>(AP.p),
                                                       reinterpret_cast<float*>(X), nullptr, nullptr);
      else
        unpermute_cols_k<<<g2, kBlock, 0, c->stream>>>(p, n, tile.pos.p, nullptr, nullptr,
                                                       reinterpret_cast<const double*>(AP.p),
                                                       reinterpret_cast<double*>(X));
      launched(c);
    }
    cg_true_residual_k<T><<<g2, kBlock, 0, c->stream>>>(p, n, pr, pc, gr, gc, pl0, Xt, X, part.p, st.p);
  }
  launched(c);
  host = read_back(c, st.p);
  *converged = host.rel_res <= cfg.pcg_tol ? 1 : 0;
  *iterations = host.it;
}

template void alternate_decode_device<double>(Ctx*, const double*, i64, i64, const i64*, const i64*, i64, i64,
                                              Csr*, Csr*, double, double, const cpcag_decoder_config&,
                                              double*, int*, i64*);
template void alternate_decode_device<float>(Ctx*, const float*, i64, i64, const i64*, const i64*, i64, i64,
                                             Csr*, Csr*, double, double, const cpcag_decoder_config&,
                                             float*, int*, i64*);

// ------------------------------------------------------------------ column-block primitives
// The decoder's local work for one column block [c0, c1) of a column-sharded
// solve: the caller all-gathers P between ranks and
// all-reduces the partial dots; everything here touches only this GPU.
struct DecBlock {
  Ctx* c;
  int prec;
  i64 p, n, c0, c1, rho_r;
  Csr *Lr, *Lc;
  double gr, gc;
  DevBuf<int> rsel, csel;
  DevBuf<double> part;
  DevBuf<CgState> st;
  size_t smem = 0;
  i64 cols_per_cta = 1;
  dim3 grid;
  // Band apply (iterate larger than L2); null when the staged apply is used.
  std::unique_ptr<BandApply<float>> band32;
  std::unique_ptr<BandApply<double>> band64;
  BandApply<float>* band(float*) { return band32.get(); }
  BandApply<double>* band(double*) { return band64.get(); }
};

template <typename T>
__global__ void block_rhs_k(i64 p, i64 c0, i64 c1, Plan pl, const T* __restrict__ Xt, T* __restrict__ B,
                            double* partials, CgState* st) {
  double s[1] = {0.0};
  const i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x;
  if (i < p)
    for (i64 c = c0 + blockIdx.y; c < c1; c += gridDim.y) {
      const T b = rhs_at(pl, Xt, i, c);
      B[i + (c - c0) * p] = b;
      s[0] += static_cast<double>(b) * static_cast<double>(b);
    }
  double tot[1];
  if (grid_sum_last<1>(s, partials, &st->cnt[0], tot) && threadIdx.x == 0) st->norm_b = tot[0];
}

template <typename T>
__global__ void block_residual_k(i64 N, T alpha, T* __restrict__ R, const T* __restrict__ AP, double* partials,
                                 CgState* st) {
  double s[1] = {0.0};
  for (i64 q = blockIdx.x * (i64)blockDim.x + threadIdx.x; q < N; q += (i64)gridDim.x * blockDim.x) {
    const T r = sub_rn(R[q], mul_rn(alpha, AP[q]));
    R[q] = r;
    s[0] += static_cast<double>(r) * static_cast<double>(r);
  }
  double tot[1];
  if (grid_sum_last<1>(s, partials, &st->cnt[2], tot) && threadIdx.x == 0) st->rho_next = tot[0];
}

template <typename T>
__global__ void block_update_k(i64 N, T alpha, T beta, T* __restrict__ X, T* __restrict__ P, const T* __restrict__ R) {
  for (i64 q = blockIdx.x * (i64)blockDim.x + threadIdx.x; q < N; q += (i64)gridDim.x * blockDim.x) {
    const T pv = P[q];
    X[q] = add_rn(X[q], mul_rn(alpha, pv));
    P[q] = add_rn(R[q], mul_rn(beta, pv));
  }
}

}  // namespace cpcag_cuda

using namespace cpcag_cuda;

namespace {
DecBlock* as_block(cpcag_decoder_block b) {
  if (!b) invalid("null decoder block");
  return reinterpret_cast<DecBlock*>(b);
}

template <typename T>
void block_apply(DecBlock* b, const T* Pfull, T* APblk, double* dot) {
  Ctx* c = b->c;
  const Pull<T> pr = make_pull<T>(c, b->Lr, false), pc = make_pull<T>(c, b->Lc, true);
  const Plan pl{b->rsel.p, b->csel.p, b->rho_r};
  b->st.zero(c);
  // AP indexed by global column: shift the block pointer back by c0 columns.
  T* base = APblk - b->c0 * b->p;
  if (BandApply<T>* band = b->band(static_cast<T*>(nullptr))) {
    KScope ks_(c, "cg_apply");
    band->apply(c, Pfull, base, b->c0, b->c1, pl, static_cast<T>(b->gr), static_cast<T>(b->gc), b->part.p, b->st.p, 0);
  } else {
    KScope ks_(c, "cg_apply");
    cg_apply_staged_k<T><<<b->grid, kBlock, b->smem, c->stream>>>(b->p, b->c0, b->c1, pr, pc, static_cast<T>(b->gr),
                                                                  static_cast<T>(b->gc), pl, b->cols_per_cta, Pfull,
                                                                  base, b->part.p, b->st.p);
    launched(c);
  }
  *dot = read_back(c, b->st.p).curv;
}
}  // namespace

extern "C" int cpcag_cuda_decoder_block_create(cpcag_ctx ctx, int precision, int64_t p, int64_t n, int64_t c_begin,
                                               int64_t c_end, cpcag_csr Lr, cpcag_csr Lc, const int64_t* omega_r,
                                               int64_t rho_r, const int64_t* omega_c, int64_t rho_c, double gbar_r,
                                               double gbar_c, cpcag_decoder_block* out) {
  return guard([&] {
    Ctx* c = as_ctx(ctx);
    if (!out) invalid("null output pointer");
    if (precision != CPCAG_F64 && precision != CPCAG_F32) invalid("unknown precision flag");
    Csr* A = as_csr(Lr);
    Csr* B = as_csr(Lc);
    if (A->rows != p || A->cols != p || B->rows != n || B->cols != n)
      invalid("alternate decoder: Laplacians do not match plan");
    if (c_begin < 0 || c_end > n || c_begin > c_end) invalid("decoder block: column range out of bounds");
    auto blk = std::make_unique<DecBlock>();
    blk->c = c;
    blk->prec = precision;
    blk->p = p;
    blk->n = n;
    blk->c0 = c_begin;
    blk->c1 = c_end;
    blk->rho_r = rho_r;
    blk->Lr = A;
    blk->Lc = B;
    blk->gr = gbar_r;
    blk->gc = gbar_c;
    std::vector<int> rs(static_cast<size_t>(p), -1), cs(static_cast<size_t>(n), -1);
    std::vector<i64> omr(static_cast<size_t>(rho_r)), omc(static_cast<size_t>(rho_c));
    auto fetch = [&](std::vector<i64>& dst, const int64_t* src) {
      if (dst.empty()) return;
      if (is_device_ptr(src))
        CUDA_OK(cudaMemcpy(dst.data(), src, sizeof(i64) * dst.size(), cudaMemcpyDeviceToHost));
      else
        std::copy(src, src + dst.size(), dst.begin());
    };
    fetch(omr, omega_r);
    fetch(omc, omega_c);
    for (i64 k = 0; k < rho_r; ++k) {
      if (omr[k] < 0 || omr[k] >= p || rs[omr[k]] >= 0) invalid("alternate decoder: Xt does not match plan");
      rs[omr[k]] = static_cast<int>(k);
    }
    for (i64 k = 0; k < rho_c; ++k) {
      if (omc[k] < 0 || omc[k] >= n || cs[omc[k]] >= 0) invalid("alternate decoder: Xt does not match plan");
      cs[omc[k]] = static_cast<int>(k);
    }
    blk->rsel.alloc(c, std::max<i64>(p, 1));
    blk->csel.alloc(c, std::max<i64>(n, 1));
    if (p) CUDA_OK(cudaMemcpyAsync(blk->rsel.p, rs.data(), sizeof(int) * p, cudaMemcpyHostToDevice, c->stream));
    if (n) CUDA_OK(cudaMemcpyAsync(blk->csel.p, cs.data(), sizeof(int) * n, cudaMemcpyHostToDevice, c->stream));
    // launch geometry of the staged apply over the block's columns
    const i64 nb_cols = std::max<i64>(c_end - c_begin, 1);
    const unsigned gx = blocks_for(std::max<i64>(p, 1));
    const i64 ycap = std::max<i64>(1, (static_cast<i64>(c->num_sms) * 16) / gx);
    const i64 gy = std::max<i64>(1, std::min<i64>({nb_cols, ycap, 65535}));
    blk->cols_per_cta = (nb_cols + gy - 1) / gy;
    blk->grid = dim3(gx, static_cast<unsigned>((nb_cols + blk->cols_per_cta - 1) / blk->cols_per_cta));
    std::vector<i64> rpr(static_cast<size_t>(p) + 1), rpc(static_cast<size_t>(n) + 1);
    CUDA_OK(cudaMemcpy(rpr.data(), A->rp, sizeof(i64) * (p + 1), cudaMemcpyDeviceToHost));
    CUDA_OK(cudaMemcpy(rpc.data(), B->rp, sizeof(i64) * (n + 1), cudaMemcpyDeviceToHost));
    i64 max_er = 0, max_ec = 0;
    for (unsigned b = 0; b < gx; ++b) {
      const i64 a = static_cast<i64>(b) * kBlock, e = std::min<i64>(p, a + kBlock);
      max_er = std::max(max_er, rpr[e] - rpr[a]);
    }
    for (unsigned b = 0; b < blk->grid.y; ++b) {
      const i64 a = std::min<i64>(n, c_begin + static_cast<i64>(b) * blk->cols_per_cta);
      const i64 e = std::min<i64>(c_end, a + blk->cols_per_cta);
      max_ec = std::max(max_ec, rpc[e] - rpc[a]);
    }
    const size_t es = precision == CPCAG_F64 ? sizeof(double) : sizeof(float);
    blk->smem = static_cast<size_t>(max_er + max_ec) * (es + sizeof(int)) + 16;
    std::string variant = "staged";
    if (precision == CPCAG_F64 ? BandApply<double>::preferred(p, n) : BandApply<float>::preferred(p, n))
      variant = "band";
    if (const char* e = std::getenv("CPCAG_APPLY")) variant = std::string(e) == "band" ? "band" : "staged";
    if (variant == "band" && !BandApply<float>::feasible(p)) variant = "staged";
    size_t nparts = std::max<size_t>(static_cast<size_t>(blk->grid.x) * blk->grid.y,
                                     stride_blocks(c, std::max<i64>(p * nb_cols, 1)));
    if (variant == "band") {
      if (precision == CPCAG_F64) {
        blk->band64 = std::make_unique<BandApply<double>>();
        blk->band64->build(c, A, B, rpr, false);
        nparts = std::max<size_t>(nparts, blk->band64->col_blocks(c_begin, c_end));
      } else {
        blk->band32 = std::make_unique<BandApply<float>>();
        blk->band32->build(c, A, B, rpr, false);
        nparts = std::max<size_t>(nparts, blk->band32->col_blocks(c_begin, c_end));
      }
    } else {
      if (blk->smem > 200 * 1024) invalid("decoder block: operator slice exceeds shared memory");
      if (precision == CPCAG_F64)
        ensure_smem(cg_apply_staged_k<double>, blk->smem);
      else
        ensure_smem(cg_apply_staged_k<float>, blk->smem);
    }
    blk->part.alloc(c, nparts);
    blk->st.alloc(c, 1);
    blk->st.zero(c);
    sync(c);
    *out = reinterpret_cast<cpcag_decoder_block>(blk.release());
  });
}

extern "C" int cpcag_cuda_decoder_block_destroy(cpcag_decoder_block b) {
  return guard([&] { delete as_block(b); });
}

extern "C" int cpcag_cuda_decoder_block_rhs(cpcag_decoder_block bh, const void* Xt, void* B, double* sq_norm) {
  return guard([&] {
    DecBlock* b = as_block(bh);
    Ctx* c = b->c;
    if (!Xt || !B || !sq_norm) invalid("null argument");
    const Plan pl{b->rsel.p, b->csel.p, b->rho_r};
    b->st.zero(c);
    // b->grid (columns strided over grid.y): b->part holds one partial per CTA of it
    const dim3 g = b->grid;
    if (b->prec == CPCAG_F64)
      block_rhs_k<double><<<g, kBlock, 0, c->stream>>>(b->p, b->c0, b->c1, pl, static_cast<const double*>(Xt),
                                                       static_cast<double*>(B), b->part.p, b->st.p);
    else
      block_rhs_k<float><<<g, kBlock, 0, c->stream>>>(b->p, b->c0, b->c1, pl, static_cast<const float*>(Xt),
                                                      static_cast<float*>(B), b->part.p, b->st.p);
    launched(c);
    *sq_norm = read_back(c, b->st.p).norm_b;
  });
}

extern "C" int cpcag_cuda_decoder_block_apply(cpcag_decoder_block bh, const void* P_full, void* AP_block,
                                              double* dot) {
  return guard([&] {
    DecBlock* b = as_block(bh);
    if (!P_full || !AP_block || !dot) invalid("null argument");
    if (b->prec == CPCAG_F64)
      block_apply<double>(b, static_cast<const double*>(P_full), static_cast<double*>(AP_block), dot);
    else
      block_apply<float>(b, static_cast<const float*>(P_full), static_cast<float*>(AP_block), dot);
  });
}

extern "C" int cpcag_cuda_cg_residual(cpcag_ctx ctx, int precision, int64_t count, double alpha, void* R,
                                      const void* AP, double* rr) {
  return guard([&] {
    Ctx* c = as_ctx(ctx);
    if (!rr) invalid("null argument");
    const unsigned nb = stride_blocks(c, std::max<int64_t>(count, 1));
    DevBuf<double> part(c, nb);
    DevBuf<CgState> st(c, 1);
    st.zero(c);
    if (precision == CPCAG_F64)
      block_residual_k<double><<<nb, kBlock, 0, c->stream>>>(count, alpha, static_cast<double*>(R),
                                                             static_cast<const double*>(AP), part.p, st.p);
    else if (precision == CPCAG_F32)
      block_residual_k<float><<<nb, kBlock, 0, c->stream>>>(count, static_cast<float>(alpha), static_cast<float*>(R),
                                                            static_cast<const float*>(AP), part.p, st.p);
    else
      invalid("unknown precision flag");
    launched(c);
    *rr = read_back(c, st.p).rho_next;
  });
}

extern "C" int cpcag_cuda_cg_update(cpcag_ctx ctx, int precision, int64_t count, double alpha, double beta, void* X,
                                    void* P, const void* R) {
  return guard([&] {
    Ctx* c = as_ctx(ctx);
    const unsigned nb = stride_blocks(c, std::max<int64_t>(count, 1));
    if (precision == CPCAG_F64)
      block_update_k<double><<<nb, kBlock, 0, c->stream>>>(count, alpha, beta, static_cast<double*>(X),
                                                           static_cast<double*>(P), static_cast<const double*>(R));
    else if (precision == CPCAG_F32)
      block_update_k<float><<<nb, kBlock, 0, c->stream>>>(count, static_cast<float>(alpha), static_cast<float>(beta),
                                                          static_cast<float*>(X), static_cast<float*>(P),
                                                          static_cast<const float*>(R));
    else
      invalid("unknown precision flag");
    launched(c);
  });
}

namespace cpcag_cuda {
}  // namespace cpcag_cuda

using namespace cpcag_cuda;

extern "C" int cpcag_cuda_alternate_decode(cpcag_ctx ctx, int precision, const void* Xt, int64_t rho_r,
                                           int64_t rho_c, const int64_t* omega_r, const int64_t* omega_c,
                                           int64_t p, int64_t n, cpcag_csr Lr, cpcag_csr Lc,
                                           double lambda_k1_r, double lambda_k1_c,
                                           const cpcag_decoder_config* cfg, void* X, int* converged,
                                           int64_t* iterations) {
  auto run = [&](auto tag) {
    using T = decltype(tag);
    return guard([&] {
      Ctx* c = as_ctx(ctx);
      if (!cfg || !converged || !iterations) invalid("null argument");
      std::vector<i64> omr(static_cast<size_t>(std::max<int64_t>(rho_r, 0)));
      std::vector<i64> omc(static_cast<size_t>(std::max<int64_t>(rho_c, 0)));
      auto fetch = [&](std::vector<i64>& dst, const int64_t* src) {
        if (dst.empty()) return;
        if (is_device_ptr(src))
          CUDA_OK(cudaMemcpy(dst.data(), src, sizeof(i64) * dst.size(), cudaMemcpyDeviceToHost));
        else
          std::copy(src, src + dst.size(), dst.begin());
      };
      fetch(omr, omega_r);
      fetch(omc, omega_c);
      InView<T> xt(c, static_cast<const T*>(Xt), static_cast<size_t>(rho_r * rho_c));
      OutView<T> x(c, static_cast<T*>(X), static_cast<size_t>(p * n));
      alternate_decode_device<T>(c, xt.d, rho_r, rho_c, omr.data(), omc.data(), p, n, as_csr(Lr), as_csr(Lc),
                                 lambda_k1_r, lambda_k1_c, *cfg, x.d, converged, iterations);
      x.flush(c);
      sync(c);
    });
  };
  if (precision == CPCAG_F64) return run(double{});
  if (precision == CPCAG_F32) return run(float{});
  set_last_error("unknown precision flag");
  return CPCAG_ERR_INVALID_ARGUMENT;
}
