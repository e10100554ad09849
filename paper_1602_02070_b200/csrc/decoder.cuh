// decoder.cuh -- kernels and launch geometry of the alternate decoder's CG
// (decoders.cpp:145-186), shared by the one-GPU solver (decoder.cu) and the
// column-sharded solver (sharded.cu).  See decoder.cu for the design.
#pragma once

#include <algorithm>
#include <array>
#include <cstring>
#include <numeric>
#include <string>
#include <vector>

#include "common.cuh"
#include "frpcag.cuh"

namespace cpcag_cuda {

struct CgState {
  double rho, rho_next, curv;
  double norm_b, target, rel_res;
  i64 it, max_iter;
  int done, err, zero_rhs, pad;
  i64 err_it;
  unsigned cnt[4];
};

struct Plan {
  const int* rsel;  // p: index into omega_r or -1
  const int* csel;  // n: index into omega_c or -1 (global column index)
  i64 rho_r;
};

template <typename T>
__device__ __forceinline__ T rhs_at(const Plan& pl, const T* __restrict__ Xt, i64 i, i64 c) {
  const int a = pl.rsel[i], b = pl.csel[c];
  return (a >= 0 && b >= 0) ? Xt[a + static_cast<i64>(b) * pl.rho_r] : T(0);
}

// Accumulation step: exact multiply-then-add in fp64 (the reference's
// per-entry order), fused multiply-add in fp32.
template <typename TK>
__device__ __forceinline__ TK acc(TK a, TK v, TK x) {
  if constexpr (sizeof(TK) == 8)
    return __dadd_rn(a, __dmul_rn(v, x));
  else
    return fmaf(v, x, a);
}

// Second stage of the apply: AP = gc x1 + gr x2 (+ P on the sampled grid),
// and either <P, AP> (CG step) or ||b - AP||^2 (true residual, Xt != null).
template <typename TK, typename TB>
struct Combine {
  const TK* other;     // the partial sums of the pass that ran first
  TK* AP;              // output (null: not stored)
  TK gr, gc;
  Plan pl;
  const TB* Xt;        // true-residual mode: right-hand side source
  double* partials;
  CgState* st;
};

template <typename TK, typename TI>
__device__ __forceinline__ TK combine_one(TK x1, TK x2, TK gr, TK gc, bool sampled, TI pv) {
  TK out = add_rn(mul_rn(gc, x1), mul_rn(gr, x2));
  if (sampled) out = add_rn(out, static_cast<TK>(pv));
  return out;
}

template <typename TK, typename TB>
__device__ __forceinline__ void finish_reduction(double s, const Combine<TK, TB>& cb) {
  double v[1] = {s}, tot[1];
  if (grid_sum_last<1>(v, cb.partials, &cb.st->cnt[1], tot) && threadIdx.x == 0) cb.st->curv = tot[0];
}


// Loads through the L2 with an evict_last policy: the lc pass re-reads the
// whole L_c (entries) once per row band, and the streamed band and U writes
// must not push it out of L2.
__device__ __forceinline__ uint64_t l2_keep_policy() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ float ld_keep(const float* a, uint64_t pol) {
  float v;
  asm volatile("ld.global.nc.L2::cache_hint.f32 %0, [%1], %2;" : "=f"(v) : "l"(a), "l"(pol));
  return v;
}
__device__ __forceinline__ double ld_keep(const double* a, uint64_t pol) {
  double v;
  asm volatile("ld.global.nc.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(a), "l"(pol));
  return v;
}
__device__ __forceinline__ int ld_keep(const int* a, uint64_t pol) {
  int v;
  asm volatile("ld.global.nc.L2::cache_hint.s32 %0, [%1], %2;" : "=r"(v) : "l"(a), "l"(pol));
  return v;
}

// ------------------------------------------------------------------ fused apply (iterates resident in L2)
// AP = gc P Lc + gr Lr P (+ P on the sampled grid) in one pass for problems
// whose Krylov vectors stay in L2 (config 1: 10 304 x 1 000).  CTA = 512
// rows (two per thread, sharing every staged entry) x a chunk of <= 128
// columns; the L_r rows of its rows and the L_c rows of its columns are
// staged in shared memory as (value, element offset) pairs, so a gather is one
// broadcast shared load, one address add, one coalesced global load (lanes =
// consecutive rows) and one multiply-add.  Per entry the reference's order
// (decoders.cpp:160-170).  Residual mode (cb.Xt): ||b - A x||^2 instead of
// <P, AP>.
template <typename TV>
struct alignas(sizeof(TV) == 8 ? 16 : 8) OffEnt {
  TV v;
  int off;
};

template <typename TI, typename TK, typename TV, typename TB>
__global__ void __launch_bounds__(256, 4) fused_k(int p, int n, Pull<TV> Lr, Pull<TV> Lc, int cols_per_cta,
                                                 const TI* __restrict__ P, Combine<TK, TB> cb) {
  pdl_wait();  // P and the solver state come from the previous kernel on the stream
  pdl_trigger();
  if (cb.st && cb.st->done) return;
  extern __shared__ __align__(16) unsigned char smraw[];
  constexpr int RB = 512;
  const int i0 = blockIdx.x * RB;
  const int i1 = min(p, i0 + RB);
  const int cb0 = blockIdx.y * cols_per_cta;
  const int ce = min(n, cb0 + cols_per_cta);
  const i64 kr_base = Lr.rp[i0];
  const int er = static_cast<int>(Lr.rp[i1] - kr_base);
  const i64 kc_base = cb0 < ce ? Lc.rp[cb0] : 0;
  const int ec = cb0 < ce ? static_cast<int>(Lc.rp[ce] - kc_base) : 0;
  OffEnt<TV>* Er = reinterpret_cast<OffEnt<TV>*>(smraw);
  OffEnt<TV>* Ec = Er + er;
  int* crp = reinterpret_cast<int*>(Ec + ec);
  for (int k = threadIdx.x; k < er; k += blockDim.x) Er[k] = OffEnt<TV>{Lr.v[kr_base + k], Lr.ci[kr_base + k]};
  for (int k = threadIdx.x; k < ec; k += blockDim.x) Ec[k] = OffEnt<TV>{Lc.v[kc_base + k], Lc.ci[kc_base + k] * p};
  for (int q = threadIdx.x; q <= ce - cb0; q += blockDim.x) crp[q] = static_cast<int>(Lc.rp[cb0 + q] - kc_base);
  __syncthreads();
  double s = 0.0;
  const int ia = i0 + threadIdx.x, ib = ia + 256;
  const bool va = ia < p, vb = ib < p;
  if (va) {
    const int a0 = static_cast<int>(Lr.rp[ia] - kr_base), a1 = static_cast<int>(Lr.rp[ia + 1] - kr_base);
    const int b0 = vb ? static_cast<int>(Lr.rp[ib] - kr_base) : 0, b1 = vb ? static_cast<int>(Lr.rp[ib + 1] - kr_base) : 0;
    const bool sa = cb.pl.rsel[ia] >= 0, sb = vb && cb.pl.rsel[ib] >= 0;
    const TI* Pa = P + ia;
    for (int c = cb0; c < ce; ++c) {
      TK xa = TK(0), xb = TK(0);
      const int k0 = crp[c - cb0], k1 = crp[c - cb0 + 1];
#pragma unroll 4
      for (int k = k0; k < k1; ++k) {
        const OffEnt<TV> e = Ec[k];
        xa = acc<TK>(xa, static_cast<TK>(e.v), static_cast<TK>(Pa[e.off]));
        if (vb) xb = acc<TK>(xb, static_cast<TK>(e.v), static_cast<TK>(Pa[e.off + 256]));
      }
      const TI* pc = P + static_cast<i64>(c) * p;
      TK ya = TK(0), yb = TK(0);
#pragma unroll 4
      for (int k = a0; k < a1; ++k) {
        const OffEnt<TV> e = Er[k];
        ya = acc<TK>(ya, static_cast<TK>(e.v), static_cast<TK>(pc[e.off]));
      }
#pragma unroll 4
      for (int k = b0; k < b1; ++k) {
        const OffEnt<TV> e = Er[k];
        yb = acc<TK>(yb, static_cast<TK>(e.v), static_cast<TK>(pc[e.off]));
      }
      const bool cs = cb.pl.csel[c] >= 0;
      const i64 ata = ia + static_cast<i64>(c) * p;
      {
        const TI pv = pc[ia];
        const TK out = combine_one<TK>(xa, ya, cb.gr, cb.gc, sa && cs, pv);
        if (cb.Xt) {
          const double d = static_cast<double>(sub_rn(static_cast<TK>(rhs_at(cb.pl, cb.Xt, ia, c)), out));
          s += d * d;
        } else {
          cb.AP[ata] = out;
          s += static_cast<double>(pv) * static_cast<double>(out);
        }
      }
      if (vb) {
        const TI pv = pc[ib];
        const TK out = combine_one<TK>(xb, yb, cb.gr, cb.gc, sb && cs, pv);
        if (cb.Xt) {
          const double d = static_cast<double>(sub_rn(static_cast<TK>(rhs_at(cb.pl, cb.Xt, ib, c)), out));
          s += d * d;
        } else {
          cb.AP[ata + 256] = out;
          s += static_cast<double>(pv) * static_cast<double>(out);
        }
      }
    }
  }
  finish_reduction(s, cb);
}

// ------------------------------------------------------------------ slab apply (fp32 iterates, small n)
// AP = gc P Lc + gr Lr P (+ P on the sampled grid) and <P, AP> in one pass
// when a slab of 32 rows x all n columns fits in shared memory (config 1:
// 10 304 x 1 000 fp32, 125 KB).  CTA = one slab (or one of `parts` column
// ranges of it); the slab is copied once (cp.async, 16 bytes a thread).
//  * L_c: a warp works on "quads" of 4 output columns of similar degree; lane
//    (g, s) = (lane / 8, lane % 8) owns rows 4s .. 4s + 3 of column g, so one
//    entry is one 16-byte shared load of the neighbour column's segment and
//    four multiply-adds into independent sums.  A quad's entries are
//    interleaved records (64 bytes: two (value, byte offset) entries of each
//    of the 4 columns), zero padded to the longest column, streamed through
//    a 4-chunk ring of 512 bytes (one 16-byte cp.async per lane per chunk)
//    and read back by one 16-byte load per two entries (4 addresses a warp,
//    broadcast).  Quads longer than the ring allows are split into steps.
//  * The sums move to a per-warp scratch and come back lane = row for L_r,
//    the combine and the coalesced store.
//  * L_r: the rows a slab's L_r rows reference (for the pixel grid: the slab
//    and the +-w stencil rows, <= 32 aligned 16-byte chunks of a column) are
//    staged per quad into a per-warp window (one cp.async per lane per
//    column), issued after the previous quad's L_r so the copy overlaps the
//    next L_c loop; each lane keeps its row's entries in registers as
//    (value, shared address in the window).
// Per entry the reference's order (decoders.cpp:160-170).
template <typename TV>
struct alignas(sizeof(TV) == 8 ? 16 : 8) SEnt {
  TV v;
  int off;  // byte offset of the neighbour column's segment in the band / slab
};

struct SlabStep {  // 32 bytes, everything precomputed at plan time
  int rec;       // byte offset of the step's records (multiple of 64)
  int rows;      // 64-byte record rows (two entries of each column)
  int flags;     // 1: first step of its quad, 2: last, 4: its records were issued this step; bit 8 + g: column g real
  int issue_hi;  // ring chunks up to this index are issued at the start of the step
  int col[4];    // output columns (missing ones repeat a real column)
};
static_assert(sizeof(SlabStep) == 32, "SlabStep is one 32-byte record");

struct SlabPlan {
  const unsigned char* rec;  // interleaved (value, byte offset) records
  const SlabStep* steps;
  const int* wsteps;  // [parts][kSlabWarps + 1] step ranges (indices into steps)
  int max_steps;      // steps of the largest part (their shared-memory copy)
  const int* win;     // [slabs][32]: first row (relative to the slab) of each window chunk, or kNoChunk
  const float* lv;    // [EVR][p]: L_r row entries, zero padded
  const int* lo;      // [EVR][p]: byte offset of the entry's row in a column's window
};

constexpr int kSlabWarps = 16;
constexpr int kSlabThreads = kSlabWarps * 32;
constexpr int kSlabRing = 4;  // 512-byte record chunks per warp
constexpr int kNoChunk = 0x40000000;
constexpr size_t kSlabWarpBytes = kSlabRing * 512 + 4 * 512 + 1024;  // ring, 4 windows, scratch

__device__ __forceinline__ void cp_async16(unsigned dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ float lds_f32(unsigned a) {
  float v;
  asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ float4 lds_f128(unsigned a) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a));
  return v;
}
__device__ __forceinline__ int4 lds_i128(unsigned a) {
  int4 v;
  asm volatile("ld.shared.v4.s32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a));
  return v;
}

// O32: p n < 2^31, element offsets in 32 bits (no 64-bit multiplies per column).
template <typename TK, int EVR, bool kResid, typename TB, bool O32 = false>
__global__ void __launch_bounds__(kSlabThreads, 1) slab_k(int p, int n, int parts, SlabPlan sp,
                                                           const float* __restrict__ P, Combine<TK, TB> cb) {
  pdl_wait();  // P and the solver state come from the previous kernel on the stream
  pdl_trigger();
  if (cb.st && cb.st->done) return;
  auto colp = [p](int c) -> i64 {
    if constexpr (O32)
      return static_cast<i64>(static_cast<unsigned>(c) * static_cast<unsigned>(p));
    else
      return static_cast<i64>(c) * p;
  };
  extern __shared__ __align__(16) unsigned char smraw[];
  float* Pb = reinterpret_cast<float*>(smraw);  // [n][32]
  const unsigned sbase = static_cast<unsigned>(__cvta_generic_to_shared(Pb));
  const unsigned stbase = sbase + static_cast<unsigned>(static_cast<size_t>(n) * 128);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g4 = lane >> 3, s4 = lane & 7;  // quad layout: column g4, rows 4 s4 .. 4 s4 + 3
  const unsigned wbase = stbase + static_cast<unsigned>(sp.max_steps) * 32u +
                         static_cast<unsigned>(warp) * static_cast<unsigned>(kSlabWarpBytes);
  const unsigned rbase = wbase, hbase = wbase + kSlabRing * 512, xbase = hbase + 4 * 512;
  // persistent: this CTA's contiguous range of (slab, column part) items; the
  // slab is copied again only when the slab changes
  const int items = ((p + 31) / 32) * parts;
  const int ia = static_cast<int>(static_cast<i64>(items) * blockIdx.x / gridDim.x);
  const int ib = static_cast<int>(static_cast<i64>(items) * (blockIdx.x + 1) / gridDim.x);
  double s = 0.0;
  int cur_slab = -1, i0 = 0, rows = 0, i = 0;
  bool vrow = false, wcopy = false, rs = false;
  float lv[EVR];
  unsigned lo[EVR];  // shared address of the entry's row in window 0
  const float* wsrc = P;
  TK* APi = nullptr;
  for (int item = ia; item < ib; ++item) {
  const int slab = item / parts, part = item % parts;
  __syncthreads();  // the previous item is done with the slab, steps, rings and windows
  if (slab != cur_slab) {
    cur_slab = slab;
    i0 = slab * 32;
    rows = min(32, p - i0);
    if (rows == 32) {
      for (int q = threadIdx.x; q < n * 8; q += kSlabThreads)
        cp_async16(sbase + static_cast<unsigned>(q) * 16u, P + colp(q >> 3) + i0 + (q & 7) * 4);
      asm volatile("cp.async.commit_group;" ::: "memory");
    } else {
      for (int q = threadIdx.x; q < n * 32; q += kSlabThreads) {
        const int c = q >> 5, r = q & 31;
        Pb[q] = r < rows ? P[colp(c) + i0 + r] : 0.f;
      }
    }
    vrow = lane < rows;
    i = i0 + (vrow ? lane : 0);
#pragma unroll
    for (int e = 0; e < EVR; ++e) {
      lv[e] = vrow ? sp.lv[static_cast<i64>(e) * p + i] : 0.f;
      lo[e] = hbase + (vrow ? static_cast<unsigned>(sp.lo[static_cast<i64>(e) * p + i]) : 0u);
    }
    const int wrow = sp.win[slab * 32 + lane];  // this lane's window chunk (rows wrow .. wrow + 3)
    wcopy = wrow != kNoChunk;
    wsrc = P + i0 + (wcopy ? wrow : 0);
    rs = vrow && cb.pl.rsel[i] >= 0;
    if constexpr (!kResid) APi = cb.AP + i;
  }
  // the part's step list next to the slab
  const int pst0 = sp.wsteps[part * (kSlabWarps + 1)], pst1 = sp.wsteps[part * (kSlabWarps + 1) + kSlabWarps];
  {
    const unsigned char* src = reinterpret_cast<const unsigned char*>(sp.steps + pst0);
    for (int q = threadIdx.x; q < (pst1 - pst0) * 2; q += kSlabThreads) cp_async16(stbase + q * 16u, src + q * 16);
    asm volatile("cp.async.commit_group;" ::: "memory");
  }
  const SlabStep* S = reinterpret_cast<const SlabStep*>(smraw + (stbase - sbase)) - pst0;  // indexed by step
  const int st0 = sp.wsteps[part * (kSlabWarps + 1) + warp], st1 = sp.wsteps[part * (kSlabWarps + 1) + warp + 1];
  asm volatile("cp.async.wait_all;" ::: "memory");
  __syncthreads();
  if (st0 < st1) {
    unsigned issued = static_cast<unsigned>(S[st0].rec) / 512u;
    const unsigned char* gsrc = sp.rec + lane * 16;
    auto window = [&](const SlabStep& q) {  // the quad's L_r windows (one commit group)
      if (wcopy)
#pragma unroll
        for (int g = 0; g < 4; ++g) cp_async16(hbase + g * 512 + lane * 16, wsrc + colp(q.col[g]));
      asm volatile("cp.async.commit_group;" ::: "memory");
    };
    window(S[st0]);
    float4 acc4 = make_float4(0.f, 0.f, 0.f, 0.f);
    TK accd[4] = {TK(0), TK(0), TK(0), TK(0)};
    for (int st = st0; st < st1; ++st) {
      const SlabStep cur = S[st];
      int csq[4];  // plan positions of the quad's columns, loaded ahead of the combine
#pragma unroll
      for (int g = 0; g < 4; ++g) csq[g] = cb.pl.csel[cur.col[g]];
      __syncwarp();  // ring chunks of earlier steps are free
      for (; static_cast<int>(issued) <= cur.issue_hi; ++issued)
        cp_async16(rbase + (issued % kSlabRing) * 512u + lane * 16u, gsrc + static_cast<i64>(issued) * 512);
      asm volatile("cp.async.commit_group;" ::: "memory");
      if (cur.flags & 4)
        asm volatile("cp.async.wait_group 0;" ::: "memory");
      else
        asm volatile("cp.async.wait_group 2;" ::: "memory");
      __syncwarp();
      // L_c: record rows of this step
      const unsigned rb0 = rbase + g4 * 16;
#pragma unroll 4
      for (int k = 0; k < cur.rows; ++k) {
        const unsigned rb = static_cast<unsigned>(cur.rec + k * 64);
        const int4 e = lds_i128(rb0 + (rb % (kSlabRing * 512u)));
        const float4 x0 = lds_f128(sbase + static_cast<unsigned>(e.y) + s4 * 16);
        const float4 x1 = lds_f128(sbase + static_cast<unsigned>(e.w) + s4 * 16);
        const float v0 = __int_as_float(e.x), v1 = __int_as_float(e.z);
        if constexpr (sizeof(TK) == 4) {
          acc4.x = fmaf(v0, x0.x, acc4.x);
          acc4.y = fmaf(v0, x0.y, acc4.y);
          acc4.z = fmaf(v0, x0.z, acc4.z);
          acc4.w = fmaf(v0, x0.w, acc4.w);
          acc4.x = fmaf(v1, x1.x, acc4.x);
          acc4.y = fmaf(v1, x1.y, acc4.y);
          acc4.z = fmaf(v1, x1.z, acc4.z);
          acc4.w = fmaf(v1, x1.w, acc4.w);
        } else {
          accd[0] = acc<TK>(accd[0], v0, x0.x);
          accd[1] = acc<TK>(accd[1], v0, x0.y);
          accd[2] = acc<TK>(accd[2], v0, x0.z);
          accd[3] = acc<TK>(accd[3], v0, x0.w);
          accd[0] = acc<TK>(accd[0], v1, x1.x);
          accd[1] = acc<TK>(accd[1], v1, x1.y);
          accd[2] = acc<TK>(accd[2], v1, x1.z);
          accd[3] = acc<TK>(accd[3], v1, x1.w);
        }
      }
      if (cur.flags & 2) {
        // sums to lane = row through the scratch
        TK a[4];
        if constexpr (sizeof(TK) == 4) {
          asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(xbase + g4 * 128 + s4 * 16), "f"(acc4.x),
                       "f"(acc4.y), "f"(acc4.z), "f"(acc4.w)
                       : "memory");
          __syncwarp();
#pragma unroll
          for (int g = 0; g < 4; ++g) a[g] = lds_f32(xbase + g * 128 + lane * 4);
        } else {
          TK* X = reinterpret_cast<TK*>(smraw + (xbase - sbase));  // 4 x 32 sums
#pragma unroll
          for (int t = 0; t < 4; ++t) X[g4 * 32 + s4 * 4 + t] = accd[t];
          __syncwarp();
#pragma unroll
          for (int g = 0; g < 4; ++g) a[g] = X[g * 32 + lane];
        }
        asm volatile("cp.async.wait_group 1;" ::: "memory");  // this quad's windows
        __syncwarp();
        TK y[4] = {TK(0), TK(0), TK(0), TK(0)};
#pragma unroll
        for (int e = 0; e < EVR; ++e)
#pragma unroll
          for (int g = 0; g < 4; ++g) y[g] = acc<TK>(y[g], static_cast<TK>(lv[e]), static_cast<TK>(lds_f32(lo[e] + g * 512)));
#pragma unroll
        for (int g = 0; g < 4; ++g) {
          const bool real = vrow && ((cur.flags >> (8 + g)) & 1);
          const float pv = lds_f32(sbase + static_cast<unsigned>(cur.col[g] * 32 + lane) * 4u);
          const TK out = combine_one<TK>(a[g], y[g], cb.gr, cb.gc, rs && csq[g] >= 0, pv);
          if constexpr (kResid) {
            const double d = real ? static_cast<double>(sub_rn(static_cast<TK>(rhs_at(cb.pl, cb.Xt, i, cur.col[g])), out))
                                  : 0.0;
            s += d * d;
          } else {
            if (real) APi[colp(cur.col[g])] = out;
            s += real ? static_cast<double>(pv) * static_cast<double>(out) : 0.0;
          }
        }
        __syncwarp();  // windows and scratch are free
        if (st + 1 < st1) window(S[st + 1]);
        else asm volatile("cp.async.commit_group;" ::: "memory");
        acc4 = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
        for (int t = 0; t < 4; ++t) accd[t] = TK(0);
      } else {
        asm volatile("cp.async.commit_group;" ::: "memory");  // keep two groups per step
      }
      issued = max(issued, static_cast<unsigned>(cur.issue_hi + 1));
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
  }
  }  // items
  finish_reduction(s, cb);
}

// ------------------------------------------------------------------ lc pass, band in shared memory
// One CTA per band of S = 128 B / sizeof(TI) rows: the band's segment of all
// n_local columns (n x 128 B) is copied to shared memory once.  A (half) warp
// of S lanes (lane = row of the band) owns a contiguous range of output
// columns; the L_c row of each column is staged as (value, byte offset of the
// neighbour's band segment) in a per-worker double buffer, loaded while the
// previous column is gathered, then read back by broadcast 16-byte loads, so
// an entry costs one gather, one add and one multiply-add.  Rows are padded
// in the buffer to a multiple of 4 with zero entries pointing at column 0
// (a zero product leaves the sum unchanged; CSR order is kept).
template <typename TV>
__device__ __forceinline__ void lds_ent4(const SEnt<TV>* e, TV (&v)[4], int (&o)[4]) {
  if constexpr (sizeof(TV) == 4) {
    const int4 a = reinterpret_cast<const int4*>(e)[0], b = reinterpret_cast<const int4*>(e)[1];
    v[0] = __int_as_float(a.x);
    o[0] = a.y;
    v[1] = __int_as_float(a.z);
    o[1] = a.w;
    v[2] = __int_as_float(b.x);
    o[2] = b.y;
    v[3] = __int_as_float(b.z);
    o[3] = b.w;
  } else {
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int4 a = reinterpret_cast<const int4*>(e)[u];
      v[u] = __hiloint2double(a.y, a.x);
      o[u] = a.z;
    }
  }
}

constexpr int kLcSmemThreads = 1024;
template <typename TI, typename TV>
constexpr size_t lc_smem_ent_bytes() {
  return static_cast<size_t>(kLcSmemThreads / 32) * (32 / (128 / sizeof(TI))) * 2 * 32 * sizeof(SEnt<TV>);
}

template <typename TI, typename TK, typename TV, bool kCombine, typename TB>
__global__ void __launch_bounds__(kLcSmemThreads) lc_smem_k(int p, int ncols, int nload, Pull<TV> L,
                                                            const TI* __restrict__ P, TK* __restrict__ U,
                                                            i64 col_base, Combine<TK, TB> cb) {
  constexpr int S = 128 / sizeof(TI);
  constexpr int G = 32 / S;
  extern __shared__ __align__(16) unsigned char smraw[];
  TI* Pb = reinterpret_cast<TI*>(smraw);  // [nload][S]
  SEnt<TV>* ents = reinterpret_cast<SEnt<TV>*>(smraw + ((static_cast<size_t>(nload) * 128 + 15) / 16) * 16);
  if (cb.st && cb.st->done) return;
  const int i0 = blockIdx.x * S;
  const int rows = min(S, p - i0);
  const bool vec = rows == S && (reinterpret_cast<uintptr_t>(P) % 16 == 0) &&
                   ((static_cast<i64>(p) * sizeof(TI)) % 16 == 0);
  if (vec) {
    constexpr int CH = 128 / 16;
    const unsigned sbase = static_cast<unsigned>(__cvta_generic_to_shared(Pb));
    for (int q = threadIdx.x; q < nload * CH; q += blockDim.x) {
      const int c = q / CH, k = q % CH;
      const TI* src = P + static_cast<i64>(c) * p + i0 + k * (16 / sizeof(TI));
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sbase + static_cast<unsigned>(q) * 16u),
                   "l"(src)
                   : "memory");
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  } else {
    for (int q = threadIdx.x; q < nload * S; q += blockDim.x) {
      const int c = q / S, r = q % S;
      Pb[q] = r < rows ? P[static_cast<i64>(c) * p + i0 + r] : TI(0);
    }
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  const int half = lane / S, r = lane % S;
  const unsigned hmask = S == 32 ? 0xffffffffu : (0xffffu << (16 * half));
  const bool vrow = r < rows;
  const i64 i = i0 + (vrow ? r : 0);
  const unsigned char* Prb = reinterpret_cast<const unsigned char*>(Pb + r);
  const int nwk = nwarps * G, wk = warp * G + half;
  const int wa = static_cast<int>((static_cast<i64>(ncols) * wk) / nwk);
  const int wb = static_cast<int>((static_cast<i64>(ncols) * (wk + 1)) / nwk);
  SEnt<TV>* buf = ents + static_cast<size_t>(wk) * 64;
  constexpr int kSegBytes = S * static_cast<int>(sizeof(TI));
  // stage column c's first 32 entries (padded to a multiple of 4) into buf[b]
  auto stage = [&](int b, i64 k0, int deg, TV v0, int j0, TV v1, int j1) {
    const int dp = min(32, (deg + 3) & ~3);
    SEnt<TV>* d = buf + b * 32;
    if (r < dp) d[r] = SEnt<TV>{r < deg ? v0 : TV(0), r < deg ? j0 * kSegBytes : 0};
    if (r + S < dp) d[r + S] = SEnt<TV>{r + S < deg ? v1 : TV(0), r + S < deg ? j1 * kSegBytes : 0};
  };
  auto load = [&](i64 k0, int deg, TV& v0, int& j0, TV& v1, int& j1) {
    v0 = TV(0), v1 = TV(0), j0 = 0, j1 = 0;
    if (r < deg) {
      v0 = L.v[k0 + r];
      j0 = L.ci[k0 + r];
    }
    if (r + S < deg && r + S < 32) {
      v1 = L.v[k0 + r + S];
      j1 = L.ci[k0 + r + S];
    }
  };
  if (vec) asm volatile("cp.async.wait_all;" ::: "memory");
  __syncthreads();
  double s = 0.0;
  for (int c0 = wa; c0 < wb; c0 += S) {
    const int cnt = min(S, wb - c0);
    const i64 kst_l = r < cnt ? L.rp[c0 + r] : 0;
    const i64 ken_l = r < cnt ? L.rp[c0 + r + 1] : 0;
    i64 k0 = __shfl_sync(hmask, kst_l, 0, S);
    int deg = static_cast<int>(__shfl_sync(hmask, ken_l, 0, S) - k0);
    {
      TV v0, v1;
      int j0, j1;
      load(k0, deg, v0, j0, v1, j1);
      stage(0, k0, deg, v0, j0, v1, j1);
    }
    __syncwarp(hmask);
    int b = 0;
    for (int cc = 0; cc < cnt; ++cc) {
      i64 k0n = 0;
      int degn = 0;
      TV v0n = TV(0), v1n = TV(0);
      int j0n = 0, j1n = 0;
      if (cc + 1 < cnt) {
        k0n = __shfl_sync(hmask, kst_l, cc + 1, S);
        degn = static_cast<int>(__shfl_sync(hmask, ken_l, cc + 1, S) - k0n);
        load(k0n, degn, v0n, j0n, v1n, j1n);
      }
      TK a = TK(0);
      const SEnt<TV>* e = buf + b * 32;
      const int dp = min(32, (deg + 3) & ~3);
      for (int t = 0; t < dp; t += 4) {
        TV v[4];
        int o[4];
        lds_ent4(e + t, v, o);
        TI x[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) x[u] = *reinterpret_cast<const TI*>(Prb + o[u]);
#pragma unroll
        for (int u = 0; u < 4; ++u) a = acc<TK>(a, static_cast<TK>(v[u]), static_cast<TK>(x[u]));
      }
      for (int t0 = 32; t0 < deg; t0 += S) {  // hub columns beyond the buffer: shuffle path
        TV vc = TV(0);
        int jc = 0;
        if (t0 + r < deg) {
          vc = L.v[k0 + t0 + r];
          jc = L.ci[k0 + t0 + r];
        }
        const int dn = min(S, deg - t0);
        for (int t = 0; t < dn; ++t) {
          const TV v = __shfl_sync(hmask, vc, t, S);
          const int j = __shfl_sync(hmask, jc, t, S);
          a = acc<TK>(a, static_cast<TK>(v), static_cast<TK>(Pb[j * S + r]));
        }
      }
      const int c = c0 + cc;
      if (vrow) {
        const i64 at = i + static_cast<i64>(c) * p;
        if constexpr (kCombine) {
          const bool sampled = cb.pl.rsel[i] >= 0 && cb.pl.csel[col_base + c] >= 0;
          const TI pv = Pb[c * S + r];
          const TK out = combine_one<TK>(a, cb.other[at], cb.gr, cb.gc, sampled, pv);
          if (cb.AP) cb.AP[at] = out;
          s += static_cast<double>(pv) * static_cast<double>(out);
        } else {
          U[at] = a;
        }
      }
      if (cc + 1 < cnt) {
        stage(b ^ 1, k0n, degn, v0n, j0n, v1n, j1n);
        __syncwarp(hmask);
      }
      b ^= 1;
      k0 = k0n;
      deg = degn;
    }
  }
  if constexpr (kCombine) finish_reduction(s, cb);
}

// ------------------------------------------------------------------ lc pass, band resident in L2
// U = P Lc when the band of all columns does not fit in shared memory
// (config 3/4): bands of 32 rows, the grid band-major (blockIdx.x = band *
// chunks + chunk) so the CTAs in flight share one band of 32 rows x all
// columns (<= 51 MB in fp64), which stays resident in L2; lane = row, one
// warp per output column, each gather a 128/256-byte line group.  Each warp
// owns a contiguous range of columns: the row pointers of 32 columns at a time
// sit one per lane, and the L_c row of the next column is loaded (one entry
// per lane, two slots, with an L2 evict_last policy so the whole L_c stays
// cached across bands) while the current one is gathered in batches of 8
// independent loads; entries are broadcast by shuffle, accumulated in CSR
// order.
template <typename TI, typename TK, typename TV, bool kCombine, typename TB>
__global__ void __launch_bounds__(256, 4) lc_k(int p, int ncols, int chunks, int cpc, Pull<TV> L,
                                            const TI* __restrict__ P, TK* __restrict__ U, i64 col_base,
                                            Combine<TK, TB> cb) {
  if (cb.st && cb.st->done) return;
  const int band = blockIdx.x / chunks, chunk = blockIdx.x % chunks;
  const int i0 = band * 32;
  const int rows = min(32, p - i0);
  const int r = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  const bool vrow = r < rows;
  const i64 i = i0 + (vrow ? r : 0);
  const TI* Pr = P + i;
  const i64 jstride = p;
  const int ca0 = chunk * cpc, ca1 = min(ncols, ca0 + cpc);
  const uint64_t keep = l2_keep_policy();
  auto ldv = [&](i64 k) { return ld_keep(L.v + k, keep); };
  auto ldj = [&](i64 k) { return ld_keep(L.ci + k, keep); };
  const int wa = ca0 + static_cast<int>((static_cast<i64>(ca1 - ca0) * warp) / nwarps);
  const int wb = ca0 + static_cast<int>((static_cast<i64>(ca1 - ca0) * (warp + 1)) / nwarps);
  double s = 0.0;
  for (int c0 = wa; c0 < wb; c0 += 32) {
    const int cnt = min(32, wb - c0);
    const i64 kst_l = r < cnt ? L.rp[c0 + r] : 0;
    const i64 ken_l = r < cnt ? L.rp[c0 + r + 1] : 0;
    i64 k0 = __shfl_sync(0xffffffffu, kst_l, 0);
    int deg = static_cast<int>(__shfl_sync(0xffffffffu, ken_l, 0) - k0);
    TV va = TV(0), vb = TV(0);
    int ja = 0, jb = 0;
    if (r < deg) {
      va = ldv(k0 + r);
      ja = ldj(k0 + r);
    }
    if (r + 32 < deg) {
      vb = ldv(k0 + r + 32);
      jb = ldj(k0 + r + 32);
    }
    for (int cc = 0; cc < cnt; ++cc) {
      i64 k0n = 0;
      int degn = 0;
      TV van = TV(0), vbn = TV(0);
      int jan = 0, jbn = 0;
      if (cc + 1 < cnt) {
        k0n = __shfl_sync(0xffffffffu, kst_l, cc + 1);
        degn = static_cast<int>(__shfl_sync(0xffffffffu, ken_l, cc + 1) - k0n);
        if (r < degn) {
          van = ldv(k0n + r);
          jan = ldj(k0n + r);
        }
        if (r + 32 < degn) {
          vbn = ldv(k0n + r + 32);
          jbn = ldj(k0n + r + 32);
        }
      }
      TK a = TK(0);
      auto slot = [&](TV vs, int js, int cnt_s) {
        for (int t0 = 0; t0 < cnt_s; t0 += 8) {
          TV v[8];
          TI x[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            v[u] = __shfl_sync(0xffffffffu, vs, (t0 + u) & 31);
            const int j = __shfl_sync(0xffffffffu, js, (t0 + u) & 31);
            x[u] = __ldg(Pr + j * jstride);
          }
#pragma unroll
          for (int u = 0; u < 8; ++u)
            if (t0 + u < cnt_s) a = acc<TK>(a, static_cast<TK>(v[u]), static_cast<TK>(x[u]));
        }
      };
      slot(va, ja, min(deg, 32));
      if (deg > 32) slot(vb, jb, min(deg, 64) - 32);
      for (int t0 = 64; t0 < deg; t0 += 32) {  // hub columns: further slots on demand
        TV vc = TV(0);
        int jc = 0;
        if (t0 + r < deg) {
          vc = ldv(k0 + t0 + r);
          jc = ldj(k0 + t0 + r);
        }
        slot(vc, jc, min(32, deg - t0));
      }
      const int c = c0 + cc;
      if (vrow) {
        const i64 at = i + static_cast<i64>(c) * p;
        if constexpr (kCombine) {
          const bool sampled = cb.pl.rsel[i] >= 0 && cb.pl.csel[col_base + c] >= 0;
          const TI pv = P[at];
          const TK out = combine_one<TK>(a, cb.other[at], cb.gr, cb.gc, sampled, pv);
          if (cb.AP) cb.AP[at] = out;
          s += static_cast<double>(pv) * static_cast<double>(out);
        } else {
          __stcs(U + at, a);  // streamed: keep the L2 for the band
        }
      }
      k0 = k0n;
      deg = degn;
      va = van;
      vb = vbn;
      ja = jan;
      jb = jbn;
    }
  }
  if constexpr (kCombine) finish_reduction(s, cb);
}

// ------------------------------------------------------------------ lr pass
// CTA = (row range, tile of C columns).  The rows the range's L_r entries
// reference, [w0, w1), of the C columns are staged in shared memory as one
// C-wide record per row; each thread takes rows of the range (in `order`,
// degree-sorted for hub-heavy graphs so a warp's rows have similar length),
// streams its row's L_r entries once for all C columns and gathers the C-wide
// records.  kCombine: AP = gc U + gr (Lr P) (+ P), <P, AP>; otherwise the x2
// sums go to U (the lc pass combines).
struct RowRange {
  int r0, r1;  // positions in `order`
  int w0, w1;  // staged rows
};

template <typename TI, int C>
struct alignas(C * sizeof(TI) >= 16 ? 16 : C * sizeof(TI)) Rec {
  TI v[C];
};

template <typename TI, typename TK, typename TV, int C, bool kCombine, typename TB>
__global__ void __launch_bounds__(512) lr_k(int p, int ncols, const RowRange* __restrict__ ranges,
                                            const int* __restrict__ order, Pull<TV> Lr, const TI* __restrict__ P,
                                            TK* __restrict__ U, i64 col_base, Combine<TK, TB> cb) {
  if (cb.st && cb.st->done) return;
  extern __shared__ __align__(16) unsigned char smraw[];
  Rec<TI, C>* W = reinterpret_cast<Rec<TI, C>*>(smraw);
  const RowRange rr = ranges[blockIdx.y];
  const int c0 = blockIdx.x * C;
  const int nw = rr.w1 - rr.w0;
  for (int q = threadIdx.x; q < nw; q += blockDim.x) {
    Rec<TI, C> rec;
#pragma unroll
    for (int cc = 0; cc < C; ++cc)
      rec.v[cc] = (c0 + cc < ncols) ? P[rr.w0 + q + static_cast<i64>(c0 + cc) * p] : TI(0);
    W[q] = rec;
  }
  __syncthreads();
  double s = 0.0;
  for (int t = rr.r0 + threadIdx.x; t < rr.r1; t += blockDim.x) {
    const int i = order ? order[t] : t;
    const i64 k0 = Lr.rp[i], k1 = Lr.rp[i + 1];
    TK a[C];
#pragma unroll
    for (int cc = 0; cc < C; ++cc) a[cc] = TK(0);
#pragma unroll 4
    for (i64 k = k0; k < k1; ++k) {
      const TK v = static_cast<TK>(Lr.v[k]);
      const Rec<TI, C> x = W[Lr.ci[k] - rr.w0];
#pragma unroll
      for (int cc = 0; cc < C; ++cc) a[cc] = acc<TK>(a[cc], v, static_cast<TK>(x.v[cc]));
    }
    const bool rs = cb.pl.rsel ? cb.pl.rsel[i] >= 0 : false;
    const Rec<TI, C> own = W[i - rr.w0];
#pragma unroll
    for (int cc = 0; cc < C; ++cc) {
      const int c = c0 + cc;
      if (c >= ncols) break;
      const i64 at = i + static_cast<i64>(c) * p;
      if constexpr (kCombine) {
        const bool sampled = rs && cb.pl.csel[col_base + c] >= 0;
        const TK out = combine_one<TK>(cb.other[at], a[cc], cb.gr, cb.gc, sampled, own.v[cc]);
        if (cb.Xt) {
          const double e = static_cast<double>(sub_rn(static_cast<TK>(rhs_at(cb.pl, cb.Xt, i, col_base + c)), out));
          s += e * e;
        } else {
          if (cb.AP) cb.AP[at] = out;
          s += static_cast<double>(own.v[cc]) * static_cast<double>(out);
        }
      } else {
        U[at] = a[cc];
      }
    }
  }
  if constexpr (kCombine) finish_reduction(s, cb);
}

// ------------------------------------------------------------------ lr pass, register-resident rows
// The rows of L_r (in natural order, or degree-sorted for hub-heavy graphs)
// are cut into "vrows" of at most EV entries (hub rows span several), packed
// into groups of at most T vrows; thread t of a CTA keeps vrow t of its group
// in registers for the whole kernel (ELL-interleaved, zero-padded).  A CTA =
// (group, column stripe) walks the stripe's tiles of C columns: the group's
// window of rows [w0, w1) of the tile is staged in shared memory (column-major,
// cp.async, double buffered), every thread gathers its EV entries from it,
// split rows add their vrows' partial sums in order, and the row's output is
// combined.  Each L_r entry is read from HBM once per kernel, not once per
// column tile.  Unsplit rows keep the CSR order exactly (fp64 bit-identical);
// split rows (fp32 data only) sum chunk partials.
struct LrGroup {
  int v0, nv;  // first vrow, vrow count (<= T)
  int w0, wl;  // staged rows [w0, w0 + wl), w0 aligned to 16 bytes
  int split;   // any row of the group spans several vrows
};

// Stages rows [w0, w0 + wl) of the C columns [c0, c0 + C) as one C-wide
// record per row (element-sized cp.async copies, so the copy stays
// asynchronous while the layout turns row-major): a gather then reads all C
// columns of a row with one 8/16-byte shared load, which halves the bank
// conflicts of random 8-byte reads.
template <typename TI, int C>
__device__ __forceinline__ void stage_tile(Rec<TI, C>* W, int wl, const TI* __restrict__ P, i64 p, int w0, int c0,
                                           int ncols) {
  const unsigned sb = static_cast<unsigned>(__cvta_generic_to_shared(W));
  for (int q = threadIdx.x; q < C * wl; q += blockDim.x) {
    const int cc = q / wl, k = q % wl;
    const unsigned dst = sb + static_cast<unsigned>((k * C + cc) * sizeof(TI));
    const int col = min(c0 + cc, ncols - 1);  // columns past the end: a valid duplicate, never combined
    const TI* src = P + static_cast<i64>(col) * p + w0 + k;
    if constexpr (sizeof(TI) == 8)
      asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(dst), "l"(src) : "memory");
    else
      asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(dst), "l"(src) : "memory");
  }
  asm volatile("cp.async.commit_group;" ::: "memory");
}

template <typename TI, typename TK, typename TV, int C, int EV, int T, bool kCombine, typename TB>
__global__ void __launch_bounds__(T, 1) lr_reg_k(int p, int ncols, int stripes, const LrGroup* __restrict__ groups,
                                                 const int* __restrict__ vrow_row, const int* __restrict__ vrow_np,
                                                 const TV* __restrict__ ev, const int* __restrict__ ej, int wl_max,
                                                 const TI* __restrict__ P, TK* __restrict__ U, i64 col_base,
                                                 Combine<TK, TB> cb) {
  if (cb.st && cb.st->done) return;
  extern __shared__ __align__(16) unsigned char smraw[];
  const int g = blockIdx.x / stripes, stripe = blockIdx.x % stripes;
  const LrGroup gr = groups[g];
  Rec<TI, C>* W0 = reinterpret_cast<Rec<TI, C>*>(smraw);
  Rec<TI, C>* W1 = W0 + wl_max;
  TK* part = reinterpret_cast<TK*>(W1 + wl_max);  // [T][C] when split
  const int t = threadIdx.x;
  const bool active = t < gr.nv;
  TV v[EV];
  int jj[EV];
#pragma unroll
  for (int e = 0; e < EV; ++e) {
    const i64 at = (static_cast<i64>(g) * EV + e) * T + t;
    v[e] = ev[at];
    jj[e] = ej[at];
  }
  const int row = active ? vrow_row[gr.v0 + t] : 0;
  const int np = active ? vrow_np[gr.v0 + t] : 0;  // parts of a leader vrow, 0 for a follower
  const bool rs = active && np > 0 && cb.pl.rsel[row] >= 0;
  const int ntiles = (ncols + C - 1) / C;
  double s = 0.0;
  int tile = stripe;
  if (tile < ntiles) stage_tile<TI, C>(W0, gr.wl, P, p, gr.w0, tile * C, ncols);
  int b = 0;
  for (; tile < ntiles; tile += stripes, b ^= 1) {
    const Rec<TI, C>* W = b ? W1 : W0;
    const int nxt = tile + stripes;
    if (nxt < ntiles) {
      stage_tile<TI, C>(b ? W0 : W1, gr.wl, P, p, gr.w0, nxt * C, ncols);
      asm volatile("cp.async.wait_group 1;" ::: "memory");
    } else {
      asm volatile("cp.async.wait_group 0;" ::: "memory");
    }
    __syncthreads();
    const int c0 = tile * C;
    TK o[C];  // the other pass's sums for this row, loaded ahead of the gathers
    if constexpr (kCombine) {
#pragma unroll
      for (int cc = 0; cc < C; ++cc)
        o[cc] = (np > 0 && c0 + cc < ncols) ? cb.other[row + static_cast<i64>(c0 + cc) * p] : TK(0);
    }
    TK a[C];
#pragma unroll
    for (int cc = 0; cc < C; ++cc) a[cc] = TK(0);
#pragma unroll
    for (int e = 0; e < EV; ++e) {
      const Rec<TI, C> x = W[jj[e]];
#pragma unroll
      for (int cc = 0; cc < C; ++cc) a[cc] = acc<TK>(a[cc], static_cast<TK>(v[e]), static_cast<TK>(x.v[cc]));
    }
    if (gr.split) {
#pragma unroll
      for (int cc = 0; cc < C; ++cc) part[t * C + cc] = a[cc];
      __syncthreads();
      if (np > 1)
        for (int q = 1; q < np; ++q)
#pragma unroll
          for (int cc = 0; cc < C; ++cc) a[cc] = add_rn(a[cc], part[(t + q) * C + cc]);
    }
    if (np > 0) {
#pragma unroll
      for (int cc = 0; cc < C; ++cc) {
        const int c = c0 + cc;
        if (c >= ncols) break;
        const i64 at = row + static_cast<i64>(c) * p;
        if constexpr (kCombine) {
          const TI pv = W[row - gr.w0].v[cc];
          const bool sampled = rs && cb.pl.csel[col_base + c] >= 0;
          const TK out = combine_one<TK>(o[cc], a[cc], cb.gr, cb.gc, sampled, pv);
          if (cb.Xt) {
            const double d = static_cast<double>(sub_rn(static_cast<TK>(rhs_at(cb.pl, cb.Xt, row, col_base + c)), out));
            s += d * d;
          } else {
            if (cb.AP) cb.AP[at] = out;
            s += static_cast<double>(pv) * static_cast<double>(out);
          }
        } else {
          U[at] = a[cc];
        }
      }
    }
    __syncthreads();  // the buffer is restaged two tiles on
  }
  if constexpr (kCombine) finish_reduction(s, cb);
}

// ------------------------------------------------------------------ CG vector kernels
// x = 0, r = p = b over columns [0, ncols) (global column col_base + c);
// rho = ||b||^2 (a partial sum when `partial`: the sharded caller
// all-reduces it and calls cg_start_k).
template <typename TK, typename TX, typename TB>
__global__ void cg_init_k(i64 p, i64 ncols, i64 col_base, Plan pl, const TB* __restrict__ Xt, TX* __restrict__ X,
                          TK* __restrict__ R, TK* __restrict__ P, double* partials, CgState* st) {
  double s[1] = {0.0};
  const i64 N = p * ncols;
  for (i64 q = blockIdx.x * (i64)blockDim.x + threadIdx.x; q < N; q += (i64)gridDim.x * blockDim.x) {
    const i64 c = q / p, i = q - c * p;
    const TK b = static_cast<TK>(rhs_at(pl, Xt, i, col_base + c));
    X[q] = TX(0);
    R[q] = b;
    P[q] = b;
    s[0] += static_cast<double>(b) * static_cast<double>(b);
  }
  double tot[1];
  if (grid_sum_last<1>(s, partials, &st->cnt[0], tot) && threadIdx.x == 0) st->rho = tot[0];
}

// pcg_core's set-up after ||b||^2 is known (solvers.hpp:38-50).
static __global__ void cg_start_k(CgState* st, double tol, i64 max_iter) {
  const double nb = sqrt(st->rho);
  st->norm_b = nb;
  st->it = 0;
  st->max_iter = max_iter;
  if (nb == 0.0) {
    st->zero_rhs = 1;
    st->done = 1;
    return;
  }
  st->target = tol * nb;
  if (nb <= st->target || max_iter <= 0) st->done = 1;
}

// 16-byte vectors of the iterates (W entries of T).
template <typename T>
struct V16;
template <>
struct V16<float> {
  using V = float4;
  static constexpr int W = 4;
};
template <>
struct V16<double> {
  using V = double2;
  static constexpr int W = 2;
};
template <typename T, typename V>
__device__ __forceinline__ T& lane_of(V& v, int k) {
  return reinterpret_cast<T*>(&v)[k];
}

// alpha = rho / <P, AP> (breakdown check, solvers.hpp:53-57); R -= alpha AP;
// rho_next = ||R||^2.  The element loops are device functions shared by the
// separate kernels (sharded solver) and the fused cooperative kernel below.
template <typename TK, bool kVec>
__device__ __forceinline__ double residual_loop(i64 N, TK* __restrict__ R, const TK* __restrict__ AP, TK alpha) {
  double s = 0.0;
  const i64 t0 = blockIdx.x * (i64)blockDim.x + threadIdx.x, ts = (i64)gridDim.x * blockDim.x;
  i64 from = 0;
  if constexpr (kVec) {
    using V = typename V16<TK>::V;
    constexpr int W = V16<TK>::W;
    const i64 nv = N / W;
    V* Rv = reinterpret_cast<V*>(R);
    const V* Av = reinterpret_cast<const V*>(AP);
    i64 q = t0;
    for (; q + 3 * ts < nv; q += 4 * ts) {  // four 16-byte pairs in flight per thread
      V r[4], a[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        r[u] = Rv[q + u * ts];
        a[u] = __ldcs(Av + q + u * ts);  // AP is dead after this pass: evict-first
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
#pragma unroll
        for (int k = 0; k < W; ++k) {
          TK& x = lane_of<TK>(r[u], k);
          x = sub_rn(x, mul_rn(alpha, reinterpret_cast<const TK*>(&a[u])[k]));
          s += static_cast<double>(x) * static_cast<double>(x);
        }
        Rv[q + u * ts] = r[u];
      }
    }
    for (; q < nv; q += ts) {
      V r = Rv[q];
      const V a = __ldcs(Av + q);
#pragma unroll
      for (int k = 0; k < W; ++k) {
        TK& x = lane_of<TK>(r, k);
        x = sub_rn(x, mul_rn(alpha, reinterpret_cast<const TK*>(&a)[k]));
        s += static_cast<double>(x) * static_cast<double>(x);
      }
      Rv[q] = r;
    }
    from = nv * W;
  }
  for (i64 q = from + t0; q < N; q += ts) {
    const TK r = sub_rn(R[q], mul_rn(alpha, AP[q]));
    R[q] = r;
    s += static_cast<double>(r) * static_cast<double>(r);
  }
  return s;
}

// X += alpha P, P = R + beta P.
template <typename TK, typename TX, bool kVec>
__device__ __forceinline__ void update_loop(i64 N, TX* __restrict__ X, TK* __restrict__ P, const TK* __restrict__ R,
                                            TK alpha, TK beta) {
  const i64 t0 = blockIdx.x * (i64)blockDim.x + threadIdx.x, ts = (i64)gridDim.x * blockDim.x;
  i64 from = 0;
  if constexpr (kVec && sizeof(TX) == sizeof(TK)) {
    using V = typename V16<TK>::V;
    constexpr int W = V16<TK>::W;
    const i64 nv = N / W;
    V* Xv = reinterpret_cast<V*>(X);
    V* Pv = reinterpret_cast<V*>(P);
    const V* Rv = reinterpret_cast<const V*>(R);
    auto one = [&](V& x, const V& pv, const V& r, V& pn) {
#pragma unroll
      for (int k = 0; k < W; ++k) {
        lane_of<TK>(x, k) = add_rn(lane_of<TK>(x, k), mul_rn(alpha, reinterpret_cast<const TK*>(&pv)[k]));
        lane_of<TK>(pn, k) = add_rn(reinterpret_cast<const TK*>(&r)[k], mul_rn(beta, reinterpret_cast<const TK*>(&pv)[k]));
      }
    };
    i64 q = t0;
    // X is touched by this pass only: streamed (evict-first) loads and stores,
    // so the L2 keeps R, P and AP for the passes that share them (config 1:
    // 3 x 41 MB of Krylov vectors against 126 MB of L2)
    auto ldx = [&](i64 k) { return __ldcs(Xv + k); };
    auto stx = [&](i64 k, const V& v) { __stcs(Xv + k, v); };
    for (; q + 3 * ts < nv; q += 4 * ts) {  // four 16-byte triples in flight per thread
      V x[4], pv[4], r[4], pn[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        x[u] = ldx(q + u * ts);
        pv[u] = Pv[q + u * ts];
        r[u] = Rv[q + u * ts];
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        one(x[u], pv[u], r[u], pn[u]);
        stx(q + u * ts, x[u]);
        Pv[q + u * ts] = pn[u];
      }
    }
    for (; q < nv; q += ts) {
      V x = ldx(q), pv = Pv[q], pn;
      const V r = Rv[q];
      one(x, pv, r, pn);
      stx(q, x);
      Pv[q] = pn;
    }
    from = nv * W;
  } else if constexpr (kVec) {
    // fp32 X, fp64 Krylov vectors: 4 entries per step (16-byte X, 2 x 16-byte P / R)
    const i64 nv = N / 4;
    float4* Xv = reinterpret_cast<float4*>(X);
    double2* Pv = reinterpret_cast<double2*>(P);
    const double2* Rv = reinterpret_cast<const double2*>(R);
    for (i64 q = t0; q < nv; q += ts) {
      float4 x = Xv[q];
      double2 p0 = Pv[2 * q], p1 = Pv[2 * q + 1];
      const double2 r0 = Rv[2 * q], r1 = Rv[2 * q + 1];
      x.x = static_cast<float>(add_rn(static_cast<double>(x.x), mul_rn(static_cast<double>(alpha), p0.x)));
      x.y = static_cast<float>(add_rn(static_cast<double>(x.y), mul_rn(static_cast<double>(alpha), p0.y)));
      x.z = static_cast<float>(add_rn(static_cast<double>(x.z), mul_rn(static_cast<double>(alpha), p1.x)));
      x.w = static_cast<float>(add_rn(static_cast<double>(x.w), mul_rn(static_cast<double>(alpha), p1.y)));
      p0.x = add_rn(r0.x, mul_rn(static_cast<double>(beta), p0.x));
      p0.y = add_rn(r0.y, mul_rn(static_cast<double>(beta), p0.y));
      p1.x = add_rn(r1.x, mul_rn(static_cast<double>(beta), p1.x));
      p1.y = add_rn(r1.y, mul_rn(static_cast<double>(beta), p1.y));
      Xv[q] = x;
      Pv[2 * q] = p0;
      Pv[2 * q + 1] = p1;
    }
    from = nv * 4;
  }
  for (i64 q = from + t0; q < N; q += ts) {
    const TK pv = P[q];
    X[q] = static_cast<TX>(add_rn(static_cast<TK>(X[q]), mul_rn(alpha, pv)));
    P[q] = add_rn(R[q], mul_rn(beta, pv));
  }
}

// breakdown check (solvers.hpp:53-57), uniform over the grid; true when the
// iteration stops here
__device__ __forceinline__ bool cg_breakdown(CgState* st) {
  const double curv = st->curv;
  if (!isfinite(curv) || curv <= 0.0) {
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      st->err = 1;
      st->err_it = st->it;
      st->done = 1;
    }
    return true;
  }
  return false;
}

template <typename TK, bool kVec>
__global__ void cg_residual_k(i64 N, TK* __restrict__ R, const TK* __restrict__ AP, double* partials,
                              CgState* st) {
  pdl_wait();
  pdl_trigger();
  if (st->done || cg_breakdown(st)) return;
  const TK alpha = static_cast<TK>(st->rho / st->curv);
  double s[1] = {residual_loop<TK, kVec>(N, R, AP, alpha)};
  double tot[1];
  if (grid_sum_last<1>(s, partials, &st->cnt[2], tot) && threadIdx.x == 0) st->rho_next = tot[0];
}

// X += alpha P, P = R + beta P (beta = rho_next / rho); the last block
// advances the iteration and applies the loop-top stop test.
template <typename TK, typename TX, bool kVec>
__global__ void cg_update_k(i64 N, TX* __restrict__ X, TK* __restrict__ P, const TK* __restrict__ R, CgState* st) {
  pdl_wait();
  pdl_trigger();
  if (st->done) return;
  const TK alpha = static_cast<TK>(st->rho / st->curv);
  const TK beta = static_cast<TK>(st->rho_next / st->rho);
  update_loop<TK, TX, kVec>(N, X, P, R, alpha, beta);
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
    if (sqrt(st->rho) <= st->target || st->it >= st->max_iter) st->done = 1;
  }
}

static __global__ void fill_sel_k(i64 len, int* sel) {
  const i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x;
  if (i < len) sel[i] = -1;
}
static __global__ void scatter_sel_k(const i64* __restrict__ om, i64 rho, int* sel) {
  const i64 k = blockIdx.x * (i64)blockDim.x + threadIdx.x;
  if (k < rho) sel[om[k]] = static_cast<int>(k);
}

static __global__ void gather_int_k(i64 len, const int* __restrict__ src, const int* __restrict__ idx, int* dst) {
  const i64 k = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x;
  if (k < len) dst[k] = src[idx[k]];
}

// X(i, c) <- X(pos[i], c) for every column, in place through shared memory.
template <typename TX>
__global__ void __launch_bounds__(1024) unpermute_rows_k(i64 p, i64 n, const int* __restrict__ pos, TX* X) {
  extern __shared__ __align__(16) unsigned char smraw[];
  TX* s = reinterpret_cast<TX*>(smraw);
  for (i64 col = blockIdx.x; col < n; col += gridDim.x) {
    TX* x = X + col * p;
    for (i64 i = threadIdx.x; i < p; i += blockDim.x) s[i] = x[i];
    __syncthreads();
    for (i64 i = threadIdx.x; i < p; i += blockDim.x) x[i] = s[pos[i]];
    __syncthreads();
  }
}


// The solve's row order.  Hub-heavy row graphs on the two-pass path: the
// row-group pass wants rows of similar degree side by side (32 natural rows
// would pad the entries by > 30 %).  Rather than indirecting every row access
// through a sorted order (scattered 8-byte reads of U and writes of AP: 4x
// their bytes in 32-byte sectors), the whole system is solved in the sorted
// row order -- L_r's rows and column indices renamed (each row's entries keep
// their order, so every sum is the same chain), rsel permuted, X put back at
// the end.  `ord` new -> old row, `pos` old -> new.
template <typename TV>
struct RowOrder {
  bool on = false;
  i64 p = 0;
  DevBuf<int> ord, pos;
  DevBuf<i64> rp;
  DevBuf<int> ci;
  DevBuf<TV> v;
  Pull<TV> pull{};

  // Decides (two-pass path, padding > 30 %, a column of X fits shared memory)
  // and, when on, renames the host CSR in place and uploads it (`pull`).
  bool build(Ctx* c, i64 p_, bool two_pass, size_t x_bytes, std::vector<i64>& rpr, std::vector<int>& cir,
             std::vector<TV>& vr) {
    p = p_;
    i64 tot = 0, pad_nat = 0;
    for (i64 w = 0; w < p; w += 32) {
      i64 mx = 0;
      for (i64 i = w; i < std::min<i64>(p, w + 32); ++i) {
        mx = std::max(mx, rpr[i + 1] - rpr[i]);
        tot += rpr[i + 1] - rpr[i];
      }
      pad_nat += mx * std::min<i64>(32, p - w);
    }
    if (!(two_pass && tot > 0 && pad_nat > tot + tot / 3 && p * static_cast<i64>(x_bytes) <= 160 * 1024)) return false;
    std::vector<int> o(static_cast<size_t>(p)), q(static_cast<size_t>(p));
    std::iota(o.begin(), o.end(), 0);
    std::stable_sort(o.begin(), o.end(), [&](int a, int b) { return rpr[a + 1] - rpr[a] > rpr[b + 1] - rpr[b]; });
    for (i64 t = 0; t < p; ++t) q[o[t]] = static_cast<int>(t);
    std::vector<i64> rp2(static_cast<size_t>(p) + 1, 0);
    std::vector<int> ci2(cir.size());
    std::vector<TV> v2(vr.size());
    for (i64 t = 0; t < p; ++t) {
      const i64 a = rpr[o[t]], b = rpr[o[t] + 1];
      rp2[t + 1] = rp2[t] + (b - a);
      for (i64 k = a; k < b; ++k) {
        ci2[rp2[t] + (k - a)] = q[cir[k]];
        v2[rp2[t] + (k - a)] = vr[k];
      }
    }
    ord.alloc(c, static_cast<size_t>(p));
    pos.alloc(c, static_cast<size_t>(p));
    rp.alloc(c, rp2.size());
    ci.alloc(c, std::max<size_t>(ci2.size(), 1));
    v.alloc(c, std::max<size_t>(v2.size(), 1));
    CUDA_OK(cudaMemcpyAsync(ord.p, o.data(), sizeof(int) * p, cudaMemcpyHostToDevice, c->stream));
    CUDA_OK(cudaMemcpyAsync(pos.p, q.data(), sizeof(int) * p, cudaMemcpyHostToDevice, c->stream));
    CUDA_OK(cudaMemcpyAsync(rp.p, rp2.data(), sizeof(i64) * rp2.size(), cudaMemcpyHostToDevice, c->stream));
    CUDA_OK(cudaMemcpyAsync(ci.p, ci2.data(), sizeof(int) * ci2.size(), cudaMemcpyHostToDevice, c->stream));
    CUDA_OK(cudaMemcpyAsync(v.p, v2.data(), sizeof(TV) * v2.size(), cudaMemcpyHostToDevice, c->stream));
    sync(c);  // the host arrays go out of scope below
    pull = Pull<TV>{rp.p, ci.p, v.p};
    rpr.swap(rp2);
    cir.swap(ci2);
    vr.swap(v2);
    on = true;
    return true;
  }
  // rsel in the solve's order (out owns the storage)
  const int* permute_rsel(Ctx* c, const int* rsel, DevBuf<int>& out) const {
    out.alloc(c, static_cast<size_t>(p));
    gather_int_k<<<blocks_for(p), kBlock, 0, c->stream>>>(p, rsel, ord.p, out.p);
    launched(c);
    return out.p;
  }
  // rows of X (p x ncols) back to the caller's order, column by column in place
  template <typename TX>
  void restore_rows(Ctx* c, TX* X, i64 ncols) const {
    if (ncols <= 0) return;
    const size_t bytes = static_cast<size_t>(p) * sizeof(TX);
    ensure_smem(unpermute_rows_k<TX>, bytes);
    const unsigned g = static_cast<unsigned>(std::max<i64>(1, std::min<i64>(ncols, static_cast<i64>(c->num_sms) * 2)));
    unpermute_rows_k<TX><<<g, 1024, bytes, c->stream>>>(p, ncols, pos.p, X);
    launched(c);
  }
};

// ------------------------------------------------------------------ the apply engine
// Geometry of both passes for one operator pair, built once per decode.  The
// lc pass works on a local column space of n_local columns ([own | halo] for
// the sharded decoder) and produces columns [0, ncols).
struct ApplyPlan {
  i64 p = 0, ncols = 0, n_local = 0, col_base = 0;
  // slab apply (slab_k): fp32 iterates, a 32-row slab of all columns in shared memory
  bool slab = false;
  int s_parts = 1, s_evr = 9, s_max_steps = 0, s_grid = 1;
  size_t s_smem = 0;
  DevBuf<unsigned char> s_rec, s_steps;  // interleaved L_c records, SlabStep list
  DevBuf<int> s_wsteps, s_win, s_lo;
  DevBuf<float> s_lv;
  // fused one-pass apply (fused_k) for L2-resident iterates
  bool fused = false;
  dim3 f_grid;
  int f_cpc = 1;
  size_t f_smem = 0;
  bool lc_smem = true;
  size_t lc_smem_bytes = 0;
  int lc_chunks = 1, lc_cpc = 1;
  // lr pass, register-resident rows (lr_reg_k)
  bool lr_reg = false;
  int lr_C = 1, lr_EV = 16, lr_T = 512, lr_stripes = 1, lr_groups = 0, lr_wl_max = 0;
  size_t lr_smem = 0;
  DevBuf<LrGroup> groups;
  DevBuf<int> vrow_row, vrow_np, ej;
  DevBuf<unsigned char> ev;  // TV values, ELL-interleaved
  // lr pass, generic fallback (lr_k)
  DevBuf<RowRange> ranges;
  int n_ranges = 0;
  DevBuf<int> order;
  bool use_order = false;
  int gen_C = 1;
  size_t gen_smem = 0;
};

constexpr size_t kSmemMax = 200 * 1024;

// exact: fp64 data -- rows may not be split (bit-identical sums).
// rpc (L_c row pointers, host): when given and the Krylov vectors fit in L2,
// the fused one-pass apply is planned instead of the two passes.
inline int __float_as_int_host(float f) {
  int i;
  std::memcpy(&i, &f, sizeof(i));
  return i;
}

// Host copy of the L_c pull (for the one-pass plans).
template <typename TV>
struct HostPull {
  std::vector<i64> rp;
  std::vector<int> ci;
  std::vector<TV> v;
};

// Slab apply geometry (slab_k): fp32 iterates (p a multiple of 4), the slab
// (n * 128 B) and the warps' rings and windows within one CTA's shared
// memory, L_r rows of <= 16 entries whose referenced rows fit 32 aligned
// 16-byte chunks per slab, L_c pull rows of <= (kSlabRing - 1) chunks.
// Returns false when it does not apply.
template <typename TI, typename TV>
bool plan_slab(Ctx* c, ApplyPlan& ap, i64 p, i64 n, const std::vector<i64>& rpr, const std::vector<int>& cir,
               const std::vector<TV>& vr, const HostPull<TV>& lc) {
  if constexpr (sizeof(TI) != 4 || sizeof(TV) != 4) {
    return false;
  } else {
    const size_t smem = ((static_cast<size_t>(n) * 128 + 15) / 16) * 16 + (kSlabThreads / 32) * kSlabWarpBytes;
    if (p <= 0 || n <= 0 || p % 4 != 0 || smem > 227 * 1024) return false;
    i64 mr = 0;
    for (i64 i = 0; i < p; ++i) mr = std::max(mr, rpr[i + 1] - rpr[i]);
    if (mr > 16) return false;
    const int EVR = mr <= 9 ? 9 : 16;
    trace_mark(c, "slab plan: enter");
    // L_r windows
    const i64 slabs = (p + 31) / 32;
    std::vector<int> win(static_cast<size_t>(slabs) * 32, kNoChunk);
    std::vector<float> lv(static_cast<size_t>(EVR) * p, 0.f);
    std::vector<int> lo(static_cast<size_t>(EVR) * p, 0);
    std::vector<int> ch;
    std::vector<uint64_t> bits;
    std::vector<int> rank;
    for (i64 sl = 0; sl < slabs; ++sl) {
      const i64 i0 = sl * 32, i1 = std::min(p, i0 + 32);
      // distinct 4-row chunks the slab's rows reference, in order (bitmap over their range)
      int lo_c = INT32_MAX, hi_c = -1;
      for (i64 i = i0; i < i1; ++i) {
        lo_c = std::min(lo_c, static_cast<int>(i >> 2));
        hi_c = std::max(hi_c, static_cast<int>(i >> 2));
        for (i64 k = rpr[i]; k < rpr[i + 1]; ++k) {
          lo_c = std::min(lo_c, cir[k] >> 2);
          hi_c = std::max(hi_c, cir[k] >> 2);
        }
      }
      if (hi_c - lo_c >= 65536) return false;  // rows scattered over more than 256 K rows
      const size_t words = static_cast<size_t>(hi_c - lo_c) / 64 + 1;
      bits.assign(words, 0);
      auto mark = [&](int row) {
        const int q = (row >> 2) - lo_c;
        bits[q >> 6] |= uint64_t{1} << (q & 63);
      };
      for (i64 i = i0; i < i1; ++i) {
        mark(static_cast<int>(i));
        for (i64 k = rpr[i]; k < rpr[i + 1]; ++k) mark(cir[k]);
      }
      ch.clear();
      for (size_t w = 0; w < words && ch.size() <= 32; ++w)
        for (uint64_t b = bits[w]; b; b &= b - 1)
          ch.push_back((lo_c + static_cast<int>(w * 64 + __builtin_ctzll(b))) * 4);
      if (ch.size() > 32) return false;
      for (size_t t = 0; t < ch.size(); ++t) win[sl * 32 + t] = ch[t] - static_cast<int>(i0);
      rank.assign(static_cast<size_t>(hi_c - lo_c) + 1, 0);
      for (size_t t = 0; t < ch.size(); ++t) rank[(ch[t] >> 2) - lo_c] = static_cast<int>(t);
      auto where = [&](i64 j) { return (rank[(j >> 2) - lo_c] * 4 + static_cast<int>(j & 3)) * 4; };
      for (i64 i = i0; i < i1; ++i) {
        for (int e = 0; e < EVR; ++e) {
          const i64 k = rpr[i] + e;
          const bool in = k < rpr[i + 1];
          lv[static_cast<size_t>(e) * p + i] = in ? static_cast<float>(vr[k]) : 0.f;
          lo[static_cast<size_t>(e) * p + i] = where(in ? cir[k] : i);
        }
      }
    }
    trace_mark(c, "slab plan: windows");
    // column parts per slab: the persistent CTAs take contiguous runs of
    // (slab, part) items, so finer parts balance the SMs; each part keeps
    // >= ~4 quads per warp for the warps' own balance
    const int best = n >= 768 ? 4 : n >= 384 ? 2 : 1;
    // L_c quads: per part, columns sorted by degree, 4 at a time, dealt to the
    // warps round-robin; each warp's steps (<= (kSlabRing - 1) chunks of
    // records) laid out contiguously
    constexpr int kMaxRows = (kSlabRing - 1) * 512 / 64;
    std::vector<SlabStep> steps;
    std::vector<int> wsteps;
    std::vector<int4> rec;  // 16-byte groups
    for (int part = 0; part < best; ++part) {
      const i64 pa = n * part / best, pb = n * (part + 1) / best;
      std::vector<int> cols(static_cast<size_t>(pb - pa));
      std::iota(cols.begin(), cols.end(), static_cast<int>(pa));
      auto deg = [&](int q) { return lc.rp[q + 1] - lc.rp[q]; };
      std::stable_sort(cols.begin(), cols.end(), [&](int x, int y) { return deg(x) > deg(y); });
      const i64 nq = (static_cast<i64>(cols.size()) + 3) / 4;
      // quads to warps: longest first to the least loaded warp (record rows + a fixed per-quad cost)
      std::vector<std::vector<i64>> wq(kSlabWarps);
      {
        std::vector<i64> load(kSlabWarps, 0);
        for (i64 q = 0; q < nq; ++q) {
          const int w = static_cast<int>(std::min_element(load.begin(), load.end()) - load.begin());
          wq[w].push_back(q);
          load[w] += (deg(cols[q * 4]) + 1) / 2 + 6;
        }
      }
      for (int w = 0; w < kSlabWarps; ++w) {
        wsteps.push_back(static_cast<int>(steps.size()));
        for (const i64 q : wq[w]) {
          int cq[4];
          i64 dmax = 0;
          for (int g = 0; g < 4; ++g) {
            const i64 at = q * 4 + g;
            cq[g] = at < static_cast<i64>(cols.size()) ? cols[at] : -1;
            if (cq[g] >= 0) dmax = std::max(dmax, deg(cq[g]));
          }
          const int rows_q = static_cast<int>((dmax + 1) / 2);
          int mask = 0, any = -1;
          for (int g = 0; g < 4; ++g)
            if (cq[g] >= 0) mask |= 1 << g, any = any < 0 ? cq[g] : any;
          int k = 0;
          do {
            const int r = std::min(kMaxRows, rows_q - k);
            SlabStep st{};
            st.rec = static_cast<int>(rec.size() * 16);
            st.rows = r;
            st.flags = (k == 0 ? 1 : 0) | (k + r == rows_q ? 2 : 0) | (mask << 8);
            for (int g = 0; g < 4; ++g) st.col[g] = cq[g] >= 0 ? cq[g] : any;
            for (int kr = k; kr < k + r; ++kr)
              for (int g = 0; g < 4; ++g) {
                int4 e{0, 0, 0, 0};
                if (cq[g] >= 0) {
                  const i64 b0 = lc.rp[cq[g]], d = deg(cq[g]);
                  if (2 * kr < d) {
                    e.x = __float_as_int_host(static_cast<float>(lc.v[b0 + 2 * kr]));
                    e.y = lc.ci[b0 + 2 * kr] * 128;
                  }
                  if (2 * kr + 1 < d) {
                    e.z = __float_as_int_host(static_cast<float>(lc.v[b0 + 2 * kr + 1]));
                    e.w = lc.ci[b0 + 2 * kr + 1] * 128;
                  }
                }
                rec.push_back(e);
              }
            steps.push_back(st);
            k += r;
          } while (k < rows_q);
        }
        // the warp's ring schedule: at each step issue the chunks up to
        // min(last, first chunk of the step + kSlabRing - 1); a step whose last
        // chunk is issued in that same step waits for it at once
        const size_t w0 = static_cast<size_t>(wsteps.back());
        if (w0 < steps.size()) {
          const int clast = (steps.back().rec + steps.back().rows * 64 - 1) / 512;
          int issued = steps[w0].rec / 512;
          for (size_t t = w0; t < steps.size(); ++t) {
            SlabStep& st = steps[t];
            const int c0 = st.rec / 512, cl = (st.rec + st.rows * 64 - 1) / 512;
            st.issue_hi = std::max(issued - 1, std::min(clast, c0 + kSlabRing - 1));
            if (st.rows > 0 && cl >= issued) st.flags |= 4;
            issued = std::max(issued, st.issue_hi + 1);
          }
        }
      }
      wsteps.push_back(static_cast<int>(steps.size()));
    }
    trace_mark(c, "slab plan: quads");
    int max_steps = 0;
    for (int part = 0; part < best; ++part)
      max_steps = std::max(max_steps, wsteps[part * (kSlabWarps + 1) + kSlabWarps] - wsteps[part * (kSlabWarps + 1)]);
    const size_t smem_all = smem + static_cast<size_t>(max_steps) * sizeof(SlabStep);
    if (rec.size() * 16 >= (size_t{1} << 31) || smem_all > 227 * 1024) return false;
    rec.resize(((rec.size() + 31) / 32 + 1) * 32, int4{0, 0, 0, 0});  // whole 512-byte chunks, one spare
    ap.slab = true;
    ap.s_parts = best;
    ap.s_grid = static_cast<int>(std::min<i64>(c->num_sms, slabs * best));
    ap.s_evr = EVR;
    ap.s_smem = smem_all;
    ap.s_max_steps = max_steps;
    ap.s_rec.alloc(c, rec.size() * 16);
    ap.s_steps.alloc(c, steps.size() * sizeof(SlabStep));
    ap.s_wsteps.alloc(c, wsteps.size());
    ap.s_win.alloc(c, win.size());
    ap.s_lv.alloc(c, lv.size());
    ap.s_lo.alloc(c, lo.size());
    CUDA_OK(cudaMemcpyAsync(ap.s_rec.p, rec.data(), rec.size() * 16, cudaMemcpyHostToDevice, c->stream));
    CUDA_OK(cudaMemcpyAsync(ap.s_steps.p, steps.data(), steps.size() * sizeof(SlabStep), cudaMemcpyHostToDevice,
                            c->stream));
    CUDA_OK(cudaMemcpyAsync(ap.s_wsteps.p, wsteps.data(), sizeof(int) * wsteps.size(), cudaMemcpyHostToDevice, c->stream));
    CUDA_OK(cudaMemcpyAsync(ap.s_win.p, win.data(), sizeof(int) * win.size(), cudaMemcpyHostToDevice, c->stream));
    CUDA_OK(cudaMemcpyAsync(ap.s_lv.p, lv.data(), sizeof(float) * lv.size(), cudaMemcpyHostToDevice, c->stream));
    CUDA_OK(cudaMemcpyAsync(ap.s_lo.p, lo.data(), sizeof(int) * lo.size(), cudaMemcpyHostToDevice, c->stream));
    sync(c);
    return true;
  }
}

template <typename TI, typename TK, typename TV>
void plan_apply(Ctx* c, ApplyPlan& ap, i64 p, i64 ncols, i64 n_local, i64 col_base, const std::vector<i64>& rpr,
                const std::vector<int>& cir, const std::vector<TV>& vr, bool exact,
                const HostPull<TV>* lcp = nullptr) {
  ap.p = p;
  ap.ncols = ncols;
  ap.n_local = n_local;
  ap.col_base = col_base;
  const std::vector<i64>* rpc = lcp ? &lcp->rp : nullptr;
  const bool l2_resident = p * ncols * static_cast<i64>(sizeof(TK)) <= (i64{96} << 20);
  if (lcp && ncols == n_local && (c->apply_path == 3 || (c->apply_path == 0 && l2_resident)) &&
      plan_slab<TI, TV>(c, ap, p, ncols, rpr, cir, vr, *lcp)) {
    c->last_apply_path = 3;
    return;
  }
  c->last_apply_path = 1;
  if (rpc && (c->apply_path >= 2 || (c->apply_path == 0 && l2_resident)) && p * ncols < (i64{1} << 31) && p > 0 &&
      ncols > 0) {
    const i64 gx = (p + 511) / 512;
    const i64 ycap = std::max<i64>(1, (static_cast<i64>(c->num_sms) * 8) / gx);
    const i64 ny = std::min<i64>(ncols, ycap);
    const i64 cpc = std::max<i64>({i64{1}, std::min<i64>((ncols + ny - 1) / ny, 128), (ncols + 65534) / 65535});
    const i64 gy = (ncols + cpc - 1) / cpc;
    i64 mer = 0, mec = 0;
    for (i64 b = 0; b < gx; ++b) mer = std::max(mer, rpr[std::min<i64>(p, (b + 1) * 512)] - rpr[b * 512]);
    for (i64 b = 0; b < gy; ++b) mec = std::max(mec, (*rpc)[std::min<i64>(ncols, (b + 1) * cpc)] - (*rpc)[b * cpc]);
    const size_t smem = static_cast<size_t>(mer + mec) * sizeof(OffEnt<TV>) + sizeof(int) * (cpc + 2) + 16;
    if (smem <= 96 * 1024) {
      ap.fused = true;
      ap.f_grid = dim3(static_cast<unsigned>(gx), static_cast<unsigned>(gy));
      ap.f_cpc = static_cast<int>(cpc);
      ap.f_smem = smem;
      c->last_apply_path = 2;
      return;
    }
  }
  const size_t band_bytes = static_cast<size_t>(n_local) * 128;
  ap.lc_smem = band_bytes + lc_smem_ent_bytes<TI, TV>() <= 220 * 1024;
  ap.lc_smem_bytes = std::max<size_t>(band_bytes, 16);
  ap.lc_cpc = 8 * 32;  // L2 mode: 8 warps x 32 columns (one row-pointer load per warp)
  ap.lc_chunks = static_cast<int>(std::max<i64>(1, (ncols + ap.lc_cpc - 1) / ap.lc_cpc));
  // row order: degree-sorted when natural warps would pad the rows > 30 %
  std::vector<int> deg(static_cast<size_t>(p));
  int maxdeg = 0;
  i64 tot = 0;
  for (i64 i = 0; i < p; ++i) {
    deg[i] = static_cast<int>(rpr[i + 1] - rpr[i]);
    maxdeg = std::max(maxdeg, deg[i]);
    tot += deg[i];
  }
  i64 pad_nat = 0;
  for (i64 w = 0; w < p; w += 32) {
    int mx = 0;
    for (i64 i = w; i < std::min<i64>(p, w + 32); ++i) mx = std::max(mx, deg[i]);
    pad_nat += static_cast<i64>(mx) * std::min<i64>(32, p - w);
  }
  std::vector<int> ord(static_cast<size_t>(p));
  std::iota(ord.begin(), ord.end(), 0);
  ap.use_order = tot > 0 && pad_nat > tot + tot / 3;
  if (ap.use_order) std::stable_sort(ord.begin(), ord.end(), [&](int a, int b) { return deg[a] > deg[b]; });
  constexpr int E = 16 / sizeof(TI);
  // --- register-resident rows
  const int EV = maxdeg <= 9 ? 9 : 16;
  const int T = sizeof(TV) == 4 ? 1024 : 512;
  if (!(exact && maxdeg > EV) && p > 0) {
    std::vector<int> vrow_row, vrow_np;
    std::vector<LrGroup> grp;
    std::vector<std::array<int, 2>> vrow_k;  // entry range of each vrow
    for (i64 t = 0; t < p; ++t) {
      const int i = ord[t];
      const int parts = std::max(1, (deg[i] + EV - 1) / EV);
      if (grp.empty() || grp.back().nv + parts > T) grp.push_back({static_cast<int>(vrow_row.size()), 0, 0, 0, 0});
      for (int q = 0; q < parts; ++q) {
        const i64 k0 = rpr[i] + static_cast<i64>(q) * EV;
        const int k1 = static_cast<int>(std::min<i64>(rpr[i + 1], k0 + EV));
        vrow_row.push_back(i);
        vrow_np.push_back(q == 0 ? parts : 0);
        vrow_k.push_back({static_cast<int>(k0), k1});
      }
      grp.back().nv += parts;
      if (parts > 1) grp.back().split = 1;
    }
    int wl_max = 0;
    for (auto& g : grp) {
      int lo = INT32_MAX, hi = -1;
      for (int t = g.v0; t < g.v0 + g.nv; ++t) {
        lo = std::min(lo, vrow_row[t]);
        hi = std::max(hi, vrow_row[t]);
        for (int k = vrow_k[t][0]; k < vrow_k[t][1]; ++k) {
          lo = std::min(lo, cir[k]);
          hi = std::max(hi, cir[k]);
        }
      }
      lo = (lo / E) * E;
      hi = static_cast<int>(std::min<i64>(p, ((hi + 1 + E - 1) / E) * E));
      g.w0 = lo;
      g.wl = hi - lo;
      wl_max = std::max(wl_max, g.wl);
    }
    const bool any_split = std::any_of(grp.begin(), grp.end(), [](const LrGroup& g) { return g.split; });
    int C = 8;
    auto bytes = [&](int Cc) {
      return 2 * static_cast<size_t>(Cc) * wl_max * sizeof(TI) + (any_split ? static_cast<size_t>(T) * Cc * sizeof(TK) : 0);
    };
    while (C > 1 && bytes(C) > kSmemMax) C /= 2;
    if (bytes(C) <= kSmemMax) {
      ap.lr_reg = true;
      ap.lr_C = C;
      ap.lr_EV = EV;
      ap.lr_T = T;
      ap.lr_groups = static_cast<int>(grp.size());
      ap.lr_wl_max = wl_max;
      ap.lr_smem = std::max<size_t>(bytes(C), 16);
      const int per_sm = ap.lr_smem <= 100 * 1024 && T <= 1024 ? (T == 512 ? 2 : 1) : 1;
      const i64 tiles = (ncols + C - 1) / C;
      // one wave: stripes x groups <= resident CTAs
      ap.lr_stripes = static_cast<int>(
          std::max<i64>(1, std::min<i64>(tiles, (static_cast<i64>(c->num_sms) * per_sm) / ap.lr_groups)));
      const size_t ne = static_cast<size_t>(grp.size()) * EV * T;
      std::vector<TV> hv(ne, TV(0));
      std::vector<int> hj(ne, 0);
      for (size_t g = 0; g < grp.size(); ++g)
        for (int t = 0; t < grp[g].nv; ++t) {
          const int q = grp[g].v0 + t;
          const int own = vrow_row[q] - grp[g].w0;
          for (int e = 0; e < EV; ++e) {
            const size_t at = (g * EV + e) * static_cast<size_t>(T) + t;
            const int k = vrow_k[q][0] + e;
            if (k < vrow_k[q][1]) {
              hv[at] = vr[k];
              hj[at] = cir[k] - grp[g].w0;
            } else {
              hj[at] = own;
            }
          }
        }
      // Bank-aware entry order (fp32 data; fp64 data keeps the CSR order for
      // bit parity).  Step e of a warp is one shared-memory gather: the lanes
      // of a phase (128 bytes of requests: 8 lanes of 16-byte records, 16 of
      // 8-byte) read records of unrelated rows, and every extra distinct
      // record in one bank group is another wavefront (measured ~2.8 per
      // ideal one with the entries in CSR order).  The entries of a vrow may
      // be summed in any order here, so each lane's entries are dealt to the
      // steps greedily -- at every step a lane takes, among the entries it
      // has left, the one whose bank group is least loaded in its phase.
      if (!exact) {
        const int rb = C * static_cast<int>(sizeof(TI));       // record bytes
        const int aw = std::min(rb, 16);                        // bytes per shared load
        const int phase = 128 / aw;                             // lanes served by one wavefront
        const int ngr = 128 / aw;                               // bank groups
        auto group_of = [&](int j) { return ((static_cast<i64>(j) * rb) % 128) / aw; };
        std::vector<int> load(static_cast<size_t>(ngr));
        std::vector<std::vector<int>> seen(static_cast<size_t>(ngr));
        std::vector<unsigned char> used(static_cast<size_t>(32) * EV);
        for (size_t g = 0; g < grp.size(); ++g)
          for (int w0 = 0; w0 < T; w0 += 32) {
            std::fill(used.begin(), used.end(), 0);
            // the warp's entries, before reordering
            std::vector<TV> ov(static_cast<size_t>(32) * EV);
            std::vector<int> oj(static_cast<size_t>(32) * EV);
            for (int l = 0; l < 32; ++l)
              for (int e = 0; e < EV; ++e) {
                const size_t at = (g * EV + e) * static_cast<size_t>(T) + w0 + l;
                ov[l * EV + e] = hv[at];
                oj[l * EV + e] = hj[at];
              }
            for (int e = 0; e < EV; ++e)
              for (int ph = 0; ph < 32; ph += phase) {
                std::fill(load.begin(), load.end(), 0);
                for (auto& sj : seen) sj.clear();
                for (int l = ph; l < ph + phase; ++l) {
                  int best = -1, best_cost = INT32_MAX;
                  for (int x = 0; x < EV; ++x) {
                    if (used[l * EV + x]) continue;
                    const int j = oj[l * EV + x];
                    const int gq = static_cast<int>(group_of(j));
                    const bool dup = std::find(seen[gq].begin(), seen[gq].end(), j) != seen[gq].end();
                    const int cost = dup ? -1 : load[gq];
                    if (cost < best_cost) best_cost = cost, best = x;
                  }
                  used[l * EV + best] = 1;
                  const int j = oj[l * EV + best];
                  const int gq = static_cast<int>(group_of(j));
                  if (std::find(seen[gq].begin(), seen[gq].end(), j) == seen[gq].end()) {
                    seen[gq].push_back(j);
                    ++load[gq];
                  }
                  const size_t at = (g * EV + e) * static_cast<size_t>(T) + w0 + l;
                  hv[at] = ov[l * EV + best];
                  hj[at] = j;
                }
              }
          }
      }
      ap.groups.alloc(c, grp.size());
      ap.vrow_row.alloc(c, vrow_row.size());
      ap.vrow_np.alloc(c, vrow_np.size());
      ap.ev.alloc(c, ne * sizeof(TV));
      ap.ej.alloc(c, ne);
      CUDA_OK(cudaMemcpyAsync(ap.groups.p, grp.data(), sizeof(LrGroup) * grp.size(), cudaMemcpyHostToDevice, c->stream));
      CUDA_OK(cudaMemcpyAsync(ap.vrow_row.p, vrow_row.data(), sizeof(int) * vrow_row.size(), cudaMemcpyHostToDevice,
                              c->stream));
      CUDA_OK(cudaMemcpyAsync(ap.vrow_np.p, vrow_np.data(), sizeof(int) * vrow_np.size(), cudaMemcpyHostToDevice,
                              c->stream));
      CUDA_OK(cudaMemcpyAsync(ap.ev.p, hv.data(), sizeof(TV) * ne, cudaMemcpyHostToDevice, c->stream));
      CUDA_OK(cudaMemcpyAsync(ap.ej.p, hj.data(), sizeof(int) * ne, cudaMemcpyHostToDevice, c->stream));
      sync(c);
      return;
    }
  }
  // --- generic fallback: row ranges with windows, CSR entries streamed per tile
  auto window = [&](i64 a, i64 e, int& w0, int& w1) {
    int lo = INT32_MAX, hi = -1;
    for (i64 t = a; t < e; ++t) {
      const int i = ord[t];
      lo = std::min(lo, i);
      hi = std::max(hi, i);
      for (i64 k = rpr[i]; k < rpr[i + 1]; ++k) {
        lo = std::min(lo, cir[k]);
        hi = std::max(hi, cir[k]);
      }
    }
    w0 = lo;
    w1 = hi + 1;
  };
  const i64 RB = 1024;
  std::vector<RowRange> rr;
  int maxw = 0;
  if (p > 0) {
    int w0, w1;
    window(0, p, w0, w1);
    i64 sum_w = 0;
    std::vector<RowRange> split;
    for (i64 a = 0; a < p; a += RB) {
      const i64 e = std::min<i64>(p, a + RB);
      int x0, x1;
      window(a, e, x0, x1);
      split.push_back({static_cast<int>(a), static_cast<int>(e), x0, x1});
      sum_w += x1 - x0;
    }
    if (split.size() > 1 && sum_w < 2 * (w1 - w0))
      rr = split;
    else
      rr.push_back({0, static_cast<int>(p), w0, w1});
    for (const auto& r : rr) maxw = std::max(maxw, r.w1 - r.w0);
  }
  int C = 8;
  while (C > 1 && static_cast<size_t>(maxw) * C * sizeof(TI) > kSmemMax) C /= 2;
  if (static_cast<size_t>(maxw) * C * sizeof(TI) > kSmemMax)
    invalid("alternate decoder: row graph window exceeds shared memory (p too large)");
  ap.gen_C = C;
  ap.gen_smem = std::max<size_t>(static_cast<size_t>(maxw) * C * sizeof(TI), 16);
  ap.n_ranges = static_cast<int>(rr.size());
  ap.ranges.alloc(c, std::max<size_t>(rr.size(), 1));
  if (!rr.empty())
    CUDA_OK(cudaMemcpyAsync(ap.ranges.p, rr.data(), sizeof(RowRange) * rr.size(), cudaMemcpyHostToDevice, c->stream));
  if (ap.use_order) {
    ap.order.alloc(c, static_cast<size_t>(p));
    CUDA_OK(cudaMemcpyAsync(ap.order.p, ord.data(), sizeof(int) * p, cudaMemcpyHostToDevice, c->stream));
  }
  sync(c);
}

// Number of CTAs (reduction partials) of a pass.
inline size_t lc_blocks(const ApplyPlan& ap, int S) {
  return ap.lc_smem ? static_cast<size_t>((ap.p + S - 1) / S)
                    : static_cast<size_t>((ap.p + 31) / 32) * ap.lc_chunks;
}
inline size_t lr_blocks(const ApplyPlan& ap) {
  if (ap.slab) return static_cast<size_t>(ap.s_grid);
  if (ap.fused) return static_cast<size_t>(ap.f_grid.x) * ap.f_grid.y;
  return ap.lr_reg ? static_cast<size_t>(ap.lr_groups) * ap.lr_stripes
                   : static_cast<size_t>(ap.n_ranges) * ((ap.ncols + ap.gen_C - 1) / ap.gen_C);
}

template <typename TI, typename TK, typename TV, typename TB>
void launch_lc(Ctx* c, const ApplyPlan& ap, Pull<TV> L, const TI* P, TK* U, const Combine<TK, TB>& cb, bool combine) {
  KScope ks_(c, "cg_apply_lc");
  if (ap.ncols == 0 || ap.p == 0) return;
  constexpr int S = 128 / sizeof(TI);
  const unsigned bands = static_cast<unsigned>((ap.p + S - 1) / S);
  if (ap.lc_smem) {
    auto k = combine ? lc_smem_k<TI, TK, TV, true, TB> : lc_smem_k<TI, TK, TV, false, TB>;
    const size_t bytes = ((ap.n_local * 128 + 15) / 16) * 16 + lc_smem_ent_bytes<TI, TV>();
    ensure_smem(k, bytes);
    k<<<bands, kLcSmemThreads, bytes, c->stream>>>(static_cast<int>(ap.p), static_cast<int>(ap.ncols),
                                                   static_cast<int>(ap.n_local), L, P, U, ap.col_base, cb);
  } else {
    auto k = combine ? lc_k<TI, TK, TV, true, TB> : lc_k<TI, TK, TV, false, TB>;
    const unsigned bands32 = static_cast<unsigned>((ap.p + 31) / 32);
    k<<<bands32 * ap.lc_chunks, 256, 0, c->stream>>>(static_cast<int>(ap.p), static_cast<int>(ap.ncols),
                                                     ap.lc_chunks, ap.lc_cpc, L, P, U, ap.col_base, cb);
  }
  launched(c);
}

template <typename TI, typename TK, typename TV, int C, int EV, int T, typename TB>
void launch_lr_reg(Ctx* c, const ApplyPlan& ap, const TI* P, TK* U, const Combine<TK, TB>& cb, bool combine) {
  auto k = combine ? lr_reg_k<TI, TK, TV, C, EV, T, true, TB> : lr_reg_k<TI, TK, TV, C, EV, T, false, TB>;
  ensure_smem(k, ap.lr_smem);
  k<<<static_cast<unsigned>(ap.lr_groups * ap.lr_stripes), T, ap.lr_smem, c->stream>>>(
      static_cast<int>(ap.p), static_cast<int>(ap.ncols), ap.lr_stripes, ap.groups.p, ap.vrow_row.p, ap.vrow_np.p,
      reinterpret_cast<const TV*>(ap.ev.p), ap.ej.p, ap.lr_wl_max, P, U, ap.col_base, cb);
}

template <typename TI, typename TK, typename TV, int C, typename TB>
void launch_lr_gen(Ctx* c, const ApplyPlan& ap, Pull<TV> Lr, const TI* P, TK* U, const Combine<TK, TB>& cb,
                   bool combine) {
  auto k = combine ? lr_k<TI, TK, TV, C, true, TB> : lr_k<TI, TK, TV, C, false, TB>;
  ensure_smem(k, ap.gen_smem);
  const dim3 g(static_cast<unsigned>((ap.ncols + C - 1) / C), static_cast<unsigned>(ap.n_ranges));
  k<<<g, 512, ap.gen_smem, c->stream>>>(static_cast<int>(ap.p), static_cast<int>(ap.ncols), ap.ranges.p,
                                        ap.use_order ? ap.order.p : nullptr, Lr, P, U, ap.col_base, cb);
}

template <typename TI, typename TK, typename TV, int EV, int T, typename TB>
void launch_lr_reg_c(Ctx* c, const ApplyPlan& ap, const TI* P, TK* U, const Combine<TK, TB>& cb, bool combine) {
  switch (ap.lr_C) {
    case 8: launch_lr_reg<TI, TK, TV, 8, EV, T>(c, ap, P, U, cb, combine); break;
    case 4: launch_lr_reg<TI, TK, TV, 4, EV, T>(c, ap, P, U, cb, combine); break;
    case 2: launch_lr_reg<TI, TK, TV, 2, EV, T>(c, ap, P, U, cb, combine); break;
    default: launch_lr_reg<TI, TK, TV, 1, EV, T>(c, ap, P, U, cb, combine); break;
  }
}

template <typename TI, typename TK, typename TV, typename TB>
void launch_lr(Ctx* c, const ApplyPlan& ap, Pull<TV> Lr, const TI* P, TK* U, const Combine<TK, TB>& cb, bool combine) {
  KScope ks_(c, "cg_apply_lr");
  if (ap.ncols == 0 || ap.p == 0) return;
  constexpr int T = sizeof(TV) == 4 ? 1024 : 512;
  if (ap.lr_reg) {
    if (ap.lr_EV == 9)
      launch_lr_reg_c<TI, TK, TV, 9, T>(c, ap, P, U, cb, combine);
    else
      launch_lr_reg_c<TI, TK, TV, 16, T>(c, ap, P, U, cb, combine);
  } else {
    switch (ap.gen_C) {
      case 8: launch_lr_gen<TI, TK, TV, 8>(c, ap, Lr, P, U, cb, combine); break;
      case 4: launch_lr_gen<TI, TK, TV, 4>(c, ap, Lr, P, U, cb, combine); break;
      case 2: launch_lr_gen<TI, TK, TV, 2>(c, ap, Lr, P, U, cb, combine); break;
      default: launch_lr_gen<TI, TK, TV, 1>(c, ap, Lr, P, U, cb, combine); break;
    }
  }
  launched(c);
}

// The whole operator: fused one-pass apply, or the lc pass (x1 -> U) then the
// lr pass combining (AP, <P, AP> or the true residual).
template <typename TI, typename TK, typename TV, typename TB>
void launch_apply(Ctx* c, const ApplyPlan& ap, Pull<TV> Lr, Pull<TV> Lc, const TI* P, TK* U,
                  const Combine<TK, TB>& cb) {
  if constexpr (sizeof(TI) == 4 && sizeof(TV) == 4) {
    if (ap.slab) {
      KScope ks_(c, "cg_apply");
      const bool o32 = ap.p * ap.ncols < (i64{1} << 31);
      auto k = cb.Xt ? (ap.s_evr == 9 ? (o32 ? slab_k<TK, 9, true, TB, true> : slab_k<TK, 9, true, TB>)
                                      : (o32 ? slab_k<TK, 16, true, TB, true> : slab_k<TK, 16, true, TB>))
                     : (ap.s_evr == 9 ? (o32 ? slab_k<TK, 9, false, TB, true> : slab_k<TK, 9, false, TB>)
                                      : (o32 ? slab_k<TK, 16, false, TB, true> : slab_k<TK, 16, false, TB>));
      ensure_smem(k, ap.s_smem);
      const SlabPlan sp{ap.s_rec.p,  reinterpret_cast<const SlabStep*>(ap.s_steps.p), ap.s_wsteps.p, ap.s_max_steps,
                        ap.s_win.p, ap.s_lv.p, ap.s_lo.p};
      // persistent, one CTA per SM (less the SMs a side-stream job holds)
      const unsigned grid = static_cast<unsigned>(std::max(1, std::min(ap.s_grid, c->num_sms - c->sm_reserve)));
      launch_pdl(k, dim3(grid), dim3(kSlabThreads), ap.s_smem, c->stream, static_cast<int>(ap.p),
                 static_cast<int>(ap.ncols), ap.s_parts, sp, P, cb);
      launched(c);
      return;
    }
  }
  if (ap.fused) {
    KScope ks_(c, "cg_apply");
    auto k = fused_k<TI, TK, TV, TB>;
    ensure_smem(k, ap.f_smem);
    launch_pdl(k, ap.f_grid, dim3(256), ap.f_smem, c->stream, static_cast<int>(ap.p), static_cast<int>(ap.ncols), Lr,
               Lc, ap.f_cpc, P, cb);
    launched(c);
    return;
  }
  const Combine<TK, TB> none{nullptr, nullptr, cb.gr, cb.gc, cb.pl, nullptr, nullptr, cb.st};
  Combine<TK, TB> cb2 = cb;
  cb2.other = U;
  launch_lc<TI, TK, TV, TB>(c, ap, Lc, P, U, none, false);
  launch_lr<TI, TK, TV, TB>(c, ap, Lr, P, nullptr, cb2, true);
}

// Host copy of a device pull (row pointers, columns and optionally values).
template <typename TV>
void host_pull(Ctx* c, const Pull<TV>& pv, i64 rows, i64 nnz, std::vector<i64>& rp, std::vector<int>& ci,
               std::vector<TV>* v) {
  rp.resize(static_cast<size_t>(rows) + 1);
  ci.resize(static_cast<size_t>(nnz));
  CUDA_OK(cudaMemcpyAsync(rp.data(), pv.rp, sizeof(i64) * (rows + 1), cudaMemcpyDeviceToHost, c->stream));
  if (nnz) CUDA_OK(cudaMemcpyAsync(ci.data(), pv.ci, sizeof(int) * nnz, cudaMemcpyDeviceToHost, c->stream));
  if (v) {
    v->resize(static_cast<size_t>(nnz));
    if (nnz) CUDA_OK(cudaMemcpyAsync(v->data(), pv.v, sizeof(TV) * nnz, cudaMemcpyDeviceToHost, c->stream));
  }
  sync(c);
}

}  // namespace cpcag_cuda
