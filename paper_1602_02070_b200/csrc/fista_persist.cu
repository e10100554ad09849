// fista_persist.cu -- the whole FISTA solve (frpcag.cpp:62-112, Algorithm 1
// of the paper) as ONE cooperative kernel, for the fp32
// path with dense Kron-reduced Laplacians (config 1: 1031 x 100, L~_r 56 %
// full, L~_c 100 % full).
//
// Why: at config-1 size one iteration is ~230 MFLOP and ~400 KB of state, so
// the per-kernel path (4 launches per iteration, split-K partial sums through
// HBM) is launch- and latency-bound at ~47 us per iteration.  Here the grid
// is one CTA per SM, each CTA owns an output tile (TM rows x TN columns) of
// every m-sized array for the whole solve, and an iteration costs one grid
// barrier:
//
//   phase A (tile-local)  S_j = prox(Z_j - step * 2 H(Z_j), Y, step)
//                         -> tile of S_j to global (column- and row-major)
//   grid barrier          (S_j complete; partial sums of iteration j-1 visible)
//   reduce j-1            objective, finite check, trace, stop test of j-1
//   phase B (tile GEMM)   H(S_j) = g_r L~_r S_j + g_c S_j L~_c for the tile:
//                         g_r L~_r rows resident in shared memory, S_j column
//                         panel streamed in k-chunks with cp.async (L2 -> smem)
//   phase B (tile-local)  objective partials, t_{j+1}, Z_{j+1} = S + coef
//                         (S - S_prev), H(Z_{j+1}) by linearity,
//                         ||Z_j||^2, ||Z_{j+1} - Z_j||^2 partials
//
// H = g_c S L~_c + g_r L~_r S is the only combination the solve reads: the
// gradient is 2 H(Z) (frpcag.cpp:53-60 with s = 2 g) and the two objective
// penalties are sum H(S) o S (frpcag.cpp:27-33; L~_c is exactly symmetric,
// so (L~_c S^T) o S^T sums like (S L~_c) o S).  The operators are pre-scaled
// by their weights once.  All reductions are fixed-order (per-CTA block
// sums, partials summed in block order by every CTA), so the run is
// deterministic and every CTA takes the same stop decision.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <string>

#include "common.cuh"
#include "fista_persist.cuh"
#include "frpcag.cuh"

namespace cpcag_cuda {

namespace {

constexpr int kPT = 256;      // threads per CTA
constexpr int kMaxGrid = 160;      // CTAs (one per SM)
constexpr int kPsm = 4 * kMaxGrid;  // doubles of the partial-sum staging area

template <typename T>
struct PersistArgs {
  int rr, rc, ldS, ldT;
  int TM, TN, C, KS, KC;
  int ldA, ldB;  // shared-memory row strides of the k-major A (TM) and B (TN) panels
  int use_r, use_c, loss;
  int dbg;  // diagnostics (CPCAG_FISTA_PERSIST_DBG): 1 = no B chunk loads, 2 = no chunk FMAs
  T step;
  double tol;
  i64 max_iter;
  double gamma_r, gamma_c;
  const T* Dr;  // rr x rr dense, exactly symmetric
  const T* Dc;  // rc x rc dense, exactly symmetric
  const T* Y;   // rr x rc column-major
  T* Sg[2];     // S_j column-major, ldS rows (padding rows stay 0)
  T* SgT[2];    // S_j row-major, ldT columns (padding stays 0)
  double* part;     // [2][grid][4] per-CTA partial sums by iteration parity
  double* trace;    // objective per iteration
  T* X;         // output, rr x rc column-major
  FistaPersistOut* out;
  unsigned* bar;    // grid barrier count, generation
};

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

__device__ __forceinline__ unsigned long long gtimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ float4 lds4(const float* p) { return *reinterpret_cast<const float4*>(p); }

// four consecutive values (16-byte aligned) of either precision
__device__ __forceinline__ void ld4v(const float* p, float (&v)[4]) {
  const float4 x = *reinterpret_cast<const float4*>(p);
  v[0] = x.x;
  v[1] = x.y;
  v[2] = x.z;
  v[3] = x.w;
}
__device__ __forceinline__ void ld4v(const double* p, double (&v)[4]) {
  const double2 x = *reinterpret_cast<const double2*>(p);
  const double2 y = *reinterpret_cast<const double2*>(p + 2);
  v[0] = x.x;
  v[1] = x.y;
  v[2] = y.x;
  v[3] = y.y;
}


// acc += sum over cnt k-steps of a(k) b(k)^T, a/b 4-value strips at strides
// sa/sb, k ascending, accumulated in fp64 for either storage precision: the
// products of fp32 operands are exact in fp64, and H = g L~ S sums ~1e3
// terms of magnitude up to ~1e4 that cancel to O(10) (Laplacian rows sum to
// zero), so an fp32 accumulator left ~4e-4 relative error in the config-1
// FISTA output after 300 iterations (above the 1e-4 bar; fp64: 1e-6).
// (Prefetching the operands four k-steps ahead measured slower: the loop is
// bound by shared-memory wavefronts, ncu: 4.4 per LDS.128.)
template <typename T>
__device__ __forceinline__ void strip_gemm(double (&acc)[4][4], const T* ap, int sa, const T* bp, int sb, int cnt) {
#pragma unroll 4
  for (int q = 0; q < cnt; ++q) {
    T av[4], bv[4];
    ld4v(ap + q * sa, av);
    ld4v(bp + q * sb, bv);
#pragma unroll
    for (int x = 0; x < 4; ++x)
#pragma unroll
      for (int y = 0; y < 4; ++y)
        acc[x][y] = fma(static_cast<double>(av[x]), static_cast<double>(bv[y]), acc[x][y]);
  }
}

// acc[x 8 + y] += a[x] b[y] for one k (8-float strips of A and B).
__device__ __forceinline__ void fma88(float (&acc)[64], const float* ap, const float* bp) {
  const float4 a0 = lds4(ap), a1 = lds4(ap + 4), b0 = lds4(bp), b1 = lds4(bp + 4);
  const float av[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
  const float bv[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
#pragma unroll
  for (int x = 0; x < 8; ++x)
#pragma unroll
    for (int y = 0; y < 8; ++y) acc[x * 8 + y] = fmaf(av[x], bv[y], acc[x * 8 + y]);
}

// Sum of the 64 partial entries over the 32 lanes, scattered: after five
// halving rounds (partner lane ^ 16, 8, 4, 2, 1; the lane with the bit set
// keeps the upper half) lane l holds entries 2 l and 2 l + 1 in acc[0..1].
// The summation tree is fixed, so the result is deterministic.
__device__ __forceinline__ void reduce_scatter64(float (&acc)[64], int lane) {
#pragma unroll
  for (int r = 0; r < 5; ++r) {
    const int o = 16 >> r, half = 32 >> r;
    const bool up = (lane & o) != 0;
#pragma unroll
    for (int i = 0; i < half; ++i) {
      const float send = up ? acc[i] : acc[i + half];
      const float keep = up ? acc[i + half] : acc[i];
      acc[i] = keep + __shfl_xor_sync(0xffffffffu, send, o);
    }
  }
}

// MODE 0: 4 x 4 micro-tiles, the k range split across thread groups (KS),
//         partial tiles summed through shared memory.
// MODE 1: 8 x 8 micro-tiles, one warp per micro-tile with the k range split
//         across its lanes, lanes reduced by a fixed shuffle reduce-scatter
//         (twice the multiply-adds per shared-memory wavefront of MODE 0).
template <typename T, int MODE>
__global__ void __launch_bounds__(MODE == 0 ? 256 : 512, 1) fista_persist_k(const PersistArgs<T> a) {
  static_assert(MODE == 0 || sizeof(T) == 4, "MODE 1 is fp32 only");
  constexpr int EPC = 16 / static_cast<int>(sizeof(T));  // values per 16-byte cp.async
  const int kPT = blockDim.x;
  // stages of the S-panel ring (MODE 0: 2 x 128-row chunks measured 16.1 us
  // per iteration vs 19.2 us for 4 x 64)
  constexpr int NST = MODE == 0 ? 2 : 4;
  extern __shared__ __align__(16) double smd[];
  double* psm = smd;  // [kPsm] partial sums of the previous iteration (4 per CTA)
  double* red = smd + kPsm;  // [KS][TE] split-k partial tiles (fp64; MODE 1: KS = 1)
  T* sm = reinterpret_cast<T*>(red + static_cast<size_t>(a.KS) * a.TM * a.TN);
  __shared__ double tot_sh[4];
  const int G = gridDim.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int TM = a.TM, TN = a.TN, TE = TM * TN, rr = a.rr, rc = a.rc, KC = a.KC, KS = a.KS;
  const int rb = blockIdx.x / a.C, cb = blockIdx.x % a.C;
  const int r0 = rb * TM, c0 = cb * TN;
  const int rn = min(TM, rr - r0), cn = min(TN, rc - c0);
  const int ldA = a.ldA, ldB = a.ldB;
  T* As = sm;                                      // [rr][ldA]  g_r L~_r(r0 + i, k)
  T* Bc = As + static_cast<size_t>(rr) * ldA;      // [rc][ldB]  g_c L~_c(k, c0 + j)
  T* A2 = Bc + static_cast<size_t>(rc) * ldB;      // [rc][ldA]  S(r0 + i, k)
  T* Bb = A2 + static_cast<size_t>(rc) * ldA;      // [2][KC][ldB]  S(k, c0 + j)
  T* Yt = Bb + NST * static_cast<size_t>(KC) * ldB;  // tile state, e = i + TM j
  T* Zt = Yt + TE;                                // Z_j
  T* HZ = Zt + TE;                                // H(Z_j)
  T* Sp = HZ + TE;                                // S_{j-1}
  T* Hp = Sp + TE;                                // H(S_{j-1})
  T* Sc = Hp + TE;                                // S_j

  // ---- one-time staging of the pre-scaled operators and the tile of Y
  if (a.use_r)
    for (int t = tid; t < rr * TM; t += kPT) {
      const int k = t / TM, i = t - k * TM;
      // L~_r(r0 + i, k) from the column-major dense copy (contiguous in i)
      As[k * ldA + i] = i < rn ? static_cast<T>(a.gamma_r * static_cast<double>(a.Dr[(r0 + i) + static_cast<i64>(k) * rr]))
                     : T(0);
    }
  if (a.use_c)
    for (int t = tid; t < rc * TN; t += kPT) {
      const int k = t / TN, j = t - k * TN;
      Bc[k * ldB + j] = j < cn ? static_cast<T>(a.gamma_c * static_cast<double>(a.Dc[(c0 + j) + static_cast<i64>(k) * rc]))
                     : T(0);
    }
  for (int e = tid; e < TE; e += kPT) {
    const int j = e / TM, i = e - j * TM;
    const bool ok = i < rn && j < cn;
    const T y = ok ? a.Y[(r0 + i) + static_cast<i64>(c0 + j) * rr] : T(0);
    Yt[e] = y;
    Zt[e] = y;  // Z_1 = Y
    Sp[e] = y;  // S_0 = Y
    Sc[e] = y;
    if (ok) {
      a.Sg[0][(r0 + i) + static_cast<i64>(c0 + j) * a.ldS] = y;
      a.SgT[0][(c0 + j) + static_cast<i64>(r0 + i) * a.ldT] = y;
    }
  }

  // ---- tile GEMM: red[s] = partial H of the tile over the k-slice of split s
  const int nmi = TM / 4, NMT = nmi * (TN / 4);
  const bool gthr = tid < NMT * KS;
  const int mt = tid % NMT, s = tid / NMT, mi = mt % nmi, ni = mt / nmi;
  const int mi8 = warp % max(TM / 8, 1), ni8 = warp / max(TM / 8, 1);
  const bool w8 = MODE == 1 && warp < (TM / 8) * (TN / 8);
  auto tile_gemm = [&](const T* Sbuf, const T* SbufT) {
    double acc[4][4];
    float acc8[MODE == 1 ? 64 : 1];
#pragma unroll
    for (int x = 0; x < 4; ++x)
#pragma unroll
      for (int y = 0; y < 4; ++y) acc[x][y] = 0.0;
#pragma unroll
    for (int q = 0; q < (MODE == 1 ? 64 : 1); ++q) acc8[q] = 0.f;
    const int q4m = TM / EPC, q4n = TN / EPC;
    if (a.use_c)  // S(r0.., k) for every k: TM contiguous floats per column k
      for (int t = tid; t < rc * q4m; t += kPT) {
        const int k = t / q4m, q = t - k * q4m;
        cp_async16(A2 + k * ldA + EPC * q, Sbuf + (r0 + EPC * q) + static_cast<i64>(k) * a.ldS);
      }
    cp_async_commit();  // group 0: A2 (and the caller's partial sums)
    const int nch = a.use_r ? (rr + KC - 1) / KC : 0;
    auto issue_chunk = [&](int ch) {
      const int k0 = ch * KC, kl = min(KC, rr - k0);
      T* dst = Bb + (ch % NST) * KC * ldB;
      for (int t = tid; t < kl * q4n; t += kPT) {
        const int k = t / q4n, q = t - k * q4n;
        cp_async16(dst + k * ldB + EPC * q, SbufT + (c0 + EPC * q) + static_cast<i64>(k0 + k) * a.ldT);
      }
    };
    // NST-stage ring: chunks 0 .. NST-2 in flight before the first one is used
#pragma unroll
    for (int q = 0; q < NST - 1; ++q) {
      if (q < nch && !(a.dbg & 1)) issue_chunk(q);
      cp_async_commit();
    }
    for (int ch = 0; ch < nch; ++ch) {
      if (ch + NST - 1 < nch && !(a.dbg & 1)) issue_chunk(ch + NST - 1);
      cp_async_commit();
      cp_async_wait<NST - 1>();  // A2 and chunk ch have landed
      __syncthreads();
      if constexpr (MODE == 0) {
        if (gthr && !(a.dbg & 2)) {
          const int k0 = ch * KC, kl = min(KC, rr - k0);
          const int cnt = s < kl ? (kl - 1 - s) / KS + 1 : 0;
          strip_gemm(acc, As + static_cast<size_t>(k0 + s) * ldA + 4 * mi, KS * ldA,
                     Bb + (ch % NST) * KC * ldB + s * ldB + 4 * ni, KS * ldB, cnt);
        }
      } else {
        if (w8) {
          if (ch == 0 && a.use_c)  // the resident S L~_c part overlaps the chunks in flight
            for (int k = lane; k < rc; k += 32) fma88(acc8, A2 + k * ldA + 8 * mi8, Bc + k * ldB + 8 * ni8);
          const int k0 = ch * KC, kl = min(KC, rr - k0);
          const float* ab = As + static_cast<size_t>(k0) * ldA + 8 * mi8;
          const float* bb = Bb + (ch % NST) * KC * ldB + 8 * ni8;
          for (int k = lane; k < kl; k += 32) fma88(acc8, ab + k * ldA, bb + k * ldB);
        }
      }
      __syncthreads();
    }
    if (nch == 0) {
      cp_async_wait<0>();
      __syncthreads();
    }
    if constexpr (MODE == 0) {
      if (a.use_c && gthr) {
        const int cnt = s < rc ? (rc - 1 - s) / KS + 1 : 0;
        strip_gemm(acc, A2 + s * ldA + 4 * mi, KS * ldA, Bc + s * ldB + 4 * ni, KS * ldB, cnt);
      }
      if (gthr) {
        double* o = red + static_cast<size_t>(s) * TE;
#pragma unroll
        for (int x = 0; x < 4; ++x)
#pragma unroll
          for (int y = 0; y < 4; ++y) o[(4 * mi + x) + TM * (4 * ni + y)] = acc[x][y];
      }
    } else {
      if (w8) {
        if (a.use_c && nch == 0)
          for (int k = lane; k < rc; k += 32) fma88(acc8, A2 + k * ldA + 8 * mi8, Bc + k * ldB + 8 * ni8);
        reduce_scatter64(acc8, lane);  // lane now holds entries 2 lane, 2 lane + 1 of the micro-tile
        const int x = lane >> 2, y = (2 * lane) & 7;
        double* o = red + (8 * mi8 + x) + TM * (8 * ni8 + y);
        o[0] = acc8[0];
        o[TM] = acc8[1];
      }
    }
    __syncthreads();
  };
  auto tile_h = [&](int e) {
    double h = 0.0;
    for (int q = 0; q < KS; ++q) h += red[q * TE + e];
    return static_cast<T>(h);
  };

  // ---- H(Y): Z_1 = S_0 = Y, so H(Z_1) = H(S_0)
  grid_barrier(&a.bar[0], &a.bar[1]);
  tile_gemm(a.Sg[0], a.SgT[0]);
  for (int e = tid; e < TE; e += kPT) {
    const float h = tile_h(e);
    HZ[e] = h;
    Hp[e] = h;
  }
  __syncthreads();

  const T step = a.step;
  // phase timers (CTA 0, thread 0; read by tools/fista_diag.py)
  unsigned long long pt[5] = {0, 0, 0, 0, 0}, tq = gtimer_ns();
  auto mark = [&](int ph) {
    if (tid == 0) {
      const unsigned long long now = gtimer_ns();
      pt[ph] += now - tq;
      tq = now;
    }
  };
  double t = 1.0;
  i64 J = 0;
  int conv = 0, err = 0;
  double frc = 0.0;
  for (i64 j = 1;; ++j) {
    const int b = static_cast<int>(j & 1);
    if (j <= a.max_iter) {
      // ---- phase A: gradient step + prox (frpcag.cpp:82-88)
      T* Sgb = a.Sg[b];
      T* SgTb = a.SgT[b];
      for (int e = tid; e < TE; e += kPT) {
        const int jj = e / TM, i = e - jj * TM;
        if (i < rn && jj < cn) {
          const T g = T(2) * HZ[e];
          const T arg = sub_rn(Zt[e], mul_rn(step, g));
          const T y = Yt[e];
          const T sv = a.loss == CPCAG_LOSS_L2 ? prox_l2_elem(arg, y, step) : prox_l1_elem(arg, y, step);
          Sc[e] = sv;
          Sgb[(r0 + i) + static_cast<i64>(c0 + jj) * a.ldS] = sv;
          SgTb[(c0 + jj) + static_cast<i64>(r0 + i) * a.ldT] = sv;
        }
      }
    }
    mark(0);
    grid_barrier(&a.bar[0], &a.bar[1]);
    mark(1);
    // partial sums of iteration j-1: cp.async (L2 -> shared, bypassing L1)
    // issued now, joining the GEMM's first copy group, consumed after the
    // tile GEMM (their L2 latency hides behind it)
    if (j >= 2 && warp == 0) {
      const double* pp = a.part + static_cast<size_t>((j - 1) & 1) * G * 4;
      for (int q = lane; q < 2 * G; q += 32) cp_async16(psm + 2 * q, pp + 2 * q);
    }
    // ---- phase B GEMM: H(S_j) (frpcag.cpp:89-90 penalties, linearity for Z)
    if (j <= a.max_iter) tile_gemm(a.Sg[b], a.SgT[b]);
    cp_async_commit();
    cp_async_wait<0>();
    __syncthreads();
    mark(3);
    if (j >= 2) {
      // ---- iteration j-1: objective, divergence, trace, stop test
      //      (frpcag.cpp:89-106)
      if (warp == 0) {
        double v[4] = {0.0, 0.0, 0.0, 0.0};
        for (int q = lane; q < G; q += 32)
#pragma unroll
          for (int u = 0; u < 4; ++u) v[u] += psm[q * 4 + u];
#pragma unroll
        for (int u = 0; u < 4; ++u) v[u] = warp_sum(v[u]);
        if (lane == 0)
#pragma unroll
          for (int u = 0; u < 4; ++u) tot_sh[u] = v[u];
      }
      __syncthreads();
      const double obj = tot_sh[0] + tot_sh[1];
      const double denom = tot_sh[2], change = tot_sh[3];
      __syncthreads();
      J = j - 1;
      if (!isfinite(obj)) {
        err = 1;
        break;
      }
      if (blockIdx.x == 0 && tid == 0) a.trace[j - 2] = obj;
      frc = denom > 0.0 ? change / denom : change;
      if (change < a.tol * denom) {
        conv = 1;
        break;
      }
    }
    if (j > a.max_iter) break;
    mark(2);

    // ---- phase B element-wise: objective partials, momentum (frpcag.cpp:89-110)
    const double tn = 0.5 * (1.0 + sqrt(1.0 + 4.0 * t * t));
    const T coef = static_cast<T>((t - 1.0) / tn);
    t = tn;
    double acc4[4] = {0.0, 0.0, 0.0, 0.0};
    for (int e = tid; e < TE; e += kPT) {
      const int jj = e / TM, i = e - jj * TM;
      if (i < rn && jj < cn) {
        const T h = tile_h(e);
        const T sv = Sc[e];
        const double d = static_cast<double>(Yt[e]) - static_cast<double>(sv);
        acc4[0] += a.loss == CPCAG_LOSS_L2 ? d * d : fabs(d);
        acc4[1] += static_cast<double>(h) * static_cast<double>(sv);
        const T zn = add_rn(sv, mul_rn(coef, sub_rn(sv, Sp[e])));
        const T hz = add_rn(h, mul_rn(coef, sub_rn(h, Hp[e])));
        const T z = Zt[e];
        const double zd = static_cast<double>(z), dd = static_cast<double>(sub_rn(zn, z));
        acc4[2] += zd * zd;
        acc4[3] += dd * dd;
        Sp[e] = sv;
        Hp[e] = h;
        Zt[e] = zn;
        HZ[e] = hz;
      }
    }
    block_sum<4>(acc4);
    if (tid == 0) {
      double* pp = a.part + static_cast<size_t>(j & 1) * G * 4 + static_cast<size_t>(blockIdx.x) * 4;
#pragma unroll
      for (int u = 0; u < 4; ++u) pp[u] = acc4[u];
    }
    mark(4);
  }
  // ---- output: the last prox result S_J (frpcag.cpp:111), own tile
  if (J >= 1 && !err) {
    const T* Sgb = a.Sg[J & 1];
    for (int e = tid; e < TE; e += kPT) {
      const int jj = e / TM, i = e - jj * TM;
      if (i < rn && jj < cn)
        a.X[(r0 + i) + static_cast<i64>(c0 + jj) * rr] = Sgb[(r0 + i) + static_cast<i64>(c0 + jj) * a.ldS];
    }
  }
  if (blockIdx.x == 0 && tid == 0) {
    a.out->iterations = J;
    a.out->converged = conv;
    a.out->err = err;
    a.out->frc = frc;
#pragma unroll
    for (int u = 0; u < 5; ++u) a.out->prof_ns[u] = pt[u];
  }
}

struct Geom {
  int mode, TM, TN, R, C, KS, KC, ldA, ldB, threads;
  size_t smem;
};

size_t geom_smem(i64 rr, i64 rc, int TM, int TN, int ldA, int ldB, int KS, int KC, int nst, size_t w = 4) {
  const size_t TE = static_cast<size_t>(TM) * TN;
  return 8 * kPsm + 8 * static_cast<size_t>(KS) * TE +
         w * (static_cast<size_t>(rr) * ldA + static_cast<size_t>(rc) * ldB + static_cast<size_t>(rc) * ldA +
              static_cast<size_t>(nst) * KC * ldB + 6 * TE);
}

// MODE 1 (preferred): TM, TN multiples of 8, one warp per 8 x 8 micro-tile
// (at most 16 warps), k-major panels padded by 4 floats so that lanes at
// different k hit distinct 16-byte bank groups; minimises the per-scheduler
// multiply-add work max(warps, 4) (rr + rc) within the shared-memory budget.
bool plan_mode1(Ctx* c, i64 rr, i64 rc, size_t budget, Geom* out) {
  bool found = false;
  double best = 0.0;
  const i64 sms = c->num_sms;
  const int fix_m = 0, fix_n = 0;
  for (i64 TM = 8; TM <= std::max<i64>(8, (rr + 7) / 8 * 8); TM += 8)
    for (i64 TN = 8; TN <= std::max<i64>(8, (rc + 7) / 8 * 8); TN += 8) {
      const i64 R = (rr + TM - 1) / TM, C = (rc + TN - 1) / TN;
      const i64 warps = (TM / 8) * (TN / 8);
      if (R * C > sms || warps > 16) continue;
      if (fix_m && (TM != fix_m || TN != fix_n)) continue;
      const int ldA = static_cast<int>(TM + 4), ldB = static_cast<int>(TN + 4);
      int KC = 64;
      size_t sm = geom_smem(rr, rc, static_cast<int>(TM), static_cast<int>(TN), ldA, ldB, 1, KC, 4);
      if (sm > budget) {
        KC = 32;
        sm = geom_smem(rr, rc, static_cast<int>(TM), static_cast<int>(TN), ldA, ldB, 1, KC, 4);
      }
      if (sm > budget) continue;
      // per-scheduler multiply-add work, plus the exposed latency of the S
      // panel ring: each of the ceil(rr / KC) chunks must cover ~1 us of L2
      // latency spread over the 3 chunks in flight (measured: a 8 x 104 tile
      // with 2 k-steps per lane per chunk ran latency-bound)
      const double work = static_cast<double>(std::max<i64>(warps, 4)) * static_cast<double>(rr + rc) * 64.0 / 4.0;
      const double chunk_work = static_cast<double>(std::max<i64>(warps, 4)) * KC * 64.0 / 4.0 / 32.0;
      const double cost = work + static_cast<double>((rr + KC - 1) / KC) * std::max(0.0, 700.0 - chunk_work) +
                          1e-3 * static_cast<double>(sm);
      if (!found || cost < best) {
        found = true;
        best = cost;
        *out = Geom{1, static_cast<int>(TM), static_cast<int>(TN), static_cast<int>(R), static_cast<int>(C), 1, KC,
                    ldA, ldB, static_cast<int>(std::max<i64>(warps, 4) * 32), sm};
      }
    }
  return found;
}

// MODE 0: R x C CTAs (at most one per SM), TM/TN multiples of 4, the k range
// split over thread groups; minimises the per-CTA multiply-add count TM TN
// (rr + rc) within the shared-memory budget.
bool plan_mode0(Ctx* c, i64 rr, i64 rc, size_t budget, Geom* out, size_t w = 4) {
  bool found = false;
  double best = 0.0;
  const i64 sms = c->num_sms;
  for (i64 TN = 4; TN <= ((rc + 3) / 4) * 4; TN += 4) {
    const i64 C = (rc + TN - 1) / TN;
    if (C > sms) continue;
    if ((rc + C - 1) / C + 3 < TN) continue;  // same C with a smaller TN exists
    const i64 Rmax = sms / C;
    i64 TM = ((rr + Rmax - 1) / Rmax + 3) / 4 * 4;
    for (; TM <= ((rr + 3) / 4) * 4; TM += 4) {
      const i64 NMT = (TM / 4) * (TN / 4);
      if (NMT > kPT) break;
      const int KS = static_cast<int>(std::min<i64>(8, kPT / NMT));
      int KC = 128;
      size_t sm = geom_smem(rr, rc, static_cast<int>(TM), static_cast<int>(TN), static_cast<int>(TM),
                            static_cast<int>(TN), KS, KC, 2, w);
      if (sm > budget) {
        KC = 32;
        sm = geom_smem(rr, rc, static_cast<int>(TM), static_cast<int>(TN), static_cast<int>(TM), static_cast<int>(TN),
                       KS, KC, 2, w);
      }
      if (sm > budget) break;  // a taller tile only needs more
      const i64 R = (rr + TM - 1) / TM;
      const double cost = static_cast<double>(TM * TN) * static_cast<double>(rr + rc) /
                          static_cast<double>(NMT * KS) + 64.0 * static_cast<double>(rr) / KC;
      if (!found || cost < best) {
        found = true;
        best = cost;
        *out = Geom{0, static_cast<int>(TM), static_cast<int>(TN), static_cast<int>(R), static_cast<int>(C), KS, KC,
                    static_cast<int>(TM), static_cast<int>(TN), kPT, sm};
      }
      break;  // the smallest feasible TM for this TN is the cheapest
    }
  }
  return found;
}

}  // namespace

bool fista_persist_enabled() {
  const char* e = std::getenv("CPCAG_FISTA_PERSIST");
  return !(e && std::string(e) == "0");
}

template <typename T>
bool fista_persist_run(Ctx* c, const T* Y, i64 rr, i64 rc, const T* Dr, const T* Dc, const cpcag_frpcag_config& cfg,
                       double step, T* X, double* trace_dev, FistaPersistOut* res) {
  if (rr < 1 || rc < 1 || rr > (1 << 20) || rc > (1 << 20)) return false;
  int optin = 0;
  CUDA_OK(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, c->device));
  const size_t budget = static_cast<size_t>(optin) > 4096 ? static_cast<size_t>(optin) - 4096 : 0;
  Geom g;
  // MODE 0 (wide row panels); the MODE 1 micro-tile variant measured no
  // faster at config 1 (16.6 vs 16.1 us per tile GEMM) and is not selected.
  const bool want1 = false;
  if (!(want1 && plan_mode1(c, rr, rc, budget, &g)) && !plan_mode0(c, rr, rc, budget, &g, sizeof(T))) return false;
  const void* kfn;
  if constexpr (sizeof(T) == 4) {
    kfn = g.mode == 1 ? reinterpret_cast<const void*>(fista_persist_k<T, 1>)
                      : reinterpret_cast<const void*>(fista_persist_k<T, 0>);
    if (g.mode == 1)
      ensure_smem(fista_persist_k<T, 1>, g.smem);
    else
      ensure_smem(fista_persist_k<T, 0>, g.smem);
  } else {
    kfn = reinterpret_cast<const void*>(fista_persist_k<T, 0>);
    ensure_smem(fista_persist_k<T, 0>, g.smem);
  }
  int per_sm = 0;
  CUDA_OK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kfn, g.threads, g.smem));
  const i64 grid = static_cast<i64>(g.R) * g.C;
  if (per_sm < 1 || grid > static_cast<i64>(per_sm) * c->num_sms || grid > kMaxGrid) return false;

  const i64 ldS = static_cast<i64>(g.R) * g.TM, ldT = static_cast<i64>(g.C) * g.TN;
  const size_t sz = static_cast<size_t>(ldS * ldT);
  DevBuf<T> sbuf(c, 4 * sz);
  sbuf.zero(c);
  DevBuf<double> part(c, 2 * 4 * static_cast<size_t>(grid));
  DevBuf<unsigned> bar(c, 2);
  bar.zero(c);
  DevBuf<FistaPersistOut> out(c, 1);
  out.zero(c);
  PersistArgs<T> a{};
  a.rr = static_cast<int>(rr);
  a.rc = static_cast<int>(rc);
  a.ldS = static_cast<int>(ldS);
  a.ldT = static_cast<int>(ldT);
  a.TM = g.TM;
  a.TN = g.TN;
  a.C = g.C;
  a.KS = g.KS;
  a.KC = g.KC;
  a.ldA = g.ldA;
  a.ldB = g.ldB;
  a.use_r = cfg.gamma_r != 0.0;
  a.use_c = cfg.gamma_c != 0.0;
  a.loss = cfg.loss;
  a.step = static_cast<T>(step);
  a.tol = cfg.tol;
  a.max_iter = cfg.max_iter;
  a.gamma_r = cfg.gamma_r;
  a.gamma_c = cfg.gamma_c;
  a.Dr = Dr;
  a.Dc = Dc;
  a.Y = Y;
  a.Sg[0] = sbuf.p;
  a.Sg[1] = sbuf.p + sz;
  a.SgT[0] = sbuf.p + 2 * sz;
  a.SgT[1] = sbuf.p + 3 * sz;
  a.part = part.p;
  a.trace = trace_dev;
  a.X = X;
  a.out = out.p;
  a.bar = bar.p;
  void* args[] = {(void*)&a};
  {
    KScope ks_(c, "fista_persist");
    CUDA_OK(cudaLaunchCooperativeKernel(kfn, dim3(static_cast<unsigned>(grid)), dim3(g.threads), args, g.smem,
                                        c->stream));
    launched(c);
  }
  *res = read_back(c, out.p);
  if (std::getenv("CPCAG_TRACE"))
    std::fprintf(stderr,
                 "[fista_persist] mode %d grid %lld (%d x %d tiles of %d x %d, KS %d, KC %d, %d threads, smem %zu) "
                 "its %lld: phaseA %.1f barrier %.1f reduce %.1f gemm %.1f elem %.1f us\n",
                 g.mode, static_cast<long long>(grid), g.R, g.C, g.TM, g.TN, g.KS, g.KC, g.threads, g.smem,
                 static_cast<long long>(res->iterations), res->prof_ns[0] * 1e-3, res->prof_ns[1] * 1e-3,
                 res->prof_ns[2] * 1e-3, res->prof_ns[3] * 1e-3, res->prof_ns[4] * 1e-3);
  return true;
}

template bool fista_persist_run<float>(Ctx*, const float*, i64, i64, const float*, const float*,
                                       const cpcag_frpcag_config&, double, float*, double*, FistaPersistOut*);
template bool fista_persist_run<double>(Ctx*, const double*, i64, i64, const double*, const double*,
                                        const cpcag_frpcag_config&, double, double*, double*, FistaPersistOut*);

}  // namespace cpcag_cuda
