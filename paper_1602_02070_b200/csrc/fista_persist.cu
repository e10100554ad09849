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
#include <type_traits>

#include "common.cuh"
#include "fista_persist.cuh"
#include "frpcag.cuh"

namespace cpcag_cuda {

namespace {

constexpr int kPT = 256;      // threads per CTA
constexpr int kMaxGrid = 160;      // CTAs (one per SM)
constexpr int kPsm = 4 * kMaxGrid;  // doubles of the partial-sum staging area
constexpr int kNst1 = 2;            // MODE 1 ring stages (A and S chunks)

template <typename T>
struct PersistArgs {
  int rr, rc, ldS, ldT;
  int TM, TN, C, KS, KC;
  int ldA, ldB;  // shared-memory row strides of the k-major A (TM) and B (TN) panels
  int use_r, use_c, loss;
  T step;
  double tol;
  i64 max_iter;
  double gamma_r, gamma_c;
  const T* Dr;  // rr x rr dense, exactly symmetric
  const T* Drs;  // MODE 1: g_r L~_r k-major with ldS rows per k (A panels streamed from it), padding rows 0
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

// fp64 tensor-core multiply-add (DMMA): D(8 x 8) += A(8 x 4) B(4 x 8), lane
// (g, t) = (lane / 4, lane % 4) supplies A(g, t) and B(t, g) and holds
// D(g, 2t), D(g, 2t + 1) (layout checked against a scalar product in
// tools/micro/dmma_peak.cu; 37 TFLOP/s measured vs 34 for DFMA).
__device__ __forceinline__ void dmma884(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
               : "+d"(d[0]), "+d"(d[1])
               : "d"(a), "d"(b));
}

// Swizzled k-major panel index for MODE 1: row k, column i.  Columns are
// XOR-ed by multiples of 8 elements per k (4 k-rows for fp32, 2 for fp64), so
// a DMMA operand load (8 columns x 4 k-rows) hits distinct banks; 16-byte
// groups stay contiguous (cp.async copies keep working).
template <typename T>
__device__ __forceinline__ int swz(int k, int i, int ld) {
  constexpr int W = sizeof(T) == 4 ? 3 : 1;
  return k * ld + (i ^ ((k & W) << 3));
}

// MODE 1 k-loop: acc (a 16 x 16 block at (m0, n0) as 2 x 2 DMMA tiles) +=
// A(m0.., k) B(k, n0..) for the k4 steps q = s, s + KS, ... < nk4 (k-split
// s).  A and B are shared byte addresses of swizzled k-major panels whose rows
// past the data are zero up to a multiple of 4, so the loop needs no bounds:
// lane (g, t) reads row 4 q + t, whose swizzle (t << 3) is loop-invariant.
template <typename T>
__device__ __forceinline__ T lds_t(unsigned a) {
  if constexpr (sizeof(T) == 4) {
    float v;
    asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(a));
    return v;
  } else {
    double v;
    asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(a));
    return v;
  }
}

template <typename T>
__device__ __forceinline__ void dmma_block(double (&acc)[2][2][2], unsigned A, int lda, unsigned B, int ldb, int nk4,
                                           int m0, int n0, int s, int KS, int lane) {
  constexpr unsigned E = sizeof(T);
  const int g = lane >> 2, t = lane & 3;
  const int sw = (t & (E == 4 ? 3 : 1)) << 3;
  const int k = 4 * s + t;
  unsigned a0 = A + static_cast<unsigned>(k * lda + ((m0 + g) ^ sw)) * E;
  unsigned a1 = A + static_cast<unsigned>(k * lda + ((m0 + 8 + g) ^ sw)) * E;
  unsigned b0 = B + static_cast<unsigned>(k * ldb + ((n0 + g) ^ sw)) * E;
  unsigned b1 = B + static_cast<unsigned>(k * ldb + ((n0 + 8 + g) ^ sw)) * E;
  const unsigned da = static_cast<unsigned>(4 * KS * lda) * E, db = static_cast<unsigned>(4 * KS * ldb) * E;
#pragma unroll 2
  for (int q = s; q < nk4; q += KS) {
    const double x0 = static_cast<double>(lds_t<T>(a0)), x1 = static_cast<double>(lds_t<T>(a1));
    const double y0 = static_cast<double>(lds_t<T>(b0)), y1 = static_cast<double>(lds_t<T>(b1));
    dmma884(acc[0][0], x0, y0);
    dmma884(acc[0][1], x0, y1);
    dmma884(acc[1][0], x1, y0);
    dmma884(acc[1][1], x1, y1);
    a0 += da;
    a1 += da;
    b0 += db;
    b1 += db;
  }
}

// MODE 0: 4 x 4 SIMT micro-tiles (fp64 DFMA on widened operands), the k range
//         split across thread groups (KS), partial tiles summed through shared
//         memory.
// MODE 1: fp64 tensor cores (DMMA m8n8k4): one warp per 16 x 16 block and
//         k-split s, operands widened once per load, k-major panels swizzled
//         (swz); partial tiles summed through shared memory as MODE 0.
template <typename T, int MODE>
__global__ void __launch_bounds__(MODE == 0 ? 256 : 512, 1) fista_persist_k(const PersistArgs<T> a) {
  constexpr int EPC = 16 / static_cast<int>(sizeof(T));  // values per 16-byte cp.async
  const int kPT = blockDim.x;
  // stages of the S-panel ring (MODE 0: 2 x 128-row chunks measured 16.1 us
  // per iteration vs 19.2 us for 4 x 64)
  constexpr int NST = MODE == 0 ? 2 : kNst1;
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
  // MODE 0 keeps g_r L~_r resident (As); MODE 1 streams it chunk by chunk (Ab)
  T* As = sm;                                                        // [rr][ldA]  g_r L~_r(r0 + i, k)
  T* Bc = As + (MODE == 0 ? static_cast<size_t>(rr) * ldA : 0);      // [rc4][ldB]  g_c L~_c(k, c0 + j)
  const int rc4 = (rc + 3) / 4 * 4;                                  // MODE 1: zero rows up to a multiple of 4
  T* A2 = Bc + static_cast<size_t>(rc4) * ldB;                       // [rc4][ldA]  S(r0 + i, k)
  T* Bb = A2 + static_cast<size_t>(rc4) * ldA;                       // [NST][KC][ldB]  S(k, c0 + j)
  T* Ab = Bb + NST * static_cast<size_t>(KC) * ldB;                  // MODE 1: [NST][KC][ldA]  g_r L~_r(r0 + i, k)
  T* Yt = Ab + (MODE == 1 ? NST * static_cast<size_t>(KC) * ldA : 0);  // tile state, e = i + TM j
  T* Zt = Yt + TE;                                // Z_j
  T* HZ = Zt + TE;                                // H(Z_j)
  T* Sp = HZ + TE;                                // S_{j-1}
  T* Hp = Sp + TE;                                // H(S_{j-1})
  T* Sc = Hp + TE;                                // S_j

  // ---- one-time staging of the pre-scaled operators and the tile of Y
  auto pidx = [&](int k, int i, int ld) { return MODE == 1 ? swz<T>(k, i, ld) : k * ld + i; };
  auto sh = [](const T* p) { return static_cast<unsigned>(__cvta_generic_to_shared(p)); };
  if (MODE == 0 && a.use_r)
    for (int t = tid; t < rr * TM; t += kPT) {
      const int k = t / TM, i = t - k * TM;
      // L~_r(r0 + i, k) from the column-major dense copy (contiguous in i)
      As[pidx(k, i, ldA)] =
          i < rn ? static_cast<T>(a.gamma_r * static_cast<double>(a.Dr[(r0 + i) + static_cast<i64>(k) * rr])) : T(0);
    }
  for (int t = tid; t < (rc4 - rc) * (TM > TN ? TM : TN); t += kPT) {  // padding rows of A2 and Bc
    const int k = rc + t / (TM > TN ? TM : TN), i = t % (TM > TN ? TM : TN);
    if (i < TM) A2[k * ldA + i] = T(0);
    if (i < TN) Bc[k * ldB + i] = T(0);
  }
  if (a.use_c)
    for (int t = tid; t < rc * TN; t += kPT) {
      const int k = t / TN, j = t - k * TN;
      Bc[pidx(k, j, ldB)] =
          j < cn ? static_cast<T>(a.gamma_c * static_cast<double>(a.Dc[(c0 + j) + static_cast<i64>(k) * rc])) : T(0);
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
  // MODE 1: warp -> (16 x 16 block, k-split)
  const int nbm = TM / 16, nblk = nbm * (TN / 16);
  const bool wd = MODE == 1 && warp < nblk * KS;
  const int wb = warp % max(nblk, 1), ws = warp / max(nblk, 1);
  const int m16 = 16 * (wb % max(nbm, 1)), n16 = 16 * (wb / max(nbm, 1));
  auto tile_gemm = [&](const T* Sbuf, const T* SbufT) {
    double acc[4][4];
    double accd[2][2][2];
#pragma unroll
    for (int x = 0; x < 4; ++x)
#pragma unroll
      for (int y = 0; y < 4; ++y) acc[x][y] = 0.0;
#pragma unroll
    for (int x = 0; x < 2; ++x)
#pragma unroll
      for (int y = 0; y < 2; ++y) accd[x][y][0] = accd[x][y][1] = 0.0;
    const int q4m = TM / EPC;
    if (a.use_c)  // S(r0.., k) for every k: TM contiguous floats per column k
      for (int t = tid; t < rc * q4m; t += kPT) {
        const int k = t / q4m, q = t - k * q4m;
        cp_async16(A2 + pidx(k, EPC * q, ldA), Sbuf + (r0 + EPC * q) + static_cast<i64>(k) * a.ldS);
      }
    cp_async_commit();  // group 0: A2 (and the caller's partial sums)
    const int nch = a.use_r ? (rr + KC - 1) / KC : 0;
    const int q4n = TN / EPC;
    auto issue_chunk = [&](int ch) {
      const int k0 = ch * KC, kl = min(KC, rr - k0);
      T* dst = Bb + (ch % NST) * KC * ldB;
      for (int t = tid; t < kl * q4n; t += kPT) {
        const int k = t / q4n, q = t - k * q4n;
        cp_async16(dst + pidx(k, EPC * q, ldB), SbufT + (c0 + EPC * q) + static_cast<i64>(k0 + k) * a.ldT);
      }
      if constexpr (MODE == 1) {
        T* dsa = Ab + (ch % NST) * KC * ldA;
        for (int t = tid; t < kl * q4m; t += kPT) {
          const int k = t / q4m, q = t - k * q4m;
          cp_async16(dsa + pidx(k, EPC * q, ldA), a.Drs + (r0 + EPC * q) + static_cast<i64>(k0 + k) * a.ldS);
        }
        const int kl4 = (kl + 3) / 4 * 4;  // rows past the data up to a multiple of 4: zeros
        for (int t = tid; t < (kl4 - kl) * (TM > TN ? TM : TN); t += kPT) {
          const int k = kl + t / (TM > TN ? TM : TN), i = t % (TM > TN ? TM : TN);
          if (i < TM) dsa[k * ldA + i] = T(0);
          if (i < TN) dst[k * ldB + i] = T(0);
        }
      }
    };
    // NST-stage ring: chunks 0 .. NST-2 in flight before the first one is used;
    // one CTA barrier per chunk: after it, every warp is done with chunk
    // ch - 1, whose slot the chunk issued next (ch + NST - 1) reuses
#pragma unroll
    for (int q = 0; q < NST - 1; ++q) {
      if (q < nch) issue_chunk(q);
      cp_async_commit();
    }
    for (int ch = 0; ch < nch; ++ch) {
      cp_async_wait<NST - 2>();  // A2 and chunk ch have landed
      __syncthreads();
      if (ch + NST - 1 < nch) issue_chunk(ch + NST - 1);
      cp_async_commit();
      if constexpr (MODE == 0) {
        if (gthr) {
          const int k0 = ch * KC, kl = min(KC, rr - k0);
          const int cnt = s < kl ? (kl - 1 - s) / KS + 1 : 0;
          strip_gemm(acc, As + static_cast<size_t>(k0 + s) * ldA + 4 * mi, KS * ldA,
                     Bb + (ch % NST) * KC * ldB + s * ldB + 4 * ni, KS * ldB, cnt);
        }
      } else {
        if (wd) {
          if (ch == 0 && a.use_c)  // the resident S L~_c part overlaps the chunks in flight
            dmma_block<T>(accd, sh(A2), ldA, sh(Bc), ldB, rc4 / 4, m16, n16, ws, KS, lane);
          const int k0 = ch * KC, kl = min(KC, rr - k0);
          dmma_block<T>(accd, sh(Ab + (ch % NST) * KC * ldA), ldA, sh(Bb + (ch % NST) * KC * ldB), ldB, (kl + 3) / 4,
                        m16, n16, ws, KS, lane);
        }
      }
    }
    __syncthreads();
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
      if (wd) {
        if (a.use_c && nch == 0) dmma_block<T>(accd, sh(A2), ldA, sh(Bc), ldB, rc4 / 4, m16, n16, ws, KS, lane);
        const int g = lane >> 2, t = lane & 3;
        double* o = red + static_cast<size_t>(ws) * TE;
#pragma unroll
        for (int x = 0; x < 2; ++x)
#pragma unroll
          for (int y = 0; y < 2; ++y)
#pragma unroll
            for (int q = 0; q < 2; ++q) o[(m16 + 8 * x + g) + TM * (n16 + 8 * y + 2 * t + q)] = accd[x][y][q];
      }
    }
    __syncthreads();
  };
  auto tile_h = [&](int e) {
    double h = 0.0;
    for (int q = 0; q < KS; ++q) h += red[q * TE + e];
    return static_cast<T>(h);
  };

  unsigned bar_g = 0;  // grid barriers passed (a.bar is zeroed before the launch)
  // ---- H(Y): Z_1 = S_0 = Y, so H(Z_1) = H(S_0)
  grid_barrier_mono(&a.bar[0], bar_g);
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
    grid_barrier_mono(&a.bar[0], bar_g);
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

// Drs[k ldS + i] = g_r Dr(i, k) rounded to T (the value MODE 0 stages), 0 for i >= rr.
template <typename T>
__global__ void scale_panel_k(i64 rr, i64 ldS, double g, const T* __restrict__ Dr, T* __restrict__ Drs) {
  const i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x;
  if (i >= ldS) return;
  for (i64 k = blockIdx.y; k < rr; k += gridDim.y)
    Drs[k * ldS + i] = i < rr ? static_cast<T>(g * static_cast<double>(Dr[i + k * rr])) : T(0);
}

struct Geom {
  int mode, TM, TN, R, C, KS, KC, ldA, ldB, threads;
  size_t smem;
};

size_t geom_smem(i64 rr, i64 rc, int TM, int TN, int ldA, int ldB, int KS, int KC, int nst, size_t w = 4,
                 int mode = 0) {
  const size_t TE = static_cast<size_t>(TM) * TN;
  const size_t rc4 = static_cast<size_t>((rc + 3) / 4 * 4);
  const size_t a_panel = mode == 0 ? static_cast<size_t>(rr) * ldA : static_cast<size_t>(nst) * KC * ldA;
  return 8 * kPsm + 8 * static_cast<size_t>(KS) * TE +
         w * (a_panel + rc4 * ldB + rc4 * ldA + static_cast<size_t>(nst) * KC * ldB + 6 * TE);
}

// MODE 1 (DMMA): TM a multiple of 32 (fp32; 16 for fp64) and TN of 32 (16),
// so the swizzled panels stay in range; one warp per 16 x 16 block and
// k-split (at most 16 warps).  The tensor pipe is shared per SM, so the
// per-CTA time follows TM TN (rr + rc): take the smallest tile area the SM
// count allows, then the most k-splits (latency hiding) and the longest S
// chunks the shared memory holds.
bool plan_mode1(Ctx* c, i64 rr, i64 rc, size_t budget, Geom* out, size_t w) {
  const i64 mq = w == 4 ? 32 : 16, nq = w == 4 ? 32 : 16;
  bool found = false;
  double best = 0.0;
  const i64 sms = c->num_sms;
  for (i64 TM = mq; TM <= std::max<i64>(mq, (rr + mq - 1) / mq * mq); TM += mq)
    for (i64 TN = nq; TN <= std::max<i64>(nq, (rc + nq - 1) / nq * nq); TN += nq) {
      const i64 R = (rr + TM - 1) / TM, C = (rc + TN - 1) / TN;
      if (R * C > sms) continue;
      const i64 blocks = (TM / 16) * (TN / 16);
      if (blocks > 16) continue;
      for (int KS = static_cast<int>(std::min<i64>(4, 16 / blocks)); KS >= 1; KS /= 2) {
        int KC = 0;
        size_t sm = 0;
        for (int kc : {256, 128, 64, 32}) {
          sm = geom_smem(rr, rc, static_cast<int>(TM), static_cast<int>(TN), static_cast<int>(TM), static_cast<int>(TN),
                         KS, kc, kNst1, w, 1);
          if (sm <= budget) {
            KC = kc;
            break;
          }
        }
        if (!KC) continue;
        const double cost = static_cast<double>(TM * TN) * static_cast<double>(rr + rc) * (1.0 + 0.25 / KS) +
                            64.0 * static_cast<double>(rr) / KC;
        if (!found || cost < best) {
          found = true;
          best = cost;
          *out = Geom{1, static_cast<int>(TM), static_cast<int>(TN), static_cast<int>(R), static_cast<int>(C), KS, KC,
                      static_cast<int>(TM), static_cast<int>(TN), static_cast<int>(blocks * KS * 32), sm};
        }
        break;  // the most k-splits that fit
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
  // MODE 1 (fp64 tensor cores) when its tiling fits, else MODE 0 (SIMT DFMA)
  const bool simt = c->fista_simt != 0;  // test hook: force the SIMT tile GEMM
  if (!(!simt && plan_mode1(c, rr, rc, budget, &g, sizeof(T))) && !plan_mode0(c, rr, rc, budget, &g, sizeof(T)))
    return false;
  const void* kfn = g.mode == 1 ? reinterpret_cast<const void*>(fista_persist_k<T, 1>)
                                : reinterpret_cast<const void*>(fista_persist_k<T, 0>);
  if (g.mode == 1)
    ensure_smem(fista_persist_k<T, 1>, g.smem);
  else
    ensure_smem(fista_persist_k<T, 0>, g.smem);
  int per_sm = 0;
  CUDA_OK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kfn, g.threads, g.smem));
  const i64 grid = static_cast<i64>(g.R) * g.C;
  if (per_sm < 1 || grid > static_cast<i64>(per_sm) * c->num_sms || grid > kMaxGrid) return false;

  const i64 ldS = static_cast<i64>(g.R) * g.TM, ldT = static_cast<i64>(g.C) * g.TN;
  const size_t sz = static_cast<size_t>(ldS * ldT);
  DevBuf<T> drs(c, g.mode == 1 ? static_cast<size_t>(rr) * ldS : 1);
  if (g.mode == 1 && cfg.gamma_r != 0.0) {
    dim3 gs(static_cast<unsigned>((ldS + 255) / 256), static_cast<unsigned>(std::min<i64>(rr, 65535)));
    scale_panel_k<T><<<gs, 256, 0, c->stream>>>(rr, ldS, cfg.gamma_r, Dr, drs.p);
    launched(c);
  }
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
  a.Drs = drs.p;
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
