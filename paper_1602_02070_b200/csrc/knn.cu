// knn.cu -- kNN graph construction (graph.cpp:47-135), graph_from_adjacency
// (graph.cpp:137-154) and the Laplacian assembly (graph.cpp:16-43).
//
// Neighbour selection is exact with respect to the reference's canonical
// fp64 distance d2(i,j) = max(0, (g_ii + g_jj) - 2 g_ij) where every Gram
// entry is the k-ascending sum of products with separate rounding (no FMA):
// the tiled Gram kernel keeps one accumulator per pair and walks k in order,
// so the value is bit-identical to the oracle's (and symmetric in i, j
// because products commute).  Per-row top-K is kept under the lexicographic
// (d2, j) order, i.e. ties go to the lower index (graph.cpp:93-96).
//
// Layout: points are gathered point-major (n x d fp64, each point
// contiguous) so a 64-point x 16-k tile is 64 coalesced 128-byte reads.  A
// CTA owns 64 query points and sweeps a range of 64-point candidate tiles;
// the candidate range is split across CTAs when n/64 alone cannot fill the
// 148 SMs, and the per-split top-K lists are merged afterwards.
//
// Graph assembly: 2nK directed (row, col, d2) records -> one radix sort on
// (row << 32 | col) -> duplicates dropped (union symmetrisation) ->
// Gaussian weights (w == 0 dropped) -> CSR W -> degrees -> CSR L.
#include <algorithm>
#include <cstdio>
#include <cub/cub.cuh>
#include <math_constants.h>

#include <cstdlib>
#include <memory>
#include <string>

#include "common.cuh"

namespace cpcag_cuda {

constexpr int kTile = 64;   // points per tile side
constexpr int kKc = 16;     // k-chunk staged in shared memory
constexpr int kMaxK = 64;   // largest supported neighbour count
constexpr size_t kKnnSmem = (2 * kKc + kTile) * (kTile + 1) * sizeof(double) +
                            kTile * (kMaxK + 1) * (sizeof(double) + sizeof(int));

template <typename T>
__global__ void gather_points_k(const T* __restrict__ X, i64 x_rows, i64 n, i64 d, int axis_rows,
                                double* __restrict__ Pm) {
  const i64 t = blockIdx.x * (i64)blockDim.x + threadIdx.x;
  if (t >= n * d) return;
  const i64 i = t / d, k = t % d;
  Pm[t] = static_cast<double>(axis_rows ? X[i + k * x_rows] : X[k + i * x_rows]);
}

// g_ii summed over k in order (the canonical Gram diagonal).  A warp owns 32
// points; each 32-wide k slab is loaded coalesced (one point row per load)
// and transposed through shared memory so lane r accumulates point r's slab
// in k order.
__global__ void __launch_bounds__(256) sqnorm_k(const double* __restrict__ Pm, i64 n, i64 d,
                                                double* __restrict__ sq) {
  // one warp per point: 32-value chunks of its row read coalesced one chunk
  // ahead, the sum over k in order with separate rounding (the canonical
  // g_ii) run redundantly by every lane on shuffled values
  const i64 i = (blockIdx.x * (i64)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (i >= n) return;
  const double* r = Pm + i * d;
  double s = 0.0;
  double cur = lane < d ? r[lane] : 0.0;
  for (i64 k0 = 0; k0 < d; k0 += 32) {
    const double nxt = k0 + 32 + lane < d ? r[k0 + 32 + lane] : 0.0;
    const int cnt = static_cast<int>(min(static_cast<i64>(32), d - k0));
#pragma unroll 8
    for (int u = 0; u < cnt; ++u) {
      const double x = __shfl_sync(0xffffffffu, cur, u);
      s = __dadd_rn(s, __dmul_rn(x, x));
    }
    cur = nxt;
  }
  if (lane == 0) sq[i] = s;
}

__device__ __forceinline__ bool lex_less(double da, int ja, double db, int jb) {
  return da < db || (da == db && ja < jb);
}

// One CTA: 64 query points x candidate tiles [jt0, jt1).  Output: per query
// point the K best (d2, j) of the range, ascending, into cand[split].
// qidx (optional): the query points are qidx[0..nq) instead of 0..n-1 (used
// for the rows the tensor-core filter could not certify); outputs are indexed
// by query position.
__global__ void __launch_bounds__(256) knn_tile_k(const double* __restrict__ Pm, const double* __restrict__ sq,
                                                  i64 n, i64 d, int K, int tiles_per_split,
                                                  double* __restrict__ cand_d, int* __restrict__ cand_j,
                                                  int* __restrict__ dup, const int* __restrict__ qidx, i64 nq) {
  extern __shared__ __align__(16) unsigned char smem[];
  double(*As)[kTile + 1] = reinterpret_cast<double(*)[kTile + 1]>(smem);
  double(*Bs)[kTile + 1] = As + kKc;
  double(*Dt)[kTile + 1] = Bs + kKc;
  double(*best_d)[kMaxK + 1] = reinterpret_cast<double(*)[kMaxK + 1]>(Dt + kTile);
  int(*best_j)[kMaxK + 1] = reinterpret_cast<int(*)[kMaxK + 1]>(best_d + kTile);

  const int tid = threadIdx.x;
  const int tx = tid & 15, ty = tid >> 4;
  const i64 i0 = static_cast<i64>(blockIdx.x) * kTile;
  const int split = blockIdx.y;
  const i64 n_tiles = (n + kTile - 1) / kTile;
  const i64 jt0 = static_cast<i64>(split) * tiles_per_split;
  const i64 jt1 = min(n_tiles, jt0 + tiles_per_split);

  if (tid < kTile)
    for (int q = 0; q < K; ++q) {
      best_d[tid][q] = CUDART_INF;
      best_j[tid][q] = INT32_MAX;
    }
  __syncthreads();

  for (i64 jt = jt0; jt < jt1; ++jt) {
    const i64 j0 = jt * kTile;
    double acc[4][4];
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
      for (int s = 0; s < 4; ++s) acc[r][s] = 0.0;

    for (i64 k0 = 0; k0 < d; k0 += kKc) {
      // Stage 64 x 16 of A (queries) and B (candidates), transposed.
#pragma unroll
      for (int q = 0; q < (kTile * kKc) / 256; ++q) {
        const int idx = tid + 256 * q;
        const int pt = idx / kKc, kk = idx % kKc;
        const i64 k = k0 + kk;
        const i64 qa = i0 + pt, jb = j0 + pt;
        const i64 ia = qa < nq ? (qidx ? qidx[qa] : qa) : n;
        As[kk][pt] = (ia < n && k < d) ? Pm[ia * d + k] : 0.0;
        Bs[kk][pt] = (jb < n && k < d) ? Pm[jb * d + k] : 0.0;
      }
      __syncthreads();
#pragma unroll
      for (int kk = 0; kk < kKc; ++kk) {
        double a[4], b[4];
#pragma unroll
        for (int r = 0; r < 4; ++r) a[r] = As[kk][ty + 16 * r];
#pragma unroll
        for (int s = 0; s < 4; ++s) b[s] = Bs[kk][tx + 16 * s];
#pragma unroll
        for (int r = 0; r < 4; ++r)
#pragma unroll
          for (int s = 0; s < 4; ++s) acc[r][s] = __dadd_rn(acc[r][s], __dmul_rn(a[r], b[s]));
      }
      __syncthreads();
    }
    // d2 tile (graph.cpp:63), masked outside the matrix and on the diagonal.
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
      for (int s = 0; s < 4; ++s) {
        const int li = ty + 16 * r, lj = tx + 16 * s;
        const i64 qi = i0 + li, gj = j0 + lj;
        const i64 gi = qi < nq ? (qidx ? qidx[qi] : qi) : n;
        double v = CUDART_INF;
        if (gi < n && gj < n && gi != gj) {
          const double t = __dsub_rn(__dadd_rn(sq[gi], sq[gj]), __dmul_rn(2.0, acc[r][s]));
          v = t > 0.0 ? t : 0.0;
        }
        Dt[li][lj] = v;
      }
    __syncthreads();
    if (tid < kTile) {
      const i64 qi = i0 + tid;
      const i64 gi = qi < nq ? (qidx ? qidx[qi] : qi) : n;
      if (gi < n) {
        for (int lj = 0; lj < kTile; ++lj) {
          const double v = Dt[tid][lj];
          const int gj = static_cast<int>(j0 + lj);
          if (v == 0.0 && gj < gi && gj < n && !dup[gi]) {
            // Coincident candidate: exact coordinate test (graph.cpp:68-84).
            const double* a = Pm + gi * d;
            const double* b = Pm + static_cast<i64>(gj) * d;
            bool same = true;
            for (i64 k = 0; k < d && same; ++k) same = a[k] == b[k];
            if (same) dup[gi] = 1;
          }
          if (!lex_less(v, gj, best_d[tid][K - 1], best_j[tid][K - 1])) continue;
          int q = K - 1;
          while (q > 0 && lex_less(v, gj, best_d[tid][q - 1], best_j[tid][q - 1])) {
            best_d[tid][q] = best_d[tid][q - 1];
            best_j[tid][q] = best_j[tid][q - 1];
            --q;
          }
          best_d[tid][q] = v;
          best_j[tid][q] = gj;
        }
      }
    }
    __syncthreads();
  }
  if (tid < kTile) {
    const i64 qi = i0 + tid;
    if (qi < nq) {
      double* od = cand_d + (static_cast<i64>(split) * nq + qi) * K;
      int* oj = cand_j + (static_cast<i64>(split) * nq + qi) * K;
      for (int q = 0; q < K; ++q) {
        od[q] = best_d[tid][q];
        oj[q] = best_j[tid][q];
      }
    }
  }
}

// All-points search over the upper triangle of 64-point tile pairs: g_ij and
// g_ji are the same bits (products commute, same k order), so one CTA per
// pair (it <= jt) forms the 64 x 64 d2 tile once and feeds both top-K
// lists: queries of `it` over candidates of `jt` (threads 0-63) and, off the
// diagonal, queries of `jt` over candidates of `it` (threads 64-127, reading
// the tile transposed).  Half the Gram work of knn_tile_k.  Output list
// (source tile s, query i) goes to cand[(s n + i) K]: every (s, i) is written
// by exactly one CTA.  The k-chunks are double-buffered through registers
// (one barrier per chunk): the 166 KB of shared memory leaves one CTA per SM.
constexpr int kKcS = 64;  // k-chunk of the symmetric kernel (one barrier per 64 k)
constexpr size_t kKnnSymStage = 4 * kKcS * (kTile + 1) * sizeof(double);
constexpr size_t kKnnSymTail = kTile * (kTile + 1) * sizeof(double) +
                               2 * kTile * (kMaxK + 1) * (sizeof(double) + sizeof(int));
constexpr size_t kKnnSymSmem = kKnnSymStage > kKnnSymTail ? kKnnSymStage : kKnnSymTail;

__device__ __forceinline__ void topk_insert(double* bd, int* bj, int K, double v, int j) {
  if (!lex_less(v, j, bd[K - 1], bj[K - 1])) return;
  int q = K - 1;
  while (q > 0 && lex_less(v, j, bd[q - 1], bj[q - 1])) {
    bd[q] = bd[q - 1];
    bj[q] = bj[q - 1];
    --q;
  }
  bd[q] = v;
  bj[q] = j;
}

// coincident candidate j < i of query i (d2 == 0): exact coordinate test (graph.cpp:68-84)
__device__ __forceinline__ void dup_check(const double* __restrict__ Pm, i64 d, i64 i, i64 j, int* dup) {
  if (dup[i]) return;
  const double* a = Pm + i * d;
  const double* b = Pm + j * d;
  bool same = true;
  for (i64 k = 0; k < d && same; ++k) same = a[k] == b[k];
  if (same) dup[i] = 1;
}

template <int kThreads>
__global__ void __launch_bounds__(kThreads) knn_sym_k(const double* __restrict__ Pm, const double* __restrict__ sq,
                                                 i64 n, i64 d, int K, int T, double* __restrict__ cand_d,
                                                 int* __restrict__ cand_j, int* __restrict__ dup) {
  extern __shared__ __align__(16) unsigned char smem[];
  using Row = double[kTile + 1];
  Row* As = reinterpret_cast<Row*>(smem);  // [2][kKcS]
  Row* Bs = As + 2 * kKcS;                 // [2][kKcS]
  Row* Dt = reinterpret_cast<Row*>(smem);  // [kTile], over the staging buffers once the Gram is done
  double(*best_d)[kMaxK + 1] = reinterpret_cast<double(*)[kMaxK + 1]>(Dt + kTile);  // [2 kTile]
  int(*best_j)[kMaxK + 1] = reinterpret_cast<int(*)[kMaxK + 1]>(best_d + 2 * kTile);

  const int tid = threadIdx.x;
  const int tx = tid & 15, ty = tid >> 4;
  int pr = blockIdx.x, it = 0;
  while (pr >= T - it) {
    pr -= T - it;
    ++it;
  }
  const int jt = it + pr;
  const i64 i0 = static_cast<i64>(it) * kTile, j0 = static_cast<i64>(jt) * kTile;

  constexpr int kPer = (kTile * kKcS) / kThreads;
  constexpr int kRows = kTile / (kThreads / 16);  // accumulator rows per thread (16 column groups of 4)
  constexpr int kRs = kThreads / 16;              // row stride
  double ra[kPer], rb[kPer];
  auto load = [&](i64 k0) {
#pragma unroll
    for (int q = 0; q < kPer; ++q) {
      const int idx = tid + kThreads * q, pt = idx / kKcS;
      const i64 k = k0 + idx % kKcS;
      ra[q] = (i0 + pt < n && k < d) ? Pm[(i0 + pt) * d + k] : 0.0;
      rb[q] = (j0 + pt < n && k < d) ? Pm[(j0 + pt) * d + k] : 0.0;
    }
  };
  auto store = [&](int buf) {
#pragma unroll
    for (int q = 0; q < kPer; ++q) {
      const int idx = tid + kThreads * q, pt = idx / kKcS, kk = idx % kKcS;
      As[buf * kKcS + kk][pt] = ra[q];
      Bs[buf * kKcS + kk][pt] = rb[q];
    }
  };
  double acc[kRows][4];
#pragma unroll
  for (int r = 0; r < kRows; ++r)
#pragma unroll
    for (int s = 0; s < 4; ++s) acc[r][s] = 0.0;
  const i64 nch = (d + kKcS - 1) / kKcS;
  load(0);
  store(0);
  __syncthreads();
  for (i64 ch = 0; ch < nch; ++ch) {
    const int buf = static_cast<int>(ch & 1);
    if (ch + 1 < nch) load((ch + 1) * kKcS);  // next chunk in flight during this one's products
    const Row* A = As + buf * kKcS;
    const Row* B = Bs + buf * kKcS;
#pragma unroll
    for (int kk = 0; kk < kKcS; ++kk) {
      double a[kRows], b[4];
#pragma unroll
      for (int r = 0; r < kRows; ++r) a[r] = A[kk][ty + kRs * r];
#pragma unroll
      for (int s = 0; s < 4; ++s) b[s] = B[kk][tx + 16 * s];
#pragma unroll
      for (int r = 0; r < kRows; ++r)
#pragma unroll
        for (int s = 0; s < 4; ++s) acc[r][s] = __dadd_rn(acc[r][s], __dmul_rn(a[r], b[s]));
    }
    if (ch + 1 < nch) store(buf ^ 1);
    __syncthreads();
  }
  // d2 tile (graph.cpp:63), masked outside the matrix and on the diagonal
  // (the loop's last barrier retired every read of the staging buffers)
  if (tid < 2 * kTile)
    for (int q = 0; q < K; ++q) {
      best_d[tid][q] = CUDART_INF;
      best_j[tid][q] = INT32_MAX;
    }
#pragma unroll
  for (int r = 0; r < kRows; ++r)
#pragma unroll
    for (int s = 0; s < 4; ++s) {
      const int li = ty + kRs * r, lj = tx + 16 * s;
      const i64 gi = i0 + li, gj = j0 + lj;
      double v = CUDART_INF;
      if (gi < n && gj < n && gi != gj) {
        const double t = __dsub_rn(__dadd_rn(sq[gi], sq[gj]), __dmul_rn(2.0, acc[r][s]));
        v = t > 0.0 ? t : 0.0;
      }
      Dt[li][lj] = v;
    }
  __syncthreads();
  if (tid < kTile) {  // queries of tile it, candidates of tile jt
    const i64 gi = i0 + tid;
    if (gi < n) {
      for (int lj = 0; lj < kTile; ++lj) {
        const double v = Dt[tid][lj];
        const i64 gj = j0 + lj;
        if (v == 0.0 && gj < gi && gj < n) dup_check(Pm, d, gi, gj, dup);
        topk_insert(best_d[tid], best_j[tid], K, v, static_cast<int>(gj < n ? gj : INT32_MAX));
      }
      double* od = cand_d + (static_cast<i64>(jt) * n + gi) * K;
      int* oj = cand_j + (static_cast<i64>(jt) * n + gi) * K;
      for (int q = 0; q < K; ++q) {
        od[q] = best_d[tid][q];
        oj[q] = best_j[tid][q];
      }
    }
  } else if (tid < 2 * kTile && it != jt) {  // queries of tile jt, candidates of tile it
    const int q0 = tid - kTile;
    const i64 gq = j0 + q0;
    if (gq < n) {
      for (int li = 0; li < kTile; ++li) {
        const double v = Dt[li][q0];
        const i64 gc = i0 + li;
        if (v == 0.0 && gc < gq && gc < n) dup_check(Pm, d, gq, gc, dup);
        topk_insert(best_d[tid], best_j[tid], K, v, static_cast<int>(gc < n ? gc : INT32_MAX));
      }
      double* od = cand_d + (static_cast<i64>(it) * n + gq) * K;
      int* oj = cand_j + (static_cast<i64>(it) * n + gq) * K;
      for (int q = 0; q < K; ++q) {
        od[q] = best_d[tid][q];
        oj[q] = best_j[tid][q];
      }
    }
  }
}

// Merge the per-split sorted lists of each point; mean d2 in ascending order.
__global__ void knn_merge_k(i64 n, int K, int splits, const double* __restrict__ cand_d,
                            const int* __restrict__ cand_j, int64_t* __restrict__ nbr,
                            double* __restrict__ nbr_d2, double* __restrict__ mean_d2,
                            const int* __restrict__ qidx) {
  const i64 qq = blockIdx.x * (i64)blockDim.x + threadIdx.x;
  if (qq >= n) return;
  const i64 i = qq;                         // position in the candidate arrays
  const i64 o = qidx ? qidx[qq] : qq;       // output row
  int pos[64];
  const int S = splits < 64 ? splits : 64;
  for (int s = 0; s < S; ++s) pos[s] = 0;
  double m = 0.0;
  for (int q = 0; q < K; ++q) {
    int bs = -1;
    double bd = CUDART_INF;
    int bj = INT32_MAX;
    for (int s = 0; s < S; ++s) {
      if (pos[s] >= K) continue;
      const i64 at = (static_cast<i64>(s) * n + i) * K + pos[s];
      const double dv = cand_d[at];
      const int jv = cand_j[at];
      if (bs < 0 || lex_less(dv, jv, bd, bj)) {
        bs = s;
        bd = dv;
        bj = jv;
      }
    }
    pos[bs]++;
    nbr[o * K + q] = bj;
    nbr_d2[o * K + q] = bd;
    m = __dadd_rn(m, bd);
  }
  mean_d2[o] = m;
}

// sigma2 = sum_i (mean_i / K) / n, summed in point order (graph.cpp:104-107).
// sigma^2 = (sum_i mean_d2[i] / K) / n with the reference's left-to-right
// sum (graph.cpp:104,107).  The divisions are independent (q_i, parallel);
// only the additions form the sequential chain.
__global__ void sigma2_div_k(i64 n, int K, const double* __restrict__ mean_d2, double* __restrict__ q) {
  const i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x;
  if (i < n) q[i] = __ddiv_rn(mean_d2[i], static_cast<double>(K));
}
__global__ void sigma2_k(i64 n, const double* __restrict__ q, double override_, double* out) {
  if (blockIdx.x || threadIdx.x) return;
  double s = 0.0;
  i64 i = 0;
  for (; i + 8 <= n; i += 8) {
    double v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) v[u] = q[i + u];
#pragma unroll
    for (int u = 0; u < 8; ++u) s = __dadd_rn(s, v[u]);
  }
  for (; i < n; ++i) s = __dadd_rn(s, q[i]);
  *out = override_ > 0.0 ? override_ : __ddiv_rn(s, static_cast<double>(n));
}

__global__ void count_dup_k(i64 n, const int* __restrict__ dup, unsigned long long* cnt) {
  const i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x;
  if (i < n && dup[i]) atomicAdd(cnt, 1ull);
}

// 2nK directed records keyed (row << 32 | col).
__global__ void edge_records_k(i64 n, int K, const int64_t* __restrict__ nbr, const double* __restrict__ nbr_d2,
                               unsigned long long* __restrict__ keys, double* __restrict__ vals) {
  const i64 t = blockIdx.x * (i64)blockDim.x + threadIdx.x;
  if (t >= n * K) return;
  const unsigned long long i = static_cast<unsigned long long>(t / K);
  const unsigned long long j = static_cast<unsigned long long>(nbr[t]);
  keys[2 * t] = (i << 32) | j;
  keys[2 * t + 1] = (j << 32) | i;
  vals[2 * t] = nbr_d2[t];
  vals[2 * t + 1] = nbr_d2[t];
}

// Unique edges with a nonzero Gaussian weight (graph.cpp:116-124).
__global__ void edge_weight_k(i64 m, const unsigned long long* __restrict__ keys, const double* __restrict__ d2,
                              const double* __restrict__ sigma2, double* __restrict__ w, i64* __restrict__ keep) {
  const i64 t = blockIdx.x * (i64)blockDim.x + threadIdx.x;
  if (t >= m) return;
  const bool first = t == 0 || keys[t] != keys[t - 1];
  const double dv = d2[t];
  const double wv = dv == 0.0 ? 1.0 : exp(__ddiv_rn(-dv, *sigma2));
  w[t] = wv;
  keep[t] = (first && wv != 0.0) ? 1 : 0;
}

__global__ void edge_rowptr_k(i64 n, i64 m, const unsigned long long* __restrict__ keys,
                              const i64* __restrict__ incl, i64* __restrict__ rp) {
  const i64 r = blockIdx.x * (i64)blockDim.x + threadIdx.x;
  if (r > n) return;
  // first record with row >= r
  i64 lo = 0, hi = m;
  const unsigned long long key = static_cast<unsigned long long>(r) << 32;
  while (lo < hi) {
    const i64 mid = (lo + hi) >> 1;
    if (keys[mid] < key) lo = mid + 1; else hi = mid;
  }
  rp[r] = lo == 0 ? 0 : incl[lo - 1];
}

__global__ void edge_fill_k(i64 m, const unsigned long long* __restrict__ keys, const double* __restrict__ w,
                            const i64* __restrict__ keep, const i64* __restrict__ incl, int* __restrict__ ci,
                            double* __restrict__ v) {
  const i64 t = blockIdx.x * (i64)blockDim.x + threadIdx.x;
  if (t >= m || !keep[t]) return;
  const i64 o = incl[t] - 1;
  ci[o] = static_cast<int>(keys[t] & 0xffffffffull);
  v[o] = w[t];
}

// Row sums in CSR order (sparse.cpp:159-168).
__global__ void row_sums_k(i64 n, const i64* __restrict__ rp, const double* __restrict__ v, double* __restrict__ out) {
  const i64 r = blockIdx.x * (i64)blockDim.x + threadIdx.x;
  if (r >= n) return;
  double s = 0.0;
  for (i64 k = rp[r]; k < rp[r + 1]; ++k) s = __dadd_rn(s, v[k]);
  out[r] = s;
}

// Laplacian rows (graph.cpp:16-43): combinatorial D - W (diagonal iff
// deg != 0) or normalised I - D^-1/2 W D^-1/2 (entries -w dis_r dis_c,
// exact zeros dropped).
__device__ __forceinline__ double lap_off(int kind, double w, const double* dis, i64 r, int c) {
  return kind == CPCAG_COMBINATORIAL ? -w : __dmul_rn(__dmul_rn(-w, dis[r]), dis[c]);
}

__global__ void dis_k(i64 n, const double* __restrict__ deg, double* __restrict__ dis) {
  const i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x;
  if (i < n) dis[i] = deg[i] > 0.0 ? __ddiv_rn(1.0, __dsqrt_rn(deg[i])) : 0.0;
}

__global__ void lap_count_k(i64 n, int kind, const i64* __restrict__ rp, const int* __restrict__ ci,
                            const double* __restrict__ v, const double* __restrict__ deg,
                            const double* __restrict__ dis, i64* __restrict__ cnt) {
  const i64 r = blockIdx.x * (i64)blockDim.x + threadIdx.x;
  if (r >= n) return;
  i64 c = (kind == CPCAG_COMBINATORIAL ? deg[r] != 0.0 : deg[r] > 0.0) ? 1 : 0;
  for (i64 k = rp[r]; k < rp[r + 1]; ++k) c += lap_off(kind, v[k], dis, r, ci[k]) != 0.0;
  cnt[r] = c;
}

__global__ void lap_fill_k(i64 n, int kind, const i64* __restrict__ rp, const int* __restrict__ ci,
                           const double* __restrict__ v, const double* __restrict__ deg,
                           const double* __restrict__ dis, const i64* __restrict__ orp, int* __restrict__ oci,
                           double* __restrict__ ov) {
  const i64 r = blockIdx.x * (i64)blockDim.x + threadIdx.x;
  if (r >= n) return;
  const bool has_diag = kind == CPCAG_COMBINATORIAL ? deg[r] != 0.0 : deg[r] > 0.0;
  const double dval = kind == CPCAG_COMBINATORIAL ? deg[r] : 1.0;
  i64 o = orp[r];
  bool placed = !has_diag;
  for (i64 k = rp[r]; k < rp[r + 1]; ++k) {
    const int c = ci[k];
    if (!placed && c > r) {
      oci[o] = static_cast<int>(r);
      ov[o] = dval;
      ++o;
      placed = true;
    }
    const double x = lap_off(kind, v[k], dis, r, c);
    if (x != 0.0) {
      oci[o] = c;
      ov[o] = x;
      ++o;
    }
  }
  if (!placed) {
    oci[o] = static_cast<int>(r);
    ov[o] = dval;
  }
}

i64 scan_counts(Ctx* c, const i64* cnt, i64 rows, i64* rp);  // kron.cu

Csr* build_laplacian(Ctx* c, Csr* W, const double* deg, int kind) {
  const i64 n = W->rows;
  Csr* L = csr_alloc(c, n, n, 0);
  std::unique_ptr<Csr> own(L);
  DevBuf<double> dis(c, std::max<i64>(n, 1));
  DevBuf<i64> cnt(c, std::max<i64>(n, 1));
  if (n) {
    dis_k<<<blocks_for(n), kBlock, 0, c->stream>>>(n, deg, dis.p);
    launched(c);
    lap_count_k<<<blocks_for(n), kBlock, 0, c->stream>>>(n, kind, W->rp, W->ci, W->v, deg, dis.p, cnt.p);
    launched(c);
  }
  L->nnz = scan_counts(c, cnt.p, n, L->rp);
  if (L->nnz) {
    L->ci = static_cast<int*>(csr_malloc(c, sizeof(int) * L->nnz));
    L->v = static_cast<double*>(csr_malloc(c, sizeof(double) * L->nnz));
    lap_fill_k<<<blocks_for(n), kBlock, 0, c->stream>>>(n, kind, W->rp, W->ci, W->v, deg, dis.p, L->rp, L->ci, L->v);
    launched(c);
  }
  L->sym = W->sym == 1 ? 1 : -1;
  return own.release();
}

// ------------------------------------------------------------------ kNN
struct KnnLists {
  DevBuf<int64_t> nbr;
  DevBuf<double> d2, mean;
  i64 n = 0, d = 0;
  DevBuf<double> Pm;
  i64 tc_rows = 0;  // points certified by the tensor-core filter
};

// ---- tensor-core filter + certified exact re-rank ------------------------
constexpr int kCandTc = 32;  // == kCand in gram_tc.cu

void split_points(Ctx* c, const double* Pm, i64 n, i64 d, i64 dp, float* H, float* L);  // gram_tc.cu
void knn_tc_filter2(Ctx* c, const float* H, const float* L, const double* sq, i64 n, i64 dp, i64 q_tiles, i64 splits,
                    i64 tps, float* cd, int* cj, const unsigned long long* max_norm_bits);
void knn_tc_filter2_rows(Ctx* c, const float* Hq, const float* Lq, const int* qidx, i64 nq, const float* H,
                         const float* L, const double* sq, i64 n, i64 dp, i64 splits, float* cd, int* cj,
                         const unsigned long long* max_norm_bits);
void gather_point_rows(Ctx* c, const float* H, const float* L, const int* qidx, i64 nq, i64 dp, float* Hq, float* Lq);

__global__ void max_norm_k(const double* __restrict__ sq, i64 n, unsigned long long* out) {
  const i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x;
  if (i < n) atomicMax(out, static_cast<unsigned long long>(__double_as_longlong(sqrt(sq[i]))));
}

// Merge the per-split sorted approximate lists of each query (first KC).
template <int KC>
__global__ void tc_merge_k(i64 nq, int splits, const float* __restrict__ cd, const int* __restrict__ cj,
                           float* __restrict__ md, int* __restrict__ mj) {
  const i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x;
  if (i >= nq) return;
  int pos[64];
  for (int s = 0; s < splits; ++s) pos[s] = 0;
  for (int q = 0; q < KC; ++q) {
    int bs = -1;
    float bd = CUDART_INF_F;
    int bj = INT32_MAX;
    for (int s = 0; s < splits; ++s) {
      if (pos[s] >= KC) continue;
      const i64 at = (static_cast<i64>(s) * nq + i) * KC + pos[s];
      const float dv = cd[at];
      const int jv = cj[at];
      if (bs < 0 || dv < bd || (dv == bd && jv < bj)) {
        bs = s;
        bd = dv;
        bj = jv;
      }
    }
    pos[bs]++;
    md[i * KC + q] = bd;
    mj[i * KC + q] = bj;
  }
}

// One warp per query, lane l holds candidates l, l + 32, ... (KC / 32 per
// lane).  The window [.., D_K + 2E] with E a rigorous bound of the 3xTF32
// distance error contains every true top-K neighbour; if the whole list lies
// inside the window some candidate may be missing and the point is deferred
// (overflow[q] = 1: a second pass with longer lists, then the exact path).
// Otherwise the candidates inside the window get the canonical fp64 distance
// (sequential k, no FMA) and the K smallest (d2, j) are selected exactly.
// qidx (null = identity) maps query q to its point; rows of nbr / nbr_d2 /
// mean_d2 / dup are indexed by point.
template <int KC>
__global__ void tc_rerank_k(const double* __restrict__ Pm, const double* __restrict__ sq, i64 nq,
                            const int* __restrict__ qidx, i64 d, int K, double cg,
                            const unsigned long long* __restrict__ maxnorm_bits, const float* __restrict__ md,
                            const int* __restrict__ mj, int64_t* __restrict__ nbr, double* __restrict__ nbr_d2,
                            double* __restrict__ mean_d2, int* __restrict__ overflow, int* __restrict__ dup) {
  constexpr int QPL = KC / 32;
  const i64 q = (blockIdx.x * (i64)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (q >= nq) return;
  const i64 i = qidx ? static_cast<i64>(qidx[q]) : q;
  const double maxnorm = __longlong_as_double(static_cast<long long>(*maxnorm_bits));
  float dq[QPL];
  int jq[QPL];
#pragma unroll
  for (int t = 0; t < QPL; ++t) {
    dq[t] = md[q * KC + t * 32 + lane];
    jq[t] = mj[q * KC + t * 32 + lane];
  }
  const double DK = static_cast<double>(__shfl_sync(0xffffffffu, dq[0], K - 1));  // K <= 32
  const double last = static_cast<double>(__shfl_sync(0xffffffffu, dq[QPL - 1], 31));
  const double E = 2.0 * cg * sqrt(sq[i]) * maxnorm;
  const double W = DK + fabs(DK) * 0x1.0p-22 + 2.0 * E;  // + float rounding of the stored d~
  const bool ovf = last - fabs(last) * 0x1.0p-22 <= W;
  if (ovf) {
    if (lane == 0) overflow[q] = 1;
    return;
  }
  double ex[QPL];
  int jc[QPL];
#pragma unroll
  for (int t = 0; t < QPL; ++t) {
    const double dql = static_cast<double>(dq[t]) - fabs(static_cast<double>(dq[t])) * 0x1.0p-22;
    ex[t] = CUDART_INF;
    jc[t] = INT32_MAX;
    if (jq[t] != INT32_MAX && dql <= W) {
      const double* a = Pm + i * d;
      const double* b = Pm + static_cast<i64>(jq[t]) * d;
      double g = 0.0;
      for (i64 k = 0; k < d; ++k) g = __dadd_rn(g, __dmul_rn(a[k], b[k]));
      const double tt = __dsub_rn(__dadd_rn(sq[i], sq[jq[t]]), __dmul_rn(2.0, g));
      ex[t] = tt > 0.0 ? tt : 0.0;
      jc[t] = jq[t];
      if (ex[t] == 0.0 && jq[t] < i) {
        bool same = true;
        for (i64 k = 0; k < d && same; ++k) same = a[k] == b[k];
        if (same) dup[i] = 1;
      }
    }
  }
  // K rounds of a lexicographic warp argmin.
  double m = 0.0;
  for (int r = 0; r < K; ++r) {
    double bv = CUDART_INF;
    int bj = INT32_MAX;
#pragma unroll
    for (int t = 0; t < QPL; ++t)
      if (ex[t] < bv || (ex[t] == bv && jc[t] < bj)) {
        bv = ex[t];
        bj = jc[t];
      }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
      const int oj = __shfl_xor_sync(0xffffffffu, bj, o);
      if (ov < bv || (ov == bv && oj < bj)) {
        bv = ov;
        bj = oj;
      }
    }
    if (lane == 0) {
      nbr[i * K + r] = bj;
      nbr_d2[i * K + r] = bv;
    }
    m = __dadd_rn(m, bv);
#pragma unroll
    for (int t = 0; t < QPL; ++t)
      if (jc[t] == bj) {
        ex[t] = CUDART_INF;
        jc[t] = INT32_MAX;
      }
  }
  if (lane == 0) mean_d2[i] = m;
}

// Exact fp64 tiled search for the queries qidx[0..nq) (all points when qidx
// is null), writing their rows of nbr / nbr_d2 / mean.
void knn_exact_rows(Ctx* c, const double* Pm, const double* sq, i64 n, i64 d, i64 K, const int* qidx, i64 nq,
                    int* dup, int64_t* nbr, double* nbr_d2, double* mean) {
  if (nq == 0) return;
  const i64 q_tiles = (nq + kTile - 1) / kTile;
  const i64 n_tiles = (n + kTile - 1) / kTile;
  if (!qidx && nq == n && n_tiles <= 64) {  // all points: the upper triangle of tile pairs
    DevBuf<double> cand_d(c, n_tiles * n * K);
    DevBuf<int> cand_j(c, n_tiles * n * K);
    constexpr int kSymThreads = 256;
    ensure_smem(knn_sym_k<kSymThreads>, kKnnSymSmem);
    {
      KScope ks_(c, "knn_tile");
      knn_sym_k<kSymThreads><<<static_cast<unsigned>(n_tiles * (n_tiles + 1) / 2), kSymThreads, kKnnSymSmem, c->stream>>>(
          Pm, sq, n, d, static_cast<int>(K), static_cast<int>(n_tiles), cand_d.p, cand_j.p, dup);
      launched(c);
    }
    knn_merge_k<<<blocks_for(n, 128), 128, 0, c->stream>>>(n, static_cast<int>(K), static_cast<int>(n_tiles),
                                                           cand_d.p, cand_j.p, nbr, nbr_d2, mean, nullptr);
    launched(c);
    return;
  }
  i64 splits = std::max<i64>(1, (2 * static_cast<i64>(c->num_sms) + q_tiles - 1) / q_tiles);
  splits = std::min<i64>({splits, n_tiles, 64});
  const i64 tps = (n_tiles + splits - 1) / splits;
  splits = (n_tiles + tps - 1) / tps;
  DevBuf<double> cand_d(c, splits * nq * K);
  DevBuf<int> cand_j(c, splits * nq * K);
  dim3 g(static_cast<unsigned>(q_tiles), static_cast<unsigned>(splits));
  ensure_smem(knn_tile_k, kKnnSmem);
  {
    KScope ks_(c, "knn_tile");
    knn_tile_k<<<g, 256, kKnnSmem, c->stream>>>(Pm, sq, n, d, static_cast<int>(K), static_cast<int>(tps), cand_d.p,
                                                cand_j.p, dup, qidx, nq);
    launched(c);
  }
  knn_merge_k<<<blocks_for(nq, 128), 128, 0, c->stream>>>(nq, static_cast<int>(K), static_cast<int>(splits),
                                                           cand_d.p, cand_j.p, nbr, nbr_d2, mean, qidx);
  launched(c);
}

static bool tc_knn_enabled(i64 n, i64 d, i64 K) {
  const char* e = std::getenv("CPCAG_KNN");
  if (e && std::string(e) == "exact") return false;
  const bool forced = e && std::string(e) == "tc";
  if (K + 4 > kCandTc || d < 1) return false;
  return forced || (n >= 4096 && d <= 1024);
}

template <typename T>
void knn_lists(Ctx* c, const T* X, i64 x_rows, i64 x_cols, bool axis_rows, i64 K, KnnLists* out) {
  if (K < 1) invalid("knn graph: K must be >= 1");
  const i64 n = axis_rows ? x_rows : x_cols;
  const i64 d = axis_rows ? x_cols : x_rows;
  if (n < K + 1) invalid("knn graph: need at least K+1 points, got " + std::to_string(n));
  if (K > kMaxK) invalid("knn graph: K above " + std::to_string(kMaxK) + " is not supported on the device");
  if (n > INT32_MAX) invalid("knn graph: more than 2^31-1 points are not supported");
  out->n = n;
  out->d = d;
  out->Pm.alloc(c, std::max<i64>(n * d, 1));
  DevBuf<double> sq(c, n);
  trace_mark(c, "knn: enter");
  if (n * d) {
    gather_points_k<T><<<blocks_for(n * d), kBlock, 0, c->stream>>>(X, x_rows, n, d, axis_rows ? 1 : 0, out->Pm.p);
    launched(c);
  } else {
    out->Pm.zero(c);
  }
  sqnorm_k<<<static_cast<unsigned>((n * 32 + 255) / 256), 256, 0, c->stream>>>(out->Pm.p, n, d, sq.p);
  launched(c);
  out->nbr.alloc(c, n * K);
  out->d2.alloc(c, n * K);
  out->mean.alloc(c, n);
  DevBuf<int> dup(c, n);
  dup.zero(c);
  out->tc_rows = 0;
  if (tc_knn_enabled(n, d, K)) {
    // Filter on the tensor cores, certify, re-rank exactly.
    const i64 dp = std::max<i64>(32, (d + 31) / 32 * 32);
    DevBuf<float> H(c, n * dp), L(c, n * dp);
    split_points(c, out->Pm.p, n, d, dp, H.p, L.p);
    const i64 q_tiles = (n + 127) / 128, n_tiles = (n + 127) / 128;
    i64 splits = std::max<i64>(1, (2 * static_cast<i64>(c->num_sms) + q_tiles - 1) / q_tiles);
    splits = std::min<i64>({splits, n_tiles, 64});
    const i64 tps = (n_tiles + splits - 1) / splits;
    splits = (n_tiles + tps - 1) / tps;
    DevBuf<float> cd(c, splits * n * kCandTc), md(c, n * kCandTc);
    DevBuf<int> cj(c, splits * n * kCandTc), mj(c, n * kCandTc), ovf(c, n);
    ovf.zero(c);
    DevBuf<unsigned long long> mxn(c, 1);
    mxn.zero(c);
    max_norm_k<<<blocks_for(n), kBlock, 0, c->stream>>>(sq.p, n, mxn.p);
    launched(c);
    {
      KScope ks_(c, "knn_tc_filter");
      knn_tc_filter2(c, H.p, L.p, sq.p, n, dp, q_tiles, splits, tps, cd.p, cj.p, mxn.p);
    }
    tc_merge_k<kCandTc><<<blocks_for(n, 128), 128, 0, c->stream>>>(n, static_cast<int>(splits), cd.p, cj.p, md.p, mj.p);
    launched(c);
    // Rigorous bound on |G~ - G| / (|x_i| |x_j|): split error 3 * 2^-22 plus
    // fp32 accumulation of 3 d exact tf32 products, 2^-23 per addition
    // (truncating accumulation), doubled for margin.
    const double cg = 2.0 * (3.0 + 3.0 * static_cast<double>(d)) * 0x1.0p-23;
    {
      KScope ks_(c, "knn_tc_rerank");
      tc_rerank_k<kCandTc><<<blocks_for(n * 32, 256), 256, 0, c->stream>>>(out->Pm.p, sq.p, n, nullptr, d,
                                                                          static_cast<int>(K), cg, mxn.p, md.p, mj.p,
                                                                          out->nbr.p, out->d2.p, out->mean.p, ovf.p,
                                                                          dup.p);
      launched(c);
    }
    trace_mark(c, "knn: tc filter+merge+rerank");
    std::vector<int> of(static_cast<size_t>(n));
    CUDA_OK(cudaMemcpyAsync(of.data(), ovf.p, sizeof(int) * n, cudaMemcpyDeviceToHost, c->stream));
    sync(c);
    std::vector<int> rows;
    for (i64 i = 0; i < n; ++i)
      if (of[i]) rows.push_back(static_cast<int>(i));
    const size_t pass1_rows = rows.size();
    const char* p2 = std::getenv("CPCAG_KNN_PASS2");
    if (!rows.empty() && !(p2 && std::string(p2) == "0") && K <= 32) {
      // Second pass for the uncertified points: their rows again on the
      // tensor cores with 64-candidate lists, then the same certified re-rank.
      trace_mark(c, "knn: pass-1 readback");
      const i64 nq = static_cast<i64>(rows.size());
      DevBuf<int> qd(c, nq), ovf2(c, nq);
      CUDA_OK(cudaMemcpyAsync(qd.p, rows.data(), sizeof(int) * nq, cudaMemcpyHostToDevice, c->stream));
      ovf2.zero(c);
      DevBuf<float> Hq(c, nq * dp), Lq(c, nq * dp);
      gather_point_rows(c, H.p, L.p, qd.p, nq, dp, Hq.p, Lq.p);
      const i64 q2 = (nq + 127) / 128;
      i64 s2 = std::max<i64>(1, static_cast<i64>(c->num_sms) / q2);
      s2 = std::min<i64>({s2, n_tiles, 64});
      const i64 tps2 = (n_tiles + s2 - 1) / s2;
      s2 = (n_tiles + tps2 - 1) / tps2;
      DevBuf<float> cd2(c, s2 * nq * 64), md2(c, nq * 64);
      DevBuf<int> cj2(c, s2 * nq * 64), mj2(c, nq * 64);
      {
        KScope ks_(c, "knn_tc_filter_pass2");
        knn_tc_filter2_rows(c, Hq.p, Lq.p, qd.p, nq, H.p, L.p, sq.p, n, dp, s2, cd2.p, cj2.p, mxn.p);
      }
      tc_merge_k<64><<<blocks_for(nq, 128), 128, 0, c->stream>>>(nq, static_cast<int>(s2), cd2.p, cj2.p, md2.p, mj2.p);
      launched(c);
      {
        KScope ks_(c, "knn_tc_rerank");
        tc_rerank_k<64><<<blocks_for(nq * 32, 256), 256, 0, c->stream>>>(out->Pm.p, sq.p, nq, qd.p, d,
                                                                        static_cast<int>(K), cg, mxn.p, md2.p, mj2.p,
                                                                        out->nbr.p, out->d2.p, out->mean.p, ovf2.p,
                                                                        dup.p);
        launched(c);
      }
      std::vector<int> of2(static_cast<size_t>(nq));
      CUDA_OK(cudaMemcpyAsync(of2.data(), ovf2.p, sizeof(int) * nq, cudaMemcpyDeviceToHost, c->stream));
      sync(c);
      std::vector<int> rest;
      for (i64 q = 0; q < nq; ++q)
        if (of2[q]) rest.push_back(rows[q]);
      rows.swap(rest);
      trace_mark(c, "knn: tc pass 2");
    }
    out->tc_rows = n - static_cast<i64>(rows.size());
    if (std::getenv("CPCAG_TRACE"))
      std::fprintf(stderr, "[knn] %lld points, %lld certified by the tensor-core filter (%zu left by pass 1), "
                   "%zu exact fallback rows\n", static_cast<long long>(n), static_cast<long long>(out->tc_rows),
                   pass1_rows, rows.size());
    if (!rows.empty()) {
      DevBuf<int> qd(c, rows.size());
      CUDA_OK(cudaMemcpyAsync(qd.p, rows.data(), sizeof(int) * rows.size(), cudaMemcpyHostToDevice, c->stream));
      knn_exact_rows(c, out->Pm.p, sq.p, n, d, K, qd.p, static_cast<i64>(rows.size()), dup.p, out->nbr.p,
                     out->d2.p, out->mean.p);
      sync(c);
    }
    trace_mark(c, "knn: exact fallback rows");
  } else {
    knn_exact_rows(c, out->Pm.p, sq.p, n, d, K, nullptr, n, dup.p, out->nbr.p, out->d2.p, out->mean.p);
  }
  DevBuf<unsigned long long> ndup(c, 1);
  ndup.zero(c);
  count_dup_k<<<blocks_for(n), kBlock, 0, c->stream>>>(n, dup.p, ndup.p);
  launched(c);
  const unsigned long long nd = read_back(c, ndup.p);
  const i64 distinct = n - static_cast<i64>(nd);
  trace_mark(c, "knn: lists done");
  if (distinct < K)
    invalid("knn graph: fewer distinct points (" + std::to_string(distinct) + ") than K (" + std::to_string(K) + ")");
}

template <typename T>
void knn_graph_device(Ctx* c, const T* X, i64 x_rows, i64 x_cols, bool axis_rows, i64 K, int kind,
                      double sigma2_override, Csr** Wout, Csr** Lout, double* degrees_dev, double* sigma2) {
  KnnLists kl;
  knn_lists<T>(c, X, x_rows, x_cols, axis_rows, K, &kl);
  const i64 n = kl.n;
  DevBuf<double> s2(c, 1), q(c, std::max<i64>(n, 1));
  sigma2_div_k<<<blocks_for(std::max<i64>(n, 1)), kBlock, 0, c->stream>>>(n, static_cast<int>(K), kl.mean.p, q.p);
  launched(c);
  sigma2_k<<<1, 1, 0, c->stream>>>(n, q.p, sigma2_override, s2.p);
  launched(c);

  const i64 m = 2 * n * K;
  DevBuf<unsigned long long> keys(c, m), keys_s(c, m);
  DevBuf<double> vals(c, m), vals_s(c, m);
  edge_records_k<<<blocks_for(n * K), kBlock, 0, c->stream>>>(n, static_cast<int>(K), kl.nbr.p, kl.d2.p, keys.p, vals.p);
  launched(c);
  int end_bit = 32;
  while ((1ll << (end_bit - 32)) < n && end_bit < 64) ++end_bit;
  size_t tmp = 0;
  CUDA_OK(cub::DeviceRadixSort::SortPairs(nullptr, tmp, keys.p, keys_s.p, vals.p, vals_s.p, static_cast<int>(m), 0,
                                          end_bit, c->stream));
  {
    DevBuf<char> ws(c, tmp);
    CUDA_OK(cub::DeviceRadixSort::SortPairs(ws.p, tmp, keys.p, keys_s.p, vals.p, vals_s.p, static_cast<int>(m), 0,
                                            end_bit, c->stream));
    launched(c);
  }
  DevBuf<double> w(c, m);
  DevBuf<i64> keep(c, m), incl(c, m);
  edge_weight_k<<<blocks_for(m), kBlock, 0, c->stream>>>(m, keys_s.p, vals_s.p, s2.p, w.p, keep.p);
  launched(c);
  {
    size_t t2 = 0;
    CUDA_OK(cub::DeviceScan::InclusiveSum(nullptr, t2, keep.p, incl.p, static_cast<int>(m), c->stream));
    DevBuf<char> ws(c, t2);
    CUDA_OK(cub::DeviceScan::InclusiveSum(ws.p, t2, keep.p, incl.p, static_cast<int>(m), c->stream));
    launched(c);
  }
  i64 nnz = 0;
  CUDA_OK(cudaMemcpyAsync(&nnz, incl.p + (m - 1), sizeof(i64), cudaMemcpyDeviceToHost, c->stream));
  sync(c);
  Csr* W = csr_alloc(c, n, n, nnz);
  std::unique_ptr<Csr> ownW(W);
  edge_rowptr_k<<<blocks_for(n + 1), kBlock, 0, c->stream>>>(n, m, keys_s.p, incl.p, W->rp);
  launched(c);
  if (nnz) {
    edge_fill_k<<<blocks_for(m), kBlock, 0, c->stream>>>(m, keys_s.p, w.p, keep.p, incl.p, W->ci, W->v);
    launched(c);
  }
  W->sym = 1;
  row_sums_k<<<blocks_for(n), kBlock, 0, c->stream>>>(n, W->rp, W->v, degrees_dev);
  launched(c);
  Csr* L = build_laplacian(c, W, degrees_dev, kind);
  L->sym = 1;
  *sigma2 = read_back(c, s2.p);
  trace_mark(c, "knn: union, W, L");
  *Wout = ownW.release();
  *Lout = L;
}

template void knn_graph_device<double>(Ctx*, const double*, i64, i64, bool, i64, int, double, Csr**, Csr**, double*,
                                       double*);
template void knn_graph_device<float>(Ctx*, const float*, i64, i64, bool, i64, int, double, Csr**, Csr**, double*,
                                      double*);

// ------------------------------------------------------------------ adjacency
__global__ void adj_check_k(i64 n, const i64* __restrict__ rp, const int* __restrict__ ci,
                            const double* __restrict__ v, int* flags) {
  const i64 r = blockIdx.x * (i64)blockDim.x + threadIdx.x;
  if (r >= n) return;
  for (i64 k = rp[r]; k < rp[r + 1]; ++k) {
    if (ci[k] == r) atomicOr(flags, 1);  // nonzero diagonal (stored entries are nonzero)
    if (v[k] < 0.0) atomicOr(flags, 2);
  }
}

void graph_from_adjacency_device(Ctx* c, Csr* W, int kind, Csr** Lout, double* degrees_dev) {
  if (W->rows != W->cols) invalid("adjacency must be square");
  if (!csr_symmetric(c, W)) invalid("adjacency must be symmetric");
  const i64 n = W->rows;
  if (n) {
    DevBuf<int> flags(c, 1);
    flags.zero(c);
    adj_check_k<<<blocks_for(n), kBlock, 0, c->stream>>>(n, W->rp, W->ci, W->v, flags.p);
    launched(c);
    const int f = read_back(c, flags.p);
    if (f & 1) invalid("adjacency must have zero diagonal");
    if (f & 2) invalid("adjacency weights must be nonnegative");
    row_sums_k<<<blocks_for(n), kBlock, 0, c->stream>>>(n, W->rp, W->v, degrees_dev);
    launched(c);
  }
  *Lout = build_laplacian(c, W, degrees_dev, kind);
  (*Lout)->sym = 1;
}

}  // namespace cpcag_cuda

using namespace cpcag_cuda;

extern "C" int cpcag_cuda_knn_graph(cpcag_ctx ctx, int precision, const void* X, int64_t x_rows, int64_t x_cols,
                                    int axis, int64_t K, int kind, double sigma2_override, cpcag_csr* adjacency,
                                    cpcag_csr* laplacian, double* degrees, double* sigma2) {
  auto run = [&](auto tag) {
    using T = decltype(tag);
    return guard([&] {
      Ctx* c = as_ctx(ctx);
      if (!adjacency || !laplacian || !sigma2) invalid("null output pointer");
      if (axis != CPCAG_AXIS_ROWS && axis != CPCAG_AXIS_COLS) invalid("knn graph: unknown axis");
      if (kind != CPCAG_COMBINATORIAL && kind != CPCAG_NORMALIZED) invalid("knn graph: unknown laplacian kind");
      const bool rows = axis == CPCAG_AXIS_ROWS;
      if (K < 1) invalid("knn graph: K must be >= 1");
      const i64 n = rows ? x_rows : x_cols;
      InView<T> xin(c, static_cast<const T*>(X), static_cast<size_t>(x_rows * x_cols));
      DevBuf<double> deg_scratch;
      double* deg_d = nullptr;
      const bool dev_deg = degrees && is_device_ptr(degrees);
      if (dev_deg) {
        deg_d = degrees;
      } else {
        deg_scratch.alloc(c, std::max<i64>(n, 1));
        deg_d = deg_scratch.p;
      }
      Csr *W = nullptr, *L = nullptr;
      knn_graph_device<T>(c, xin.d, x_rows, x_cols, rows, K, kind, sigma2_override, &W, &L, deg_d, sigma2);
      if (degrees && !dev_deg && n)
        CUDA_OK(cudaMemcpyAsync(degrees, deg_d, sizeof(double) * n, cudaMemcpyDeviceToHost, c->stream));
      sync(c);
      *adjacency = reinterpret_cast<cpcag_csr>(W);
      *laplacian = reinterpret_cast<cpcag_csr>(L);
    });
  };
  if (precision == CPCAG_F64) return run(double{});
  if (precision == CPCAG_F32) return run(float{});
  set_last_error("unknown precision flag");
  return CPCAG_ERR_INVALID_ARGUMENT;
}

extern "C" int cpcag_cuda_knn(cpcag_ctx ctx, int precision, const void* X, int64_t x_rows, int64_t x_cols, int axis,
                              int64_t K, int64_t* nbr, double* nbr_d2) {
  auto run = [&](auto tag) {
    using T = decltype(tag);
    return guard([&] {
      Ctx* c = as_ctx(ctx);
      if (axis != CPCAG_AXIS_ROWS && axis != CPCAG_AXIS_COLS) invalid("knn graph: unknown axis");
      const bool rows = axis == CPCAG_AXIS_ROWS;
      InView<T> xin(c, static_cast<const T*>(X), static_cast<size_t>(x_rows * x_cols));
      KnnLists kl;
      knn_lists<T>(c, xin.d, x_rows, x_cols, rows, K, &kl);
      OutView<int64_t> on(c, nbr, static_cast<size_t>(kl.n * K));
      OutView<double> od(c, nbr_d2, static_cast<size_t>(kl.n * K));
      if (on.d) CUDA_OK(cudaMemcpyAsync(on.d, kl.nbr.p, sizeof(int64_t) * kl.n * K, cudaMemcpyDeviceToDevice, c->stream));
      if (od.d) CUDA_OK(cudaMemcpyAsync(od.d, kl.d2.p, sizeof(double) * kl.n * K, cudaMemcpyDeviceToDevice, c->stream));
      on.flush(c);
      od.flush(c);
      sync(c);
    });
  };
  if (precision == CPCAG_F64) return run(double{});
  if (precision == CPCAG_F32) return run(float{});
  set_last_error("unknown precision flag");
  return CPCAG_ERR_INVALID_ARGUMENT;
}

extern "C" int cpcag_cuda_graph_from_adjacency(cpcag_ctx ctx, cpcag_csr W, int kind, cpcag_csr* laplacian,
                                               double* degrees) {
  return guard([&] {
    Ctx* c = as_ctx(ctx);
    if (!laplacian) invalid("null output pointer");
    Csr* Wc = as_csr(W);
    OutView<double> deg(c, degrees, static_cast<size_t>(Wc->rows));
    DevBuf<double> scratch;
    double* dd = deg.d;
    if (!dd) {
      scratch.alloc(c, std::max<i64>(Wc->rows, 1));
      dd = scratch.p;
    }
    Csr* L = nullptr;
    graph_from_adjacency_device(c, Wc, kind, &L, dd);
    deg.flush(c);
    sync(c);
    *laplacian = reinterpret_cast<cpcag_csr>(L);
  });
}
