// cluster.cu -- the clustering decoder path:
//   kmeans on the columns of X~ (clustering.cpp:40-137), decode_labels =
//   graph_upsample of the sampled-column indicator + row-wise max pooling
//   (clustering.cpp:139-160), clustering_error (clustering.cpp:165-238).
//
// kmeans keeps the reference's sequential semantics so its assignments are
// bit-identical to the oracle restatement: squared distances are sums over
// the rows in order (one thread per point), the k-means++ total and the
// sampling scan are sequential (one warp: coalesced loads, lane 0 folds them
// in order), centroid sums accumulate points in ascending index (one thread
// per row, private per-cluster accumulators), and an emptied cluster is
// re-seeded from the farthest point with the reference's in-order loop over
// clusters.  The counter RNG (rng.hpp:11-68) runs on the device.
#include <algorithm>
#include <limits>
#include <string>
#include <vector>

#include "common.cuh"

namespace cpcag_cuda {

namespace {

struct DevRng {
  unsigned long long seed, ctr;
};

__device__ __forceinline__ unsigned long long rng_mix(unsigned long long z) {
  z += 0x9e3779b97f4a7c15ULL;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}
__device__ __forceinline__ unsigned long long rng_u64(DevRng& r) { return rng_mix(r.seed + 0x632be59bd9b4e019ULL * ++r.ctr); }
__device__ __forceinline__ double rng_double(DevRng& r) { return static_cast<double>(rng_u64(r) >> 11) * 0x1.0p-53; }
__device__ __forceinline__ unsigned long long rng_below(DevRng& r, unsigned long long n) {
  const unsigned long long lim = ~0ULL - (~0ULL) % n;
  unsigned long long v = rng_u64(r);
  while (v >= lim) v = rng_u64(r);
  return v % n;
}

__device__ __forceinline__ double col_d2(const double* __restrict__ X, i64 rows, i64 j, const double* __restrict__ c) {
  const double* x = X + j * rows;
  double s = 0.0;
  for (i64 i = 0; i < rows; ++i) {
    const double d = x[i] - c[i];
    s = __dadd_rn(s, __dmul_rn(d, d));  // no FMA contraction: the oracle's order and rounding
  }
  return s;
}

__global__ void widen_k(i64 n, const float* __restrict__ src, double* __restrict__ dst) {
  for (i64 i = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x; i < n; i += gridDim.x * (i64)blockDim.x)
    dst[i] = static_cast<double>(src[i]);
}

__global__ void fill_inf_k(i64 n, double* v) {
  for (i64 i = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x; i < n; i += gridDim.x * (i64)blockDim.x)
    v[i] = __longlong_as_double(0x7ff0000000000000LL);
}

// min_d2[j] = min(min_d2[j], ||x_j - c||^2)   (clustering.cpp:47-48)
__global__ void km_mind2_k(const double* __restrict__ X, i64 rows, i64 n, const double* __restrict__ c,
                           double* __restrict__ min_d2) {
  const i64 j = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x;
  if (j >= n) return;
  const double d = col_d2(X, rows, j, c);
  const double m = min_d2[j];
  min_d2[j] = d < m ? d : m;  // std::min(m, d)
}

// Sequential fold of v[0..n) in index order by lane 0 of one warp (the
// warp loads 32 values at a time, lane 0 consumes them through shuffles).
// mode 0: returns sum; mode 1: the k-means++ scan (clustering.cpp:51-59).
__device__ double warp_seq_sum(const double* __restrict__ v, i64 n) {
  const int lane = threadIdx.x & 31;
  double s = 0.0;
  for (i64 b = 0; b < n; b += 32) {
    const double x = b + lane < n ? v[b + lane] : 0.0;
    const int m = static_cast<int>(n - b < 32 ? n - b : 32);
    for (int q = 0; q < m; ++q) s += __shfl_sync(0xffffffffu, x, q);
  }
  return s;
}

// k-means++ seeding step c (clustering.cpp:44, 49-65): picks the next
// centroid and copies X[:, pick] into cent[:, c].  One warp.
__global__ void km_pick_k(const double* __restrict__ X, i64 rows, i64 n, const double* __restrict__ min_d2, i64 c,
                          DevRng* rng, double* __restrict__ cent) {
  const int lane = threadIdx.x;
  __shared__ long long pick_s;
  if (c == 0) {
    if (lane == 0) {
      DevRng r = *rng;
      pick_s = static_cast<long long>(rng_below(r, static_cast<unsigned long long>(n)));
      *rng = r;
    }
  } else {
    const double total = warp_seq_sum(min_d2, n);
    if (total > 0.0) {
      double target = 0.0;
      if (lane == 0) {
        DevRng r = *rng;
        target = rng_double(r) * total;
        *rng = r;
      }
      target = __shfl_sync(0xffffffffu, target, 0);
      long long pick = 0;
      bool found = false;
      for (i64 b = 0; b < n && !found; b += 32) {
        const double x = b + lane < n ? min_d2[b + lane] : 0.0;
        const int m = static_cast<int>(n - b < 32 ? n - b : 32);
        for (int q = 0; q < m; ++q) {
          const double y = __shfl_sync(0xffffffffu, x, q);
          target -= y;
          pick = b + q;
          if (target <= 0.0) {
            found = true;
            break;
          }
        }
      }
      if (lane == 0) pick_s = pick;
    } else if (lane == 0) {
      DevRng r = *rng;
      pick_s = static_cast<long long>(rng_below(r, static_cast<unsigned long long>(n)));
      *rng = r;
    }
  }
  __syncwarp();
  const i64 pk = pick_s;
  for (i64 i = lane; i < rows; i += 32) cent[i + c * rows] = X[i + pk * rows];
}

// assignment step (clustering.cpp:72-79): nearest centroid, strict <.
__global__ void km_assign_k(const double* __restrict__ X, i64 rows, i64 n, i64 k, const double* __restrict__ cent,
                            int* __restrict__ a, int* changed) {
  const i64 j = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x;
  if (j >= n) return;
  int best = 0;
  double bd = __longlong_as_double(0x7ff0000000000000LL);
  for (i64 c = 0; c < k; ++c) {
    const double d = col_d2(X, rows, j, cent + c * rows);
    if (d < bd) {
      bd = d;
      best = static_cast<int>(c);
    }
  }
  if (best != a[j]) {
    a[j] = best;
    *changed = 1;
  }
}

// centroid sums, points in ascending index (clustering.cpp:82-87): one
// thread per row, private accumulators for KMAX clusters.
template <int KMAX>
__global__ void km_sums_k(const double* __restrict__ X, i64 rows, i64 n, i64 k, const int* __restrict__ a,
                          double* __restrict__ sums) {
  const i64 i = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x;
  if (i >= rows) return;
  double acc[KMAX];
#pragma unroll
  for (int c = 0; c < KMAX; ++c) acc[c] = 0.0;
  for (i64 j = 0; j < n; ++j) {
    const int c = a[j];
    const double x = X[i + j * rows];
#pragma unroll
    for (int q = 0; q < KMAX; ++q)
      if (q == c) acc[q] += x;
  }
  for (i64 c = 0; c < k; ++c) sums[i + c * rows] = acc[c];
}

// k > 64: the same order, accumulating in global memory.
__global__ void km_sums_global_k(const double* __restrict__ X, i64 rows, i64 n, i64 k, const int* __restrict__ a,
                                 double* __restrict__ sums) {
  const i64 i = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x;
  if (i >= rows) return;
  for (i64 c = 0; c < k; ++c) sums[i + c * rows] = 0.0;
  for (i64 j = 0; j < n; ++j) sums[i + static_cast<i64>(a[j]) * rows] += X[i + j * rows];
}

__global__ void km_counts_k(i64 n, i64 k, const int* __restrict__ a, long long* __restrict__ counts) {
  const i64 c = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x;
  if (c >= k) return;
  long long m = 0;
  for (i64 j = 0; j < n; ++j) m += a[j] == c;
  counts[c] = m;
}

// centroid update in cluster order, farthest-point re-seed of an emptied
// cluster (clustering.cpp:88-105).  One CTA.
__global__ void __launch_bounds__(1024) km_finalize_k(const double* __restrict__ X, i64 rows, i64 n, i64 k,
                                                      const double* __restrict__ sums,
                                                      const long long* __restrict__ counts, double* __restrict__ cent,
                                                      int* __restrict__ a) {
  __shared__ double bd_s[32];
  __shared__ long long bj_s[32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (i64 c = 0; c < k; ++c) {
    if (counts[c] > 0) {
      const double cn = static_cast<double>(counts[c]);
      for (i64 i = threadIdx.x; i < rows; i += blockDim.x) cent[i + c * rows] = sums[i + c * rows] / cn;
    } else {
      double bd = -1.0;
      long long bj = 0;
      for (i64 j = threadIdx.x; j < n; j += blockDim.x) {
        const double d = col_d2(X, rows, j, cent + static_cast<i64>(a[j]) * rows);
        if (d > bd) {  // j ascends per thread: keeps the lowest index on ties
          bd = d;
          bj = j;
        }
      }
      for (int o = 16; o > 0; o >>= 1) {
        const double od = __shfl_xor_sync(0xffffffffu, bd, o);
        const long long oj = __shfl_xor_sync(0xffffffffu, bj, o);
        if (od > bd || (od == bd && oj < bj)) {
          bd = od;
          bj = oj;
        }
      }
      if (lane == 0) {
        bd_s[wid] = bd;
        bj_s[wid] = bj;
      }
      __syncthreads();
      if (threadIdx.x == 0) {
        for (int q = 1; q < nw; ++q)
          if (bd_s[q] > bd_s[0] || (bd_s[q] == bd_s[0] && bj_s[q] < bj_s[0])) {
            bd_s[0] = bd_s[q];
            bj_s[0] = bj_s[q];
          }
      }
      __syncthreads();
      const long long far = bj_s[0];
      for (i64 i = threadIdx.x; i < rows; i += blockDim.x) cent[i + c * rows] = X[i + far * rows];
      __syncthreads();
      if (threadIdx.x == 0) a[far] = static_cast<int>(c);
    }
    __syncthreads();
  }
}

__global__ void km_pointd2_k(const double* __restrict__ X, i64 rows, i64 n, const double* __restrict__ cent,
                             const int* __restrict__ a, double* __restrict__ d2) {
  const i64 j = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x;
  if (j >= n) return;
  d2[j] = col_d2(X, rows, j, cent + static_cast<i64>(a[j]) * rows);
}

__global__ void km_wcss_k(const double* __restrict__ d2, i64 n, double* out) {
  const double s = warp_seq_sum(d2, n);
  if (threadIdx.x == 0) *out = s;
}

// decode_labels max pooling (clustering.cpp:151-158): first maximum of each
// row of C (n x k, column-major).
__global__ void max_pool_k(i64 n, i64 k, const double* __restrict__ C, int* __restrict__ out) {
  const i64 i = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x;
  if (i >= n) return;
  int arg = 0;
  double best = C[i];
  for (i64 j = 1; j < k; ++j)
    if (C[i + j * n] > best) {
      best = C[i + j * n];
      arg = static_cast<int>(j);
    }
  out[i] = arg;
}

__global__ void indicator_k(i64 m, i64 k, const int* __restrict__ lab, double* __restrict__ C) {
  const i64 i = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x;
  if (i >= m) return;
  for (i64 j = 0; j < k; ++j) C[i + j * m] = lab[i] == j ? 1.0 : 0.0;
}

}  // namespace

// kmeans (clustering.cpp:124-137) on the device; X fp64 device (rows x n).
void kmeans_device(Ctx* c, const double* X, i64 rows, i64 n, i64 k, i64 restarts, uint64_t seed, i64 max_iter,
                   int* assignments_dev, double* wcss_out) {
  if (k < 1) invalid("kmeans: k must be >= 1");
  if (k > n) invalid("kmeans: more clusters than points");
  if (restarts < 1) invalid("kmeans: restarts must be >= 1");
  DevBuf<double> cent(c, static_cast<size_t>(rows * k)), sums(c, static_cast<size_t>(rows * k)),
      min_d2(c, static_cast<size_t>(n)), d2(c, static_cast<size_t>(n)), wc(c, 1);
  DevBuf<int> a(c, static_cast<size_t>(n)), changed(c, 1);
  DevBuf<long long> counts(c, static_cast<size_t>(k));
  DevBuf<DevRng> rng(c, 1);
  const unsigned gp = blocks_for(n), gr = blocks_for(rows);
  double best = std::numeric_limits<double>::infinity();
  for (i64 r = 0; r < restarts; ++r) {
    const HostRng hr = HostRng::derive(seed, static_cast<uint64_t>(r));
    const DevRng dr{hr.seed, 0};
    CUDA_OK(cudaMemcpyAsync(rng.p, &dr, sizeof(dr), cudaMemcpyHostToDevice, c->stream));
    fill_inf_k<<<stride_blocks(c, n), kBlock, 0, c->stream>>>(n, min_d2.p);
    launched(c);
    km_pick_k<<<1, 32, 0, c->stream>>>(X, rows, n, min_d2.p, 0, rng.p, cent.p);
    launched(c);
    for (i64 q = 1; q < k; ++q) {
      km_mind2_k<<<gp, kBlock, 0, c->stream>>>(X, rows, n, cent.p + (q - 1) * rows, min_d2.p);
      launched(c);
      km_pick_k<<<1, 32, 0, c->stream>>>(X, rows, n, min_d2.p, q, rng.p, cent.p);
      launched(c);
    }
    a.zero(c);
    for (i64 it = 0; it < max_iter; ++it) {
      changed.zero(c);
      km_assign_k<<<gp, kBlock, 0, c->stream>>>(X, rows, n, k, cent.p, a.p, changed.p);
      launched(c);
      if (!read_back(c, changed.p) && it > 0) break;
      if (k <= 8)
        km_sums_k<8><<<gr, kBlock, 0, c->stream>>>(X, rows, n, k, a.p, sums.p);
      else if (k <= 64)
        km_sums_k<64><<<gr, kBlock, 0, c->stream>>>(X, rows, n, k, a.p, sums.p);
      else
        km_sums_global_k<<<gr, kBlock, 0, c->stream>>>(X, rows, n, k, a.p, sums.p);
      launched(c);
      km_counts_k<<<blocks_for(k), kBlock, 0, c->stream>>>(n, k, a.p, counts.p);
      launched(c);
      km_finalize_k<<<1, 1024, 0, c->stream>>>(X, rows, n, k, sums.p, counts.p, cent.p, a.p);
      launched(c);
    }
    km_pointd2_k<<<gp, kBlock, 0, c->stream>>>(X, rows, n, cent.p, a.p, d2.p);
    launched(c);
    km_wcss_k<<<1, 32, 0, c->stream>>>(d2.p, n, wc.p);
    launched(c);
    const double w = read_back(c, wc.p);
    if (w < best) {  // strict: ties keep the earlier restart (clustering.cpp:133)
      best = w;
      CUDA_OK(cudaMemcpyAsync(assignments_dev, a.p, sizeof(int) * n, cudaMemcpyDeviceToDevice, c->stream));
    }
  }
  if (!(best < std::numeric_limits<double>::infinity())) {
    // every restart had a non-finite wcss: the reference keeps the empty
    // initial run; its assignments are then all zero
    CUDA_OK(cudaMemsetAsync(assignments_dev, 0, sizeof(int) * n, c->stream));
  }
  if (wcss_out) *wcss_out = best;
  sync(c);
}

// decode_labels (clustering.cpp:139-160) on device data: sampled labels
// (rho_c ints, device, values in [0, k)) -> labels (n ints, device).
void decode_labels_device(Ctx* c, Csr* Lc, const std::vector<i64>& om_c, const int* sampled_dev, i64 k,
                          double pcg_tol, i64 pcg_max_iter, i64 n, int* labels_dev) {
  const i64 rho_c = static_cast<i64>(om_c.size());
  if (Lc->rows != n) invalid("decode_labels: column Laplacian does not match plan");
  DevBuf<double> Ct(c, static_cast<size_t>(std::max<i64>(rho_c * k, 1))), C(c, static_cast<size_t>(std::max<i64>(n * k, 1)));
  indicator_k<<<blocks_for(rho_c), kBlock, 0, c->stream>>>(rho_c, k, sampled_dev, Ct.p);  // ClusterLabels::indicator
  launched(c);
  graph_upsample_device(c, Lc, om_c, Ct.p, k, pcg_tol, pcg_max_iter, C.p);
  max_pool_k<<<blocks_for(n), kBlock, 0, c->stream>>>(n, k, C.p, labels_dev);
  launched(c);
}

}  // namespace cpcag_cuda

using namespace cpcag_cuda;

namespace {

// clustering.cpp:165-218 (host: k x k).
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

extern "C" int cpcag_cuda_kmeans(cpcag_ctx ctx, int precision, const void* X, int64_t rows, int64_t n, int64_t k,
                                 int64_t restarts, uint64_t seed, int64_t max_iter, int* assignments, double* wcss) {
  return guard([&] {
    Ctx* c = as_ctx(ctx);
    if (precision != CPCAG_F32 && precision != CPCAG_F64) invalid("unknown precision flag");
    if (!assignments || (rows * n > 0 && !X)) invalid("null argument");
    if (rows < 0 || n < 0) invalid("kmeans: negative dimensions");
    const size_t w = precision == CPCAG_F64 ? 8 : 4;
    DevBuf<double> Xd(c, static_cast<size_t>(std::max<i64>(rows * n, 1)));
    if (rows * n > 0) {
      if (precision == CPCAG_F64) {
        CUDA_OK(cudaMemcpyAsync(Xd.p, X, w * rows * n, cudaMemcpyDefault, c->stream));
      } else {
        DevBuf<float> Xf(c, static_cast<size_t>(rows * n));
        CUDA_OK(cudaMemcpyAsync(Xf.p, X, w * rows * n, cudaMemcpyDefault, c->stream));
        widen_k<<<stride_blocks(c, rows * n), kBlock, 0, c->stream>>>(rows * n, Xf.p, Xd.p);
        launched(c);
      }
    }
    DevBuf<int> a(c, static_cast<size_t>(std::max<i64>(n, 1)));
    kmeans_device(c, Xd.p, rows, n, k, restarts, seed, max_iter, a.p, wcss);
    CUDA_OK(cudaMemcpyAsync(assignments, a.p, sizeof(int) * n, cudaMemcpyDefault, c->stream));
    sync(c);
  });
}

extern "C" int cpcag_cuda_decode_labels(cpcag_ctx ctx, const int* sampled, int64_t rho_c, int64_t k,
                                        const int64_t* omega_c, int64_t n, cpcag_csr Lc, double pcg_tol,
                                        int64_t pcg_max_iter, int* labels) {
  return guard([&] {
    Ctx* c = as_ctx(ctx);
    Csr* L = as_csr(Lc);
    if (!sampled || !omega_c || !labels) invalid("null argument");
    if (k < 1) invalid("labels: k must be >= 1");
    std::vector<int> lab(static_cast<size_t>(rho_c));
    CUDA_OK(cudaMemcpy(lab.data(), sampled, sizeof(int) * rho_c, cudaMemcpyDefault));
    for (int x : lab)
      if (x < 0 || x >= k) invalid("labels: assignment out of range");
    if (L->rows != n) invalid("decode_labels: column Laplacian does not match plan");
    std::vector<i64> om(static_cast<size_t>(rho_c));
    CUDA_OK(cudaMemcpy(om.data(), omega_c, sizeof(i64) * rho_c, cudaMemcpyDefault));
    DevBuf<int> ld(c, static_cast<size_t>(std::max<i64>(rho_c, 1)));
    CUDA_OK(cudaMemcpyAsync(ld.p, lab.data(), sizeof(int) * rho_c, cudaMemcpyHostToDevice, c->stream));
    DevBuf<int> out(c, static_cast<size_t>(std::max<i64>(n, 1)));
    decode_labels_device(c, L, om, ld.p, k, pcg_tol, pcg_max_iter, n, out.p);
    CUDA_OK(cudaMemcpyAsync(labels, out.p, sizeof(int) * n, cudaMemcpyDefault, c->stream));
    sync(c);
  });
}

extern "C" int cpcag_clustering_error(const int* pred, const int* truth, int64_t n, int64_t k_pred, int64_t k_truth,
                                      double* out) {
  return guard([&] {
    if (!pred || !truth || !out) invalid("null argument");
    if (k_pred != k_truth) invalid("clustering error: cluster counts differ");
    if (n == 0) invalid("clustering error: empty labels");
    const i64 k = k_pred;
    std::vector<double> cont(static_cast<size_t>(k * k), 0.0);
    for (i64 i = 0; i < n; ++i) {
      if (pred[i] < 0 || pred[i] >= k || truth[i] < 0 || truth[i] >= k) invalid("labels: assignment out of range");
      cont[pred[i] + static_cast<i64>(truth[i]) * k] += 1.0;
    }
    const std::vector<i64> perm = max_assignment(cont, k);
    double agree = 0.0;
    for (i64 c = 0; c < k; ++c) agree += cont[c + perm[c] * k];
    *out = 1.0 - agree / static_cast<double>(n);
  });
}
