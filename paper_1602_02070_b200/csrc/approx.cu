// approx.cu -- the approximate (subspace-upsampling) decoder, Algorithm 2 of
// the paper as the reference implements it (decoders.cpp:188-225), with its
// building blocks thin_svd (eigs.cpp:53-57) and detect_rank (eigs.cpp:59-64).
//
//   Xt = U~ S~ V~^T (thin SVD, fp64, cuSOLVER gesvdj on the small sampled
//   matrix);  k = #{i : s_i / s_1 >= rank_threshold};
//   U = graph_upsample(L_r, Omega_r, U~(:, :k)),  V = graph_upsample(L_c, ...)
//   (multi-RHS Jacobi PCG on the interior block, kron.cu);
//   unit-normalise the columns, make the largest-|.| entry of each U column
//   positive (V flips with it), S = sqrt(np / (rho_r rho_c (1 - delta))) S~,
//   X = U S V^T.
// The factors are fp64; X is written in the working precision.
#include <cusolverDn.h>

#include <algorithm>
#include <cmath>
#include <memory>
#include <mutex>
#include <string>
#include <unordered_map>
#include <vector>

#include "common.cuh"

namespace cpcag_cuda {

namespace {

void solver_ok(cusolverStatus_t st, const char* what) {
  if (st != CUSOLVER_STATUS_SUCCESS)
    fail(CPCAG_ERR_CUDA, std::string("cusolver ") + what + " failed (status " + std::to_string(static_cast<int>(st)) + ")");
}

// One cuSOLVER handle per (thread, device); the stream is set per call.
cusolverDnHandle_t solver_handle(Ctx* c) {
  thread_local std::unordered_map<int, cusolverDnHandle_t> handles;
  auto it = handles.find(c->device);
  if (it == handles.end()) {
    cusolverDnHandle_t h = nullptr;
    solver_ok(cusolverDnCreate(&h), "create");
    it = handles.emplace(c->device, h).first;
  }
  solver_ok(cusolverDnSetStream(it->second, c->stream), "set stream");
  return it->second;
}

}  // namespace

__global__ void nonfinite_k(i64 n, const double* __restrict__ a, int* flag) {
  for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < n; i += (i64)gridDim.x * blockDim.x)
    if (!isfinite(a[i])) *flag = 1;
}

template <typename T>
__global__ void to_f64_k(i64 n, const T* __restrict__ a, double* __restrict__ b) {
  for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < n; i += (i64)gridDim.x * blockDim.x)
    b[i] = static_cast<double>(a[i]);
}

// Column norms sqrt(sum x^2) of an m x k column-major matrix, one CTA per
// column (fixed reduction tree).
__global__ void col_norms_k(i64 m, const double* __restrict__ A, double* __restrict__ out) {
  const i64 j = blockIdx.x;
  double s[1] = {0.0};
  for (i64 i = threadIdx.x; i < m; i += blockDim.x) {
    const double x = A[i + j * m];
    s[0] += x * x;
  }
  block_sum<1>(s);
  if (threadIdx.x == 0) out[j] = sqrt(s[0]);
}

// A(:, j) /= nrm[j] (decoders.cpp:213-214).
__global__ void col_div_k(i64 m, i64 k, double* __restrict__ A, const double* __restrict__ nrm) {
  const i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x;
  if (i >= m) return;
  for (i64 j = blockIdx.y; j < k; j += gridDim.y) A[i + j * m] = __ddiv_rn(A[i + j * m], nrm[j]);
}

// Index of the first largest |U(i, j)| per column (decoders.cpp:35-49).
__global__ void col_argmax_abs_k(i64 m, const double* __restrict__ U, i64* __restrict__ arg) {
  __shared__ double bv[1024];
  __shared__ i64 bi[1024];
  const i64 j = blockIdx.x;
  double best = -1.0;
  i64 at = 0;
  for (i64 i = threadIdx.x; i < m; i += blockDim.x) {
    const double a = fabs(U[i + j * m]);
    if (a > best) {
      best = a;
      at = i;
    }
  }
  bv[threadIdx.x] = best;
  bi[threadIdx.x] = at;
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) {
      const double ov = bv[threadIdx.x + s];
      const i64 oi = bi[threadIdx.x + s];
      if (ov > bv[threadIdx.x] || (ov == bv[threadIdx.x] && oi < bi[threadIdx.x])) {
        bv[threadIdx.x] = ov;
        bi[threadIdx.x] = oi;
      }
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) arg[j] = bi[0];
}

__global__ void pivot_sign_k(i64 p, i64 k, const double* __restrict__ U, const i64* __restrict__ arg,
                             int* __restrict__ flip) {
  const i64 j = blockIdx.x * (i64)blockDim.x + threadIdx.x;
  if (j < k) flip[j] = U[arg[j] + j * p] < 0.0 ? 1 : 0;
}

__global__ void flip_cols_k(i64 m, i64 k, double* __restrict__ A, const int* __restrict__ flip) {
  const i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x;
  if (i >= m) return;
  for (i64 j = blockIdx.y; j < k; j += gridDim.y)
    if (flip[j]) A[i + j * m] = -A[i + j * m];
}

// X(i, c) = sum_j (U(i, j) s_j) V(c, j), j ascending (decoders.cpp:220).
template <typename T>
__global__ void lowrank_k(i64 p, i64 n, i64 k, const double* __restrict__ U, const double* __restrict__ s,
                          const double* __restrict__ V, T* __restrict__ X) {
  const i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x;
  if (i >= p) return;
  for (i64 c = blockIdx.y; c < n; c += gridDim.y) {
    double x = 0.0;
    for (i64 j = 0; j < k; ++j) x = __dadd_rn(x, __dmul_rn(__dmul_rn(U[i + j * p], s[j]), V[c + j * n]));
    X[i + c * p] = static_cast<T>(x);
  }
}

// eigs.cpp:53-57.  A is m x n (device, fp64, col-major); U m x q, sigma q
// (descending), V n x q with q = min(m, n).  Column signs are the solver's.
void thin_svd_device(Ctx* c, const double* A, i64 m, i64 n, double* U, double* sigma, double* V) {
  const i64 mn = m * n;
  if (mn) {
    DevBuf<int> flag(c, 1);
    flag.zero(c);
    nonfinite_k<<<stride_blocks(c, mn), kBlock, 0, c->stream>>>(mn, A, flag.p);
    launched(c);
    if (read_back(c, flag.p)) invalid("thin_svd: non-finite input");
  }
  const i64 q = std::min(m, n);
  if (q == 0) return;
  if (m > INT32_MAX || n > INT32_MAX) invalid("thin_svd: matrix too large");
  cusolverDnHandle_t h = solver_handle(c);
  gesvdjInfo_t params = nullptr;
  solver_ok(cusolverDnCreateGesvdjInfo(&params), "gesvdj info");
  std::unique_ptr<std::remove_pointer<gesvdjInfo_t>::type, void (*)(gesvdjInfo_t)> own(
      params, [](gesvdjInfo_t p) { cusolverDnDestroyGesvdjInfo(p); });
  solver_ok(cusolverDnXgesvdjSetSortEig(params, 1), "gesvdj sort");
  DevBuf<double> W(c, mn);  // gesvdj overwrites its input
  CUDA_OK(cudaMemcpyAsync(W.p, A, sizeof(double) * mn, cudaMemcpyDeviceToDevice, c->stream));
  const int mi = static_cast<int>(m), ni = static_cast<int>(n);
  int lwork = 0;
  solver_ok(cusolverDnDgesvdj_bufferSize(h, CUSOLVER_EIG_MODE_VECTOR, 1, mi, ni, W.p, mi, sigma, U, mi, V, ni,
                                         &lwork, params),
            "gesvdj buffer");
  DevBuf<double> work(c, std::max(lwork, 1));
  DevBuf<int> info(c, 1);
  solver_ok(cusolverDnDgesvdj(h, CUSOLVER_EIG_MODE_VECTOR, 1, mi, ni, W.p, mi, sigma, U, mi, V, ni, work.p, lwork,
                              info.p, params),
            "gesvdj");
  const int inf = read_back(c, info.p);
  if (inf != 0) runtime("thin_svd: solver did not converge (info " + std::to_string(inf) + ")");
}

// ---------------------------------------------------------------- Gram SVD
// The decoder only needs the leading singular triplets of the small sampled
// matrix (k at sigma_k / sigma_1 >= rank_threshold), so it goes through the
// Gram matrix of the short side: G = A^T A (n <= m) or A A^T, eigenpairs by
// cuSOLVER syevd, sigma = sqrt(lambda), and the long-side vectors as
// A v / sigma for the k requested columns.  The error of a used vector is
// ~eps (sigma_1 / sigma_k)^2 <= 1e-14 at the default threshold 0.1.
__global__ void gram_k(i64 m, i64 n, bool tall, const double* __restrict__ A, double* __restrict__ G) {
  // tall: G (n x n) = A^T A, else G (m x m) = A A^T; fixed sequential order.
  const i64 q = tall ? n : m;
  const i64 a = blockIdx.x * (i64)blockDim.x + threadIdx.x, b = blockIdx.y;
  if (a >= q || b > a) return;
  double s = 0.0;
  if (tall)
    for (i64 i = 0; i < m; ++i) s += A[i + a * m] * A[i + b * m];
  else
    for (i64 j = 0; j < n; ++j) s += A[a + j * m] * A[b + j * m];
  G[a + b * q] = s;
  G[b + a * q] = s;
}

// Reverse eigenpairs to descending order; sigma = sqrt(max(lambda, 0)).
__global__ void eig_to_svd_k(i64 q, i64 kvec, const double* __restrict__ lam, const double* __restrict__ E,
                             double* __restrict__ sigma, double* __restrict__ W) {
  const i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x;
  if (i < q) sigma[i] = sqrt(fmax(lam[q - 1 - i], 0.0));
  for (i64 j = blockIdx.y; j < kvec; j += gridDim.y)
    if (i < q) W[i + j * q] = E[i + (q - 1 - j) * q];
}

// Out (len x k) = op(A) W diag(1 / sigma): tall -> A (m x n) W (n x k);
// wide -> A^T (n x m) W (m x k).
__global__ void project_k(i64 m, i64 n, bool tall, i64 k, const double* __restrict__ A, const double* __restrict__ W,
                          const double* __restrict__ sigma, double* __restrict__ Out) {
  const i64 len = tall ? m : n, q = tall ? n : m;
  const i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x;
  if (i >= len) return;
  for (i64 j = blockIdx.y; j < k; j += gridDim.y) {
    double s = 0.0;
    for (i64 t = 0; t < q; ++t) s += (tall ? A[i + t * m] : A[t + i * m]) * W[t + j * q];
    Out[i + j * len] = s / sigma[j];
  }
}

// sigma (q = min(m, n), descending); U (m x kvec) and V (n x kvec) when
// kvec > 0 (every used sigma must be > 0).
void gram_svd_device(Ctx* c, const double* A, i64 m, i64 n, i64 kvec, double* sigma, double* U, double* V) {
  const i64 q = std::min(m, n);
  if (q == 0) return;
  {
    DevBuf<int> flag(c, 1);
    flag.zero(c);
    nonfinite_k<<<stride_blocks(c, m * n), kBlock, 0, c->stream>>>(m * n, A, flag.p);
    launched(c);
    if (read_back(c, flag.p)) invalid("thin_svd: non-finite input");
  }
  if (q > INT32_MAX) invalid("thin_svd: matrix too large");
  const bool tall = m >= n;
  DevBuf<double> G(c, q * q), lam(c, q);
  gram_k<<<dim3(blocks_for(q), static_cast<unsigned>(std::min<i64>(q, 65535))), kBlock, 0, c->stream>>>(m, n, tall, A,
                                                                                                        G.p);
  launched(c);
  cusolverDnHandle_t h = solver_handle(c);
  const cusolverEigMode_t mode = kvec > 0 ? CUSOLVER_EIG_MODE_VECTOR : CUSOLVER_EIG_MODE_NOVECTOR;
  const int qi = static_cast<int>(q);
  int lwork = 0;
  solver_ok(cusolverDnDsyevd_bufferSize(h, mode, CUBLAS_FILL_MODE_LOWER, qi, G.p, qi, lam.p, &lwork), "syevd buffer");
  DevBuf<double> work(c, std::max(lwork, 1));
  DevBuf<int> info(c, 1);
  solver_ok(cusolverDnDsyevd(h, mode, CUBLAS_FILL_MODE_LOWER, qi, G.p, qi, lam.p, work.p, lwork, info.p), "syevd");
  if (read_back(c, info.p) != 0) runtime("thin_svd: eigensolver did not converge");
  DevBuf<double> Wv(c, std::max<i64>(q * kvec, 1));
  eig_to_svd_k<<<dim3(blocks_for(q), static_cast<unsigned>(std::max<i64>(1, std::min<i64>(kvec, 65535)))), kBlock, 0,
                 c->stream>>>(q, kvec, lam.p, G.p, sigma, Wv.p);
  launched(c);
  if (kvec == 0) return;
  // short-side vectors are the eigenvectors; the long side is projected
  double* shortv = tall ? V : U;
  double* longv = tall ? U : V;
  CUDA_OK(cudaMemcpyAsync(shortv, Wv.p, sizeof(double) * q * kvec, cudaMemcpyDeviceToDevice, c->stream));
  const i64 len = tall ? m : n;
  project_k<<<dim3(blocks_for(len), static_cast<unsigned>(std::min<i64>(kvec, 65535))), kBlock, 0, c->stream>>>(
      m, n, tall, kvec, A, Wv.p, sigma, longv);
  launched(c);
}

template <typename T>
void to_f64_device(Ctx* c, const T* a, i64 n, double* out) {
  if (!n) return;
  to_f64_k<T><<<stride_blocks(c, n), kBlock, 0, c->stream>>>(n, a, out);
  launched(c);
}
template void to_f64_device<float>(Ctx*, const float*, i64, double*);
template void to_f64_device<double>(Ctx*, const double*, i64, double*);

// ---------------------------------------------------------------- sym_eig
// eigs.cpp:34-51: densify, symmetrise 0.5 (D + D^T), dense symmetric
// eigensolver (cuSOLVER syevd, eigenvalues ascending), the first k pairs, and
// each eigenvector column's sign fixed so its first entry above 1e-12 times
// the column peak is positive.  Dense by design (the reference's own
// desk-scale solver): n is limited by memory (n^2 doubles).
__global__ void densify_sym_k(i64 n, const i64* __restrict__ rp, const int* __restrict__ ci,
                              const double* __restrict__ v, double* __restrict__ D) {
  const i64 r = blockIdx.x * (i64)blockDim.x + threadIdx.x;
  if (r >= n) return;
  for (i64 k = rp[r]; k < rp[r + 1]; ++k) D[r + static_cast<i64>(ci[k]) * n] = v[k];
}
__global__ void symmetrize_k(i64 n, const double* __restrict__ D, double* __restrict__ S) {
  const i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x;
  if (i >= n) return;
  for (i64 j = blockIdx.y; j < n; j += gridDim.y) S[i + j * n] = 0.5 * (D[i + j * n] + D[j + i * n]);
}
// One CTA per column: peak = max |x|, then the first index with |x| > 1e-12 peak.
__global__ void fix_signs_k(i64 n, double* __restrict__ E) {
  __shared__ double red[1024];
  __shared__ i64 first;
  const i64 j = blockIdx.x;
  double* x = E + j * n;
  double m = 0.0;
  for (i64 i = threadIdx.x; i < n; i += blockDim.x) m = fmax(m, fabs(x[i]));
  red[threadIdx.x] = m;
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) red[threadIdx.x] = fmax(red[threadIdx.x], red[threadIdx.x + s]);
    __syncthreads();
  }
  const double peak = red[0];
  if (threadIdx.x == 0) first = n;
  __syncthreads();
  if (peak == 0.0) return;
  for (i64 i = threadIdx.x; i < n; i += blockDim.x)
    if (fabs(x[i]) > 1e-12 * peak) atomicMin(reinterpret_cast<unsigned long long*>(&first), static_cast<unsigned long long>(i));
  __syncthreads();
  const bool flip = first < n && x[first] < 0.0;
  __syncthreads();
  if (flip)
    for (i64 i = threadIdx.x; i < n; i += blockDim.x) x[i] = -x[i];
}

void sym_eig_device(Ctx* c, Csr* A, i64 k, double* evals, double* evecs) {
  if (A->rows != A->cols) invalid("sym_eig: square matrix required");
  const i64 n = A->rows;
  if (k < 1 || k > n)
    invalid("sym_eig: order k out of range (k = " + std::to_string(k) + ", dim = " + std::to_string(n) + ")");
  if (n > 46340) invalid("sym_eig: dense eigensolver limited to n <= 46340 on the device");
  DevBuf<double> D(c, n * n), S(c, n * n), lam(c, n);
  D.zero(c);
  densify_sym_k<<<blocks_for(n), kBlock, 0, c->stream>>>(n, A->rp, A->ci, A->v, D.p);
  launched(c);
  symmetrize_k<<<dim3(blocks_for(n), static_cast<unsigned>(std::min<i64>(n, 65535))), kBlock, 0, c->stream>>>(n, D.p,
                                                                                                          S.p);
  launched(c);
  D.release();
  cusolverDnHandle_t h = solver_handle(c);
  const cusolverEigMode_t mode = evecs ? CUSOLVER_EIG_MODE_VECTOR : CUSOLVER_EIG_MODE_NOVECTOR;
  const int ni = static_cast<int>(n);
  int lwork = 0;
  solver_ok(cusolverDnDsyevd_bufferSize(h, mode, CUBLAS_FILL_MODE_LOWER, ni, S.p, ni, lam.p, &lwork), "syevd buffer");
  DevBuf<double> work(c, std::max(lwork, 1));
  DevBuf<int> info(c, 1);
  solver_ok(cusolverDnDsyevd(h, mode, CUBLAS_FILL_MODE_LOWER, ni, S.p, ni, lam.p, work.p, lwork, info.p), "syevd");
  if (read_back(c, info.p) != 0) runtime("sym_eig: eigensolver failed");
  CUDA_OK(cudaMemcpyAsync(evals, lam.p, sizeof(double) * k, cudaMemcpyDefault, c->stream));
  if (evecs) {
    fix_signs_k<<<static_cast<unsigned>(k), 1024, 0, c->stream>>>(n, S.p);
    launched(c);
    CUDA_OK(cudaMemcpyAsync(evecs, S.p, sizeof(double) * n * k, cudaMemcpyDefault, c->stream));
  }
  sync(c);
}

// graph.cpp:237-249.
cpcag_spectral_gap spectral_gap_host(const double* evals, i64 order, i64 k) {
  if (k < 1 || order < k + 1) invalid("spectral gap: need at least k+1 eigenvalues");
  cpcag_spectral_gap g;
  g.k = k;
  g.lambda_k = std::max(0.0, evals[k - 1]);
  g.lambda_k1 = std::max(0.0, evals[k]);
  if (g.lambda_k1 <= 1e-14) runtime("gap undefined: graph has > k components");
  g.ratio = g.lambda_k / g.lambda_k1;
  return g;
}

// eigs.cpp:59-64.
// ---------------------------------------------------------------- rank job
// The pipeline's detected rank (pipeline.cpp:319-321): singular values of the
// compressed solution Xt = sqrt of the eigenvalues of its Gram matrix.  The
// eigenvalues come from a parallel cyclic Jacobi in ONE CTA (the Gram matrix
// of config 1 is 100 x 100: 80 KB in shared memory), so the whole job runs
// on the side stream beside the decoder and the host reads the result after
// the decode; no library solver on the timed path.
constexpr int kJacobiThreads = 1024;

__global__ void __launch_bounds__(kJacobiThreads) jacobi_eigvals_k(int n, const double* __restrict__ G,
                                                                    double* __restrict__ lam, int max_sweeps) {
  extern __shared__ double A[];  // m x m, m = n rounded up to even (padding index: zero row/column)
  const int m = n + (n & 1);
  double* cs = A + static_cast<size_t>(m) * m;  // [m/2][2] rotation (c, s) per pair
  int* pr = reinterpret_cast<int*>(cs + m);      // [m] pair members of the current step
  __shared__ double red[2][32];
  __shared__ int stop;
  for (int e = threadIdx.x; e < m * m; e += blockDim.x) {
    const int i = e % m, j = e / m;
    A[e] = (i < n && j < n) ? G[i + static_cast<i64>(j) * n] : 0.0;
  }
  if (threadIdx.x == 0) stop = 0;
  __syncthreads();
  const int half = m / 2, lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int sweep = 0; sweep < max_sweeps; ++sweep) {
    // convergence: off-diagonal vs diagonal Frobenius norms (fixed-order sums)
    double off = 0.0, dia = 0.0;
    for (int e = threadIdx.x; e < m * m; e += blockDim.x) {
      const int i = e % m, j = e / m;
      const double x = A[e];
      if (i == j)
        dia += x * x;
      else
        off += x * x;
    }
    off = warp_sum(off);
    dia = warp_sum(dia);
    if (lane == 0) {
      red[0][wid] = off;
      red[1][wid] = dia;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      double o = 0.0, d = 0.0;
      for (int w = 0; w < static_cast<int>(blockDim.x >> 5); ++w) o += red[0][w], d += red[1][w];
      stop = !(o > 1e-26 * d) || o == 0.0;  // off-diagonal below 1e-13 of the diagonal (Frobenius)
    }
    __syncthreads();
    if (stop) break;
    for (int step = 0; step < m - 1; ++step) {
      // round-robin pairing: index 0 fixed, the others rotate
      for (int k = threadIdx.x; k < half; k += blockDim.x) {
        const int a = k == 0 ? 0 : 1 + (k - 1 + step) % (m - 1);
        const int b = 1 + (m - 2 - k + step) % (m - 1);
        const int p = a < b ? a : b, q = a < b ? b : a;
        pr[2 * k] = p;
        pr[2 * k + 1] = q;
        const double apq = A[p + q * m], app = A[p + p * m], aqq = A[q + q * m];
        double c = 1.0, s = 0.0;
        if (apq != 0.0) {
          const double th = (aqq - app) / (2.0 * apq);
          const double t = (th >= 0.0 ? 1.0 : -1.0) / (fabs(th) + sqrt(th * th + 1.0));
          c = 1.0 / sqrt(t * t + 1.0);
          s = t * c;
        }
        cs[2 * k] = c;
        cs[2 * k + 1] = s;
      }
      __syncthreads();
      // rows p, q <- rotated (disjoint across pairs)
      for (int e = threadIdx.x; e < half * m; e += blockDim.x) {
        const int k = e / m, col = e % m;
        const int p = pr[2 * k], q = pr[2 * k + 1];
        const double c = cs[2 * k], s = cs[2 * k + 1];
        const double xp = A[p + col * m], xq = A[q + col * m];
        A[p + col * m] = c * xp - s * xq;
        A[q + col * m] = s * xp + c * xq;
      }
      __syncthreads();
      // columns p, q <- rotated
      for (int e = threadIdx.x; e < half * m; e += blockDim.x) {
        const int k = e / m, row = e % m;
        const int p = pr[2 * k], q = pr[2 * k + 1];
        const double c = cs[2 * k], s = cs[2 * k + 1];
        const double xp = A[row + p * m], xq = A[row + q * m];
        A[row + p * m] = c * xp - s * xq;
        A[row + q * m] = s * xp + c * xq;
      }
      __syncthreads();
    }
  }
  for (int i = threadIdx.x; i < n; i += blockDim.x) lam[i] = A[i + i * m];
}

void rank_job_start(Ctx* c, RankJob& job, const double* Xt64, i64 m, i64 n, cudaStream_t s) {
  job.q = std::min(m, n);
  if (job.q == 0) return;
  if (job.q > 110) invalid("rank job: Gram order above 110");
  const bool tall = m >= n;
  job.G.alloc(c, job.q * job.q);
  job.lam.alloc(c, job.q);
  job.flag.alloc(c, 1);
  job.flag.zero(c);
  if (!job.host) CUDA_OK(cudaMallocHost(&job.host, sizeof(double) * 128));
  CUDA_OK(cudaEventRecord(c->fork_ev, c->stream));
  CUDA_OK(cudaStreamWaitEvent(s, c->fork_ev, 0));
  nonfinite_k<<<stride_blocks(c, m * n), kBlock, 0, s>>>(m * n, Xt64, job.flag.p);
  launched(c);
  gram_k<<<dim3(blocks_for(job.q), static_cast<unsigned>(job.q)), kBlock, 0, s>>>(m, n, tall, Xt64, job.G.p);
  launched(c);
  const int mm = static_cast<int>(job.q + (job.q & 1));
  const size_t smem = sizeof(double) * (static_cast<size_t>(mm) * mm + mm) + sizeof(int) * mm;
  ensure_smem(jacobi_eigvals_k, smem);
  jacobi_eigvals_k<<<1, kJacobiThreads, smem, s>>>(static_cast<int>(job.q), job.G.p, job.lam.p, 60);
  launched(c);
  CUDA_OK(cudaMemcpyAsync(job.host, job.lam.p, sizeof(double) * job.q, cudaMemcpyDeviceToHost, s));
  CUDA_OK(cudaMemcpyAsync(reinterpret_cast<int*>(reinterpret_cast<double*>(job.host) + 120), job.flag.p, sizeof(int),
                          cudaMemcpyDeviceToHost, s));
  CUDA_OK(cudaEventRecord(c->join_ev, s));
  job.side = s;
  job.running = true;
  c->side_job_running = true;
}

// Joins the job (the main stream waits for the side stream) and returns the
// singular values, descending.
std::vector<double> rank_job_finish(Ctx* c, RankJob& job) {
  std::vector<double> sv;
  if (!job.running) return sv;
  CUDA_OK(cudaStreamWaitEvent(c->stream, c->join_ev, 0));
  CUDA_OK(cudaEventSynchronize(c->join_ev));
  job.running = false;
  c->side_job_running = false;
  c->sm_reserve = 0;
  const double* h = reinterpret_cast<const double*>(job.host);
  if (*reinterpret_cast<const int*>(h + 120)) invalid("thin_svd: non-finite input");
  sv.resize(static_cast<size_t>(job.q));
  for (i64 i = 0; i < job.q; ++i) sv[i] = std::sqrt(std::max(h[i], 0.0));
  std::sort(sv.begin(), sv.end(), [](double a, double b) { return a > b; });
  return sv;
}

RankJob::~RankJob() {
  if (running && side) cudaStreamSynchronize(side);  // an exception left the job in flight
  if (host) cudaFreeHost(host);
}

i64 detect_rank_host(const std::vector<double>& s, double thr) {
  if (s.empty() || !(s[0] > 0.0)) return 0;
  i64 k = 0;
  while (k < static_cast<i64>(s.size()) && s[k] / s[0] >= thr) ++k;
  return k;
}

template <typename T>
void approx_decode_device(Ctx* c, const T* Xt, i64 rho_r, i64 rho_c, const std::vector<i64>& om_r,
                          const std::vector<i64>& om_c, i64 p, i64 n, Csr* Lr, Csr* Lc,
                          const cpcag_approx_config& cfg, T* X, double* U_out, double* s_out, double* V_out,
                          i64 k_cap, i64* k_out) {
  if (Lr->rows != p || Lc->rows != n) invalid("approximate decoder: Laplacians do not match plan");
  if (!(cfg.rank_threshold > 0.0 && cfg.rank_threshold < 1.0))
    invalid("approximate decoder: rank threshold must be in (0,1)");
  const i64 q = std::min(rho_r, rho_c);
  DevBuf<double> A(c, std::max<i64>(rho_r * rho_c, 1)), Ut(c, std::max<i64>(rho_r * q, 1)),
      Vt(c, std::max<i64>(rho_c * q, 1)), st(c, std::max<i64>(q, 1));
  if (rho_r * rho_c) {
    to_f64_k<T><<<stride_blocks(c, rho_r * rho_c), kBlock, 0, c->stream>>>(rho_r * rho_c, Xt, A.p);
    launched(c);
  }
  gram_svd_device(c, A.p, rho_r, rho_c, 0, st.p, nullptr, nullptr);
  std::vector<double> s(static_cast<size_t>(q));
  if (q) CUDA_OK(cudaMemcpyAsync(s.data(), st.p, sizeof(double) * q, cudaMemcpyDeviceToHost, c->stream));
  sync(c);
  const i64 k = detect_rank_host(s, cfg.rank_threshold);
  if (k == 0) runtime("approximate decoder: no singular value above the rank threshold");
  gram_svd_device(c, A.p, rho_r, rho_c, k, st.p, Ut.p, Vt.p);

  DevBuf<double> U(c, p * k), V(c, n * k);
  graph_upsample_device(c, Lr, om_r, Ut.p, k, cfg.pcg_tol, cfg.pcg_max_iter, U.p);
  graph_upsample_device(c, Lc, om_c, Vt.p, k, cfg.pcg_tol, cfg.pcg_max_iter, V.p);

  DevBuf<double> nu(c, k), nv(c, k);
  col_norms_k<<<static_cast<unsigned>(k), kBlock, 0, c->stream>>>(p, U.p, nu.p);
  launched(c);
  col_norms_k<<<static_cast<unsigned>(k), kBlock, 0, c->stream>>>(n, V.p, nv.p);
  launched(c);
  std::vector<double> hnu(static_cast<size_t>(k)), hnv(static_cast<size_t>(k));
  CUDA_OK(cudaMemcpyAsync(hnu.data(), nu.p, sizeof(double) * k, cudaMemcpyDeviceToHost, c->stream));
  CUDA_OK(cudaMemcpyAsync(hnv.data(), nv.p, sizeof(double) * k, cudaMemcpyDeviceToHost, c->stream));
  sync(c);
  for (i64 j = 0; j < k; ++j)
    if (hnu[j] <= 1e-14 || hnv[j] <= 1e-14)
      runtime("approximate decoder: zero column " + std::to_string(j) + " after upsampling (rank overestimated)");
  const unsigned ky = static_cast<unsigned>(std::min<i64>(k, 65535));
  col_div_k<<<dim3(blocks_for(p), ky), kBlock, 0, c->stream>>>(p, k, U.p, nu.p);
  launched(c);
  col_div_k<<<dim3(blocks_for(n), ky), kBlock, 0, c->stream>>>(n, k, V.p, nv.p);
  launched(c);
  // align_factor_signs (decoders.cpp:33-50)
  DevBuf<i64> arg(c, k);
  DevBuf<int> flip(c, k);
  col_argmax_abs_k<<<static_cast<unsigned>(k), 1024, 0, c->stream>>>(p, U.p, arg.p);
  launched(c);
  pivot_sign_k<<<blocks_for(k), kBlock, 0, c->stream>>>(p, k, U.p, arg.p, flip.p);
  launched(c);
  flip_cols_k<<<dim3(blocks_for(p), ky), kBlock, 0, c->stream>>>(p, k, U.p, flip.p);
  launched(c);
  flip_cols_k<<<dim3(blocks_for(n), ky), kBlock, 0, c->stream>>>(n, k, V.p, flip.p);
  launched(c);
  // scaling_constant (decoders.cpp:27-31, sampling.cpp:12-15)
  const double delta = cfg.delta_for_scaling;
  if (!(delta >= 0.0 && delta < 1.0)) invalid("decoder: delta_for_scaling must be in [0,1)");
  const double norm_const = (static_cast<double>(n) * static_cast<double>(p)) /
                            (static_cast<double>(rho_r) * static_cast<double>(rho_c));
  const double scale = std::sqrt(norm_const / (1.0 - delta));
  std::vector<double> sig(static_cast<size_t>(k));
  for (i64 j = 0; j < k; ++j) sig[j] = scale * s[j];
  DevBuf<double> sd(c, k);
  CUDA_OK(cudaMemcpyAsync(sd.p, sig.data(), sizeof(double) * k, cudaMemcpyHostToDevice, c->stream));
  if (p && n) {
    dim3 g(blocks_for(p), static_cast<unsigned>(std::min<i64>(n, 65535)));
    lowrank_k<T><<<g, kBlock, 0, c->stream>>>(p, n, k, U.p, sd.p, V.p, X);
    launched(c);
  }
  *k_out = k;
  if (k_cap > 0 && k <= k_cap) {
    if (U_out) CUDA_OK(cudaMemcpyAsync(U_out, U.p, sizeof(double) * p * k, cudaMemcpyDefault, c->stream));
    if (V_out) CUDA_OK(cudaMemcpyAsync(V_out, V.p, sizeof(double) * n * k, cudaMemcpyDefault, c->stream));
    if (s_out) CUDA_OK(cudaMemcpyAsync(s_out, sd.p, sizeof(double) * k, cudaMemcpyDefault, c->stream));
  }
  sync(c);
}

template void approx_decode_device<double>(Ctx*, const double*, i64, i64, const std::vector<i64>&,
                                           const std::vector<i64>&, i64, i64, Csr*, Csr*, const cpcag_approx_config&,
                                           double*, double*, double*, double*, i64, i64*);
template void approx_decode_device<float>(Ctx*, const float*, i64, i64, const std::vector<i64>&,
                                          const std::vector<i64>&, i64, i64, Csr*, Csr*, const cpcag_approx_config&,
                                          float*, double*, double*, double*, i64, i64*);

}  // namespace cpcag_cuda

using namespace cpcag_cuda;

namespace {
std::vector<i64> fetch_idx(const int64_t* src, i64 count) {
  std::vector<i64> v(static_cast<size_t>(std::max<i64>(count, 0)));
  if (v.empty()) return v;
  if (!src) invalid("null argument");
  if (is_device_ptr(src))
    CUDA_OK(cudaMemcpy(v.data(), src, sizeof(i64) * v.size(), cudaMemcpyDeviceToHost));
  else
    std::copy(src, src + v.size(), v.begin());
  return v;
}
}  // namespace

extern "C" int cpcag_cuda_thin_svd(cpcag_ctx ctx, const double* A, int64_t m, int64_t n, double* U, double* sigma,
                                   double* V) {
  return guard([&] {
    Ctx* c = as_ctx(ctx);
    if (m < 0 || n < 0) invalid("thin_svd: negative size");
    const i64 q = std::min(m, n);
    if ((m * n && !A) || (q && (!U || !sigma || !V))) invalid("null argument");
    InView<double> a(c, A, static_cast<size_t>(m * n));
    OutView<double> u(c, U, static_cast<size_t>(m * q)), s(c, sigma, static_cast<size_t>(q)),
        v(c, V, static_cast<size_t>(n * q));
    thin_svd_device(c, a.d, m, n, u.d, s.d, v.d);
    u.flush(c);
    s.flush(c);
    v.flush(c);
    sync(c);
  });
}

extern "C" int cpcag_cuda_approx_decode(cpcag_ctx ctx, int precision, const void* Xt, int64_t rho_r, int64_t rho_c,
                                        const int64_t* omega_r, const int64_t* omega_c, int64_t p, int64_t n,
                                        cpcag_csr Lr, cpcag_csr Lc, const cpcag_approx_config* cfg, void* X,
                                        double* U, double* sigma, double* V, int64_t k_cap, int64_t* k) {
  auto run = [&](auto tag) {
    using T = decltype(tag);
    return guard([&] {
      Ctx* c = as_ctx(ctx);
      if (!cfg || !k || (p * n && !X) || (rho_r * rho_c && !Xt)) invalid("null argument");
      const std::vector<i64> omr = fetch_idx(omega_r, rho_r), omc = fetch_idx(omega_c, rho_c);
      InView<T> xt(c, static_cast<const T*>(Xt), static_cast<size_t>(rho_r * rho_c));
      OutView<T> x(c, static_cast<T*>(X), static_cast<size_t>(p * n));
      approx_decode_device<T>(c, xt.d, rho_r, rho_c, omr, omc, p, n, as_csr(Lr), as_csr(Lc), *cfg, x.d, U, sigma, V,
                              k_cap, k);
      x.flush(c);
      sync(c);
    });
  };
  if (precision == CPCAG_F64) return run(double{});
  if (precision == CPCAG_F32) return run(float{});
  set_last_error("unknown precision flag");
  return CPCAG_ERR_INVALID_ARGUMENT;
}

extern "C" int cpcag_cuda_sym_eig(cpcag_ctx ctx, cpcag_csr A, int64_t k, double* eigenvalues, double* eigenvectors) {
  return guard([&] {
    Ctx* c = as_ctx(ctx);
    Csr* a = as_csr(A);
    if (!eigenvalues) invalid("null argument");
    OutView<double> ev(c, eigenvalues, static_cast<size_t>(std::max<int64_t>(k, 0)));
    OutView<double> ex(c, eigenvectors, eigenvectors ? static_cast<size_t>(a->rows * std::max<int64_t>(k, 0)) : 0);
    sym_eig_device(c, a, k, ev.d, eigenvectors ? ex.d : nullptr);
    ev.flush(c);
    if (eigenvectors) ex.flush(c);
    sync(c);
  });
}
