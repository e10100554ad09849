// lanczos.cu -- the k smallest eigenvalues of a large sparse symmetric
// matrix (graph Laplacian) for the spectral gap of the alternate decoder
// (replaces the dense sym_eig of eigs.cpp:34-51 where the
// reference's dense solver is infeasible: the 2e5- and 1e6-node graphs of
// configs 3/4, pipeline.cpp:343-349).
//
// Lanczos on B = sigma I - A with sigma the Gershgorin bound (B is PSD and
// its LARGEST eigenvalues are sigma - the smallest of A), full
// reorthogonalisation by classical Gram-Schmidt applied twice (two cuBLAS
// GEMV pairs per step against the stored basis), scalars kept on the device.
// Every `check` steps the host reads alpha/beta, diagonalises the tridiagonal
// T_j by implicit QL tracking only the last row of its eigenvector matrix,
// and stops when the k largest Ritz values have residual |beta_j s_ji| <=
// tol * sigma (or the Krylov space is invariant).  Deterministic for a given
// seed (start vector from the reference RNG, fixed kernel/GEMV order).
#include <cublas_v2.h>

#include <algorithm>
#include <cmath>
#include <string>
#include <unordered_map>
#include <vector>

#include "common.cuh"

namespace cpcag_cuda {

namespace {

cublasHandle_t blas_handle(Ctx* c) {
  thread_local std::unordered_map<int, cublasHandle_t> handles;
  auto it = handles.find(c->device);
  cublasHandle_t h;
  if (it == handles.end()) {
    if (cublasCreate(&h) != CUBLAS_STATUS_SUCCESS) fail(CPCAG_ERR_CUDA, "cublas: handle creation failed");
    handles.emplace(c->device, h);
  } else {
    h = it->second;
  }
  cublasSetStream(h, c->stream);
  return h;
}

void blas_ok(cublasStatus_t s, const char* what) {
  if (s != CUBLAS_STATUS_SUCCESS)
    fail(CPCAG_ERR_CUDA, std::string("cublas ") + what + " failed (status " + std::to_string(static_cast<int>(s)) + ")");
}

// w = sigma v - A v, warp per row.
__global__ void shifted_spmv_k(i64 n, const i64* __restrict__ rp, const int* __restrict__ ci,
                               const double* __restrict__ val, double sigma, const double* __restrict__ v,
                               double* __restrict__ w) {
  const int lane = threadIdx.x & 31;
  const i64 r = (blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x) >> 5;
  if (r >= n) return;
  double acc = 0.0;
  for (i64 k = rp[r] + lane; k < rp[r + 1]; k += 32) acc += val[k] * v[ci[k]];
  acc = warp_sum(acc);
  if (lane == 0) w[r] = sigma * v[r] - acc;
}

// Gershgorin bound max_i sum_j |A_ij| (block partial maxima).
__global__ void row_abs_max_k(i64 n, const i64* __restrict__ rp, const double* __restrict__ val,
                              double* __restrict__ out) {
  double m = 0.0;
  for (i64 r = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x; r < n; r += gridDim.x * (i64)blockDim.x) {
    double s = 0.0;
    for (i64 k = rp[r]; k < rp[r + 1]; ++k) s += fabs(val[k]);
    m = fmax(m, s);
  }
  for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  __shared__ double sh[32];
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int q = 0; q < (blockDim.x + 31) / 32; ++q) t = fmax(t, sh[q]);
    out[blockIdx.x] = t;
  }
}

__global__ void alpha_k(const double* __restrict__ h1, const double* __restrict__ h2, i64 j, double* alpha) {
  alpha[j] = h1[j] + h2[j];
}

// v_next = w / beta (beta on the device; an exact zero leaves v_next = 0 and
// the host stops on the invariant subspace).
__global__ void scale_k(i64 n, const double* __restrict__ w, const double* __restrict__ beta, double* __restrict__ out) {
  const double b = *beta;
  for (i64 i = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x; i < n; i += gridDim.x * (i64)blockDim.x)
    out[i] = b > 0.0 ? __ddiv_rn(w[i], b) : 0.0;
}

// Implicit QL on the symmetric tridiagonal (d, e), e[i] between i and i+1;
// z tracks the LAST row of the eigenvector matrix.  d becomes the
// eigenvalues (unsorted), z[i] the last component of eigenvector i.
void tql_lastrow(std::vector<double>& d, std::vector<double> e, std::vector<double>& z) {
  const int n = static_cast<int>(d.size());
  z.assign(static_cast<size_t>(n), 0.0);
  if (n == 0) return;
  z[static_cast<size_t>(n - 1)] = 1.0;
  e.resize(static_cast<size_t>(n));
  e[static_cast<size_t>(n - 1)] = 0.0;
  for (int l = 0; l < n; ++l) {
    int iter = 0, m;
    do {
      for (m = l; m < n - 1; ++m) {
        const double dd = std::fabs(d[m]) + std::fabs(d[m + 1]);
        if (std::fabs(e[m]) <= 1e-16 * dd) break;
      }
      if (m != l) {
        if (iter++ == 200) runtime("lanczos: tridiagonal eigensolver did not converge");
        double g = (d[l + 1] - d[l]) / (2.0 * e[l]);
        double r = std::hypot(g, 1.0);
        g = d[m] - d[l] + e[l] / (g + std::copysign(r, g));
        double s = 1.0, c = 1.0, p = 0.0;
        int i;
        bool underflow = false;
        for (i = m - 1; i >= l; --i) {
          double f = s * e[i];
          const double b = c * e[i];
          r = std::hypot(f, g);
          e[i + 1] = r;
          if (r == 0.0) {
            d[i + 1] -= p;
            e[m] = 0.0;
            underflow = true;
            break;
          }
          s = f / r;
          c = g / r;
          g = d[i + 1] - p;
          r = (d[i] - g) * s + 2.0 * c * b;
          p = s * r;
          d[i + 1] = g + p;
          g = c * r - b;
          f = z[i + 1];
          z[i + 1] = s * z[i] + c * f;
          z[i] = c * z[i] - s * f;
        }
        if (underflow) continue;
        d[l] -= p;
        e[l] = g;
        e[m] = 0.0;
      }
    } while (m != l);
  }
}

}  // namespace

void sym_eigvals_lanczos(Ctx* c, Csr* A, i64 k, double tol, i64 max_iter, uint64_t seed, double* evals,
                         i64* iterations) {
  if (A->rows != A->cols) invalid("sym_eig: square matrix required");
  const i64 n = A->rows;
  if (k < 1 || k > n)
    invalid("sym_eig: order k out of range (k = " + std::to_string(k) + ", dim = " + std::to_string(n) + ")");
  if (!(tol > 0.0)) invalid("lanczos: tolerance must be positive");
  const i64 m_max = std::min<i64>(n, std::max<i64>(max_iter, k + 1));
  // sigma: Gershgorin bound (B = sigma I - A is PSD)
  const unsigned gb = static_cast<unsigned>(std::min<i64>(1024, (n + 255) / 256));
  DevBuf<double> gpart(c, gb);
  row_abs_max_k<<<gb, 256, 0, c->stream>>>(n, A->rp, A->v, gpart.p);
  launched(c);
  std::vector<double> gh(gb);
  CUDA_OK(cudaMemcpyAsync(gh.data(), gpart.p, sizeof(double) * gb, cudaMemcpyDeviceToHost, c->stream));
  sync(c);
  double sigma = 0.0;
  for (double x : gh) sigma = std::max(sigma, x);
  if (sigma == 0.0) {  // the zero matrix
    for (i64 q = 0; q < k; ++q) evals[q] = 0.0;
    if (iterations) *iterations = 0;
    return;
  }
  // Krylov basis (n x (m_max + 1)), start vector from the reference RNG
  DevBuf<double> V(c, static_cast<size_t>(n) * (m_max + 1)), w(c, n), h1(c, m_max + 1), h2(c, m_max + 1),
      al(c, m_max), be(c, m_max);
  {
    HostRng rng(HostRng::mix(seed ^ 0x1a2c705ULL));
    std::vector<double> v0(static_cast<size_t>(n));
    double nv = 0.0;
    for (auto& x : v0) {
      x = rng.gaussian();
      nv += x * x;
    }
    nv = std::sqrt(nv);
    for (auto& x : v0) x /= nv;
    CUDA_OK(cudaMemcpyAsync(V.p, v0.data(), sizeof(double) * n, cudaMemcpyHostToDevice, c->stream));
    sync(c);
  }
  cublasHandle_t h = blas_handle(c);
  const double one = 1.0, zero = 0.0, mone = -1.0;
  const unsigned sb = static_cast<unsigned>(std::min<i64>((n * 32 + 255) / 256, i64{1} << 30));
  const unsigned eb = stride_blocks(c, n);
  const i64 check = 20;
  std::vector<double> ah, bh, d, z;
  i64 j = 0;
  bool done = false;
  std::vector<double> theta;
  for (; j < m_max && !done; ++j) {
    const double* vj = V.p + static_cast<size_t>(j) * n;
    shifted_spmv_k<<<sb, 256, 0, c->stream>>>(n, A->rp, A->ci, A->v, sigma, vj, w.p);
    launched(c);
    const int cols = static_cast<int>(j + 1);
    const int nn = static_cast<int>(n);
    blas_ok(cublasSetPointerMode(h, CUBLAS_POINTER_MODE_HOST), "pointer mode");
    blas_ok(cublasDgemv(h, CUBLAS_OP_T, nn, cols, &one, V.p, nn, w.p, 1, &zero, h1.p, 1), "gemv");
    blas_ok(cublasDgemv(h, CUBLAS_OP_N, nn, cols, &mone, V.p, nn, h1.p, 1, &one, w.p, 1), "gemv");
    blas_ok(cublasDgemv(h, CUBLAS_OP_T, nn, cols, &one, V.p, nn, w.p, 1, &zero, h2.p, 1), "gemv");
    blas_ok(cublasDgemv(h, CUBLAS_OP_N, nn, cols, &mone, V.p, nn, h2.p, 1, &one, w.p, 1), "gemv");
    alpha_k<<<1, 1, 0, c->stream>>>(h1.p, h2.p, j, al.p);
    launched(c);
    blas_ok(cublasSetPointerMode(h, CUBLAS_POINTER_MODE_DEVICE), "pointer mode");
    blas_ok(cublasDnrm2(h, nn, w.p, 1, be.p + j), "nrm2");
    blas_ok(cublasSetPointerMode(h, CUBLAS_POINTER_MODE_HOST), "pointer mode");
    scale_k<<<eb, kBlock, 0, c->stream>>>(n, w.p, be.p + j, V.p + static_cast<size_t>(j + 1) * n);
    launched(c);
    const i64 steps = j + 1;
    if (steps % check == 0 || steps == m_max) {
      ah.resize(static_cast<size_t>(steps));
      bh.resize(static_cast<size_t>(steps));
      CUDA_OK(cudaMemcpyAsync(ah.data(), al.p, sizeof(double) * steps, cudaMemcpyDeviceToHost, c->stream));
      CUDA_OK(cudaMemcpyAsync(bh.data(), be.p, sizeof(double) * steps, cudaMemcpyDeviceToHost, c->stream));
      sync(c);
      d = ah;
      tql_lastrow(d, std::vector<double>(bh.begin(), bh.end() - 1), z);
      std::vector<i64> ord(static_cast<size_t>(steps));
      for (i64 q = 0; q < steps; ++q) ord[q] = q;
      std::sort(ord.begin(), ord.end(), [&](i64 a, i64 b) { return d[a] > d[b]; });
      const double bj = bh.back();
      const bool invariant = bj <= 1e-14 * sigma;
      bool conv = steps >= k;
      for (i64 q = 0; q < std::min(k, steps) && conv; ++q)
        conv = std::fabs(bj * z[ord[q]]) <= tol * sigma;
      if (steps == n) conv = true;  // the whole space: T_n is similar to B
      if (invariant || conv || steps == m_max) {
        if (steps < k) runtime("lanczos: Krylov space smaller than the requested order");
        if (!(conv || invariant)) runtime("lanczos: not converged after " + std::to_string(steps) + " steps");
        theta.resize(static_cast<size_t>(k));
        for (i64 q = 0; q < k; ++q) theta[q] = d[ord[q]];
        done = true;
      }
    }
  }
  if (!done) runtime("lanczos: not converged after " + std::to_string(j) + " steps");
  // eigenvalues of A, ascending (theta descending)
  for (i64 q = 0; q < k; ++q) evals[q] = sigma - theta[q];
  if (iterations) *iterations = j;
}

}  // namespace cpcag_cuda

using namespace cpcag_cuda;

extern "C" int cpcag_cuda_sym_eigvals_lanczos(cpcag_ctx ctx, cpcag_csr A, int64_t k, double tol, int64_t max_iter,
                                              uint64_t seed, double* eigenvalues, int64_t* iterations) {
  return guard([&] {
    Ctx* c = as_ctx(ctx);
    Csr* a = as_csr(A);
    if (!eigenvalues) invalid("null argument");
    std::vector<double> ev(static_cast<size_t>(std::max<int64_t>(k, 1)));
    i64 it = 0;
    sym_eigvals_lanczos(c, a, k, tol, max_iter, seed, ev.data(), &it);
    CUDA_OK(cudaMemcpy(eigenvalues, ev.data(), sizeof(double) * k, cudaMemcpyDefault));
    if (iterations) *iterations = it;
  });
}
