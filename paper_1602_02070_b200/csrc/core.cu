// core.cu -- context, device CSR operator, SpMM/SpMV, power iteration,
// sampling plan + gather, and the element-wise FRPCAG operators.
//
// Reference: proj/core/src/sparse.cpp (CSR, SpMV/SpMM), solvers.cpp:29-53
// (power iteration), sampling.cpp:35-75 (plan, subsample), frpcag.cpp:23-60
// (objective, prox, gradient).
#include <cooperative_groups.h>

#include <algorithm>
#include <chrono>
#include <mutex>
#include <cstdio>
#include <cstdlib>
#include <cub/cub.cuh>
#include <numeric>

#include "common.cuh"
#include "frpcag.cuh"

namespace cpcag_cuda {

static thread_local std::string g_last_error;
void set_last_error(const std::string& m) { g_last_error = m; }

bool is_device_ptr(const void* ptr) {
  if (!ptr) return false;
  cudaPointerAttributes a;
  cudaError_t e = cudaPointerGetAttributes(&a, ptr);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

double HostRng::gaussian() {
  if (has_spare) {
    has_spare = false;
    return spare;
  }
  double a = uniform();
  while (a <= 0.0) a = uniform();
  const double b = uniform();
  const double rad = std::sqrt(-2.0 * std::log(a));
  const double tau = 6.283185307179586476925286766559;
  spare = rad * std::sin(tau * b);
  has_spare = true;
  return rad * std::cos(tau * b);
}

void ensure_smem_impl(const void* func, size_t bytes) {
  static std::mutex mu;
  static std::vector<std::pair<const void*, size_t>> seen;
  std::lock_guard<std::mutex> lock(mu);
  for (auto& e : seen)
    if (e.first == func) {
      if (e.second >= bytes) return;
      CUDA_OK(cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(bytes)));
      e.second = bytes;
      return;
    }
  CUDA_OK(cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(bytes)));
  seen.push_back({func, bytes});
}

void run_idle_work(Ctx* c) {
  if (!c->idle_work) return;
  std::function<void()> work = std::move(c->idle_work);
  c->idle_work = nullptr;
  if (!c->aux) {
    CUDA_OK(cudaStreamCreateWithFlags(&c->aux, cudaStreamNonBlocking));
    CUDA_OK(cudaEventCreateWithFlags(&c->aux_ev, cudaEventDisableTiming));
  }
  cudaStream_t main_stream = c->stream;
  c->stream = c->aux;
  try {
    work();
  } catch (...) {
    c->stream = main_stream;
    throw;
  }
  c->stream = main_stream;
  CUDA_OK(cudaEventRecord(c->aux_ev, c->aux));
  CUDA_OK(cudaStreamWaitEvent(main_stream, c->aux_ev, 0));
}

void trace_mark(Ctx* c, const char* what) {
  static const bool on = std::getenv("CPCAG_TRACE") != nullptr;
  if (!on) return;
  static thread_local std::chrono::steady_clock::time_point last = std::chrono::steady_clock::now();
  cudaStreamSynchronize(c->stream);
  const auto now = std::chrono::steady_clock::now();
  std::fprintf(stderr, "[cpcag trace] %-28s %9.3f ms\n", what,
               std::chrono::duration<double, std::milli>(now - last).count());
  last = now;
}

// ------------------------------------------------------------------ kernel timing
static cudaEvent_t take_event(Ctx* c) {
  if (!c->kt.pool.empty()) {
    cudaEvent_t e = c->kt.pool.back();
    c->kt.pool.pop_back();
    return e;
  }
  cudaEvent_t e;
  CUDA_OK(cudaEventCreate(&e));
  return e;
}

KScope::KScope(Ctx* ctx, const char* t) : c(ctx), tag(t) {
  if (!c->timing) return;
  if (!c->timing_filter.empty()) {
    const std::string f = "," + c->timing_filter + ",";
    if (f.find("," + std::string(t) + ",") == std::string::npos) return;
  }
  a = take_event(c);
  b = take_event(c);
  cudaEventRecord(a, c->stream);
}

KScope::~KScope() {
  if (!a) return;
  cudaEventRecord(b, c->stream);
  c->kt.recs.push_back({tag, a, b});
}

static void harvest(Ctx* c) {
  if (c->kt.recs.empty()) return;
  CUDA_OK(cudaStreamSynchronize(c->stream));
  for (auto& r : c->kt.recs) {
    float ms = 0.f;
    cudaEventElapsedTime(&ms, r.a, r.b);
    bool found = false;
    for (auto& t : c->kt.totals)
      if (t.first == r.tag) {
        t.second.first += 1;
        t.second.second += ms;
        found = true;
        break;
      }
    if (!found) c->kt.totals.push_back({r.tag, {1, static_cast<double>(ms)}});
    c->kt.pool.push_back(r.a);
    c->kt.pool.push_back(r.b);
  }
  c->kt.recs.clear();
}

// ------------------------------------------------------------------ CSR
// CSR arrays live in the stream-ordered pool (cudaMallocAsync on the context
// stream): plain cudaMalloc/cudaFree map and unmap device memory on every
// graph built and dropped, which measured as 20-500 ms stalls inside the
// pipeline.  The destructor cannot know which stream last used the arrays,
// so it synchronises the device (what cudaFree would do) and returns them to
// the pool, where the next allocation reuses them without a remap.
// Exclusive prefix sum of n int64 values (out[0] = 0); returns the total
// in[0] + ... + in[n-1] (synchronises to read it).
i64 exclusive_scan_i64(Ctx* c, const i64* in, i64* out, i64 n) {
  if (n <= 0) return 0;
  size_t tmp = 0;
  CUDA_OK(cub::DeviceScan::ExclusiveSum(nullptr, tmp, in, out, static_cast<int>(n), c->stream));
  DevBuf<char> ws(c, std::max<size_t>(tmp, 1));
  CUDA_OK(cub::DeviceScan::ExclusiveSum(ws.p, tmp, in, out, static_cast<int>(n), c->stream));
  launched(c);
  i64 last_out = 0, last_in = 0;
  CUDA_OK(cudaMemcpyAsync(&last_out, out + n - 1, sizeof(i64), cudaMemcpyDeviceToHost, c->stream));
  CUDA_OK(cudaMemcpyAsync(&last_in, in + n - 1, sizeof(i64), cudaMemcpyDeviceToHost, c->stream));
  sync(c);
  return last_out + last_in;
}

void* csr_malloc(Ctx* c, size_t bytes) {
  void* p = nullptr;
  if (bytes) CUDA_OK(cudaMallocAsync(&p, bytes, c->stream));
  return p;
}

Csr::~Csr() {
  void* arrays[] = {rp, ci, v, v32, t_rp, t_ci, t_v, t_v32};
  bool any = false;
  for (void* p : arrays) any |= p != nullptr;
  if (!any) return;
  if (cudaDeviceSynchronize() != cudaSuccess) return;  // context gone (process exit)
  for (void* p : arrays)
    if (p) cudaFreeAsync(p, 0);
}

Csr* csr_alloc(Ctx* c, i64 rows, i64 cols, i64 nnz) {
  Csr* a = new Csr();
  a->rows = rows;
  a->cols = cols;
  a->nnz = nnz;
  a->device = c->device;
  try {
    a->rp = static_cast<i64*>(csr_malloc(c, sizeof(i64) * (rows + 1)));
    CUDA_OK(cudaMemsetAsync(a->rp, 0, sizeof(i64) * (rows + 1), c->stream));
    if (nnz) {
      a->ci = static_cast<int*>(csr_malloc(c, sizeof(int) * nnz));
      a->v = static_cast<double*>(csr_malloc(c, sizeof(double) * nnz));
    }
  } catch (...) {
    delete a;
    throw;
  }
  return a;
}

__global__ void to_f32_k(const double* __restrict__ a, float* __restrict__ b, i64 n) {
  for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < n; i += (i64)gridDim.x * blockDim.x)
    b[i] = static_cast<float>(a[i]);
}

template <>
const double* csr_values<double>(Ctx*, Csr* a) {
  return a->v;
}
template <>
const float* csr_values<float>(Ctx* c, Csr* a) {
  if (!a->v32 && a->nnz) {
    a->v32 = static_cast<float*>(csr_malloc(c, sizeof(float) * a->nnz));
    to_f32_k<<<stride_blocks(c, a->nnz), kBlock, 0, c->stream>>>(a->v, a->v32, a->nnz);
    launched(c);
  }
  return a->v32;
}

// Exact symmetry: every (r, c, v) has (c, r, v) with the same bits.
__global__ void sym_check_k(i64 rows, const i64* __restrict__ rp, const int* __restrict__ ci,
                            const double* __restrict__ v, int* asym) {
  const i64 r = blockIdx.x * (i64)blockDim.x + threadIdx.x;
  if (r >= rows) return;
  for (i64 k = rp[r]; k < rp[r + 1]; ++k) {
    const int c = ci[k];
    i64 lo = rp[c], hi = rp[c + 1];
    while (lo < hi) {
      const i64 mid = (lo + hi) >> 1;
      if (ci[mid] < r) lo = mid + 1; else hi = mid;
    }
    if (lo == rp[c + 1] || ci[lo] != r ||
        __double_as_longlong(v[lo]) != __double_as_longlong(v[k])) {
      *asym = 1;
      return;
    }
  }
}

int csr_symmetric(Ctx* c, Csr* a) {
  if (a->sym >= 0) return a->sym;
  if (a->rows != a->cols) return a->sym = 0;
  DevBuf<int> flag(c, 1);
  flag.zero(c);
  if (a->rows) {
    sym_check_k<<<blocks_for(a->rows), kBlock, 0, c->stream>>>(a->rows, a->rp, a->ci, a->v, flag.p);
    launched(c);
  }
  const int asym = read_back(c, flag.p);
  return a->sym = asym ? 0 : 1;
}

__global__ void expand_rows_k(i64 rows, const i64* __restrict__ rp, int* __restrict__ row_of) {
  const i64 r = blockIdx.x * (i64)blockDim.x + threadIdx.x;
  if (r >= rows) return;
  for (i64 k = rp[r]; k < rp[r + 1]; ++k) row_of[k] = static_cast<int>(r);
}

__global__ void gather_perm_k(i64 nnz, const int* __restrict__ perm, const int* __restrict__ row_of,
                              const double* __restrict__ v, int* __restrict__ t_ci,
                              double* __restrict__ t_v) {
  const i64 k = blockIdx.x * (i64)blockDim.x + threadIdx.x;
  if (k >= nnz) return;
  const int src = perm[k];
  t_ci[k] = row_of[src];
  t_v[k] = v[src];
}

__global__ void count_cols_k(i64 nnz, const int* __restrict__ sorted_cols, i64 cols, i64* t_rp) {
  // t_rp[c+1] = number of entries with column <= c, via upper bounds on the
  // sorted column list (one thread per column).
  const i64 c = blockIdx.x * (i64)blockDim.x + threadIdx.x;
  if (c > cols) return;
  if (c == 0) {
    t_rp[0] = 0;
    return;
  }
  i64 lo = 0, hi = nnz;
  const int key = static_cast<int>(c - 1);
  while (lo < hi) {
    const i64 mid = (lo + hi) >> 1;
    if (sorted_cols[mid] <= key) lo = mid + 1; else hi = mid;
  }
  t_rp[c] = lo;
}

__global__ void iota_k(i64 n, int* out) {
  const i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x;
  if (i < n) out[i] = static_cast<int>(i);
}

// A^T as CSR (stable radix sort of entries by column keeps rows ascending
// within each column: the order sparse.cpp:100-111 accumulates in).
void csr_build_transpose(Ctx* c, Csr* a) {
  if (a->t_rp) return;
  const i64 nnz = a->nnz;
  a->t_rp = static_cast<i64*>(csr_malloc(c, sizeof(i64) * (a->cols + 1)));
  if (nnz == 0) {
    CUDA_OK(cudaMemsetAsync(a->t_rp, 0, sizeof(i64) * (a->cols + 1), c->stream));
    return;
  }
  a->t_ci = static_cast<int*>(csr_malloc(c, sizeof(int) * nnz));
  a->t_v = static_cast<double*>(csr_malloc(c, sizeof(double) * nnz));
  DevBuf<int> keys_out(c, nnz), idx(c, nnz), idx_out(c, nnz), row_of(c, nnz);
  iota_k<<<blocks_for(nnz), kBlock, 0, c->stream>>>(nnz, idx.p);
  launched(c);
  expand_rows_k<<<blocks_for(a->rows), kBlock, 0, c->stream>>>(a->rows, a->rp, row_of.p);
  launched(c);
  size_t tmp = 0;
  CUDA_OK(cub::DeviceRadixSort::SortPairs(nullptr, tmp, a->ci, keys_out.p, idx.p, idx_out.p,
                                          static_cast<int>(nnz), 0, 32, c->stream));
  DevBuf<char> ws(c, tmp);
  CUDA_OK(cub::DeviceRadixSort::SortPairs(ws.p, tmp, a->ci, keys_out.p, idx.p, idx_out.p,
                                          static_cast<int>(nnz), 0, 32, c->stream));
  launched(c);
  gather_perm_k<<<blocks_for(nnz), kBlock, 0, c->stream>>>(nnz, idx_out.p, row_of.p, a->v,
                                                           a->t_ci, a->t_v);
  launched(c);
  count_cols_k<<<blocks_for(a->cols + 1), kBlock, 0, c->stream>>>(nnz, keys_out.p, a->cols, a->t_rp);
  launched(c);
}

template <>
const double* csr_t_values<double>(Ctx* c, Csr* a) {
  csr_build_transpose(c, a);
  return a->t_v;
}
template <>
const float* csr_t_values<float>(Ctx* c, Csr* a) {
  csr_build_transpose(c, a);
  if (!a->t_v32 && a->nnz) {
    a->t_v32 = static_cast<float*>(csr_malloc(c, sizeof(float) * a->nnz));
    to_f32_k<<<stride_blocks(c, a->nnz), kBlock, 0, c->stream>>>(a->t_v, a->t_v32, a->nnz);
    launched(c);
  }
  return a->t_v32;
}

// Column-pull view of A for X*A: A itself when exactly symmetric, else A^T.
template <typename T>
struct PullView {
  const i64* rp;
  const int* ci;
  const T* v;
};
template <typename T>
PullView<T> pull_view(Ctx* c, Csr* a) {
  if (csr_symmetric(c, a)) return {a->rp, a->ci, csr_values<T>(c, a)};
  const T* tv = csr_t_values<T>(c, a);
  return {a->t_rp, a->t_ci, tv};
}

// ------------------------------------------------------------------ SpMM
// Y(r, j) = sum_k v_k X(c_k, j), CSR order, explicit mul then add
// (sparse.cpp:87-98).  Threads run down a column of Y (coalesced stores).
template <typename T>
__global__ void spmm_left_k(i64 rows, i64 m, const i64* __restrict__ rp, const int* __restrict__ ci,
                            const T* __restrict__ v, const T* __restrict__ X, i64 ldx,
                            T* __restrict__ Y) {
  const i64 r = blockIdx.x * (i64)blockDim.x + threadIdx.x;
  if (r >= rows) return;
  const i64 k0 = rp[r], k1 = rp[r + 1];
  for (i64 j = blockIdx.y; j < m; j += gridDim.y) {
    Y[r + j * rows] = pull_left(k0, k1, ci, v, X + j * ldx);
  }
}

// Y(i, c) = sum over rows r of A holding column c (ascending) of A(r,c) X(i,r)
// (sparse.cpp:100-111), pulled over row c of A^T.
template <typename T>
__global__ void spmm_right_k(i64 xr, i64 cols, const i64* __restrict__ rp, const int* __restrict__ ci,
                             const T* __restrict__ v, const T* __restrict__ X, T* __restrict__ Y) {
  const i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x;
  if (i >= xr) return;
  for (i64 c = blockIdx.y; c < cols; c += gridDim.y) {
    Y[i + c * xr] = pull_right(rp[c], rp[c + 1], ci, v, X, xr, i);
  }
}

template <typename T>
void spmm_left(Ctx* c, Csr* A, const T* X, i64 m, T* Y) {
  if (A->rows == 0 || m == 0) return;
  dim3 g(blocks_for(A->rows), static_cast<unsigned>(std::min<i64>(m, 65535)));
  spmm_left_k<T><<<g, kBlock, 0, c->stream>>>(A->rows, m, A->rp, A->ci, csr_values<T>(c, A), X,
                                              A->cols, Y);
  launched(c);
}

template <typename T>
void spmm_right(Ctx* c, Csr* A, const T* X, i64 m, T* Y) {
  if (A->cols == 0 || m == 0) return;
  const PullView<T> pv = pull_view<T>(c, A);
  dim3 g(blocks_for(m), static_cast<unsigned>(std::min<i64>(A->cols, 65535)));
  spmm_right_k<T><<<g, kBlock, 0, c->stream>>>(m, A->cols, pv.rp, pv.ci, pv.v, X, Y);
  launched(c);
}

template void spmm_left<double>(Ctx*, Csr*, const double*, i64, double*);
template void spmm_left<float>(Ctx*, Csr*, const float*, i64, float*);
template void spmm_right<double>(Ctx*, Csr*, const double*, i64, double*);
template void spmm_right<float>(Ctx*, Csr*, const float*, i64, float*);

// ------------------------------------------------------------------ dots
template <typename T>
__global__ void dot_k(const T* __restrict__ a, const T* __restrict__ b, i64 n, double* partials,
                      unsigned* counter, double* out) {
  double s[1] = {0.0};
  for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < n; i += (i64)gridDim.x * blockDim.x)
    s[0] += static_cast<double>(a[i]) * static_cast<double>(b[i]);
  double t[1];
  if (grid_sum_last<1>(s, partials, counter, t) && threadIdx.x == 0) *out = t[0];
}

template <typename T>
void dot_device(Ctx* c, const T* a, const T* b, i64 n, double* out_dev) {
  const unsigned nb = stride_blocks(c, n);
  DevBuf<double> part(c, nb);
  DevBuf<unsigned> cnt(c, 1);
  cnt.zero(c);
  dot_k<T><<<nb, kBlock, 0, c->stream>>>(a, b, n, part.p, cnt.p, out_dev);
  launched(c);
}
template void dot_device<double>(Ctx*, const double*, const double*, i64, double*);
template void dot_device<float>(Ctx*, const float*, const float*, i64, double*);

// ------------------------------------------------------------------ power iteration
// solvers.cpp:29-53: w = A v, est = ||w||, v = w / est, stop when
// |est - prev| <= tol est.  v0 comes from the reference RNG on the host
// (bit-identical).  The SpMV is warp-per-row (lanes stride the row, fixed
// shuffle tree), so rows of the near-dense Kron-reduced Laplacians (~600
// nnz/row at config 1) read coalesced.
struct PowerState {
  double est;
  i64 iterations;
  unsigned bar_count, bar_gen;
};

__device__ __forceinline__ double warp_row_dot(i64 k0, i64 k1, const int* __restrict__ ci,
                                               const double* __restrict__ val, const double* x, int lane) {
  double acc = 0.0;
  for (i64 k = k0 + lane; k < k1; k += 32) acc += val[k] * x[ci[k]];
  return warp_sum(acc);
}

// Small operators: the whole iteration in one CTA, v and w in shared memory
// (and the CSR rows too when they fit: no grid barrier, no L2 round trip).
__global__ void __launch_bounds__(512) power_iter_small_k(i64 n, const i64* __restrict__ rp,
                                                           const int* __restrict__ ci,
                                                           const double* __restrict__ val,
                                                           const double* __restrict__ v0, double tol,
                                                           i64 max_iter, int mat_in_smem, PowerState* st) {
  extern __shared__ double sm[];
  double* vs = sm;
  double* ws = sm + n;
  const i64 nnz = rp[n];
  double* sval = ws + n;
  i64* srp = reinterpret_cast<i64*>(sval + (mat_in_smem ? nnz : 0));
  int* sci = reinterpret_cast<int*>(srp + (mat_in_smem ? n + 1 : 0));
  if (mat_in_smem) {
    for (i64 k = threadIdx.x; k < nnz; k += blockDim.x) {
      sval[k] = val[k];
      sci[k] = ci[k];
    }
    for (i64 i = threadIdx.x; i <= n; i += blockDim.x) srp[i] = rp[i];
  }
  const i64* RP = mat_in_smem ? srp : rp;
  const int* CI = mat_in_smem ? sci : ci;
  const double* VA = mat_in_smem ? sval : val;
  __shared__ double warp_part[32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (i64 i = threadIdx.x; i < n; i += blockDim.x) vs[i] = v0[i];
  __syncthreads();
  double est = 0.0;
  i64 it = 0;
  for (; it < max_iter; ++it) {
    double part = 0.0;
    for (i64 r = wid; r < n; r += nw) {
      const double acc = warp_row_dot(RP[r], RP[r + 1], CI, VA, vs, lane);
      if (lane == 0) {
        ws[r] = acc;
        part += acc * acc;
      }
    }
    if (lane == 0) warp_part[wid] = part;
    __syncthreads();
    double tot = lane < nw ? warp_part[lane] : 0.0;
    tot = warp_sum(tot);  // every warp computes the same total
    const double nrm = sqrt(tot);
    if (nrm == 0.0) {
      est = 0.0;
      break;
    }
    const double prev = est;
    est = nrm;
    for (i64 i = threadIdx.x; i < n; i += blockDim.x) vs[i] = __ddiv_rn(ws[i], nrm);
    __syncthreads();
    if (it > 0 && fabs(est - prev) <= tol * est) {
      ++it;
      break;
    }
  }
  if (threadIdx.x == 0) {
    st->est = est;
    st->iterations = it;
  }
}

// Large operators: cooperative grid, one CTA per SM, each CTA owning a
// contiguous slice of rows whose CSR entries stay resident in its shared
// memory for the whole iteration (when they fit), a private shared-memory copy
// of v, and ONE grid barrier per iteration: every CTA publishes its slice of
// w (double-buffered by iteration parity), then every CTA reads all of w,
// forms ||w||^2 in the same fixed order and renormalises the whole of v into
// its own shared copy (`partials` is unused).
__global__ void __launch_bounds__(512) power_iter_coop_k(i64 n, const i64* __restrict__ rp,
                                                         const int* __restrict__ ci,
                                                         const double* __restrict__ val,
                                                         double* v0, double* wbuf,
                                                         double* partials, double tol, i64 max_iter,
                                                         int slice_in_smem, int v_in_smem, PowerState* st) {
  // v0 is rewritten in place between grid barriers when it does not fit in
  // shared memory: plain (coherent) loads only, never the read-only path.
  extern __shared__ double sm[];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const unsigned nb = gridDim.x;
  const i64 r0 = (n * blockIdx.x) / nb, r1 = (n * (blockIdx.x + 1)) / nb;
  const i64 k0 = rp[r0], k1 = rp[r1];
  double* vs = sm;                                   // n doubles (if v_in_smem)
  double* sval = sm + (v_in_smem ? n : 0);           // slice values
  int* sci = reinterpret_cast<int*>(sval + (slice_in_smem ? (k1 - k0) : 0));
  if (slice_in_smem)
    for (i64 k = k0 + threadIdx.x; k < k1; k += blockDim.x) {
      sval[k - k0] = val[k];
      sci[k - k0] = ci[k];
    }
  if (v_in_smem)
    for (i64 i = threadIdx.x; i < n; i += blockDim.x) vs[i] = v0[i];
  __syncthreads();
  const double* vsrc = v_in_smem ? vs : v0;
  double est = 0.0;
  i64 it = 0;
  unsigned bar_g = 0;  // barriers passed (PowerState is zeroed before the launch)
  for (; it < max_iter; ++it) {
    double* w = wbuf + (it & 1) * n;
    for (i64 r = r0 + wid; r < r1; r += nw) {
      double acc = 0.0;
      if (slice_in_smem) {
        for (i64 k = rp[r] + lane; k < rp[r + 1]; k += 32) acc += sval[k - k0] * vsrc[sci[k - k0]];
      } else {
        for (i64 k = rp[r] + lane; k < rp[r + 1]; k += 32) acc += val[k] * vsrc[ci[k]];
      }
      acc = warp_sum(acc);
      if (lane == 0) w[r] = acc;
    }
    grid_barrier_mono(&st->bar_count, bar_g);
    // ||w||^2 straight from w, which every CTA reads anyway: one L2 round
    // trip per iteration instead of two (partials, then w).  Same data and
    // the same fixed-order block reduction in every CTA, so every CTA gets
    // the same norm and takes the same stop decision.
    double t[1] = {0.0};
    for (i64 i = threadIdx.x; i < n; i += blockDim.x) {
      const double x = __ldcg(w + i);
      if (v_in_smem) vs[i] = x;
      t[0] += x * x;
    }
    block_sum<1>(t);
    const double nrm = sqrt(t[0]);
    if (nrm == 0.0) {
      est = 0.0;
      break;
    }
    const double prev = est;
    est = nrm;
    if (v_in_smem) {
      for (i64 i = threadIdx.x; i < n; i += blockDim.x) vs[i] = __ddiv_rn(vs[i], nrm);
      __syncthreads();
    } else {
      // v lives in global memory: the grid renormalises its own rows and
      // needs a second barrier before the next product reads them.
      double* vg = v0;
      for (i64 i = r0 + threadIdx.x; i < r1; i += blockDim.x) vg[i] = __ddiv_rn(__ldcg(w + i), nrm);
    }
    if (it > 0 && fabs(est - prev) <= tol * est) {
      ++it;
      break;
    }
    if (!v_in_smem) grid_barrier_mono(&st->bar_count, bar_g);
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    st->est = est;
    st->iterations = it;
  }
}

// K products per grid barrier for operators whose powers fit beside them:
// with A2 = A A (and A3 = A2 A), dense and built once, one round forms
// w_m = A^m v, m = 1..K, from the same v.  ||w_1|| is the reference's estimate
// of this iteration; the next iterate would be v' = w_1 / ||w_1||, so
// A v' = w_2 / ||w_1|| and the next estimate is ||w_2|| / ||w_1||, the one
// after it ||w_3|| / ||w_2||, and the iterate after the round w_K / ||w_K||
// (solvers.cpp:43-51 K times, every stop test in order).  The barrier and the
// L2 round trip of w are paid once per K reference iterations; estimates
// agree with the one-product form to rounding (~1e-15 relative).
template <int K>
__global__ void __launch_bounds__(K == 3 ? 768 : 512) power_iter_coopk_k(i64 n, const i64* __restrict__ rp,
                                                          const int* __restrict__ ci,
                                                          const double* __restrict__ val,
                                                          const double* __restrict__ A2,
                                                          const double* __restrict__ A3, i64 ld,
                                                          const double* __restrict__ v0, double* wbuf, double tol,
                                                          i64 max_iter, PowerState* st) {
  extern __shared__ double sm[];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const unsigned nb = gridDim.x;
  const i64 r0 = (n * blockIdx.x) / nb, r1 = (n * (blockIdx.x + 1)) / nb;
  const int nr = static_cast<int>(r1 - r0);
  const i64 k0 = rp[r0], k1 = rp[r1];
  double* vs = sm;                     // n
  double* pws = vs + n;                // (K - 1) x nr x n: the CTA's rows of A2 (, A3)
  double* sval = pws + static_cast<i64>(K - 1) * nr * n;
  int* sci = reinterpret_cast<int*>(sval + (k1 - k0));
  for (i64 k = k0 + threadIdx.x; k < k1; k += blockDim.x) {
    sval[k - k0] = val[k];
    sci[k - k0] = ci[k];
  }
  for (i64 q = threadIdx.x; q < static_cast<i64>(nr) * n; q += blockDim.x) {
    const i64 r = q / n, j = q - r * n;
    pws[q] = A2[(r0 + r) * ld + j];
    if constexpr (K == 3) pws[static_cast<i64>(nr) * n + q] = A3[(r0 + r) * ld + j];
  }
  for (i64 i = threadIdx.x; i < n; i += blockDim.x) vs[i] = v0[i];
  __syncthreads();
  double est = 0.0;
  i64 it = 0;
  unsigned bar_g = 0, round = 0;
  while (it < max_iter) {
    double* w = wbuf + (round & 1) * K * n;  // w_1 | w_2 (| w_3)
    ++round;
    for (int task = wid; task < K * nr; task += nw) {
      double a0 = 0.0, a1 = 0.0;
      if (task < nr) {
        const i64 ra = rp[r0 + task] - k0, rb = rp[r0 + task + 1] - k0;
        i64 k = ra + lane;
        for (; k + 32 < rb; k += 64) {
          a0 += sval[k] * vs[sci[k]];
          a1 += sval[k + 32] * vs[sci[k + 32]];
        }
        if (k < rb) a0 += sval[k] * vs[sci[k]];
        a0 = warp_sum(a0 + a1);
        if (lane == 0) w[r0 + task] = a0;
      } else {
        const int m = task / nr, rr = task - m * nr;  // power m + 1, row rr
        const double* row = pws + (static_cast<i64>(m - 1) * nr + rr) * n;
        i64 j = lane;
        for (; j + 32 < n; j += 64) {
          a0 += row[j] * vs[j];
          a1 += row[j + 32] * vs[j + 32];
        }
        if (j < n) a0 += row[j] * vs[j];
        a0 = warp_sum(a0 + a1);
        if (lane == 0) w[m * n + r0 + rr] = a0;
      }
    }
    grid_barrier_mono(&st->bar_count, bar_g);
    // every CTA reads all of w and reduces the K norms in the same fixed order
    double t[K];
#pragma unroll
    for (int m = 0; m < K; ++m) t[m] = 0.0;
#pragma unroll 4
    for (i64 i = threadIdx.x; i < n; i += blockDim.x) {
      double x[K];
#pragma unroll
      for (int m = 0; m < K; ++m) x[m] = __ldcg(w + m * n + i);
      vs[i] = x[K - 1];
#pragma unroll
      for (int m = 0; m < K; ++m) t[m] += x[m] * x[m];
    }
    block_sum<K>(t);
    bool stop = false;
    double nprev = 1.0, nlast = 1.0;
#pragma unroll
    for (int m = 0; m < K; ++m) {
      const double nm = sqrt(t[m]);
      if (nm == 0.0) {  // A v = 0 for the current iterate: the reference returns 0
        est = 0.0;
        if (m > 0) ++it;
        stop = true;
        break;
      }
      const double prev = est;
      est = m == 0 ? nm : __ddiv_rn(nm, nprev);
      ++it;
      nprev = nm;
      nlast = nm;
      if ((it > 1 && fabs(est - prev) <= tol * est) || it >= max_iter) {
        stop = true;
        break;
      }
    }
    if (stop) break;
    for (i64 i = threadIdx.x; i < n; i += blockDim.x) vs[i] = __ddiv_rn(vs[i], nlast);
    __syncthreads();
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    st->est = est;
    st->iterations = it;
  }
}

// Dense copy of a CSR matrix into a zeroed ld x ld row-major array.
__global__ void csr_to_dense_k(i64 n, const i64* __restrict__ rp, const int* __restrict__ ci,
                               const double* __restrict__ val, i64 ld, double* __restrict__ D) {
  const int lane = threadIdx.x & 31;
  const i64 r = (blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x) >> 5;
  if (r >= n) return;
  for (i64 k = rp[r] + lane; k < rp[r + 1]; k += 32) D[r * ld + ci[k]] = val[k];
}

// C = A B for dense row-major ld x ld arrays (ld a multiple of 64, zero
// padded): 64 x 64 tile per CTA, 4 x 4 per thread, k ascending (each entry of
// C is one fixed-order fp64 FMA chain).
__global__ void __launch_bounds__(256) dense_mm_k(int ld, const double* __restrict__ A, const double* __restrict__ B,
                                                  double* __restrict__ C) {
  __shared__ double As[16][64 + 4];
  __shared__ __align__(16) double Bs[16][64];
  const int t = threadIdx.x, ty = t >> 4, tx = t & 15;
  const int i0 = blockIdx.y * 64, j0 = blockIdx.x * 64;
  double acc[4][4];
#pragma unroll
  for (int u = 0; u < 4; ++u)
#pragma unroll
    for (int w = 0; w < 4; ++w) acc[u][w] = 0.0;
  const int ai = t >> 2, ak = (t & 3) * 4;   // A tile: 64 rows x 16 k
  const int bk = t >> 4, bj = (t & 15) * 4;  // B tile: 16 k x 64 columns
  for (int kk = 0; kk < ld; kk += 16) {
    const double2 x0 = *reinterpret_cast<const double2*>(A + static_cast<i64>(i0 + ai) * ld + kk + ak);
    const double2 x1 = *reinterpret_cast<const double2*>(A + static_cast<i64>(i0 + ai) * ld + kk + ak + 2);
    const double2 y0 = *reinterpret_cast<const double2*>(B + static_cast<i64>(kk + bk) * ld + j0 + bj);
    const double2 y1 = *reinterpret_cast<const double2*>(B + static_cast<i64>(kk + bk) * ld + j0 + bj + 2);
    __syncthreads();
    As[ak][ai] = x0.x;
    As[ak + 1][ai] = x0.y;
    As[ak + 2][ai] = x1.x;
    As[ak + 3][ai] = x1.y;
    *reinterpret_cast<double2*>(&Bs[bk][bj]) = y0;
    *reinterpret_cast<double2*>(&Bs[bk][bj + 2]) = y1;
    __syncthreads();
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      double a[4], b[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) a[u] = As[k][ty * 4 + u];
      const double2 b0 = *reinterpret_cast<const double2*>(&Bs[k][tx * 4]);
      const double2 b1 = *reinterpret_cast<const double2*>(&Bs[k][tx * 4 + 2]);
      b[0] = b0.x, b[1] = b0.y, b[2] = b1.x, b[3] = b1.y;
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int w = 0; w < 4; ++w) acc[u][w] = fma(a[u], b[w], acc[u][w]);
    }
  }
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    double* out = C + static_cast<i64>(i0 + ty * 4 + u) * ld + j0 + tx * 4;
    *reinterpret_cast<double2*>(out) = make_double2(acc[u][0], acc[u][1]);
    *reinterpret_cast<double2*>(out + 2) = make_double2(acc[u][2], acc[u][3]);
  }
}

// One power iteration, set up and launched on `s` (the host work -- start
// vector, geometry -- happens now; the result lands in st->est).  Returns
// false when there is nothing to launch (st->est is then set on the host:
// n == 0, ||v0|| == 0 or max_iter <= 0 give 0).
struct PowerJob {
  DevBuf<double> v, w, part, dense, sq, cube;
  DevBuf<PowerState> st;
  double host_est = 0.0;
  bool launched = false;
  bool small = false;
};

static void power_prepare(Ctx* c, Csr* A, double tol, uint64_t seed, i64 max_iter, PowerJob& job, cudaStream_t s,
                          bool timed) {
  if (A->rows != A->cols) invalid("power iteration: square matrix required");
  const i64 n = A->rows;
  c->last_power_path = 0;
  if (n == 0) return;
  HostRng rng(HostRng::mix(seed ^ 0x5ca1ab1eULL));
  std::vector<double> v0(static_cast<size_t>(n));
  for (i64 i = 0; i < n; ++i) v0[i] = rng.gaussian();
  double nv = 0.0;
  for (i64 i = 0; i < n; ++i) nv += v0[i] * v0[i];
  nv = std::sqrt(nv);
  if (nv == 0.0) return;
  for (double& x : v0) x /= nv;
  if (max_iter <= 0) return;
  job.v.alloc(c, n);
  job.st.alloc(c, 1);
  job.st.zero(c);
  CUDA_OK(cudaMemcpyAsync(job.v.p, v0.data(), sizeof(double) * n, cudaMemcpyHostToDevice, c->stream));
  // one CTA when v, w and the CSR rows fit its shared memory (no grid barrier)
  const size_t small_smem = 2 * sizeof(double) * static_cast<size_t>(n);
  const size_t mat_smem = static_cast<size_t>(A->nnz) * 12 + static_cast<size_t>(n + 1) * 8 + 16;
  if (small_smem + mat_smem <= 200 * 1024 || (small_smem <= 200 * 1024 && A->nnz <= 4096)) {
    const int in_smem = small_smem + mat_smem <= 200 * 1024 ? 1 : 0;
    const size_t smem = small_smem + (in_smem ? mat_smem : 0);
    ensure_smem(power_iter_small_k, smem);
    job.small = true;
    job.launched = true;
    if (s != c->stream) {  // the side stream starts after this job's inputs
      CUDA_OK(cudaEventRecord(c->fork_ev, c->stream));
      CUDA_OK(cudaStreamWaitEvent(s, c->fork_ev, 0));
    }
    if (timed) {
      KScope ks_(c, "power_iter");
      power_iter_small_k<<<1, 512, smem, s>>>(n, A->rp, A->ci, A->v, job.v.p, tol, max_iter, in_smem, job.st.p);
    } else {
      power_iter_small_k<<<1, 512, smem, s>>>(n, A->rp, A->ci, A->v, job.v.p, tol, max_iter, in_smem, job.st.p);
    }
    launched(c);
    return;
  }
  // One CTA per SM (at most one per row): measured, the per-iteration cost is
  // the in-CTA product, so spreading it wins over the cheaper barrier of a
  // smaller grid (cfg1: 148 CTAs 7.4 ms, 40 CTAs 9.5 ms, 8 CTAs 31 ms).
  const i64 want = c->num_sms;
  const unsigned nb = static_cast<unsigned>(std::max<i64>(1, std::min<i64>({static_cast<i64>(c->num_sms), want, n})));
  std::vector<i64> rph(static_cast<size_t>(n) + 1);
  CUDA_OK(cudaMemcpyAsync(rph.data(), A->rp, sizeof(i64) * (n + 1), cudaMemcpyDeviceToHost, c->stream));
  sync(c);
  i64 max_slice = 0;
  for (unsigned b = 0; b < nb; ++b) {
    const i64 r0 = (n * b) / nb, r1 = (n * (b + 1)) / nb;
    max_slice = std::max(max_slice, rph[r1] - rph[r0]);
  }
  const size_t budget = 200 * 1024;
  int v_in_smem = static_cast<size_t>(n) * 8 <= budget / 2 ? 1 : 0;
  size_t smem = v_in_smem ? static_cast<size_t>(n) * 8 : 0;
  int slice_in_smem = smem + static_cast<size_t>(max_slice) * 12 + 16 <= budget ? 1 : 0;
  if (slice_in_smem) smem += static_cast<size_t>(max_slice) * 12 + 16;
  // K = 3 or 2 products per barrier when the CTA's rows of A^2 (and A^3) fit beside its slice
  if (s == c->stream && v_in_smem && slice_in_smem && c->power_path != 1) {
    const i64 rows_max = (n + nb - 1) / nb;
    const i64 ld = ((n + 63) / 64) * 64;
    auto smem_k = [&](int K) {
      return static_cast<size_t>(n) * 8 + static_cast<size_t>(K - 1) * rows_max * n * 8 +
             static_cast<size_t>(max_slice) * 12 + 16;
    };
    int K = 0;
    if (ld * ld * 8 <= (i64{64} << 20)) {
      if (smem_k(3) <= budget && max_iter >= 3 && c->power_path != 2) K = 3;
      else if (smem_k(2) <= budget && max_iter >= 2) K = 2;
    }
    if (K) {
      const size_t smemk = smem_k(K);
      job.dense.alloc(c, static_cast<size_t>(ld * ld));
      job.sq.alloc(c, static_cast<size_t>(ld * ld));
      if (K == 3) job.cube.alloc(c, static_cast<size_t>(ld * ld));
      job.dense.zero(c);
      job.w.alloc(c, 2 * K * n);
      void* kern = K == 3 ? (void*)power_iter_coopk_k<3> : (void*)power_iter_coopk_k<2>;
      ensure_smem_impl(kern, smemk);
      int fit = 0;
      const int threads = K == 3 ? 768 : 512;  // one warp per row task (K x ~7 rows at config 1)
      if (K == 3)
        CUDA_OK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&fit, power_iter_coopk_k<3>, threads, smemk));
      else
        CUDA_OK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&fit, power_iter_coopk_k<2>, threads, smemk));
      if (fit < 1) invalid("power iteration: kernel does not fit on an SM");
      const i64* rp = A->rp;
      const int* ci = A->ci;
      const double* val = A->v;
      const double* a2 = job.sq.p;
      const double* a3 = job.cube.p;
      const double* vp = job.v.p;
      double* wp = job.w.p;
      PowerState* sp = job.st.p;
      i64 nn = n, ldd = ld;
      void* args[] = {(void*)&nn, (void*)&rp, (void*)&ci, (void*)&val, (void*)&a2, (void*)&a3, (void*)&ldd,
                      (void*)&vp, (void*)&wp, (void*)&tol, (void*)&max_iter, (void*)&sp};
      job.launched = true;
      auto go = [&] {
        csr_to_dense_k<<<blocks_for(n * 32), kBlock, 0, s>>>(n, rp, ci, val, ld, job.dense.p);
        const unsigned gt = static_cast<unsigned>(ld / 64);
        dense_mm_k<<<dim3(gt, gt), 256, 0, s>>>(static_cast<int>(ld), job.dense.p, job.dense.p, job.sq.p);
        if (K == 3) dense_mm_k<<<dim3(gt, gt), 256, 0, s>>>(static_cast<int>(ld), job.sq.p, job.dense.p, job.cube.p);
        CUDA_OK(cudaLaunchCooperativeKernel(kern, dim3(nb), dim3(threads), args, smemk, s));
      };
      if (timed) {
        KScope ks_(c, "power_iter");
        go();
      } else {
        go();
      }
      launched(c);
      c->last_power_path = K;
      return;
    }
  }
  c->last_power_path = 1;
  ensure_smem(power_iter_coop_k, smem);
  int per_sm = 0;
  CUDA_OK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, power_iter_coop_k, 512, smem));
  if (per_sm < 1) invalid("power iteration: kernel does not fit on an SM");
  job.part.alloc(c, 2 * nb);
  job.w.alloc(c, 2 * n);
  const i64* rp = A->rp;
  const int* ci = A->ci;
  const double* val = A->v;
  const double* vp = job.v.p;
  double* wp = job.w.p;
  double* pp = job.part.p;
  PowerState* sp = job.st.p;
  i64 nn = n;
  void* args[] = {(void*)&nn, (void*)&rp, (void*)&ci, (void*)&val, (void*)&vp, (void*)&wp, (void*)&pp,
                  (void*)&tol, (void*)&max_iter, (void*)&slice_in_smem, (void*)&v_in_smem, (void*)&sp};
  job.launched = true;
  if (timed) {
    KScope ks_(c, "power_iter");
    CUDA_OK(cudaLaunchCooperativeKernel((void*)power_iter_coop_k, dim3(nb), dim3(512), args, smem, s));
  } else {
    CUDA_OK(cudaLaunchCooperativeKernel((void*)power_iter_coop_k, dim3(nb), dim3(512), args, smem, s));
  }
  launched(c);
}

static double power_result(Ctx* c, PowerJob& job) {
  return job.launched ? read_back(c, job.st.p).est : job.host_est;
}

double power_norm(Ctx* c, Csr* A, double tol, uint64_t seed, i64 max_iter) {
  PowerJob job;
  power_prepare(c, A, tol, seed, max_iter, job, c->stream, true);
  return power_result(c, job);
}

// Both FISTA norms (frpcag.cpp:72-73).  When one operator takes the
// single-CTA kernel and the other the cooperative grid, the single CTA runs
// on a side stream beside the grid (it fits next to a grid CTA on one SM).
void power_norm_pair(Ctx* c, Csr* A1, Csr* A2, double tol, uint64_t seed, i64 max_iter, double* out1,
                     double* out2) {
  PowerJob j1, j2;
  cudaStream_t side = side_stream(c);
  const bool small1 = A1->rows == A1->cols &&
                      2 * 8 * static_cast<size_t>(A1->rows) + static_cast<size_t>(A1->nnz) * 12 +
                              static_cast<size_t>(A1->rows + 1) * 8 + 16 <= 200 * 1024;
  power_prepare(c, A1, tol, seed, max_iter, j1, small1 ? side : c->stream, !small1);
  power_prepare(c, A2, tol, seed, max_iter, j2, c->stream, true);
  CUDA_OK(cudaEventRecord(c->join_ev, side));
  CUDA_OK(cudaStreamWaitEvent(c->stream, c->join_ev, 0));
  run_idle_work(c);  // host work beside the iterations (the pipeline's decoder planning)
  *out1 = power_result(c, j1);
  *out2 = power_result(c, j2);
}

// ------------------------------------------------------------------ gather / prox / grad / objective
template <typename T>
__global__ void subsample_k(const T* __restrict__ Y, i64 p, const i64* __restrict__ om_r, i64 rho_r,
                            const i64* __restrict__ om_c, i64 rho_c, T* __restrict__ out) {
  const i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x;
  if (i >= rho_r) return;
  const i64 r = om_r[i];
  for (i64 j = blockIdx.y; j < rho_c; j += gridDim.y) out[i + j * rho_r] = Y[r + om_c[j] * p];
}

template <typename T>
void subsample_device(Ctx* c, const T* Y, i64 p, const i64* om_r, i64 rho_r, const i64* om_c,
                      i64 rho_c, T* out) {
  if (rho_r == 0 || rho_c == 0) return;
  dim3 g(blocks_for(rho_r), static_cast<unsigned>(std::min<i64>(rho_c, 65535)));
  subsample_k<T><<<g, kBlock, 0, c->stream>>>(Y, p, om_r, rho_r, om_c, rho_c, out);
  launched(c);
}
template void subsample_device<double>(Ctx*, const double*, i64, const i64*, i64, const i64*, i64, double*);
template void subsample_device<float>(Ctx*, const float*, i64, const i64*, i64, const i64*, i64, float*);

template <typename T>
__global__ void prox_k(int loss, const T* __restrict__ Z, const T* __restrict__ Y, i64 n, T lam,
                       T* __restrict__ out) {
  for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < n; i += (i64)gridDim.x * blockDim.x)
    out[i] = loss == CPCAG_LOSS_L2 ? prox_l2_elem(Z[i], Y[i], lam) : prox_l1_elem(Z[i], Y[i], lam);
}

template <typename T>
__global__ void grad_k(i64 rows, i64 cols, Pull<T> Lr, Pull<T> Lc, T s_r, T s_c, int use_r,
                       int use_c, const T* __restrict__ Z, T* __restrict__ G) {
  const i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x;
  if (i >= rows) return;
  for (i64 c = blockIdx.y; c < cols; c += gridDim.y)
    G[i + c * rows] = grad_elem(Lr, Lc, s_r, s_c, use_r, use_c, Z, rows, i, c);
}

// Partial sums for objective(): phi(Y - X), sum (X Lc) o X, sum (Lr X) o X.
template <typename T>
__global__ void objective_k(i64 rows, i64 cols, Pull<T> Lr, Pull<T> Lc, int loss, int use_r,
                            int use_c, const T* __restrict__ X, const T* __restrict__ Y,
                            double* partials, unsigned* counter, double3* out) {
  double s[3] = {0.0, 0.0, 0.0};
  const i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x;
  if (i < rows) {
    for (i64 c = blockIdx.y; c < cols; c += gridDim.y) {
      const i64 at = i + c * rows;
      const double e = static_cast<double>(Y[at]) - static_cast<double>(X[at]);
      s[0] += loss == CPCAG_LOSS_L2 ? e * e : fabs(e);
      const double x = static_cast<double>(X[at]);
      if (use_c) s[1] += static_cast<double>(pull_right(Lc.rp[c], Lc.rp[c + 1], Lc.ci, Lc.v, X, rows, i)) * x;
      if (use_r) s[2] += static_cast<double>(pull_left(Lr.rp[i], Lr.rp[i + 1], Lr.ci, Lr.v, X + c * rows)) * x;
    }
  }
  double t[3];
  if (grid_sum_last<3>(s, partials, counter, t) && threadIdx.x == 0) *out = make_double3(t[0], t[1], t[2]);
}

template <typename T>
Pull<T> make_pull(Ctx* c, Csr* A, bool right) {
  if (!right) return Pull<T>{A->rp, A->ci, csr_values<T>(c, A)};
  const PullView<T> pv = pull_view<T>(c, A);
  return Pull<T>{pv.rp, pv.ci, pv.v};
}
template Pull<double> make_pull<double>(Ctx*, Csr*, bool);
template Pull<float> make_pull<float>(Ctx*, Csr*, bool);

void frpcag_check_dims(i64 rows, i64 cols, Csr* Lr, Csr* Lc) {
  if (Lr->rows != Lr->cols || Lr->rows != rows) invalid("frpcag: row Laplacian does not match X");
  if (Lc->rows != Lc->cols || Lc->rows != cols) invalid("frpcag: column Laplacian does not match X");
}

template <typename T>
double objective_device(Ctx* c, const T* X, const T* Y, i64 rows, i64 cols, Csr* Lr, Csr* Lc,
                        const cpcag_frpcag_config& cfg) {
  frpcag_check_dims(rows, cols, Lr, Lc);
  const Pull<T> pr = make_pull<T>(c, Lr, false), pc = make_pull<T>(c, Lc, true);
  dim3 g(blocks_for(rows), static_cast<unsigned>(std::min<i64>(std::max<i64>(cols, 1), 65535)));
  const unsigned nb = g.x * g.y;
  DevBuf<double> part(c, 3 * nb);
  DevBuf<unsigned> cnt(c, 1);
  cnt.zero(c);
  DevBuf<double3> out(c, 1);
  CUDA_OK(cudaMemsetAsync(out.p, 0, sizeof(double3), c->stream));
  if (rows > 0 && cols > 0) {
    objective_k<T><<<g, kBlock, 0, c->stream>>>(rows, cols, pr, pc, cfg.loss, cfg.gamma_r != 0.0,
                                                cfg.gamma_c != 0.0, X, Y, part.p, cnt.p, out.p);
    launched(c);
  }
  const double3 s = read_back(c, out.p);
  double val = s.x;
  if (cfg.gamma_c != 0.0) val += cfg.gamma_c * s.y;
  if (cfg.gamma_r != 0.0) val += cfg.gamma_r * s.z;
  return val;
}

std::vector<i64> draw_indices(i64 n, i64 take, HostRng rng) {
  std::vector<i64> pool(static_cast<size_t>(n));
  std::iota(pool.begin(), pool.end(), i64{0});
  for (i64 i = 0; i < take; ++i) {
    const i64 j = i + static_cast<i64>(rng.below(static_cast<uint64_t>(n - i)));
    std::swap(pool[static_cast<size_t>(i)], pool[static_cast<size_t>(j)]);
  }
  pool.resize(static_cast<size_t>(take));
  return pool;
}

template <typename T>
size_t esize() {
  return sizeof(T);
}

}  // namespace cpcag_cuda

using namespace cpcag_cuda;

namespace {
template <class F>
int dispatch(int precision, F&& f) {
  if (precision == CPCAG_F64) return f(double{});
  if (precision == CPCAG_F32) return f(float{});
  set_last_error("unknown precision flag");
  return CPCAG_ERR_INVALID_ARGUMENT;
}

std::vector<i64> host_list(Ctx* c, const int64_t* p, int64_t n) {
  std::vector<i64> out(static_cast<size_t>(n > 0 ? n : 0));
  if (n <= 0) return out;
  if (is_device_ptr(p)) {
    CUDA_OK(cudaMemcpyAsync(out.data(), p, sizeof(i64) * n, cudaMemcpyDeviceToHost, c->stream));
    sync(c);
  } else {
    std::memcpy(out.data(), p, sizeof(i64) * n);
  }
  return out;
}
}  // namespace


extern "C" {

const char* cpcag_cuda_last_error(void) { return g_last_error.c_str(); }

const char* cpcag_cuda_version(void) { return "cpcag-b200 0.1 sm_100a"; }

int cpcag_ctx_create(int device, cpcag_ctx* out) {
  return guard([&] {
    if (!out) invalid("null output pointer");
    int dev = device;
    if (dev < 0) CUDA_OK(cudaGetDevice(&dev));
    CUDA_OK(cudaSetDevice(dev));
    cudaDeviceProp prop;
    CUDA_OK(cudaGetDeviceProperties(&prop, dev));
    if (prop.major < 10)
      fail(CPCAG_ERR_CUDA, "cpcag_cuda: device " + std::to_string(dev) + " is sm_" +
                               std::to_string(prop.major) + std::to_string(prop.minor) +
                               "; this library is built for sm_100a only");
    Ctx* c = new Ctx();
    c->device = dev;
    c->num_sms = prop.multiProcessorCount;
    // A blocking stream: it is implicitly ordered with the legacy default
    // stream, so inputs a caller produced there (torch's default stream)
    // are complete before the context's kernels read them, and vice versa.
    CUDA_OK(cudaStreamCreateWithFlags(&c->own, cudaStreamDefault));
    c->stream = c->own;
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
      uint64_t thr = UINT64_MAX;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
    *out = reinterpret_cast<cpcag_ctx>(c);
  });
}


int cpcag_ctx_reserve(cpcag_ctx ctx, int64_t bytes) {
  return guard([&] {
    Ctx* c = as_ctx(ctx);
    if (bytes <= 0) return;
    void* p = nullptr;
    CUDA_OK(cudaMallocAsync(&p, static_cast<size_t>(bytes), c->stream));
    CUDA_OK(cudaFreeAsync(p, c->stream));
    CUDA_OK(cudaStreamSynchronize(c->stream));
  });
}

int cpcag_ctx_destroy(cpcag_ctx ctx) {
  return guard([&] {
    Ctx* c = as_ctx(ctx);
    cudaStreamSynchronize(c->stream);
    for (auto& r : c->kt.recs) {
      cudaEventDestroy(r.a);
      cudaEventDestroy(r.b);
    }
    for (auto e : c->kt.pool) cudaEventDestroy(e);
    if (c->pinned) cudaFreeHost(c->pinned);
    if (c->side) {
      cudaStreamSynchronize(c->side);
      cudaStreamDestroy(c->side);
      cudaEventDestroy(c->fork_ev);
      cudaEventDestroy(c->join_ev);
    }
    if (c->aux) {
      cudaStreamSynchronize(c->aux);
      cudaStreamDestroy(c->aux);
      cudaEventDestroy(c->aux_ev);
    }
    cudaStreamDestroy(c->own);
    delete c;
  });
}

int cpcag_ctx_set_stream(cpcag_ctx ctx, void* s) {
  return guard([&] {
    Ctx* c = as_ctx(ctx);
    c->stream = s ? reinterpret_cast<cudaStream_t>(s) : c->own;
  });
}

void* cpcag_ctx_stream(cpcag_ctx ctx) { return ctx ? reinterpret_cast<Ctx*>(ctx)->stream : nullptr; }

int cpcag_ctx_set_apply_path(cpcag_ctx ctx, int path) {
  return guard([&] {
    if (path < 0 || path > 3) invalid("apply path must be 0, 1, 2 or 3");
    as_ctx(ctx)->apply_path = path;
  });
}

int cpcag_ctx_set_fista_path(cpcag_ctx ctx, int path) {
  return guard([&] {
    if (path < 0 || path > 1) invalid("fista path must be 0 or 1");
    as_ctx(ctx)->fista_simt = path;
  });
}

int cpcag_ctx_set_power_path(cpcag_ctx ctx, int path) {
  return guard([&] {
    if (path < 0 || path > 2) invalid("power path must be 0, 1 or 2");
    as_ctx(ctx)->power_path = path;
  });
}

int cpcag_ctx_last_power_path(cpcag_ctx ctx) { return ctx ? reinterpret_cast<Ctx*>(ctx)->last_power_path : -1; }

int cpcag_ctx_last_apply_path(cpcag_ctx ctx) { return ctx ? reinterpret_cast<Ctx*>(ctx)->last_apply_path : -1; }

int cpcag_ctx_synchronize(cpcag_ctx ctx) {
  return guard([&] { sync(as_ctx(ctx)); });
}

int cpcag_ctx_enable_kernel_timing(cpcag_ctx ctx, int enable) {
  return guard([&] {
    Ctx* c = as_ctx(ctx);
    harvest(c);
    c->timing = enable != 0;
  });
}

int cpcag_ctx_kernel_timing_filter(cpcag_ctx ctx, const char* tags_csv) {
  return guard([&] {
    Ctx* c = as_ctx(ctx);
    c->timing_filter = tags_csv ? tags_csv : "";
  });
}

int cpcag_ctx_reset_kernel_timing(cpcag_ctx ctx) {
  return guard([&] {
    Ctx* c = as_ctx(ctx);
    harvest(c);
    c->kt.totals.clear();
  });
}

int cpcag_ctx_kernel_timing(cpcag_ctx ctx, int index, char* tag, int64_t tag_cap, int64_t* launches,
                            double* total_ms) {
  return guard([&] {
    Ctx* c = as_ctx(ctx);
    harvest(c);
    if (index < 0 || index >= static_cast<int>(c->kt.totals.size())) fail(CPCAG_ERR_OUT_OF_RANGE, "kernel timing index out of range");
    const auto& t = c->kt.totals[static_cast<size_t>(index)];
    if (tag && tag_cap > 0) {
      std::strncpy(tag, t.first.c_str(), static_cast<size_t>(tag_cap - 1));
      tag[tag_cap - 1] = 0;
    }
    if (launches) *launches = t.second.first;
    if (total_ms) *total_ms = t.second.second;
  });
}

int cpcag_ctx_kernel_timing_count(cpcag_ctx ctx) {
  if (!ctx) return 0;
  Ctx* c = reinterpret_cast<Ctx*>(ctx);
  try {
    harvest(c);
  } catch (...) {
    return 0;
  }
  return static_cast<int>(c->kt.totals.size());
}

int64_t cpcag_ctx_launch_count(cpcag_ctx ctx) { return ctx ? reinterpret_cast<Ctx*>(ctx)->launches : 0; }
void cpcag_ctx_reset_launch_count(cpcag_ctx ctx) {
  if (ctx) reinterpret_cast<Ctx*>(ctx)->launches = 0;
}

int cpcag_csr_create(cpcag_ctx ctx, int64_t rows, int64_t cols, int64_t nnz, const int64_t* row_ptr,
                     const int64_t* col_idx, const double* values, cpcag_csr* out) {
  return guard([&] {
    Ctx* c = as_ctx(ctx);
    if (!out) invalid("null output pointer");
    if (rows < 0 || cols < 0) invalid("sparse: negative dimensions");
    if (cols > INT32_MAX) invalid("sparse: more than 2^31-1 columns are not supported");
    // Validation of the CSR invariants (sparse.hpp:15-17) on the host copy:
    // one pass over the index arrays, done once per handle.
    std::vector<i64> rp(static_cast<size_t>(rows) + 1);
    std::vector<i64> ci(static_cast<size_t>(nnz));
    std::vector<double> v(static_cast<size_t>(nnz));
    auto fetch = [&](void* dst, const void* src, size_t bytes) {
      if (!bytes) return;
      if (is_device_ptr(src))
        CUDA_OK(cudaMemcpy(dst, src, bytes, cudaMemcpyDeviceToHost));
      else
        std::memcpy(dst, src, bytes);
    };
    fetch(rp.data(), row_ptr, sizeof(i64) * (rows + 1));
    fetch(ci.data(), col_idx, sizeof(i64) * nnz);
    fetch(v.data(), values, sizeof(double) * nnz);
    if (rp[0] != 0 || rp[rows] != nnz) invalid("sparse: row pointers do not span the entries");
    std::vector<i64> rp2(static_cast<size_t>(rows) + 1, 0);
    std::vector<int> ci2;
    std::vector<double> v2;
    ci2.reserve(static_cast<size_t>(nnz));
    v2.reserve(static_cast<size_t>(nnz));
    for (i64 r = 0; r < rows; ++r) {
      if (rp[r + 1] < rp[r]) invalid("sparse: row pointers must be nondecreasing");
      for (i64 k = rp[r]; k < rp[r + 1]; ++k) {
        if (ci[k] < 0 || ci[k] >= cols) invalid("sparse: triplet index out of range");
        if (k > rp[r] && ci[k] <= ci[k - 1]) invalid("sparse: column indices must be strictly increasing");
        if (!std::isfinite(v[k])) invalid("sparse: non-finite entry");
        if (v[k] != 0.0) {
          ci2.push_back(static_cast<int>(ci[k]));
          v2.push_back(v[k]);
        }
      }
      rp2[r + 1] = static_cast<i64>(v2.size());
    }
    Csr* a = csr_alloc(c, rows, cols, static_cast<i64>(v2.size()));
    CUDA_OK(cudaMemcpyAsync(a->rp, rp2.data(), sizeof(i64) * (rows + 1), cudaMemcpyHostToDevice, c->stream));
    if (a->nnz) {
      CUDA_OK(cudaMemcpyAsync(a->ci, ci2.data(), sizeof(int) * a->nnz, cudaMemcpyHostToDevice, c->stream));
      CUDA_OK(cudaMemcpyAsync(a->v, v2.data(), sizeof(double) * a->nnz, cudaMemcpyHostToDevice, c->stream));
    }
    sync(c);
    *out = reinterpret_cast<cpcag_csr>(a);
  });
}

int cpcag_csr_destroy(cpcag_csr a) {
  return guard([&] { delete as_csr(a); });
}

int cpcag_csr_info(cpcag_csr h, int64_t* rows, int64_t* cols, int64_t* nnz) {
  return guard([&] {
    Csr* a = as_csr(h);
    if (rows) *rows = a->rows;
    if (cols) *cols = a->cols;
    if (nnz) *nnz = a->nnz;
  });
}

__global__ void widen_k(const int* __restrict__ a, int64_t* __restrict__ b, i64 n) {
  for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < n; i += (i64)gridDim.x * blockDim.x) b[i] = a[i];
}

int cpcag_csr_export(cpcag_ctx ctx, cpcag_csr h, int64_t* row_ptr, int64_t* col_idx, double* values) {
  return guard([&] {
    Ctx* c = as_ctx(ctx);
    Csr* a = as_csr(h);
    if (row_ptr) {
      OutView<i64> o(c, row_ptr, a->rows + 1);
      CUDA_OK(cudaMemcpyAsync(o.d, a->rp, sizeof(i64) * (a->rows + 1), cudaMemcpyDeviceToDevice, c->stream));
      o.flush(c);
      sync(c);
    }
    if (col_idx && a->nnz) {
      OutView<i64> o(c, col_idx, a->nnz);
      widen_k<<<stride_blocks(c, a->nnz), kBlock, 0, c->stream>>>(a->ci, o.d, a->nnz);
      launched(c);
      o.flush(c);
      sync(c);
    }
    if (values && a->nnz) {
      OutView<double> o(c, values, a->nnz);
      CUDA_OK(cudaMemcpyAsync(o.d, a->v, sizeof(double) * a->nnz, cudaMemcpyDeviceToDevice, c->stream));
      o.flush(c);
      sync(c);
    }
  });
}

int cpcag_csr_is_symmetric(cpcag_csr h) {
  Csr* a = reinterpret_cast<Csr*>(h);
  if (!a) return 0;
  return a->sym == 1 ? 1 : 0;
}

int cpcag_cuda_spmm(cpcag_ctx ctx, cpcag_csr Ah, int side, int precision, int64_t x_rows,
                    int64_t x_cols, const void* X, void* Y) {
  return dispatch(precision, [&](auto tag) {
    using T = decltype(tag);
    return guard([&] {
      Ctx* c = as_ctx(ctx);
      Csr* A = as_csr(Ah);
      if (side == CPCAG_LEFT) {
        if (x_rows != A->cols) invalid("sparse multiply: dimension mismatch");
        InView<T> xin(c, static_cast<const T*>(X), static_cast<size_t>(x_rows * x_cols));
        OutView<T> yout(c, static_cast<T*>(Y), static_cast<size_t>(A->rows * x_cols));
        spmm_left<T>(c, A, xin.d, x_cols, yout.d);
        yout.flush(c);
        if (yout.host || xin.staged.p) sync(c);
      } else if (side == CPCAG_RIGHT) {
        if (x_cols != A->rows) invalid("sparse right_multiply: dimension mismatch");
        InView<T> xin(c, static_cast<const T*>(X), static_cast<size_t>(x_rows * x_cols));
        OutView<T> yout(c, static_cast<T*>(Y), static_cast<size_t>(x_rows * A->cols));
        spmm_right<T>(c, A, xin.d, x_rows, yout.d);
        yout.flush(c);
        if (yout.host || xin.staged.p) sync(c);
      } else {
        invalid("spmm: side must be CPCAG_LEFT or CPCAG_RIGHT");
      }
    });
  });
}

int cpcag_cuda_spmv(cpcag_ctx ctx, cpcag_csr Ah, int precision, int64_t n, const void* x, void* y) {
  return dispatch(precision, [&](auto tag) {
    using T = decltype(tag);
    return guard([&] {
      Ctx* c = as_ctx(ctx);
      Csr* A = as_csr(Ah);
      if (n != A->cols)
        invalid("spmv: dimension mismatch (" + std::to_string(A->cols) + " vs " + std::to_string(n) + ")");
      InView<T> xin(c, static_cast<const T*>(x), static_cast<size_t>(n));
      OutView<T> yout(c, static_cast<T*>(y), static_cast<size_t>(A->rows));
      spmm_left<T>(c, A, xin.d, 1, yout.d);
      yout.flush(c);
      if (yout.host || xin.staged.p) sync(c);
    });
  });
}

int cpcag_cuda_power_norm(cpcag_ctx ctx, cpcag_csr A, double tol, uint64_t seed, int64_t max_iter,
                          double* out) {
  return guard([&] {
    if (!out) invalid("null output pointer");
    *out = power_norm(as_ctx(ctx), as_csr(A), tol, seed, max_iter);
  });
}

int cpcag_cuda_draw_plan(int64_t p, int64_t n, int64_t rho_r, int64_t rho_c, uint64_t seed,
                         int64_t* omega_r, int64_t* omega_c) {
  return guard([&] {
    if (rho_r < 1 || rho_r > p) invalid("draw_plan: rho_r out of range [1, " + std::to_string(p) + "]");
    if (rho_c < 1 || rho_c > n) invalid("draw_plan: rho_c out of range [1, " + std::to_string(n) + "]");
    const auto r = draw_indices(p, rho_r, HostRng::derive(seed, 0x726f7773ULL));
    const auto cc = draw_indices(n, rho_c, HostRng::derive(seed, 0x636f6c73ULL));
    std::copy(r.begin(), r.end(), omega_r);
    std::copy(cc.begin(), cc.end(), omega_c);
  });
}

int cpcag_cuda_subsample(cpcag_ctx ctx, int precision, const void* Y, int64_t p, int64_t n,
                         const int64_t* omega_r, int64_t rho_r, const int64_t* omega_c, int64_t rho_c,
                         void* out) {
  return dispatch(precision, [&](auto tag) {
    using T = decltype(tag);
    return guard([&] {
      Ctx* c = as_ctx(ctx);
      const auto hr = host_list(c, omega_r, rho_r);
      const auto hc = host_list(c, omega_c, rho_c);
      for (i64 r : hr)
        if (r < 0 || r >= p) invalid("subsample: plan does not match matrix dimensions");
      for (i64 q : hc)
        if (q < 0 || q >= n) invalid("subsample: plan does not match matrix dimensions");
      InView<T> yin(c, static_cast<const T*>(Y), static_cast<size_t>(p * n));
      InView<i64> rin(c, omega_r, static_cast<size_t>(rho_r));
      InView<i64> cin(c, omega_c, static_cast<size_t>(rho_c));
      OutView<T> o(c, static_cast<T*>(out), static_cast<size_t>(rho_r * rho_c));
      subsample_device<T>(c, yin.d, p, rin.d, rho_r, cin.d, rho_c, o.d);
      o.flush(c);
      sync(c);
    });
  });
}

int cpcag_cuda_prox(cpcag_ctx ctx, int precision, int loss, const void* Z, const void* Y, int64_t count,
                    double lam, void* out) {
  return dispatch(precision, [&](auto tag) {
    using T = decltype(tag);
    return guard([&] {
      Ctx* c = as_ctx(ctx);
      if (lam < 0.0) invalid("prox: negative threshold");
      InView<T> z(c, static_cast<const T*>(Z), static_cast<size_t>(count));
      InView<T> y(c, static_cast<const T*>(Y), static_cast<size_t>(count));
      OutView<T> o(c, static_cast<T*>(out), static_cast<size_t>(count));
      if (count > 0) {
        prox_k<T><<<stride_blocks(c, count), kBlock, 0, c->stream>>>(loss, z.d, y.d, count, static_cast<T>(lam), o.d);
        launched(c);
      }
      o.flush(c);
      sync(c);
    });
  });
}

int cpcag_cuda_grad_g(cpcag_ctx ctx, int precision, const void* Z, int64_t rows, int64_t cols,
                      cpcag_csr Lrh, cpcag_csr Lch, const cpcag_frpcag_config* cfg, void* G) {
  return dispatch(precision, [&](auto tag) {
    using T = decltype(tag);
    return guard([&] {
      Ctx* c = as_ctx(ctx);
      Csr* Lr = as_csr(Lrh);
      Csr* Lc = as_csr(Lch);
      if (!cfg) invalid("null config");
      frpcag_check_dims(rows, cols, Lr, Lc);
      InView<T> z(c, static_cast<const T*>(Z), static_cast<size_t>(rows * cols));
      OutView<T> g(c, static_cast<T*>(G), static_cast<size_t>(rows * cols));
      if (rows > 0 && cols > 0) {
        dim3 gr(blocks_for(rows), static_cast<unsigned>(std::min<i64>(cols, 65535)));
        grad_k<T><<<gr, kBlock, 0, c->stream>>>(rows, cols, make_pull<T>(c, Lr, false), make_pull<T>(c, Lc, true),
                                                 static_cast<T>(2.0 * cfg->gamma_r), static_cast<T>(2.0 * cfg->gamma_c),
                                                 cfg->gamma_r != 0.0, cfg->gamma_c != 0.0, z.d, g.d);
        launched(c);
      }
      g.flush(c);
      sync(c);
    });
  });
}

int cpcag_cuda_objective(cpcag_ctx ctx, int precision, const void* X, const void* Y, int64_t rows,
                         int64_t cols, cpcag_csr Lr, cpcag_csr Lc, const cpcag_frpcag_config* cfg,
                         double* out) {
  return dispatch(precision, [&](auto tag) {
    using T = decltype(tag);
    return guard([&] {
      Ctx* c = as_ctx(ctx);
      if (!cfg || !out) invalid("null argument");
      InView<T> x(c, static_cast<const T*>(X), static_cast<size_t>(rows * cols));
      InView<T> y(c, static_cast<const T*>(Y), static_cast<size_t>(rows * cols));
      *out = objective_device<T>(c, x.d, y.d, rows, cols, as_csr(Lr), as_csr(Lc), *cfg);
    });
  });
}

}  // extern "C"
