// common.cuh -- shared infrastructure of libcpcag_cuda.so (sm_100a).
//
// Context (stream + stream-ordered allocator + launch counter), the device
// CSR operator, error mapping to the reference's exception classes, pointer
// staging (host or device arguments), deterministic block reductions and a
// software grid barrier for cooperative (co-resident) launches.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <cmath>
#include <cstring>
#include <functional>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/cpcag_cuda.h"

namespace cpcag_cuda {

using i64 = int64_t;

// ------------------------------------------------------------------ errors
struct Error : std::runtime_error {
  int status;
  Error(int s, const std::string& m) : std::runtime_error(m), status(s) {}
};

[[noreturn]] inline void fail(int status, const std::string& msg) { throw Error(status, msg); }
[[noreturn]] inline void invalid(const std::string& msg) { fail(CPCAG_ERR_INVALID_ARGUMENT, msg); }
[[noreturn]] inline void runtime(const std::string& msg) { fail(CPCAG_ERR_RUNTIME, msg); }

void set_last_error(const std::string& m);

#define CUDA_OK(expr)                                                                      \
  do {                                                                                     \
    cudaError_t _e = (expr);                                                               \
    if (_e != cudaSuccess)                                                                 \
      ::cpcag_cuda::fail(CPCAG_ERR_CUDA, std::string("cuda: ") + cudaGetErrorString(_e) + \
                                             " at " __FILE__ ":" + std::to_string(__LINE__)); \
  } while (0)

// Runs the body and converts exceptions to the C status code.
template <class F>
int guard(F&& body) {
  try {
    body();
    return CPCAG_OK;
  } catch (const Error& e) {
    set_last_error(e.what());
    return e.status;
  } catch (const std::bad_alloc&) {
    set_last_error("out of host memory");
    return CPCAG_ERR_RUNTIME;
  } catch (const std::exception& e) {
    set_last_error(e.what());
    return CPCAG_ERR_RUNTIME;
  }
}

// ------------------------------------------------------------------ context
// Per-kernel device timing (CUDA events on the launching stream), enabled
// on demand by the caller (bench.py) for the roofline figures.
struct KernelTimes {
  struct Rec {
    std::string tag;
    cudaEvent_t a, b;
  };
  std::vector<Rec> recs;        // in flight since the last harvest
  std::vector<cudaEvent_t> pool;
  std::vector<std::pair<std::string, std::pair<i64, double>>> totals;  // tag -> (launches, ms)
};

struct Ctx {
  int device = 0;
  int num_sms = 148;
  cudaStream_t own = nullptr;
  cudaStream_t stream = nullptr;
  i64 launches = 0;
  void* pinned = nullptr;  // small pinned staging area for scalar read-back
  size_t pinned_bytes = 0;
  bool timing = false;
  std::string timing_filter;  // comma-separated tags; empty = all
  int apply_path = 0;         // decoder operator: 0 auto, 1 two passes, 2 fused, 3 slab (tests)
  int last_apply_path = 0;    // the path the last planned operator took (1, 2 or 3; tests)
  int fista_simt = 0;         // 1: the persistent FISTA kernel's SIMT tile GEMM instead of DMMA (tests)
  int power_path = 0;         // cooperative power iteration: 0 auto, 1 one product per barrier (tests)
  int last_power_path = 0;    // 1 one product, 2 two products per barrier; 0 single-CTA kernel or none (tests)
  cudaStream_t side = nullptr;  // second stream for independent work (lazily created)
  cudaEvent_t fork_ev = nullptr, join_ev = nullptr;
  // A one-CTA job on the side stream that fills an SM (the detected-rank
  // Jacobi kernel): while it runs, persistent one-CTA-per-SM grids on the main
  // stream size themselves to the SMs that are left (join_ev marks its end).
  bool side_job_running = false;
  int sm_reserve = 0;
  // Host work deferred to the next long device wait (run_idle_work): it runs
  // with `stream` switched to `aux`, and the context stream then waits on it.
  std::function<void()> idle_work;
  cudaStream_t aux = nullptr;
  cudaEvent_t aux_ev = nullptr;
  KernelTimes kt;
};

// Runs (and clears) c->idle_work on the aux stream while the device works
// through what the context stream already holds; no-op when none is pending.
void run_idle_work(Ctx* c);

// Clears c->idle_work when the scope that set it ends (its captures die there).
struct IdleWorkScope {
  Ctx* c;
  explicit IdleWorkScope(Ctx* ctx) : c(ctx) {}
  ~IdleWorkScope() { c->idle_work = nullptr; }
};

// The context's side stream (non-blocking, created on first use) and its
// fork / join events.
inline cudaStream_t side_stream(Ctx* c) {
  if (!c->side) {
    CUDA_OK(cudaStreamCreateWithFlags(&c->side, cudaStreamNonBlocking));
    CUDA_OK(cudaEventCreateWithFlags(&c->fork_ev, cudaEventDisableTiming));
    CUDA_OK(cudaEventCreateWithFlags(&c->join_ev, cudaEventDisableTiming));
  }
  return c->side;
}

// RAII scope timing one kernel launch under `tag` when timing is enabled.
struct KScope {
  Ctx* c;
  const char* tag;
  cudaEvent_t a = nullptr, b = nullptr;
  KScope(Ctx* ctx, const char* t);
  ~KScope();
};

inline Ctx* as_ctx(cpcag_ctx c) {
  if (!c) invalid("null context");
  return reinterpret_cast<Ctx*>(c);
}

// Counts a kernel launch and checks the launch status.
inline void launched(Ctx* c) {
  c->launches++;
  CUDA_OK(cudaGetLastError());
}

// Programmatic dependent launch.  A kernel launched with launch_pdl may be
// scheduled while its predecessor on the stream still runs (once every CTA of
// the predecessor has called pdl_trigger or exited); it must call pdl_wait
// before touching anything the predecessor writes -- the wait returns when the
// predecessor has completed and its writes are visible.  Back-to-back short
// kernels (the decoder's three per CG iteration) overlap their launch latency
// and CTA ramp-up with the predecessor's tail this way.  Both calls are no-ops
// in a kernel launched the ordinary way.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

template <typename... KArgs, typename... Args>
void launch_pdl(void (*k)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  CUDA_OK(cudaLaunchKernelEx(&cfg, k, static_cast<KArgs>(args)...));
}

// Stream-ordered device buffer.
template <typename T>
struct DevBuf {
  T* p = nullptr;
  size_t n = 0;
  cudaStream_t s = nullptr;
  DevBuf() = default;
  DevBuf(Ctx* c, size_t count) { alloc(c, count); }
  void alloc(Ctx* c, size_t count) {
    release();
    s = c->stream;
    n = count;
    if (count) CUDA_OK(cudaMallocAsync(reinterpret_cast<void**>(&p), count * sizeof(T), s));
  }
  void zero(Ctx* c) {
    if (n) CUDA_OK(cudaMemsetAsync(p, 0, n * sizeof(T), c->stream));
  }
  void release() {
    if (p) cudaFreeAsync(p, s);
    p = nullptr;
    n = 0;
  }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  DevBuf(DevBuf&& o) noexcept : p(o.p), n(o.n), s(o.s) { o.p = nullptr; o.n = 0; }
  DevBuf& operator=(DevBuf&& o) noexcept {
    if (this != &o) {
      release();
      p = o.p;
      n = o.n;
      s = o.s;
      o.p = nullptr;
      o.n = 0;
    }
    return *this;
  }
  ~DevBuf() { release(); }
};

// True when ptr is device (or managed) memory.
bool is_device_ptr(const void* ptr);

// Read-only view of a caller array on the device: uses it in place when it
// already is device memory, otherwise stages a copy into HBM.
template <typename T>
struct InView {
  const T* d = nullptr;
  DevBuf<T> staged;
  InView(Ctx* c, const T* ptr, size_t count) {
    if (count == 0 || ptr == nullptr) return;
    if (is_device_ptr(ptr)) {
      d = ptr;
    } else {
      staged.alloc(c, count);
      CUDA_OK(cudaMemcpyAsync(staged.p, ptr, count * sizeof(T), cudaMemcpyHostToDevice, c->stream));
      d = staged.p;
    }
  }
};

// Writable view: device destination used in place; host destination gets a
// device scratch that flush() copies back.
template <typename T>
struct OutView {
  T* d = nullptr;
  T* host = nullptr;
  size_t n = 0;
  DevBuf<T> staged;
  OutView(Ctx* c, T* ptr, size_t count) : n(count) {
    if (count == 0 || ptr == nullptr) return;
    if (is_device_ptr(ptr)) {
      d = ptr;
    } else {
      host = ptr;
      staged.alloc(c, count);
      d = staged.p;
    }
  }
  void flush(Ctx* c) {
    if (host && n) CUDA_OK(cudaMemcpyAsync(host, d, n * sizeof(T), cudaMemcpyDeviceToHost, c->stream));
  }
};

inline void sync(Ctx* c) { CUDA_OK(cudaStreamSynchronize(c->stream)); }

// Raises (never lowers) a kernel's dynamic shared-memory limit.  The limit is
// process-wide state, so concurrent contexts must not shrink it under each
// other's launches.
void ensure_smem_impl(const void* func, size_t bytes);
template <class F>
inline void ensure_smem(F* func, size_t bytes) {
  ensure_smem_impl(reinterpret_cast<const void*>(func), bytes);
}

// Host-side phase tracing (CPCAG_TRACE=1): synchronises and prints wall time
// since the previous mark.  Off by default; used to find host overheads.
void trace_mark(Ctx* c, const char* what);

// Copies a small device struct back through pinned memory (synchronises).
template <typename T>
T read_back(Ctx* c, const T* dptr) {
  if (c->pinned_bytes < sizeof(T)) {
    if (c->pinned) cudaFreeHost(c->pinned);
    c->pinned_bytes = sizeof(T) < 4096 ? 4096 : sizeof(T);
    CUDA_OK(cudaMallocHost(&c->pinned, c->pinned_bytes));
  }
  CUDA_OK(cudaMemcpyAsync(c->pinned, dptr, sizeof(T), cudaMemcpyDeviceToHost, c->stream));
  sync(c);
  T out;
  std::memcpy(&out, c->pinned, sizeof(T));
  return out;
}

// ------------------------------------------------------------------ CSR
// Device CSR with the invariants of sparse.hpp:15-17.  Values are fp64; an
// fp32 copy is made on first fp32 use.  `sym` records exact symmetry (A ==
// A^T bit for bit), which lets X*A run as a pull over CSR rows in exactly the
// reference's accumulation order (sparse.cpp:100-111).
void* csr_malloc(Ctx* c, size_t bytes);  // stream-ordered pool (see core.cu)

struct Csr {
  i64 rows = 0, cols = 0, nnz = 0;
  i64* rp = nullptr;
  int* ci = nullptr;
  double* v = nullptr;
  float* v32 = nullptr;
  int sym = -1;  // -1 unknown, 0 no, 1 yes
  // Transpose (CSC as CSR of A^T), built on demand for non-symmetric X*A.
  i64* t_rp = nullptr;
  int* t_ci = nullptr;
  double* t_v = nullptr;
  float* t_v32 = nullptr;
  int device = 0;
  ~Csr();
};

inline Csr* as_csr(cpcag_csr a) {
  if (!a) invalid("null sparse matrix handle");
  return reinterpret_cast<Csr*>(a);
}

// Allocates an empty device CSR of the given shape (rp zeroed).
Csr* csr_alloc(Ctx* c, i64 rows, i64 cols, i64 nnz);
template <typename T>
const T* csr_values(Ctx* c, Csr* a);
template <typename T>
const T* csr_t_values(Ctx* c, Csr* a);
int csr_symmetric(Ctx* c, Csr* a);
void csr_build_transpose(Ctx* c, Csr* a);

// ------------------------------------------------------------------ math helpers
__device__ __forceinline__ double mul_rn(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ float mul_rn(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ double add_rn(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ float add_rn(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ double sub_rn(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ float sub_rn(float a, float b) { return __fsub_rn(a, b); }

// ------------------------------------------------------------------ reductions
constexpr int kBlock = 256;

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Deterministic block sum (fixed shuffle tree).  All threads get the result.
template <int NV>
__device__ __forceinline__ void block_sum(double (&v)[NV]) {
  __shared__ double sh[NV][32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int nw = (blockDim.x + 31) >> 5;
#pragma unroll
  for (int q = 0; q < NV; ++q) {
    v[q] = warp_sum(v[q]);
  }
  __syncthreads();
  if (lane == 0) {
#pragma unroll
    for (int q = 0; q < NV; ++q) sh[q][wid] = v[q];
  }
  __syncthreads();
#pragma unroll
  for (int q = 0; q < NV; ++q) {
    double x = lane < nw ? sh[q][lane] : 0.0;
    v[q] = warp_sum(x);
  }
  __syncthreads();
}

// Every block deposits its NV block sums; the last block to arrive sums all
// partials in a fixed order (deterministic for a given grid) and returns
// true with the totals in `tot` (all threads of that block).  `partials`
// holds NV * nblocks doubles; `counter` must be zero on entry and is reset.
template <int NV>
__device__ bool grid_sum_last(double (&v)[NV], double* partials, unsigned* counter,
                              double (&tot)[NV]) {
  __shared__ bool last;
  const unsigned nb = gridDim.x * gridDim.y * gridDim.z;
  const unsigned bid = blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z);
  block_sum<NV>(v);
  if (threadIdx.x == 0) {
#pragma unroll
    for (int q = 0; q < NV; ++q) partials[q * nb + bid] = v[q];
    __threadfence();
    last = atomicAdd(counter, 1u) == nb - 1;
  }
  __syncthreads();
  if (!last) return false;
  __threadfence();
#pragma unroll
  for (int q = 0; q < NV; ++q) {
    double s = 0.0;
    for (unsigned i = threadIdx.x; i < nb; i += blockDim.x) s += __ldcg(partials + q * nb + i);
    tot[q] = s;
  }
  block_sum<NV>(tot);
  if (threadIdx.x == 0) *counter = 0u;
  return true;
}

// Software grid barrier for cooperative launches (all blocks co-resident).
// Thread 0 of each CTA arrives with a gpu-scope release (after the CTA's
// __syncthreads, so the CTA's prior writes are ordered before it); the last
// arriver resets the count and bumps the generation with a release; the
// others poll the generation with gpu-scope acquire loads.  Measured on B200
// with 148 CTAs: 1.19 us per barrier vs 2.26 us for the fence + volatile-poll
// form (tools/micro/barrier_bench.cu).
__device__ __forceinline__ unsigned ld_acquire_gpu(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void grid_barrier(unsigned* count, unsigned* gen) {
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned nb = gridDim.x * gridDim.y * gridDim.z;
    const unsigned g = ld_acquire_gpu(gen);
    unsigned old;
    asm volatile("atom.add.acq_rel.gpu.global.u32 %0, [%1], 1;" : "=r"(old) : "l"(count) : "memory");
    if (old == nb - 1) {
      asm volatile("st.relaxed.gpu.global.u32 [%0], 0;" ::"l"(count) : "memory");
      asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(gen) : "memory");
    } else {
      while (ld_acquire_gpu(gen) == g) {
      }
    }
  }
  __syncthreads();
}

// The same barrier with the generation tracked in a register: `g` counts the
// barriers this CTA has passed (0 at kernel start, *gen zeroed before the
// launch), so thread 0 skips the initial load of *gen -- one L2 round trip
// less per barrier.  Every CTA must pass the same sequence of barriers.
__device__ __forceinline__ void grid_barrier_local(unsigned* count, unsigned* gen, unsigned& g) {
  __syncthreads();
  ++g;
  if (threadIdx.x == 0) {
    const unsigned nb = gridDim.x * gridDim.y * gridDim.z;
    unsigned old;
    asm volatile("atom.add.acq_rel.gpu.global.u32 %0, [%1], 1;" : "=r"(old) : "l"(count) : "memory");
    if (old == nb - 1) {
      asm volatile("st.relaxed.gpu.global.u32 [%0], 0;" ::"l"(count) : "memory");
      asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(gen), "r"(g) : "memory");
    } else {
      while (static_cast<int>(ld_acquire_gpu(gen) - g) < 0) {
      }
    }
  }
  __syncthreads();
}

// Grid barrier on a monotonic arrival counter (zeroed before the launch):
// each CTA posts one fire-and-forget release add and waits until the counter
// reaches (barriers passed) x (grid size).  No last-arriver hand-off, so one
// L2 round trip less than grid_barrier_local.  g counts this CTA's barriers.
__device__ __forceinline__ void grid_barrier_mono(unsigned* count, unsigned& g) {
  __syncthreads();
  ++g;
  if (threadIdx.x == 0) {
    const unsigned target = g * (gridDim.x * gridDim.y * gridDim.z);
    asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(count) : "memory");
    while (static_cast<int>(ld_acquire_gpu(count) - target) < 0) {
    }
  }
  __syncthreads();
}

inline unsigned blocks_for(i64 n, int block = kBlock) {
  i64 b = (n + block - 1) / block;
  if (b < 1) b = 1;
  return static_cast<unsigned>(b);
}

// Capped grid for grid-stride element-wise kernels (multiple of SM count).
inline unsigned stride_blocks(Ctx* c, i64 n, int block = kBlock) {
  i64 b = (n + block - 1) / block;
  const i64 cap = static_cast<i64>(c->num_sms) * 16;
  if (b > cap) b = cap;
  if (b < 1) b = 1;
  return static_cast<unsigned>(b);
}

// ------------------------------------------------------------------ shared kernels
// Deterministic scalar reductions over a strided pair of arrays.
template <typename T>
void dot_device(Ctx* c, const T* a, const T* b, i64 n, double* out_dev);

// Host-side counter RNG identical to the reference (rng.hpp:11-68).
struct HostRng {
  uint64_t seed, ctr = 0;
  double spare = 0.0;
  bool has_spare = false;
  explicit HostRng(uint64_t s) : seed(s) {}
  static uint64_t mix(uint64_t z) {
    z += 0x9e3779b97f4a7c15ULL;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
  }
  uint64_t u64() { return mix(seed + 0x632be59bd9b4e019ULL * ++ctr); }
  double uniform() { return static_cast<double>(u64() >> 11) * 0x1.0p-53; }
  uint64_t below(uint64_t n) {
    const uint64_t lim = UINT64_MAX - UINT64_MAX % n;
    uint64_t x = u64();
    while (x >= lim) x = u64();
    return x % n;
  }
  double gaussian();
  static HostRng derive(uint64_t s, uint64_t stream) { return HostRng(mix(s ^ mix(stream))); }
};

// Internal entry points shared between translation units.
double power_norm(Ctx* c, Csr* A, double tol, uint64_t seed, i64 max_iter);
// Singular values of a small fp64 matrix (Gram + one-CTA Jacobi) on stream s,
// read back by rank_job_finish (approx.cu).
struct RankJob {
  DevBuf<double> G, lam;
  DevBuf<int> flag;
  void* host = nullptr;  // pinned: eigenvalues [0, 110), non-finite flag at double index 120
  i64 q = 0;
  bool running = false;
  cudaStream_t side = nullptr;
  ~RankJob();
};
void rank_job_start(Ctx* c, RankJob& job, const double* Xt64, i64 m, i64 n, cudaStream_t s);
std::vector<double> rank_job_finish(Ctx* c, RankJob& job);
void power_norm_pair(Ctx* c, Csr* A1, Csr* A2, double tol, uint64_t seed, i64 max_iter, double* out1,
                     double* out2);
// kmeans / decode_labels on the device (cluster.cu).
void kmeans_device(Ctx* c, const double* X, i64 rows, i64 n, i64 k, i64 restarts, uint64_t seed, i64 max_iter,
                   int* assignments_dev, double* wcss_out);
void decode_labels_device(Ctx* c, Csr* Lc, const std::vector<i64>& om_c, const int* sampled_dev, i64 k,
                          double pcg_tol, i64 pcg_max_iter, i64 n, int* labels_dev);
// k smallest eigenvalues (ascending, host array) by Lanczos (lanczos.cu).
void sym_eigvals_lanczos(Ctx* c, Csr* A, i64 k, double tol, i64 max_iter, uint64_t seed, double* evals,
                         i64* iterations);

template <typename T>
void spmm_left(Ctx* c, Csr* A, const T* X, i64 m, T* Y);
template <typename T>
void spmm_right(Ctx* c, Csr* A, const T* X, i64 m, T* Y);

struct FistaOut {
  cpcag_solve_trace trace;
};
template <typename T>
void fista_device(Ctx* c, const T* Y, i64 rows, i64 cols, Csr* Lr, Csr* Lc,
                  const cpcag_frpcag_config& cfg, T* X, double* objective_host,
                  cpcag_solve_trace* trace);

// The alternate decoder's operator plans, built ahead of the decode (host
// planning that can overlap device work; see run_idle_work).
struct DecodePrepBase {
  virtual ~DecodePrepBase() = default;
};
template <typename T>
std::unique_ptr<DecodePrepBase> alternate_decode_prepare(Ctx* c, i64 p, i64 n, Csr* Lr, Csr* Lc,
                                                         const cpcag_decoder_config& cfg);

template <typename T>
void alternate_decode_device(Ctx* c, const T* Xt, i64 rho_r, i64 rho_c, const i64* om_r_host,
                             const i64* om_c_host, i64 p, i64 n, Csr* Lr, Csr* Lc, double lk1_r,
                             double lk1_c, const cpcag_decoder_config& cfg, T* X, int* converged,
                             i64* iterations, DecodePrepBase* prep = nullptr);

Csr* kron_reduce_device(Ctx* c, Csr* L, const std::vector<i64>& keep, double pcg_tol,
                        double prune_tol);

void thin_svd_device(Ctx* c, const double* A, i64 m, i64 n, double* U, double* sigma, double* V);
void gram_svd_device(Ctx* c, const double* A, i64 m, i64 n, i64 kvec, double* sigma, double* U, double* V);
template <typename T>
void to_f64_device(Ctx* c, const T* a, i64 n, double* out);
i64 detect_rank_host(const std::vector<double>& s, double thr);
void sym_eig_device(Ctx* c, Csr* A, i64 k, double* evals, double* evecs);
cpcag_spectral_gap spectral_gap_host(const double* evals, i64 order, i64 k);

template <typename T>
void approx_decode_device(Ctx* c, const T* Xt, i64 rho_r, i64 rho_c, const std::vector<i64>& om_r,
                          const std::vector<i64>& om_c, i64 p, i64 n, Csr* Lr, Csr* Lc,
                          const cpcag_approx_config& cfg, T* X, double* U_out, double* s_out, double* V_out,
                          i64 k_cap, i64* k_out);

// decoders.cpp:72-121: S (n x r, fp64 col-major) = harmonic extension of the
// known rows R (|known| x r, leading dimension |known|).
void graph_upsample_device(Ctx* c, Csr* L, const std::vector<i64>& known, const double* R, i64 r,
                           double pcg_tol, i64 pcg_max_iter, double* S);

template <typename T>
void knn_graph_device(Ctx* c, const T* X, i64 x_rows, i64 x_cols, bool axis_rows, i64 K,
                      int kind, double sigma2_override, Csr** W, Csr** L, double* degrees_dev,
                      double* sigma2);

void graph_from_adjacency_device(Ctx* c, Csr* W, int kind, Csr** L, double* degrees_dev);

std::vector<i64> draw_indices(i64 n, i64 take, HostRng rng);

}  // namespace cpcag_cuda
