/*
 * cpcag_cuda.h -- C-ABI of the B200 (sm_100a) implementation of the CPCA hot
 * path (Compressive PCA on graphs, arXiv 1602.02070).
 *
 * This is the drop-in boundary: every entry point replaces one public
 * function of the reference library `cpcag` (the headers under proj/core/include/cpcag,
 * cited per function) with the same argument meaning, the same defaults
 * (documented per argument) and the same error behaviour: a nonzero status
 * maps back to the reference exception type and cpcag_cuda_last_error()
 * returns the reference's message text.
 *
 * Conventions
 *   - Dense matrices are column-major (types.hpp:12-13).  Element type is
 *     double for CPCAG_F64 and float for CPCAG_F32 (`precision` argument).
 *   - Every array argument may be host memory (pageable or pinned) or
 *     device memory of the context's device; the library detects which
 *     (cudaPointerGetAttributes) and stages host arrays through HBM inside
 *     the call.  Device arrays are used in place (no copies).
 *   - Index lists are int64 (types.hpp:10,16).
 *   - Sparse matrices live on the device as cpcag_csr handles (CSR with
 *     int64 row pointers, sorted int32 column indices, fp64 values; the
 *     invariants of sparse.hpp:15-17).  Handles are created from host or
 *     device CSR arrays or returned by the graph routines, and are
 *     immutable.
 *   - Calls on one context are serialised on its stream; contexts are
 *     independent, so distinct threads may use distinct contexts
 *     concurrently.  The last-error text is thread-local.
 *   - No CPU fallback: without a usable sm_100 device every call returns
 *     CPCAG_ERR_CUDA.
 */
#ifndef CPCAG_CUDA_H
#define CPCAG_CUDA_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ------------------------------------------------------------------ status */
enum cpcag_status {
  CPCAG_OK = 0,
  CPCAG_ERR_INVALID_ARGUMENT = 1, /* std::invalid_argument in the reference */
  CPCAG_ERR_RUNTIME = 2,          /* std::runtime_error */
  CPCAG_ERR_OUT_OF_RANGE = 3,     /* std::out_of_range */
  CPCAG_ERR_CUDA = 4              /* device/driver failure (no reference analogue) */
};

enum cpcag_precision { CPCAG_F64 = 0, CPCAG_F32 = 1 };
enum cpcag_axis { CPCAG_AXIS_ROWS = 0, CPCAG_AXIS_COLS = 1 };           /* graph.hpp:11 */
enum cpcag_laplacian_kind { CPCAG_COMBINATORIAL = 0, CPCAG_NORMALIZED = 1 }; /* graph.hpp:10 */
enum cpcag_loss { CPCAG_LOSS_L1 = 0, CPCAG_LOSS_L2 = 1 };                 /* frpcag.hpp:11 */
enum cpcag_spmm_side { CPCAG_LEFT = 0 /* Y = A X */, CPCAG_RIGHT = 1 /* Y = X A */ };

typedef struct cpcag_ctx_s* cpcag_ctx;
typedef struct cpcag_csr_s* cpcag_csr;

/* Thread-local text of the last failure (the reference's exception message). */
const char* cpcag_cuda_last_error(void);
/* Library version string and the compiled device architecture ("sm_100a"). */
const char* cpcag_cuda_version(void);

/* ------------------------------------------------------------------ context */
/* device < 0 selects the current device.  The context owns a non-blocking
 * stream, a workspace cache and pinned staging buffers. */
int cpcag_ctx_create(int device, cpcag_ctx* out);
int cpcag_ctx_destroy(cpcag_ctx ctx);
/* Grows the context's stream-ordered memory pool to at least `bytes` now
 * (the pool keeps freed memory), so the first runs of a workload do not pay
 * for mapping device memory while the pool grows to its peak. */
int cpcag_ctx_reserve(cpcag_ctx ctx, int64_t bytes);
/* Use an external stream (e.g. torch.cuda.current_stream()); NULL restores
 * the context's own stream (a blocking stream, implicitly ordered with the
 * legacy default stream).  To run on the legacy default
 * stream -- torch's default stream, whose handle is 0 -- pass
 * cudaStreamLegacy ((void*)0x1), not NULL. */
int cpcag_ctx_set_stream(cpcag_ctx ctx, void* cuda_stream);
void* cpcag_ctx_stream(cpcag_ctx ctx);
int cpcag_ctx_synchronize(cpcag_ctx ctx);
/* Decoder operator path for this context (tests of both paths on small
 * cases): 0 = automatic (fp32 iterates whose 32-row slab of all columns fits
 * in shared memory: the slab pass; other L2-resident Krylov vectors: one
 * fused pass; else the two-pass band / row-group kernels), 1 = always two
 * passes, 2 = fused whenever its shared-memory slice fits, 3 = slab whenever
 * it applies. */
int cpcag_ctx_set_apply_path(cpcag_ctx ctx, int path);
/* Test hook: the persistent FISTA kernel's tile GEMM, 0 = automatic (fp64
 * tensor cores, DMMA, when the tiling fits), 1 = SIMT fp64 multiply-adds. */
int cpcag_ctx_set_fista_path(cpcag_ctx ctx, int path);
/* Environment test hooks (read by the library; results are the same on
 * either side of each, the tests compare them): CPCAG_FISTA_PERSIST=0 runs
 * dense FRPCAG through the per-kernel path instead of the one persistent
 * kernel; CPCAG_KNN=tc|simt forces the kNN tile path; CPCAG_KNN_PASS2=0 sends
 * every uncertified row of the tensor-core kNN to the exact fp64 kernel;
 * CPCAG_GAP_LANCZOS=1 takes the Lanczos spectral gap inside run_pipeline at
 * any size; CPCAG_TRACE=1 prints stage marks to stderr. */
/* Test hook: the cooperative power iteration (operators too large for one
 * CTA), 0 = automatic (three, else two products per grid barrier through the
 * dense powers of the operator when a CTA's rows of them fit in shared
 * memory), 1 = always one product per barrier, 2 = at most two.
 * last_power_path: 3 / 2 / 1 products per barrier for the most recent power
 * iteration, 0 when it ran in the single-CTA kernel. */
int cpcag_ctx_set_power_path(cpcag_ctx ctx, int path);
int cpcag_ctx_last_power_path(cpcag_ctx ctx);
/* The path (1, 2 or 3 as above) the most recently planned decoder operator
 * took; 0 before any. */
int cpcag_ctx_last_apply_path(cpcag_ctx ctx);
/* Number of kernels this context has launched since creation (or reset). */
int64_t cpcag_ctx_launch_count(cpcag_ctx ctx);
void cpcag_ctx_reset_launch_count(cpcag_ctx ctx);

/* Per-kernel device timing (CUDA events around every launch of the hot
 * kernels, on the context stream).  Used by bench.py for live roofline
 * figures; off by default. */
int cpcag_ctx_enable_kernel_timing(cpcag_ctx ctx, int enable);
/* Restrict timing to a comma-separated list of kernel tags (NULL/"" = all). */
int cpcag_ctx_kernel_timing_filter(cpcag_ctx ctx, const char* tags_csv);
int cpcag_ctx_reset_kernel_timing(cpcag_ctx ctx);
int cpcag_ctx_kernel_timing_count(cpcag_ctx ctx);
/* Entry `index` (0 <= index < count): kernel tag, launches, summed ms. */
int cpcag_ctx_kernel_timing(cpcag_ctx ctx, int index, char* tag, int64_t tag_cap, int64_t* launches,
                            double* total_ms);

/* ------------------------------------------------------------------ sparse */
/* SparseMatrix from CSR arrays (sparse.hpp:18-66).  The arrays must already
 * satisfy the CSR invariants (monotone row_ptr, strictly increasing columns
 * per row, finite values); violations return CPCAG_ERR_INVALID_ARGUMENT.
 * Exact zeros are dropped as SparseMatrix::from_triplets does. */
int cpcag_csr_create(cpcag_ctx ctx, int64_t rows, int64_t cols, int64_t nnz,
                     const int64_t* row_ptr, const int64_t* col_idx, const double* values,
                     cpcag_csr* out);
int cpcag_csr_destroy(cpcag_csr a);
int cpcag_csr_info(cpcag_csr a, int64_t* rows, int64_t* cols, int64_t* nnz);
/* Copy the CSR out (host or device destinations; any may be NULL). */
int cpcag_csr_export(cpcag_ctx ctx, cpcag_csr a, int64_t* row_ptr, int64_t* col_idx,
                     double* values);
/* 1 when A == A^T bit for bit (what every Laplacian built here satisfies). */
int cpcag_csr_is_symmetric(cpcag_csr a);

/* SparseMatrix::multiply(Matrix) / right_multiply(Matrix)
 * (sparse.hpp:41-45, sparse.cpp:87-111).  side = CPCAG_LEFT: Y = A X with X
 * (A.cols x m); CPCAG_RIGHT: Y = X A with X (m x A.rows).  Per output entry
 * the accumulation order is the reference's (CSR order, starting from 0), so
 * CPCAG_F64 results are bit-identical to the reference loop. */
int cpcag_cuda_spmm(cpcag_ctx ctx, cpcag_csr A, int side, int precision, int64_t x_rows,
                    int64_t x_cols, const void* X, void* Y);
/* SparseMatrix::multiply(Vector) (sparse.cpp:73-85). */
int cpcag_cuda_spmv(cpcag_ctx ctx, cpcag_csr A, int precision, int64_t n, const void* x, void* y);

/* power_iteration_norm (solvers.hpp:90-91, solvers.cpp:29-53); defaults in
 * the reference: tol 1e-9, seed 0, max_iter 50000. */
int cpcag_cuda_power_norm(cpcag_ctx ctx, cpcag_csr A, double tol, uint64_t seed,
                          int64_t max_iter, double* out);

/* pcg_solve(const SparseMatrix&, b, x, opt, jacobi) (solvers.hpp:82-86,
 * solvers.cpp:19-27): x is the start iterate and receives the solution. */
int cpcag_cuda_pcg_solve(cpcag_ctx ctx, cpcag_csr A, const double* b, double* x, int64_t n,
                         double tol, int64_t max_iter, int jacobi, int64_t* iterations,
                         int* converged, double* relative_residual);

/* ------------------------------------------------------------------ graphs */
/* build_knn_graph (graph.hpp:29-31, graph.cpp:47-135).  X is x_rows x x_cols;
 * axis selects whether points are rows or columns.  Defaults in the
 * reference: kind = combinatorial, sigma2_override = 0 (automatic).
 * Outputs: adjacency W and Laplacian L handles, degrees (length n, host or
 * device), sigma2.  The neighbour sets follow the reference's canonical fp64
 * distance d2 = max(0, g_ii + g_jj - 2 g_ij) with ties toward the lower
 * index, bit-exactly. */
int cpcag_cuda_knn_graph(cpcag_ctx ctx, int precision, const void* X, int64_t x_rows,
                         int64_t x_cols, int axis, int64_t K, int kind, double sigma2_override,
                         cpcag_csr* adjacency, cpcag_csr* laplacian, double* degrees,
                         double* sigma2);
/* The K nearest neighbours per point (ascending (d2, index)) without the
 * graph assembly; nbr and nbr_d2 are n x K row-major. */
int cpcag_cuda_knn(cpcag_ctx ctx, int precision, const void* X, int64_t x_rows, int64_t x_cols,
                   int axis, int64_t K, int64_t* nbr, double* nbr_d2);

/* graph_from_adjacency (graph.hpp:35-36, graph.cpp:137-154). */
int cpcag_cuda_graph_from_adjacency(cpcag_ctx ctx, cpcag_csr W, int kind, cpcag_csr* laplacian,
                                    double* degrees);

/* kron_reduce (graph.hpp:50-51, graph.cpp:170-235).  Reference defaults:
 * pcg_tol 1e-12, prune_tol 1e-12 (run_pipeline passes 1e-11). */
int cpcag_cuda_kron_reduce(cpcag_ctx ctx, cpcag_csr L, const int64_t* keep, int64_t n_keep,
                           double pcg_tol, double prune_tol, cpcag_csr* out);

/* ------------------------------------------------------------------ sampling */
/* draw_plan (sampling.hpp:39-40, sampling.cpp:48-64).  Host-side by design:
 * it is O(rho) integer work on the reference's counter RNG and its output
 * must be bit-identical; omega_r/omega_c receive the draw order. */
int cpcag_cuda_draw_plan(int64_t p, int64_t n, int64_t rho_r, int64_t rho_c, uint64_t seed,
                         int64_t* omega_r, int64_t* omega_c);
/* subsample (sampling.hpp:43, sampling.cpp:66-75): out(i,j) = Y(om_r[i], om_c[j]). */
int cpcag_cuda_subsample(cpcag_ctx ctx, int precision, const void* Y, int64_t p, int64_t n,
                         const int64_t* omega_r, int64_t rho_r, const int64_t* omega_c,
                         int64_t rho_c, void* out);

/* ------------------------------------------------------------------ FRPCAG */
typedef struct cpcag_frpcag_config { /* FrpcagConfig, frpcag.hpp:15-22 */
  double gamma_r;   /* default 1 */
  double gamma_c;   /* default 1 */
  int loss;         /* CPCAG_LOSS_L1 (default) or CPCAG_LOSS_L2 */
  double tol;       /* default 1e-10: stop when ||Z+ - Z||^2 < tol ||Z||^2 */
  int64_t max_iter; /* default 500 */
  double step;      /* 0 = auto: 1 / (2 gc ||Lc|| + 2 gr ||Lr||) */
} cpcag_frpcag_config;

typedef struct cpcag_solve_trace { /* SolveTrace, frpcag.hpp:24-30 (objective separate) */
  int64_t iterations;
  int converged;
  double final_rel_change;
  double step;
} cpcag_solve_trace;

/* objective / prox_l1 / prox_l2 / grad_g (frpcag.hpp:32-43). */
int cpcag_cuda_objective(cpcag_ctx ctx, int precision, const void* X, const void* Y,
                         int64_t rows, int64_t cols, cpcag_csr Lr, cpcag_csr Lc,
                         const cpcag_frpcag_config* cfg, double* out);
int cpcag_cuda_prox(cpcag_ctx ctx, int precision, int loss, const void* Z, const void* Y,
                    int64_t count, double lam, void* out);
int cpcag_cuda_grad_g(cpcag_ctx ctx, int precision, const void* Z, int64_t rows, int64_t cols,
                      cpcag_csr Lr, cpcag_csr Lc, const cpcag_frpcag_config* cfg, void* G);

/* fista_solve (frpcag.hpp:46-47, frpcag.cpp:62-112).  Y is rows x cols; X
 * receives the last prox output; objective (may be NULL) receives one value
 * per iteration (capacity cfg->max_iter). */
int cpcag_cuda_fista(cpcag_ctx ctx, int precision, const void* Y, int64_t rows, int64_t cols,
                     cpcag_csr Lr, cpcag_csr Lc, const cpcag_frpcag_config* cfg, void* X,
                     double* objective, cpcag_solve_trace* trace);

/* ------------------------------------------------------------------ decoder */
typedef struct cpcag_decoder_config { /* DecoderConfig fields used by alternate_decode */
  double gamma;         /* default 1; scaled by 1/lambda_{k+1} per side */
  double pcg_tol;       /* default 1e-10 */
  int64_t pcg_max_iter; /* default 5000 */
  /* Extension (not in the reference): storage of the CG Krylov vectors R, P,
   * AP for fp32 data.  0 (default): fp64 Krylov vectors, fp32 X -- within
   * 1.3e-6 of the fp64 solve at config 3, where fp32 Krylov vectors drift
   * 7-8e-4 (tools/cfg3_precision.py).  CPCAG_F32: every vector fp32 (faster;
   * for well-conditioned systems).  Ignored for fp64 data. */
  int krylov_precision;
} cpcag_decoder_config;

/* alternate_decode (decoders.hpp:59-62, decoders.cpp:145-186): CG on
 * M o X + gbar_c X Lc + gbar_r Lr X = scatter(Xt), X0 = 0, no
 * preconditioner, gbar = gamma / lambda_k1 (SpectralGap::lambda_k1).
 * Xt is rho_r x rho_c; X receives the p x n solution.  Non-convergence is a
 * flag, not an error (decoders.cpp:185). */
int cpcag_cuda_alternate_decode(cpcag_ctx ctx, int precision, const void* Xt, int64_t rho_r,
                                int64_t rho_c, const int64_t* omega_r, const int64_t* omega_c,
                                int64_t p, int64_t n, cpcag_csr Lr, cpcag_csr Lc,
                                double lambda_k1_r, double lambda_k1_c,
                                const cpcag_decoder_config* cfg, void* X, int* converged,
                                int64_t* iterations);

/* The decoder's operator (decoders.cpp:160-170): AP = gbar_c P Lc + gbar_r Lr P
 * + M o P (M = the plan's sampling mask), *dot = <P, AP>; P and AP are p x n.
 * The two kernels the CG runs per iteration (fp64: bit-identical per entry
 * to the reference loop). */
int cpcag_cuda_decoder_apply(cpcag_ctx ctx, int precision, const void* P, int64_t p, int64_t n, cpcag_csr Lr,
                             cpcag_csr Lc, const int64_t* omega_r, int64_t rho_r, const int64_t* omega_c,
                             int64_t rho_c, double gbar_r, double gbar_c, void* AP, double* dot);

/* sym_eig (eigs.hpp:22, eigs.cpp:34-51): the k smallest eigenpairs of the
 * symmetric part 0.5 (A + A^T) of a CSR matrix, by a dense eigensolver on the
 * device (like the reference's; n <= 46340).  eigenvalues (k, ascending);
 * eigenvectors (n x k col-major, may be NULL) with each column's first entry
 * above 1e-12 of its peak made positive. */
int cpcag_cuda_sym_eig(cpcag_ctx ctx, cpcag_csr A, int64_t k, double* eigenvalues, double* eigenvectors);

/* The k smallest eigenvalues of a large sparse symmetric matrix (eigenvalues
 * only; replaces the dense sym_eig of eigs.cpp:34-51 where it is infeasible,
 * i.e. the spectral gaps of pipeline.cpp:343-349 on 1e5-1e6-node graphs):
 * Lanczos with full reorthogonalisation on sigma I - A (sigma = Gershgorin
 * bound), stopping when the k extreme Ritz residuals are <= tol * sigma.
 * eigenvalues: k, ascending.  iterations (may be NULL): Lanczos steps.
 * Errors: invalid_argument for a non-square A or k out of range;
 * runtime_error "lanczos: not converged after N steps". */
int cpcag_cuda_sym_eigvals_lanczos(cpcag_ctx ctx, cpcag_csr A, int64_t k, double tol, int64_t max_iter,
                                   uint64_t seed, double* eigenvalues, int64_t* iterations);

/* SpectralGap (graph.hpp:53-58). */
typedef struct cpcag_spectral_gap {
  int64_t k;
  double lambda_k, lambda_k1, ratio;
} cpcag_spectral_gap;

/* DecoderConfig fields the approximate decoder reads (decoders.hpp:13-22). */
typedef struct cpcag_approx_config {
  double delta_for_scaling; /* default 0; sigma scale sqrt(np / (rho_r rho_c (1 - delta))) */
  double rank_threshold;    /* default 0.1; k = #{sigma_i / sigma_1 >= threshold} */
  double pcg_tol;           /* default 1e-10 (upsampling solves) */
  int64_t pcg_max_iter;     /* default 5000 */
} cpcag_approx_config;

/* thin_svd (eigs.cpp:53-57): A (m x n, fp64 col-major) = U diag(sigma) V^T
 * with q = min(m, n): U m x q, sigma q (descending), V n x q.  Column signs
 * are the solver's (the reference's JacobiSVD leaves them unspecified too).
 * Non-finite input -> CPCAG_ERR_INVALID_ARGUMENT "thin_svd: non-finite input". */
int cpcag_cuda_thin_svd(cpcag_ctx ctx, const double* A, int64_t m, int64_t n, double* U, double* sigma,
                        double* V);

/* graph_upsample (decoders.hpp:37-38, decoders.cpp:72-121): S (n x r, fp64
 * col-major) equals R (n_known x r) on the rows `known` and solves
 * L_aa S_a = -L_ab R on the rest, one Jacobi PCG per column (batched).
 * Errors as the reference: index out of range / duplicate index
 * (invalid argument); a component without a known node, an interior solve
 * that does not converge, PCG breakdown (runtime). */
int cpcag_cuda_graph_upsample(cpcag_ctx ctx, cpcag_csr L, const int64_t* known, int64_t n_known, const double* R,
                              int64_t r, double pcg_tol, int64_t pcg_max_iter, double* S);

/* approx_decode (decoders.hpp:64-72, decoders.cpp:188-225): thin SVD of Xt,
 * rank k at sigma_k / sigma_1 >= rank_threshold, graph_upsample of both
 * factors, unit columns, sign alignment, sigma rescaling, X = U S V^T (p x n,
 * `precision`).  *k receives the rank; when 0 < k <= k_cap the factors are
 * also written (fp64: U p x k, sigma k, V n x k; each pointer may be NULL). */
int cpcag_cuda_approx_decode(cpcag_ctx ctx, int precision, const void* Xt, int64_t rho_r, int64_t rho_c,
                             const int64_t* omega_r, const int64_t* omega_c, int64_t p, int64_t n, cpcag_csr Lr,
                             cpcag_csr Lc, const cpcag_approx_config* cfg, void* X, double* U, double* sigma,
                             double* V, int64_t k_cap, int64_t* k);

/* 3xTF32 tensor-core Gram matrix (tcgen05.mma kind::tf32) of n points given
 * as the rows of the n x d row-major fp64 array P; G is n x n row-major fp32.
 * The kNN filter stage's arithmetic, exposed for verification. */
int cpcag_cuda_gram_tf32x3(cpcag_ctx ctx, const double* P, int64_t n, int64_t d, float* G);

/* ------------------------------------------------------------------ column-sharded decoder */
/* alternate_decode (decoders.cpp:145-186) split over the GPUs of one node by
 * column blocks of X: one process per GPU, rank g owns
 * columns [bounds[g], bounds[g+1]) (bounds: nranks + 1 ascending entries,
 * bounds[0] = 0, bounds[nranks] = n, identical on every rank).  Per CG
 * iteration the columns of the search direction that other ranks' L_c rows
 * reference (the halo) move by one grouped ncclSend/ncclRecv, overlapped
 * with the block-local L_r pass; the two CG dot products are ncclAllReduce'd
 * on device scalars.  Xt, omega, Lr and Lc are replicated on every rank;
 * X_block receives this rank's p x (bounds[g+1] - bounds[g]) block.  Entry
 * arithmetic equals the one-GPU decoder's (fp64: bit-identical applies); only
 * the dot products' summation order differs. */
typedef struct cpcag_comm_s* cpcag_comm;
typedef struct cpcag_shard_stats {
  int64_t halo_cols;          /* columns of P this rank receives per iteration */
  int64_t send_cols;          /* columns of P this rank sends per iteration */
  double bytes_per_iteration; /* (halo_cols + send_cols) * p * sizeof(Krylov element) */
  double exchange_ms;         /* sum over iterations of the exchange (pack + NCCL) time, if measured */
  int measure_exchange;       /* in: time the exchange with events on the communication stream */
} cpcag_shard_stats;
/* ncclGetUniqueId (128 bytes) on one rank; every rank passes the same id to
 * cpcag_cuda_comm_create (the bootstrap is the caller's, e.g. torch.distributed). */
int cpcag_cuda_comm_unique_id(void* id_out);
int cpcag_cuda_comm_create(cpcag_ctx ctx, const void* id, int nranks, int rank, cpcag_comm* out);
int cpcag_cuda_comm_destroy(cpcag_comm comm);
int cpcag_cuda_alternate_decode_sharded(cpcag_ctx ctx, cpcag_comm comm, int precision, const void* Xt,
                                        int64_t rho_r, int64_t rho_c, const int64_t* omega_r,
                                        const int64_t* omega_c, int64_t p, int64_t n, cpcag_csr Lr, cpcag_csr Lc,
                                        double lambda_k1_r, double lambda_k1_c, const cpcag_decoder_config* cfg,
                                        const int64_t* bounds, void* X_block, int* converged, int64_t* iterations,
                                        cpcag_shard_stats* stats);
/* The same algorithm for `nranks` ranks emulated in one process on one GPU
 * (the exchange is device copies, the all-reduce a fixed-order sum; the ranks
 * run phase by phase, no kernel waits for another).  X receives the whole
 * p x n solution; stats describe rank 0.  For tests of the multi-rank logic. */
int cpcag_cuda_alternate_decode_sharded_emulated(cpcag_ctx ctx, int nranks, int precision, const void* Xt,
                                                 int64_t rho_r, int64_t rho_c, const int64_t* omega_r,
                                                 const int64_t* omega_c, int64_t p, int64_t n, cpcag_csr Lr,
                                                 cpcag_csr Lc, double lambda_k1_r, double lambda_k1_c,
                                                 const cpcag_decoder_config* cfg, const int64_t* bounds, void* X,
                                                 int* converged, int64_t* iterations, cpcag_shard_stats* stats);
/* fista_solve (frpcag.hpp:46-47, frpcag.cpp:62-112) with the compressed
 * matrix split into contiguous column blocks, one per rank (SURVEY.md 8e:
 * "FISTA scalars all-reduced, X~ all-gathered").  Y (rows x cols), Lr, Lc and
 * cfg are the same on every rank; bounds has nranks + 1 ascending entries
 * 0 ... cols.  Each iteration a rank forms its block of S from the full Z,
 * the blocks are all-gathered (grouped NCCL send/recv), the five scalars of
 * the objective and the stopping rule are all-reduced on the device, and
 * every rank forms the full Z_next locally.  X_block receives this rank's
 * rows x (bounds[rank + 1] - bounds[rank]) block; objective and trace as
 * cpcag_cuda_fista (identical on every rank).  S matches the single-GPU CSR
 * path bit for bit per iteration; the scalars are summed in another order.
 * Errors: the reference's fista messages, plus "sharded fista: ..." for a
 * bad partition. */
int cpcag_cuda_fista_sharded(cpcag_ctx ctx, cpcag_comm comm, int precision, const void* Y, int64_t rows,
                             int64_t cols, cpcag_csr Lr, cpcag_csr Lc, const cpcag_frpcag_config* cfg,
                             const int64_t* bounds, void* X_block, double* objective, cpcag_solve_trace* trace);
/* The same for `nranks` ranks emulated in one process on one GPU (device
 * copies for the all-gather, a rank-ordered sum for the all-reduce, ranks run
 * phase by phase).  X receives the whole rows x cols solution. */
int cpcag_cuda_fista_sharded_emulated(cpcag_ctx ctx, int nranks, int precision, const void* Y, int64_t rows,
                                      int64_t cols, cpcag_csr Lr, cpcag_csr Lc, const cpcag_frpcag_config* cfg,
                                      const int64_t* bounds, void* X, double* objective, cpcag_solve_trace* trace);
/* Host only (no device): the halo plan of `rank` for L_c's CSR structure
 * (row_ptr n + 1, col_idx).  recv_counts[q] / send_counts[q]: columns this
 * rank receives from / sends to rank q; recv_cols (capacity n): their global
 * indices grouped by owner, ascending; send_cols (capacity
 * nranks * block width): local indices (j - bounds[rank]) grouped by
 * destination.  Either column array may be NULL. */
int cpcag_halo_plan(const int64_t* row_ptr, const int64_t* col_idx, int64_t n, const int64_t* bounds, int nranks,
                    int rank, int64_t* recv_counts, int64_t* send_counts, int64_t* recv_cols, int64_t* send_cols);

/* ------------------------------------------------------------------ pipeline */
typedef struct cpcag_pipeline_config { /* PipelineConfig subset, pipeline.hpp:36-63 */
  int64_t knn;               /* default 10 */
  int laplacian;             /* default combinatorial */
  double sigma2;             /* 0 = automatic */
  int64_t a, b;              /* downsampling: rho_c = ceil(n/a), rho_r = ceil(p/b) */
  int64_t rho_r_override, rho_c_override;
  double kron_pcg_tol;       /* default 1e-11 */
  cpcag_frpcag_config frpcag;
  cpcag_decoder_config decoder;
  double lambda_k1_r, lambda_k1_c; /* SpectralGap::lambda_k1; <= 0: computed as the reference does
                                      (sym_eig of the full Laplacian, k = max(1, detected rank)) */
  uint64_t seed;
  int decoder_variant;       /* DecoderVariant (decoders.hpp:11): CPCAG_DECODER_ALTERNATE or _APPROX */
  cpcag_approx_config approx; /* the approximate decoder's DecoderConfig fields */
  int task;                  /* Task (pipeline.hpp:18): CPCAG_TASK_LOWRANK (default), _CLUSTER or _BOTH */
  int64_t n_clusters;        /* clustering: k (0 = max(1, detected rank)), pipeline.cpp:374 */
  int64_t kmeans_restarts;   /* default 10; < 1 is rejected (clustering.cpp:129) */
} cpcag_pipeline_config;

enum { CPCAG_TASK_LOWRANK = 0, CPCAG_TASK_CLUSTER = 1, CPCAG_TASK_BOTH = 2 };

enum { CPCAG_DECODER_IDEAL = 0, CPCAG_DECODER_ALTERNATE = 1, CPCAG_DECODER_APPROX = 2 };

/* ------------------------------------------------------------------ GLR1 I/O
 * The reference's binary container (io.hpp:14-30, io.cpp:16-230): magic
 * "GLR1", u64 block kind (1 dense, 2 CSR, 3 factors), u64 dimensions, raw
 * little-endian arrays.  Dense blocks stream through pinned double buffers
 * straight into/out of device memory (fp64 on disk; fp32 buffers are
 * narrowed/widened on the device).  Buffers may be host or device memory.
 * Errors are std::runtime_error with the reference's texts: "<path>: cannot
 * open for reading", "<path>: not a GLR1 container (bad magic)", "<path>: not
 * a dense-matrix block", "<path>: truncated data section", ... */
/* kind and dims of a GLR1 file (dims: 2 dense rows/cols, 3 CSR rows/cols/nnz,
 * 4 factors p/n/k/scale flag). */
int cpcag_glr1_info(const char* path, int64_t* kind, int64_t* dims);
/* load_matrix / save_matrix, format glr1 (io.cpp:88-118). */
int cpcag_cuda_load_matrix_glr1(cpcag_ctx ctx, const char* path, int precision, void* out, int64_t rows,
                                int64_t cols);
int cpcag_cuda_save_matrix_glr1(cpcag_ctx ctx, const char* path, int precision, const void* M, int64_t rows,
                                int64_t cols);
/* load_sparse / save_sparse (io.cpp:151-188); a non-canonical file is
 * rebuilt like SparseMatrix::from_triplets (sorted, duplicates summed, exact
 * zeros dropped). */
int cpcag_cuda_load_sparse_glr1(cpcag_ctx ctx, const char* path, cpcag_csr* out);
int cpcag_cuda_save_sparse_glr1(cpcag_ctx ctx, cpcag_csr A, const char* path);
/* save_factors / load_factors (io.cpp:200-230): U p x k, sigma k, V n x k. */
int cpcag_cuda_save_factors_glr1(cpcag_ctx ctx, const char* path, int64_t p, int64_t n, int64_t k,
                                 int scale_applied, const double* U, const double* sigma, const double* V);
int cpcag_cuda_load_factors_glr1(cpcag_ctx ctx, const char* path, int64_t p, int64_t n, int64_t k,
                                 int* scale_applied, double* U, double* sigma, double* V);

/* ------------------------------------------------------------------ clustering
 * kmeans (clustering.hpp:26-29, clustering.cpp:40-137) on the COLUMNS of X
 * (rows x n, col-major, fp64 or fp32 widened to fp64): k-means++ seeding,
 * Lloyd iterations, best of `restarts` by within-cluster sum of squares
 * (written to wcss, may be NULL), emptied clusters re-seeded from the
 * farthest point; deterministic for a seed (reference counter RNG streams
 * derive(seed, restart)).  assignments: n ints in [0, k).
 * Errors: "kmeans: k must be >= 1", "kmeans: more clusters than points",
 * "kmeans: restarts must be >= 1" (invalid_argument). */
int cpcag_cuda_kmeans(cpcag_ctx ctx, int precision, const void* X, int64_t rows, int64_t n, int64_t k,
                      int64_t restarts, uint64_t seed, int64_t max_iter, int* assignments, double* wcss);
/* decode_labels (clustering.hpp:31-35, clustering.cpp:139-160): upsample the
 * indicator of the sampled-column labels (rho_c, values in [0, k)) over L_c
 * with known set omega_c, then row-wise max pooling (ties: lowest column).
 * labels: n ints. */
int cpcag_cuda_decode_labels(cpcag_ctx ctx, const int* sampled, int64_t rho_c, int64_t k, const int64_t* omega_c,
                             int64_t n, cpcag_csr Lc, double pcg_tol, int64_t pcg_max_iter, int* labels);
/* clustering_error (clustering.hpp:37-39, clustering.cpp:220-238): host. */
int cpcag_clustering_error(const int* pred, const int* truth, int64_t n, int64_t k_pred, int64_t k_truth,
                           double* out);

/* Optional outputs of run_pipeline: the approximate decoder's factors
 * (PipelineReport::factors, pipeline.hpp:91): fp64 U (p x k), sigma (k),
 * V (n x k) when k <= k_cap; and the decoded cluster labels
 * (PipelineReport::labels, pipeline.hpp:89; n ints, cluster/both tasks). */
typedef struct cpcag_pipeline_factors {
  double* U;
  double* sigma;
  double* V;
  int64_t k_cap;
  int* labels;
} cpcag_pipeline_factors;

typedef struct cpcag_pipeline_report { /* PipelineReport subset, pipeline.hpp:73-94 */
  int64_t p, n, rho_r, rho_c;
  cpcag_solve_trace trace;
  int decoder_converged;
  int64_t decoder_iterations;
  int64_t detected_rank;  /* detect_rank(thin_svd(Xt).sigma, rank_threshold), pipeline.cpp:319-320 */
  int64_t factors_k;      /* approximate decoder: rank of the factors (0 otherwise) */
  int has_factors;
  double lambda_k1_r, lambda_k1_c; /* gaps the alternate decoder used (supplied or computed) */
  /* Stage timings in ms (device events), in the reference's stage order:
   * graphs, plan, subsample, kron, solve, decode (pipeline.cpp:273-350). */
  double stage_ms[6];
  double cluster_ms;      /* the "cluster" stage (cluster/both tasks) */
  int64_t n_clusters;     /* k the clustering stage used */
} cpcag_pipeline_report;

/* run_pipeline (pipeline.cpp:228-391): graphs (row graph from W_r when
 * given, else kNN over rows; column graph from W_c when given, else kNN over
 * columns) -> plan -> subsample -> Kron -> FISTA -> detected rank -> decode
 * with the alternate or the approximate decoder (lowrank/both tasks) ->
 * k-means on Xt + decode_labels (cluster/both tasks, labels into
 * factors->labels).  Y is p x n; X may be NULL for the cluster task.
 * Xt (rho_r x rho_c) and X (p x n) receive the compressed and decoded
 * solutions; omega_r/omega_c (may be NULL) receive the plan; objective (may
 * be NULL) the FISTA trace; factors (may be NULL) the approximate decoder's
 * factors. */
int cpcag_cuda_run_pipeline(cpcag_ctx ctx, int precision, const void* Y, int64_t p, int64_t n,
                            cpcag_csr W_r, cpcag_csr W_c, const cpcag_pipeline_config* cfg,
                            void* Xt, void* X, int64_t* omega_r, int64_t* omega_c,
                            double* objective, cpcag_pipeline_report* report,
                            const cpcag_pipeline_factors* factors);

#ifdef __cplusplus
}
#endif
#endif /* CPCAG_CUDA_H */
