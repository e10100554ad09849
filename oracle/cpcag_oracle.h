/*
 * cpcag_oracle.h -- C ABI of the CPU oracle.
 *
 * TEST INFRASTRUCTURE ONLY.  This is a CPU restatement of the reference
 * cpcag hot path (/root/reference/proj/core/src/ sources), used as the checker
 * for the CUDA product path.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load it.  The product
 * library (libcpcag_cuda.so) never links or calls it.
 *
 * Parity pins: the reference itself cannot be compiled here (Eigen3, doctest
 * and vendor/json.hpp are absent).  The oracle is pinned
 * against every known-answer test the reference ships for this path
 * (proj/tests/test_numeric.cpp, proj/tests/test_graph.cpp) and the SPEC.md
 * examples, transcribed in tests/test_oracle_golden.py, plus the dense
 * oracles of proj/tests/oracles.hpp restated with numpy/LAPACK.
 *
 * All dense matrices are column-major fp64 (types.hpp:12-13).  Every call
 * returns 0 on success or a status code (1 invalid_argument, 2
 * runtime_error, 3 out_of_range) with the reference's message available
 * from ora_last_error().
 */
#ifndef CPCAG_ORACLE_H
#define CPCAG_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct ora_csr ora_csr;

const char* ora_last_error(void);
void ora_set_threads(int n);
int ora_get_threads(void);

/* CSR (sparse.cpp:10-46, 48-54, 122-207) */
int ora_csr_from_triplets(int64_t rows, int64_t cols, int64_t n, const int64_t* ti,
                          const int64_t* tj, const double* tv, double drop_below, ora_csr** out);
int ora_csr_from_csr(int64_t rows, int64_t cols, const int64_t* row_ptr, const int64_t* col_idx,
                     const double* values, ora_csr** out);
int ora_csr_from_dense(const double* D, int64_t rows, int64_t cols, double drop_below,
                       ora_csr** out);
void ora_csr_free(ora_csr* a);
int64_t ora_csr_rows(const ora_csr* a);
int64_t ora_csr_cols(const ora_csr* a);
int64_t ora_csr_nnz(const ora_csr* a);
void ora_csr_export(const ora_csr* a, int64_t* row_ptr, int64_t* col_idx, double* values);
int ora_csr_submatrix(const ora_csr* a, const int64_t* rows, int64_t nr, const int64_t* cols,
                      int64_t nc, ora_csr** out);
void ora_csr_row_sums(const ora_csr* a, double* out);
int ora_csr_components(const ora_csr* a, int64_t* labels, int64_t* n_comp);

/* SpMV / SpMM (sparse.cpp:73-111) */
int ora_spmv(const ora_csr* a, const double* x, int64_t n, double* y);
int ora_spmm_left(const ora_csr* a, const double* X, int64_t xr, int64_t xc, double* Y);
int ora_spmm_right(const ora_csr* a, const double* X, int64_t xr, int64_t xc, double* Y);

/* Counter RNG (rng.hpp:11-68) */
uint64_t ora_rng_mix(uint64_t z);
void ora_rng_u64(uint64_t seed, int64_t count, uint64_t* out);
void ora_rng_gaussian(uint64_t seed, int64_t count, double* out);
uint64_t ora_rng_derive_seed(uint64_t seed, uint64_t stream);

/* Solvers (solvers.hpp:33-74, solvers.cpp:7-53) */
int ora_pcg_solve(const ora_csr* A, const double* b, double* x, int64_t n, double tol,
                  int64_t max_iter, int jacobi, int64_t* iterations, int* converged,
                  double* rel_res);
int ora_power_iteration_norm(const ora_csr* A, double tol, uint64_t seed, int64_t max_iter,
                             double* out);

/* Graphs (graph.cpp:16-154, 170-235) */
int ora_knn_graph(const double* X, int64_t rows, int64_t cols, int axis_rows, int64_t K,
                  int normalized, double sigma2_override, ora_csr** adjacency,
                  ora_csr** laplacian, double* degrees, double* sigma2);
int ora_knn_neighbors(const double* X, int64_t rows, int64_t cols, int axis_rows, int64_t K,
                      int64_t* nbr, double* nbr_d2);
int ora_graph_from_adjacency(const ora_csr* W, int normalized, ora_csr** laplacian,
                             double* degrees);
/* decoders.cpp:72-121: S (n x r, col-major) = harmonic extension of the known
 * rows R (n_known x r). */
int ora_graph_upsample(const ora_csr* L, const int64_t* known, int64_t n_known, const double* R, int64_t r,
                       double pcg_tol, int64_t pcg_max_iter, double* S);
/* Exact kNN lists of the query points only (full-size spot checks). */
int ora_knn_rows(const double* X, int64_t rows, int64_t cols, int axis_rows, int64_t K, const int64_t* query,
                 int64_t nq, int64_t* nbr, double* nbr_d2);
int ora_kron_reduce(const ora_csr* L, const int64_t* keep, int64_t nkeep, double pcg_tol,
                    double prune_tol, ora_csr** out);

/* Sampling (sampling.cpp:35-75) */
int ora_draw_plan(int64_t p, int64_t n, int64_t rho_r, int64_t rho_c, uint64_t seed,
                  int64_t* omega_r, int64_t* omega_c);
int ora_subsample(const double* Y, int64_t p, int64_t n, const int64_t* omega_r, int64_t rho_r,
                  const int64_t* omega_c, int64_t rho_c, double* out);

/* FRPCAG (frpcag.cpp:23-112) */
typedef struct ora_frpcag_cfg {
  double gamma_r, gamma_c;
  int loss_l2; /* 0 = l1, 1 = l2 */
  double tol;
  int64_t max_iter;
  double step; /* <= 0: auto */
} ora_frpcag_cfg;

int ora_objective(const double* X, const double* Y, int64_t r, int64_t c, const ora_csr* Lr,
                  const ora_csr* Lc, const ora_frpcag_cfg* cfg, double* out);
int ora_prox_l1(const double* Z, const double* Y, int64_t count, double lam, double* out);
int ora_prox_l2(const double* Z, const double* Y, int64_t count, double lam, double* out);
int ora_grad_g(const double* Z, int64_t r, int64_t c, const ora_csr* Lr, const ora_csr* Lc,
               const ora_frpcag_cfg* cfg, double* G);
int ora_fista_solve(const double* Y, int64_t r, int64_t c, const ora_csr* Lr, const ora_csr* Lc,
                    const ora_frpcag_cfg* cfg, double* X_out, double* objective,
                    int64_t* iterations, int* converged, double* final_rel_change,
                    double* step_used);

/* Alternate decoder (decoders.cpp:145-186) */
int ora_alternate_decode(const double* Xt, int64_t rho_r, int64_t rho_c, const int64_t* omega_r,
                         const int64_t* omega_c, int64_t p, int64_t n, const ora_csr* Lr,
                         const ora_csr* Lc, double lambda_k1_r, double lambda_k1_c, double gamma,
                         double pcg_tol, int64_t pcg_max_iter, double* X_out, int* converged,
                         int64_t* iterations);

/* One CG iteration budget-limited apply of the decoder normal operator, for
 * per-iteration CPU timing at sizes where a full solve is too slow. */
int ora_decoder_apply(const double* X, int64_t p, int64_t n, const int64_t* omega_r,
                      int64_t rho_r, const int64_t* omega_c, int64_t rho_c, const ora_csr* Lr,
                      const ora_csr* Lc, double gbar_r, double gbar_c, double* out);

/* kmeans (clustering.cpp:40-137): assignments n; wcss of the kept restart. */
int ora_kmeans(const double* X, int64_t rows, int64_t n, int64_t k, int64_t restarts, uint64_t seed,
               int64_t max_iter, int* assignments, double* wcss);
/* clustering_error (clustering.cpp:222-238). */
int ora_clustering_error(const int* pred, const int* truth, int64_t n, int64_t k, double* out);

#ifdef __cplusplus
}
#endif
#endif
