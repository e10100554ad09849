#include "common.cuh"
using namespace cpcag_cuda;
extern "C" {
#define NI { set_last_error("not implemented yet"); return CPCAG_ERR_RUNTIME; }
int cpcag_cuda_pcg_solve(cpcag_ctx, cpcag_csr, const double*, double*, int64_t, double, int64_t, int, int64_t*, int*, double*) NI
int cpcag_cuda_knn_graph(cpcag_ctx, int, const void*, int64_t, int64_t, int, int64_t, int, double, cpcag_csr*, cpcag_csr*, double*, double*) NI
int cpcag_cuda_knn(cpcag_ctx, int, const void*, int64_t, int64_t, int, int64_t, int64_t*, double*) NI
int cpcag_cuda_graph_from_adjacency(cpcag_ctx, cpcag_csr, int, cpcag_csr*, double*) NI
int cpcag_cuda_kron_reduce(cpcag_ctx, cpcag_csr, const int64_t*, int64_t, double, double, cpcag_csr*) NI
int cpcag_cuda_run_pipeline(cpcag_ctx, int, const void*, int64_t, int64_t, cpcag_csr, cpcag_csr, const cpcag_pipeline_config*, void*, void*, int64_t*, int64_t*, double*, cpcag_pipeline_report*) NI
}
