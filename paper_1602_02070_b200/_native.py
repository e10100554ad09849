"""ctypes binding of libcpcag_cuda.so (the C-ABI declared in include/cpcag_cuda.h).

Loading fails loudly: there is no CPU fallback anywhere in this package.  If
the library is missing (not built) or cannot initialise a CUDA device, every
entry point raises.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "lib", "libcpcag_cuda.so")

i64 = C.c_int64
u64 = C.c_uint64
dbl = C.c_double
vp = C.c_void_p
ip = C.POINTER(C.c_int64)
dp = C.POINTER(C.c_double)

# status codes (cpcag_status)
OK, ERR_INVALID, ERR_RUNTIME, ERR_RANGE, ERR_CUDA = 0, 1, 2, 3, 4
F64, F32 = 0, 1
AXIS_ROWS, AXIS_COLS = 0, 1
COMBINATORIAL, NORMALIZED = 0, 1
LOSS_L1, LOSS_L2 = 0, 1
LEFT, RIGHT = 0, 1


class FrpcagConfigC(C.Structure):
    _fields_ = [("gamma_r", dbl), ("gamma_c", dbl), ("loss", C.c_int), ("tol", dbl),
                ("max_iter", i64), ("step", dbl)]


class SolveTraceC(C.Structure):
    _fields_ = [("iterations", i64), ("converged", C.c_int), ("final_rel_change", dbl),
                ("step", dbl)]


class DecoderConfigC(C.Structure):
    _fields_ = [("gamma", dbl), ("pcg_tol", dbl), ("pcg_max_iter", i64), ("krylov_precision", C.c_int)]


class ShardStatsC(C.Structure):
    _fields_ = [("halo_cols", i64), ("send_cols", i64), ("bytes_per_iteration", dbl), ("exchange_ms", dbl),
                ("measure_exchange", C.c_int)]


DECODER_IDEAL, DECODER_ALTERNATE, DECODER_APPROX = 0, 1, 2


class ApproxConfigC(C.Structure):
    _fields_ = [("delta_for_scaling", dbl), ("rank_threshold", dbl), ("pcg_tol", dbl), ("pcg_max_iter", i64)]


class PipelineConfigC(C.Structure):
    _fields_ = [("knn", i64), ("laplacian", C.c_int), ("sigma2", dbl), ("a", i64), ("b", i64),
                ("rho_r_override", i64), ("rho_c_override", i64), ("kron_pcg_tol", dbl),
                ("frpcag", FrpcagConfigC), ("decoder", DecoderConfigC), ("lambda_k1_r", dbl),
                ("lambda_k1_c", dbl), ("seed", u64), ("decoder_variant", C.c_int), ("approx", ApproxConfigC),
                ("task", C.c_int), ("n_clusters", i64), ("kmeans_restarts", i64)]


class PipelineFactorsC(C.Structure):
    _fields_ = [("U", vp), ("sigma", vp), ("V", vp), ("k_cap", i64), ("labels", vp)]


class PipelineReportC(C.Structure):
    _fields_ = [("p", i64), ("n", i64), ("rho_r", i64), ("rho_c", i64), ("trace", SolveTraceC),
                ("decoder_converged", C.c_int), ("decoder_iterations", i64), ("detected_rank", i64),
                ("factors_k", i64), ("has_factors", C.c_int), ("lambda_k1_r", dbl), ("lambda_k1_c", dbl),
                ("stage_ms", dbl * 6), ("cluster_ms", dbl), ("n_clusters", i64)]


# (name, restype, argtypes) of every exported symbol.
SIGNATURES = {
    "cpcag_cuda_last_error": (C.c_char_p, []),
    "cpcag_cuda_version": (C.c_char_p, []),
    "cpcag_ctx_create": (C.c_int, [C.c_int, C.POINTER(vp)]),
    "cpcag_ctx_destroy": (C.c_int, [vp]),
    "cpcag_ctx_set_stream": (C.c_int, [vp, vp]),
    "cpcag_ctx_stream": (vp, [vp]),
    "cpcag_ctx_synchronize": (C.c_int, [vp]),
    "cpcag_ctx_launch_count": (i64, [vp]),
    "cpcag_ctx_reset_launch_count": (None, [vp]),
    "cpcag_ctx_enable_kernel_timing": (C.c_int, [vp, C.c_int]),
    "cpcag_ctx_reset_kernel_timing": (C.c_int, [vp]),
    "cpcag_ctx_kernel_timing_filter": (C.c_int, [vp, C.c_char_p]),
    "cpcag_ctx_kernel_timing_count": (C.c_int, [vp]),
    "cpcag_ctx_kernel_timing": (C.c_int, [vp, C.c_int, C.c_char_p, i64, ip, dp]),
    "cpcag_csr_create": (C.c_int, [vp, i64, i64, i64, vp, vp, vp, C.POINTER(vp)]),
    "cpcag_csr_destroy": (C.c_int, [vp]),
    "cpcag_csr_info": (C.c_int, [vp, ip, ip, ip]),
    "cpcag_csr_export": (C.c_int, [vp, vp, vp, vp, vp]),
    "cpcag_csr_is_symmetric": (C.c_int, [vp]),
    "cpcag_cuda_spmm": (C.c_int, [vp, vp, C.c_int, C.c_int, i64, i64, vp, vp]),
    "cpcag_cuda_spmv": (C.c_int, [vp, vp, C.c_int, i64, vp, vp]),
    "cpcag_cuda_power_norm": (C.c_int, [vp, vp, dbl, u64, i64, dp]),
    "cpcag_cuda_pcg_solve": (C.c_int, [vp, vp, vp, vp, i64, dbl, i64, C.c_int, ip,
                                       C.POINTER(C.c_int), dp]),
    "cpcag_cuda_knn_graph": (C.c_int, [vp, C.c_int, vp, i64, i64, C.c_int, i64, C.c_int, dbl,
                                       C.POINTER(vp), C.POINTER(vp), vp, dp]),
    "cpcag_cuda_knn": (C.c_int, [vp, C.c_int, vp, i64, i64, C.c_int, i64, vp, vp]),
    "cpcag_cuda_graph_from_adjacency": (C.c_int, [vp, vp, C.c_int, C.POINTER(vp), vp]),
    "cpcag_cuda_kron_reduce": (C.c_int, [vp, vp, vp, i64, dbl, dbl, C.POINTER(vp)]),
    "cpcag_cuda_draw_plan": (C.c_int, [i64, i64, i64, i64, u64, vp, vp]),
    "cpcag_cuda_subsample": (C.c_int, [vp, C.c_int, vp, i64, i64, vp, i64, vp, i64, vp]),
    "cpcag_cuda_objective": (C.c_int, [vp, C.c_int, vp, vp, i64, i64, vp, vp,
                                       C.POINTER(FrpcagConfigC), dp]),
    "cpcag_cuda_prox": (C.c_int, [vp, C.c_int, C.c_int, vp, vp, i64, dbl, vp]),
    "cpcag_cuda_grad_g": (C.c_int, [vp, C.c_int, vp, i64, i64, vp, vp,
                                    C.POINTER(FrpcagConfigC), vp]),
    "cpcag_cuda_fista": (C.c_int, [vp, C.c_int, vp, i64, i64, vp, vp, C.POINTER(FrpcagConfigC),
                                   vp, vp, C.POINTER(SolveTraceC)]),
    "cpcag_cuda_alternate_decode": (C.c_int, [vp, C.c_int, vp, i64, i64, vp, vp, i64, i64, vp, vp,
                                              dbl, dbl, C.POINTER(DecoderConfigC), vp,
                                              C.POINTER(C.c_int), ip]),
    "cpcag_ctx_reserve": (C.c_int, [vp, i64]),
    "cpcag_ctx_set_apply_path": (C.c_int, [vp, C.c_int]),
    "cpcag_ctx_last_apply_path": (C.c_int, [vp]),
    "cpcag_ctx_set_fista_path": (C.c_int, [vp, C.c_int]),
    "cpcag_ctx_set_power_path": (C.c_int, [vp, C.c_int]),
    "cpcag_ctx_last_power_path": (C.c_int, [vp]),
    "cpcag_cuda_thin_svd": (C.c_int, [vp, vp, i64, i64, vp, vp, vp]),
    "cpcag_cuda_sym_eig": (C.c_int, [vp, vp, i64, vp, vp]),
    "cpcag_cuda_sym_eigvals_lanczos": (C.c_int, [vp, vp, i64, C.c_double, i64, C.c_uint64, vp, vp]),
    "cpcag_glr1_info": (C.c_int, [C.c_char_p, vp, vp]),
    "cpcag_cuda_kmeans": (C.c_int, [vp, C.c_int, vp, i64, i64, i64, i64, C.c_uint64, i64, vp, vp]),
    "cpcag_cuda_decode_labels": (C.c_int, [vp, vp, i64, i64, vp, i64, vp, C.c_double, i64, vp]),
    "cpcag_clustering_error": (C.c_int, [vp, vp, i64, i64, i64, vp]),
    "cpcag_cuda_load_matrix_glr1": (C.c_int, [vp, C.c_char_p, C.c_int, vp, i64, i64]),
    "cpcag_cuda_save_matrix_glr1": (C.c_int, [vp, C.c_char_p, C.c_int, vp, i64, i64]),
    "cpcag_cuda_load_sparse_glr1": (C.c_int, [vp, C.c_char_p, vp]),
    "cpcag_cuda_save_sparse_glr1": (C.c_int, [vp, vp, C.c_char_p]),
    "cpcag_cuda_save_factors_glr1": (C.c_int, [vp, C.c_char_p, i64, i64, i64, C.c_int, vp, vp, vp]),
    "cpcag_cuda_load_factors_glr1": (C.c_int, [vp, C.c_char_p, i64, i64, i64, vp, vp, vp, vp]),
    "cpcag_cuda_graph_upsample": (C.c_int, [vp, vp, vp, i64, vp, i64, dbl, i64, vp]),
    "cpcag_cuda_approx_decode": (C.c_int, [vp, C.c_int, vp, i64, i64, vp, vp, i64, i64, vp, vp,
                                           C.POINTER(ApproxConfigC), vp, vp, vp, vp, i64, ip]),
    "cpcag_cuda_decoder_apply": (C.c_int, [vp, C.c_int, vp, i64, i64, vp, vp, vp, i64, vp, i64, dbl, dbl, vp, dp]),
    "cpcag_halo_plan": (C.c_int, [vp, vp, i64, vp, C.c_int, C.c_int, vp, vp, vp, vp]),
    "cpcag_cuda_comm_unique_id": (C.c_int, [vp]),
    "cpcag_cuda_comm_create": (C.c_int, [vp, vp, C.c_int, C.c_int, C.POINTER(vp)]),
    "cpcag_cuda_comm_destroy": (C.c_int, [vp]),
    "cpcag_cuda_alternate_decode_sharded": (C.c_int, [vp, vp, C.c_int, vp, i64, i64, vp, vp, i64, i64, vp, vp,
                                                      dbl, dbl, C.POINTER(DecoderConfigC), vp, vp,
                                                      C.POINTER(C.c_int), ip, C.POINTER(ShardStatsC)]),
    "cpcag_cuda_alternate_decode_sharded_emulated": (C.c_int, [vp, C.c_int, C.c_int, vp, i64, i64, vp, vp, i64, i64,
                                                               vp, vp, dbl, dbl, C.POINTER(DecoderConfigC), vp, vp,
                                                               C.POINTER(C.c_int), ip, C.POINTER(ShardStatsC)]),
    "cpcag_cuda_fista_sharded": (C.c_int, [vp, vp, C.c_int, vp, i64, i64, vp, vp, C.POINTER(FrpcagConfigC), vp, vp,
                                           vp, C.POINTER(SolveTraceC)]),
    "cpcag_cuda_fista_sharded_emulated": (C.c_int, [vp, C.c_int, C.c_int, vp, i64, i64, vp, vp,
                                                    C.POINTER(FrpcagConfigC), vp, vp, vp, C.POINTER(SolveTraceC)]),
    "cpcag_cuda_gram_tf32x3": (C.c_int, [vp, vp, i64, i64, vp]),
    "cpcag_cuda_run_pipeline": (C.c_int, [vp, C.c_int, vp, i64, i64, vp, vp,
                                          C.POINTER(PipelineConfigC), vp, vp, vp, vp, vp,
                                          C.POINTER(PipelineReportC), C.POINTER(PipelineFactorsC)]),
}

_lib = None


class CpcagError(RuntimeError):
    """Raised for CPCAG_ERR_CUDA (device/driver failure)."""


def lib():
    """Load libcpcag_cuda.so; raises if it has not been built."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; "
                "g.build()'` (nvcc, sm_100a). There is no CPU fallback.")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def check(rc: int) -> None:
    """Map a cpcag_status to the reference's exception classes."""
    if rc == OK:
        return
    msg = lib().cpcag_cuda_last_error().decode(errors="replace")
    if rc == ERR_INVALID:
        raise ValueError(msg)       # std::invalid_argument
    if rc == ERR_RANGE:
        raise IndexError(msg)       # std::out_of_range
    if rc == ERR_RUNTIME:
        raise RuntimeError(msg)     # std::runtime_error
    raise CpcagError(msg)
