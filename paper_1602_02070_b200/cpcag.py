"""Python mirror of the reference `cpcag` API for the CPCA hot path.

Same names, argument meaning, defaults and exceptions as the C++ reference
(proj/core/include/cpcag/*.hpp; file:line per function below), executed by
libcpcag_cuda.so on the GPU through the C-ABI in include/cpcag_cuda.h.

Arrays: numpy arrays (host) or torch tensors (host or CUDA) are accepted;
dense matrices are column-major as in the reference (types.hpp:12-13).
Results come back as numpy arrays for host inputs and as CUDA tensors
(column-major strides) for CUDA inputs, so a caller that keeps its data in
HBM never round-trips through the host.
"""
from __future__ import annotations

import ctypes as C
import os
import math
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from . import _native as N

__all__ = [
    "Context", "SparseMatrix", "GraphModel", "SamplingPlan", "FrpcagConfig", "SolveTrace",
    "DecoderConfig", "SpectralGap", "AlternateDecodeResult", "PcgOptions", "PcgResult",
    "PipelineConfig", "PipelineReport", "build_knn_graph", "knn", "graph_from_adjacency",
    "kron_reduce", "draw_plan", "subsample", "objective", "prox_l1", "prox_l2", "grad_g",
    "fista_solve", "alternate_decode", "power_iteration_norm", "pcg_solve", "run_pipeline",
    "default_context", "SvdResult", "thin_svd", "detect_rank", "graph_upsample", "LowRankFactors",
    "ApproxDecodeResult", "approx_decode", "EigenPairs", "sym_eig", "sym_eigvals_lanczos", "spectral_gap",
    "glr1_info", "load_matrix", "save_matrix", "load_sparse", "save_sparse", "save_factors",
    "load_factors", "plan_to_json", "plan_from_json", "save_plan", "load_plan",
    "ClusterLabels", "kmeans", "decode_labels", "clustering_error", "save_labels_csv", "load_labels_csv",
    "report_to_json", "emit_report", "decoder_apply",
]


# ------------------------------------------------------------------ arrays
def _torch():
    import torch

    return torch


def _is_torch(x) -> bool:
    return type(x).__module__.startswith("torch")


def _is_cuda(x) -> bool:
    return _is_torch(x) and x.is_cuda


def _np_dtype(precision: int):
    return np.float64 if precision == N.F64 else np.float32


CUDA_STREAM_LEGACY = 0x1  # cudaStreamLegacy (driver_types.h)

class _In:
    """Pointer to a caller array in the requested precision, column-major."""

    def __init__(self, x, precision: int, shape=None, kind="float"):
        self.keep = None
        if _is_torch(x):
            torch = _torch()
            dt = torch.int64 if kind == "index" else (torch.float64 if precision == N.F64 else torch.float32)
            t = x.detach()
            if t.dtype != dt:
                t = t.to(dt)
            if t.dim() == 2 and not (t.stride(0) == 1 and t.stride(1) == max(t.shape[0], 1)):
                t = t.t().contiguous().t()
            elif t.dim() != 2 and not t.is_contiguous():
                t = t.contiguous()
            if not t.is_cuda:
                t = t.numpy()
                self._from_numpy(t, precision, kind)
            else:
                self.keep = t
                self.ptr = t.data_ptr()
                self.shape = tuple(t.shape)
        else:
            self._from_numpy(x, precision, kind)
        if shape is not None and tuple(self.shape) != tuple(shape):
            raise ValueError(f"array shape {self.shape} does not match the expected {shape}")

    def _from_numpy(self, x, precision, kind):
        dt = np.int64 if kind == "index" else _np_dtype(precision)
        a = np.asarray(x, dtype=dt)
        a = np.asfortranarray(a) if a.ndim == 2 else np.ascontiguousarray(a)
        self.keep = a
        self.ptr = a.ctypes.data if a.size else None
        self.shape = a.shape


def _out(like_cuda, device, shape, precision: int, kind="float"):
    """Column-major output buffer: CUDA tensor when inputs are CUDA, else numpy."""
    if like_cuda:
        torch = _torch()
        dt = torch.int64 if kind == "index" else (torch.float64 if precision == N.F64 else torch.float32)
        if len(shape) == 2:
            t = torch.empty((shape[1], shape[0]), dtype=dt, device=device).t()
        else:
            t = torch.empty(shape, dtype=dt, device=device)
        return t, t.data_ptr()
    dt = np.int64 if kind == "index" else _np_dtype(precision)
    a = np.empty(shape, dtype=dt, order="F")
    return a, (a.ctypes.data if a.size else None)


def _given_out(a, shape, precision: int, name: str):
    """A caller-provided column-major output (numpy F-order array, e.g. a view
    of pinned memory, or a column-major CUDA tensor) -> (array, pointer)."""
    want = _np_dtype(precision)
    if hasattr(a, "data_ptr"):  # torch tensor
        torch = _torch()
        tdt = torch.float64 if precision == N.F64 else torch.float32
        ok = tuple(a.shape) == tuple(shape) and a.dtype == tdt and (a.numel() == 0 or a.t().is_contiguous())
        if not ok:
            raise ValueError(f"{name}: expected a column-major {tuple(shape)} {tdt} tensor")
        return a, a.data_ptr()
    a = np.asarray(a)
    if a.shape != tuple(shape) or a.dtype != want or not (a.size == 0 or a.flags.f_contiguous):
        raise ValueError(f"{name}: expected a Fortran-ordered {tuple(shape)} {np.dtype(want).name} array")
    return a, (a.ctypes.data if a.size else None)


def _precision(x, precision):
    if precision is not None:
        return N.F32 if precision in (N.F32, "f32", "float32", np.float32) else N.F64
    if _is_torch(x):
        return N.F32 if x.dtype == _torch().float32 else N.F64
    if isinstance(x, np.ndarray) and x.dtype == np.float32:
        return N.F32
    return N.F64


# ------------------------------------------------------------------ context
class Context:
    """A device, a CUDA stream and a workspace (cpcag_ctx)."""

    def __init__(self, device: int = -1):
        L = N.lib()
        h = N.vp()
        N.check(L.cpcag_ctx_create(int(device), C.byref(h)))
        self._h = h
        self.device = device

    @property
    def handle(self):
        return self._h

    def set_stream(self, stream_ptr: Optional[int]):
        """Launch on `stream_ptr` (e.g. torch.cuda.current_stream().cuda_stream).
        None restores the context's own stream.  Handle 0 is torch's default
        stream, the legacy default stream, passed as cudaStreamLegacy: the
        C-ABI reads NULL as "own stream", which is not ordered with torch."""
        if stream_ptr is not None and int(stream_ptr) == 0:
            stream_ptr = CUDA_STREAM_LEGACY
        N.check(N.lib().cpcag_ctx_set_stream(self._h, stream_ptr))

    def synchronize(self):
        N.check(N.lib().cpcag_ctx_synchronize(self._h))

    @property
    def launch_count(self) -> int:
        return int(N.lib().cpcag_ctx_launch_count(self._h))

    def reset_launch_count(self):
        N.lib().cpcag_ctx_reset_launch_count(self._h)

    def set_apply_path(self, path: str):
        """Decoder operator path: "auto", "split" (two passes), "fused" or "slab"."""
        N.check(N.lib().cpcag_ctx_set_apply_path(self.handle, {"auto": 0, "split": 1, "fused": 2, "slab": 3}[path]))

    def set_fista_path(self, path: str):
        """Persistent FISTA tile GEMM: "auto" (DMMA tensor cores) or "simt" (tests)."""
        N.check(N.lib().cpcag_ctx_set_fista_path(self.handle, {"auto": 0, "simt": 1}[path]))

    def set_power_path(self, path: str):
        """Cooperative power iteration: "auto" (three or two products per barrier when the dense powers
        of the operator fit), "single" or "double" (tests)."""
        N.check(N.lib().cpcag_ctx_set_power_path(self.handle, {"auto": 0, "single": 1, "double": 2}[path]))

    def last_power_path(self) -> str:
        """How the most recent power iteration ran."""
        return {0: "cta", 1: "single", 2: "double", 3: "triple"}[N.lib().cpcag_ctx_last_power_path(self.handle)]

    def last_apply_path(self) -> str:
        """The path the most recently planned decoder operator took."""
        return {0: "none", 1: "split", 2: "fused", 3: "slab"}[N.lib().cpcag_ctx_last_apply_path(self.handle)]

    def reserve(self, nbytes: int):
        """Grow the stream-ordered memory pool to `nbytes` up front."""
        N.check(N.lib().cpcag_ctx_reserve(self._h, int(nbytes)))

    def enable_kernel_timing(self, on: bool = True):
        """CUDA-event timing of every hot-kernel launch (for roofline figures)."""
        N.check(N.lib().cpcag_ctx_enable_kernel_timing(self._h, int(bool(on))))

    def kernel_timing_filter(self, tags=None):
        """Time only these kernel tags (None = all)."""
        csv = ",".join(tags) if tags else ""
        N.check(N.lib().cpcag_ctx_kernel_timing_filter(self._h, csv.encode()))

    def reset_kernel_timing(self):
        N.check(N.lib().cpcag_ctx_reset_kernel_timing(self._h))

    def kernel_times(self) -> dict:
        """{kernel tag: (launches, total device ms)} since the last reset."""
        L = N.lib()
        out = {}
        for k in range(int(L.cpcag_ctx_kernel_timing_count(self._h))):
            buf = C.create_string_buffer(64)
            n, ms = N.i64(), N.dbl()
            N.check(L.cpcag_ctx_kernel_timing(self._h, k, buf, 64, C.byref(n), C.byref(ms)))
            out[buf.value.decode()] = (int(n.value), float(ms.value))
        return out

    def close(self):
        if getattr(self, "_h", None) is not None and self._h.value:
            N.lib().cpcag_ctx_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


_default_ctx: Optional[Context] = None


def default_context() -> Context:
    global _default_ctx
    if _default_ctx is None:
        _default_ctx = Context(-1)
    return _default_ctx


def _ctx(ctx):
    return (ctx or default_context()).handle


def _torch_device(x):
    return x.device if _is_cuda(x) else None


# ------------------------------------------------------------------ sparse
class SparseMatrix:
    """Device CSR (sparse.hpp:18-66): int64 row pointers, sorted columns, fp64
    values, no stored zeros.  Immutable."""

    def __init__(self, handle, ctx: Optional[Context] = None):
        self._h = handle if isinstance(handle, N.vp) else N.vp(handle)
        self._ctx = ctx or default_context()

    def __del__(self):
        try:
            if self._h is not None and self._h.value:
                N.lib().cpcag_csr_destroy(self._h)
                self._h = None
        except Exception:
            pass

    @property
    def handle(self):
        return self._h

    def _info(self):
        r, c, z = N.i64(), N.i64(), N.i64()
        N.check(N.lib().cpcag_csr_info(self._h, C.byref(r), C.byref(c), C.byref(z)))
        return int(r.value), int(c.value), int(z.value)

    def rows(self) -> int:
        return self._info()[0]

    def cols(self) -> int:
        return self._info()[1]

    def nonzeros(self) -> int:
        return self._info()[2]

    @property
    def shape(self):
        r, c, _ = self._info()
        return (r, c)

    # sparse.cpp:10-46 (host-side construction utility; the CSR is then
    # uploaded once and every product runs on the device).
    @staticmethod
    def from_triplets(rows, cols, ti, tj, tv, drop_below=0.0, ctx=None) -> "SparseMatrix":
        ti = np.asarray(ti, np.int64).ravel()
        tj = np.asarray(tj, np.int64).ravel()
        tv = np.asarray(tv, np.float64).ravel()
        if rows < 0 or cols < 0:
            raise ValueError("sparse: negative dimensions")
        if ti.size and (ti.min() < 0 or ti.max() >= rows or tj.min() < 0 or tj.max() >= cols):
            raise ValueError("sparse: triplet index out of range")
        if not np.all(np.isfinite(tv)):
            raise ValueError("sparse: non-finite entry")
        order = np.lexsort((tj, ti))
        ti, tj, tv = ti[order], tj[order], tv[order]
        if ti.size:
            key = ti * max(cols, 1) + tj
            start = np.concatenate(([True], key[1:] != key[:-1]))
            grp = np.cumsum(start) - 1
            vals = np.zeros(int(grp[-1]) + 1)
            # sequential per-group sums in input order (np.add.at is unbuffered)
            np.add.at(vals, grp, tv)
            ui, uj = ti[start], tj[start]
            keep = (vals != 0.0) & (np.abs(vals) > drop_below)
            ui, uj, vals = ui[keep], uj[keep], vals[keep]
        else:
            ui, uj, vals = ti, tj, tv
        rp = np.zeros(rows + 1, np.int64)
        np.add.at(rp, ui + 1, 1)
        rp = np.cumsum(rp)
        return SparseMatrix.from_csr(rows, cols, rp, uj, vals, ctx=ctx)

    @staticmethod
    def from_csr(rows, cols, row_ptr, col_idx, values, ctx=None) -> "SparseMatrix":
        ctx = ctx or default_context()
        rp = _In(row_ptr, N.F64, kind="index")
        ci = _In(col_idx, N.F64, kind="index")
        v = _In(values, N.F64)
        nnz = int(row_ptr[-1]) if len(row_ptr) else 0
        h = N.vp()
        N.check(N.lib().cpcag_csr_create(ctx.handle, int(rows), int(cols), nnz, rp.ptr, ci.ptr, v.ptr,
                                         C.byref(h)))
        return SparseMatrix(h, ctx)

    @staticmethod
    def from_scipy(S, ctx=None) -> "SparseMatrix":
        S = S.tocsr().copy()
        S.sort_indices()
        S.sum_duplicates()
        return SparseMatrix.from_csr(S.shape[0], S.shape[1], S.indptr.astype(np.int64),
                                     S.indices.astype(np.int64), S.data.astype(np.float64), ctx=ctx)

    @staticmethod
    def from_dense(D, drop_below=0.0, ctx=None) -> "SparseMatrix":
        D = np.asarray(D, np.float64)
        i, j = np.nonzero(D)
        return SparseMatrix.from_triplets(D.shape[0], D.shape[1], i, j, D[i, j], drop_below, ctx)

    def arrays(self):
        r, c, z = self._info()
        rp = np.empty(r + 1, np.int64)
        ci = np.empty(z, np.int64)
        v = np.empty(z, np.float64)
        N.check(N.lib().cpcag_csr_export(self._ctx.handle, self._h, rp.ctypes.data,
                                         ci.ctypes.data if z else None, v.ctypes.data if z else None))
        return rp, ci, v

    def to_scipy(self):
        import scipy.sparse as sp

        rp, ci, v = self.arrays()
        return sp.csr_matrix((v, ci, rp), shape=self.shape)

    def to_dense(self) -> np.ndarray:
        return self.to_scipy().toarray()

    def is_symmetric(self) -> bool:
        return bool(N.lib().cpcag_csr_is_symmetric(self._h))

    # sparse.cpp:73-98
    def multiply(self, X, precision=None):
        prec = _precision(X, precision)
        if (X.ndim if hasattr(X, "ndim") else np.ndim(X)) == 1:
            x = _In(X, prec)
            r, c, _ = self._info()
            y, yp = _out(_is_cuda(X), _torch_device(X), (r,), prec)
            N.check(N.lib().cpcag_cuda_spmv(self._ctx.handle, self._h, prec, x.shape[0], x.ptr, yp))
            return y
        x = _In(X, prec)
        r, c, _ = self._info()
        y, yp = _out(_is_cuda(X), _torch_device(X), (r, x.shape[1]), prec)
        N.check(N.lib().cpcag_cuda_spmm(self._ctx.handle, self._h, N.LEFT, prec, x.shape[0],
                                        x.shape[1], x.ptr, yp))
        return y

    # sparse.cpp:100-111
    def right_multiply(self, X, precision=None):
        prec = _precision(X, precision)
        x = _In(X, prec)
        r, c, _ = self._info()
        y, yp = _out(_is_cuda(X), _torch_device(X), (x.shape[0], c), prec)
        N.check(N.lib().cpcag_cuda_spmm(self._ctx.handle, self._h, N.RIGHT, prec, x.shape[0],
                                        x.shape[1], x.ptr, yp))
        return y


# ------------------------------------------------------------------ solvers
@dataclass
class PcgOptions:  # solvers.hpp:13-16
    tol: float = 1e-10
    max_iter: int = 5000


@dataclass
class PcgResult:  # solvers.hpp:18-22
    iterations: int = 0
    converged: bool = False
    relative_residual: float = 0.0


def power_iteration_norm(A: SparseMatrix, tol=1e-9, seed=0, max_iter=50000, ctx=None) -> float:
    """solvers.hpp:90-91 / solvers.cpp:29-53."""
    out = N.dbl()
    N.check(N.lib().cpcag_cuda_power_norm(_ctx(ctx), A.handle, float(tol), int(seed) & (2**64 - 1),
                                          int(max_iter), C.byref(out)))
    return float(out.value)


def pcg_solve(A: SparseMatrix, b, x=None, opt: PcgOptions = PcgOptions(), jacobi=True, ctx=None):
    """solvers.hpp:85-86 / solvers.cpp:19-27.  Returns (x, PcgResult)."""
    b = np.ascontiguousarray(b, np.float64)
    xv = np.zeros_like(b) if x is None or np.size(x) != b.size else np.array(x, np.float64)
    it, cv, rr = N.i64(), C.c_int(), N.dbl()
    N.check(N.lib().cpcag_cuda_pcg_solve(_ctx(ctx), A.handle, b.ctypes.data, xv.ctypes.data, b.size,
                                         float(opt.tol), int(opt.max_iter), int(bool(jacobi)),
                                         C.byref(it), C.byref(cv), C.byref(rr)))
    return xv, PcgResult(int(it.value), bool(cv.value), float(rr.value))


# ------------------------------------------------------------------ graphs
@dataclass
class GraphModel:  # graph.hpp:13-21
    n_nodes: int
    K: int
    sigma2: float
    adjacency: SparseMatrix
    degrees: np.ndarray
    laplacian: SparseMatrix
    kind: int = N.COMBINATORIAL


def _axis(axis) -> int:
    if axis in ("rows", N.AXIS_ROWS):
        return N.AXIS_ROWS
    if axis in ("cols", N.AXIS_COLS):
        return N.AXIS_COLS
    raise ValueError("axis must be 'rows' or 'cols'")


def _kind(kind) -> int:
    if kind in ("combinatorial", N.COMBINATORIAL):
        return N.COMBINATORIAL
    if kind in ("normalized", N.NORMALIZED):
        return N.NORMALIZED
    raise ValueError("unknown laplacian kind")


def build_knn_graph(X, axis, K: int, kind="combinatorial", sigma2_override=0.0, precision=None,
                    ctx=None) -> GraphModel:
    """graph.hpp:29-31 / graph.cpp:47-135."""
    prec = _precision(X, precision)
    x = _In(X, prec)
    if len(x.shape) != 2:
        raise ValueError("knn graph: X must be a matrix")
    ax = _axis(axis)
    n = x.shape[0] if ax == N.AXIS_ROWS else x.shape[1]
    W, L = N.vp(), N.vp()
    deg = np.empty(max(n, 0))
    s2 = N.dbl()
    N.check(N.lib().cpcag_cuda_knn_graph(_ctx(ctx), prec, x.ptr, x.shape[0], x.shape[1], ax, int(K),
                                         _kind(kind), float(sigma2_override), C.byref(W), C.byref(L),
                                         deg.ctypes.data if n > 0 else None, C.byref(s2)))
    c = ctx or default_context()
    return GraphModel(n, int(K), float(s2.value), SparseMatrix(W, c), deg, SparseMatrix(L, c), _kind(kind))


def knn(X, axis, K: int, precision=None, ctx=None):
    """Neighbour lists of build_knn_graph (graph.cpp:86-105): (n x K indices, n x K d2)."""
    prec = _precision(X, precision)
    x = _In(X, prec)
    ax = _axis(axis)
    n = x.shape[0] if ax == N.AXIS_ROWS else x.shape[1]
    nbr = np.empty((n, K), np.int64)
    d2 = np.empty((n, K), np.float64)
    N.check(N.lib().cpcag_cuda_knn(_ctx(ctx), prec, x.ptr, x.shape[0], x.shape[1], ax, int(K),
                                   nbr.ctypes.data, d2.ctypes.data))
    return nbr, d2


def graph_from_adjacency(W: SparseMatrix, kind="combinatorial", ctx=None) -> GraphModel:
    """graph.hpp:35-36 / graph.cpp:137-154."""
    L = N.vp()
    n = W.rows()
    deg = np.empty(n)
    N.check(N.lib().cpcag_cuda_graph_from_adjacency(_ctx(ctx), W.handle, _kind(kind), C.byref(L),
                                                    deg.ctypes.data if n else None))
    return GraphModel(n, 0, 0.0, W, deg, SparseMatrix(L, ctx or default_context()), _kind(kind))


def kron_reduce(L: SparseMatrix, keep, pcg_tol=1e-12, prune_tol=1e-12, ctx=None) -> SparseMatrix:
    """graph.hpp:50-51 / graph.cpp:170-235."""
    k = _In(keep, N.F64, kind="index")
    out = N.vp()
    N.check(N.lib().cpcag_cuda_kron_reduce(_ctx(ctx), L.handle, k.ptr, int(k.shape[0]), float(pcg_tol),
                                           float(prune_tol), C.byref(out)))
    return SparseMatrix(out, ctx or default_context())


# ------------------------------------------------------------------ sampling
@dataclass
class SamplingPlan:  # sampling.hpp:13-26
    omega_r: np.ndarray
    omega_c: np.ndarray
    p: int = 0
    n: int = 0
    delta: float = 0.0
    epsilon: float = 0.0
    seed: int = 0

    def rho_r(self) -> int:
        return len(self.omega_r)

    def rho_c(self) -> int:
        return len(self.omega_c)

    def norm_const(self) -> float:
        return (float(self.n) * float(self.p)) / (float(self.rho_r()) * float(self.rho_c()))


def draw_plan(p, n, rho_r, rho_c, delta=0.0, epsilon=0.0, seed=0) -> SamplingPlan:
    """sampling.hpp:39-40 / sampling.cpp:48-64 (host: bit-exact counter RNG)."""
    om_r = np.empty(max(int(rho_r), 0), np.int64)
    om_c = np.empty(max(int(rho_c), 0), np.int64)
    N.check(N.lib().cpcag_cuda_draw_plan(int(p), int(n), int(rho_r), int(rho_c),
                                         int(seed) & (2**64 - 1),
                                         om_r.ctypes.data if om_r.size else None,
                                         om_c.ctypes.data if om_c.size else None))
    return SamplingPlan(om_r, om_c, int(p), int(n), float(delta), float(epsilon), int(seed))


def subsample(Y, plan: SamplingPlan, precision=None, ctx=None):
    """sampling.hpp:43 / sampling.cpp:66-75."""
    prec = _precision(Y, precision)
    y = _In(Y, prec)
    if tuple(y.shape) != (plan.p, plan.n):
        raise ValueError("subsample: plan does not match matrix dimensions")
    om_r = np.ascontiguousarray(plan.omega_r, np.int64)
    om_c = np.ascontiguousarray(plan.omega_c, np.int64)
    out, op = _out(_is_cuda(Y), _torch_device(Y), (plan.rho_r(), plan.rho_c()), prec)
    N.check(N.lib().cpcag_cuda_subsample(_ctx(ctx), prec, y.ptr, plan.p, plan.n, om_r.ctypes.data,
                                         plan.rho_r(), om_c.ctypes.data, plan.rho_c(), op))
    return out


# ------------------------------------------------------------------ FRPCAG
@dataclass
class FrpcagConfig:  # frpcag.hpp:15-22
    gamma_r: float = 1.0
    gamma_c: float = 1.0
    loss: str = "l1"
    tol: float = 1e-10
    max_iter: int = 500
    step: float = 0.0

    def c(self) -> N.FrpcagConfigC:
        return N.FrpcagConfigC(self.gamma_r, self.gamma_c, N.LOSS_L2 if self.loss == "l2" else N.LOSS_L1,
                               self.tol, int(self.max_iter), self.step)


@dataclass
class SolveTrace:  # frpcag.hpp:24-30
    objective: list = field(default_factory=list)
    iterations: int = 0
    converged: bool = False
    final_rel_change: float = 0.0
    step: float = 0.0


def objective(X, Y, Lr: SparseMatrix, Lc: SparseMatrix, cfg: FrpcagConfig, precision=None, ctx=None) -> float:
    """frpcag.hpp:32-33 / frpcag.cpp:23-35."""
    prec = _precision(X, precision)
    x, y = _In(X, prec), _In(Y, prec)
    if x.shape != y.shape:
        raise ValueError("frpcag: X and Y dimensions differ")
    out = N.dbl()
    c = cfg.c()
    N.check(N.lib().cpcag_cuda_objective(_ctx(ctx), prec, x.ptr, y.ptr, x.shape[0], x.shape[1], Lr.handle,
                                         Lc.handle, C.byref(c), C.byref(out)))
    return float(out.value)


def _prox(loss, Z, Y, lam, precision, ctx):
    prec = _precision(Z, precision)
    z, y = _In(Z, prec), _In(Y, prec)
    if z.shape != y.shape:
        raise ValueError("prox: Z and Y dimensions differ")
    out, op = _out(_is_cuda(Z), _torch_device(Z), z.shape, prec)
    N.check(N.lib().cpcag_cuda_prox(_ctx(ctx), prec, loss, z.ptr, y.ptr, int(np.prod(z.shape)), float(lam), op))
    return out


def prox_l1(Z, Y, lam, precision=None, ctx=None):
    """frpcag.hpp:36 / frpcag.cpp:37-44."""
    return _prox(N.LOSS_L1, Z, Y, lam, precision, ctx)


def prox_l2(Z, Y, lam, precision=None, ctx=None):
    """frpcag.hpp:39 / frpcag.cpp:46-51."""
    return _prox(N.LOSS_L2, Z, Y, lam, precision, ctx)


def grad_g(Z, Lr: SparseMatrix, Lc: SparseMatrix, cfg: FrpcagConfig, precision=None, ctx=None):
    """frpcag.hpp:42-43 / frpcag.cpp:53-60."""
    prec = _precision(Z, precision)
    z = _In(Z, prec)
    out, op = _out(_is_cuda(Z), _torch_device(Z), z.shape, prec)
    c = cfg.c()
    N.check(N.lib().cpcag_cuda_grad_g(_ctx(ctx), prec, z.ptr, z.shape[0], z.shape[1], Lr.handle, Lc.handle,
                                      C.byref(c), op))
    return out


def fista_solve(Y, Lr: SparseMatrix, Lc: SparseMatrix, cfg: FrpcagConfig, precision=None, ctx=None):
    """frpcag.hpp:46-47 / frpcag.cpp:62-112.  Returns (X, SolveTrace)."""
    prec = _precision(Y, precision)
    y = _In(Y, prec)
    if len(y.shape) != 2:
        raise ValueError("fista: Y must be a matrix")
    out, op = _out(_is_cuda(Y), _torch_device(Y), y.shape, prec)
    obj = np.zeros(max(int(cfg.max_iter), 1))
    tr = N.SolveTraceC()
    c = cfg.c()
    N.check(N.lib().cpcag_cuda_fista(_ctx(ctx), prec, y.ptr, y.shape[0], y.shape[1], Lr.handle, Lc.handle,
                                     C.byref(c), op, obj.ctypes.data, C.byref(tr)))
    n = int(tr.iterations)
    return out, SolveTrace(list(obj[:n]), n, bool(tr.converged), float(tr.final_rel_change), float(tr.step))


# ------------------------------------------------------------------ decoder
@dataclass
class DecoderConfig:  # decoders.hpp:13-22
    gamma: float = 1.0
    pcg_tol: float = 1e-10
    pcg_max_iter: int = 5000
    variant: str = "approx"          # decoder of run_pipeline: "approx" (reference default) | "alternate"
    delta_for_scaling: float = 0.0
    rank_threshold: float = 0.1
    # extension: CG Krylov vectors for fp32 data ("fp64", default: fp32 X with
    # fp64 R/P/AP; "fp32": every vector fp32), see cpcag_cuda.h
    krylov_precision: str = "fp64"

    def c(self) -> N.DecoderConfigC:
        if self.krylov_precision not in ("fp64", "fp32"):
            raise ValueError(f"unknown krylov_precision {self.krylov_precision!r}")
        return N.DecoderConfigC(self.gamma, self.pcg_tol, int(self.pcg_max_iter),
                                N.F32 if self.krylov_precision == "fp32" else 0)

    def approx_c(self) -> N.ApproxConfigC:
        return N.ApproxConfigC(float(self.delta_for_scaling), float(self.rank_threshold), float(self.pcg_tol),
                               int(self.pcg_max_iter))


@dataclass
class SpectralGap:  # graph.hpp:53-58
    k: int = 0
    lambda_k: float = 0.0
    lambda_k1: float = 0.0
    ratio: float = 0.0


@dataclass
class AlternateDecodeResult:  # decoders.hpp:50-54
    X: object
    converged: bool
    iterations: int


def alternate_decode(Xt, plan: SamplingPlan, Lr: SparseMatrix, Lc: SparseMatrix, gap_r: SpectralGap,
                     gap_c: SpectralGap, cfg: DecoderConfig = DecoderConfig(), precision=None,
                     ctx=None) -> AlternateDecodeResult:
    """decoders.hpp:59-62 / decoders.cpp:145-186."""
    prec = _precision(Xt, precision)
    xt = _In(Xt, prec)
    if tuple(xt.shape) != (plan.rho_r(), plan.rho_c()):
        raise ValueError("alternate decoder: Xt does not match plan")
    om_r = np.ascontiguousarray(plan.omega_r, np.int64)
    om_c = np.ascontiguousarray(plan.omega_c, np.int64)
    out, op = _out(_is_cuda(Xt), _torch_device(Xt), (plan.p, plan.n), prec)
    cv, it = C.c_int(), N.i64()
    c = cfg.c()
    N.check(N.lib().cpcag_cuda_alternate_decode(_ctx(ctx), prec, xt.ptr, plan.rho_r(), plan.rho_c(),
                                                om_r.ctypes.data if om_r.size else None,
                                                om_c.ctypes.data if om_c.size else None, plan.p, plan.n,
                                                Lr.handle, Lc.handle, float(gap_r.lambda_k1),
                                                float(gap_c.lambda_k1), C.byref(c), op, C.byref(cv),
                                                C.byref(it)))
    return AlternateDecodeResult(out, bool(cv.value), int(it.value))


# ------------------------------------------------------------------ eigen / spectral gap
def decoder_apply(P, plan: SamplingPlan, Lr: SparseMatrix, Lc: SparseMatrix, gbar_r: float, gbar_c: float,
                  precision=None, ctx=None):
    """The alternate decoder's operator (decoders.cpp:160-170) on a p x n
    matrix: returns (AP, <P, AP>)."""
    prec = _precision(P, precision)
    pv = _In(P, prec, shape=(plan.p, plan.n))
    om_r = np.ascontiguousarray(plan.omega_r, np.int64)
    om_c = np.ascontiguousarray(plan.omega_c, np.int64)
    out, op = _out(_is_cuda(P), _torch_device(P), (plan.p, plan.n), prec)
    dot = N.dbl()
    N.check(N.lib().cpcag_cuda_decoder_apply(_ctx(ctx), prec, pv.ptr, plan.p, plan.n, Lr.handle, Lc.handle,
                                             om_r.ctypes.data if om_r.size else None, len(om_r),
                                             om_c.ctypes.data if om_c.size else None, len(om_c), float(gbar_r),
                                             float(gbar_c), op, C.byref(dot)))
    return out, float(dot.value)


@dataclass
class EigenPairs:  # eigs.hpp:11-19
    eigenvalues: np.ndarray
    eigenvectors: Optional[np.ndarray]

    def order(self) -> int:
        return len(self.eigenvalues)

    def leading(self, k: int):
        if k > self.order():
            raise ValueError("EigenPairs: fewer pairs than requested")
        return self.eigenvectors[:, :k]


def sym_eig(A: SparseMatrix, k: int, vectors: bool = True, ctx=None) -> EigenPairs:
    """eigs.cpp:34-51 on the device (dense symmetric eigensolver)."""
    n = A.rows()
    ev = np.empty(max(int(k), 1), np.float64)
    vec = np.empty((n, max(int(k), 1)), np.float64, order="F") if vectors else None
    N.check(N.lib().cpcag_cuda_sym_eig(_ctx(ctx), A.handle, int(k), ev.ctypes.data,
                                       vec.ctypes.data if vectors else None))
    return EigenPairs(ev[:k].copy(), np.asfortranarray(vec[:, :k]) if vectors else None)


def sym_eigvals_lanczos(A: SparseMatrix, k: int, tol: float = 1e-10, max_iter: int = 5000, seed: int = 0,
                        ctx=None):
    """The k smallest eigenvalues (ascending) of a large sparse symmetric
    matrix by Lanczos with full reorthogonalisation on the device: the
    spectral gaps of pipeline.cpp:343-349 where the dense eigs.cpp:34-51 is
    infeasible.  Returns (eigenvalues, lanczos_steps)."""
    ev = np.empty(max(int(k), 1), np.float64)
    it = N.i64()
    N.check(N.lib().cpcag_cuda_sym_eigvals_lanczos(_ctx(ctx), A.handle, int(k), float(tol), int(max_iter), int(seed),
                                                   ev.ctypes.data, C.byref(it)))
    return ev[:k].copy(), int(it.value)


def spectral_gap(basis: EigenPairs, k: int) -> "SpectralGap":
    """graph.cpp:237-249 (host logic on the eigenvalues)."""
    if k < 1 or basis.order() < k + 1:
        raise ValueError("spectral gap: need at least k+1 eigenvalues")
    lk = max(0.0, float(basis.eigenvalues[k - 1]))
    lk1 = max(0.0, float(basis.eigenvalues[k]))
    if lk1 <= 1e-14:
        raise RuntimeError("gap undefined: graph has > k components")
    return SpectralGap(k, lk, lk1, lk / lk1)


# ------------------------------------------------------------------ approximate decoder
@dataclass
class SvdResult:  # eigs.hpp (thin_svd)
    U: object
    sigma: np.ndarray
    V: object


def thin_svd(A, ctx=None) -> SvdResult:
    """eigs.cpp:53-57 on the device (fp64).  Column signs are unspecified, as
    with the reference's JacobiSVD."""
    a = _In(A, N.F64)
    if len(a.shape) != 2:
        raise ValueError("thin_svd: matrix required")
    m, n = a.shape
    q = min(m, n)
    cuda = _is_cuda(A)
    U, up = _out(cuda, _torch_device(A), (m, q), N.F64)
    V, vp_ = _out(cuda, _torch_device(A), (n, q), N.F64)
    s = np.empty(q, np.float64)
    N.check(N.lib().cpcag_cuda_thin_svd(_ctx(ctx), a.ptr, m, n, up, s.ctypes.data if q else None, vp_))
    return SvdResult(U, s, V)


def detect_rank(sigma, threshold: float) -> int:
    """eigs.cpp:59-64 (host logic on the singular values)."""
    s = np.asarray(sigma, np.float64)
    if s.size == 0 or not s[0] > 0.0:
        return 0
    k = 0
    while k < s.size and s[k] / s[0] >= threshold:
        k += 1
    return k


def graph_upsample(L: SparseMatrix, known, R, pcg_tol: float = 1e-10, pcg_max_iter: int = 5000, ctx=None):
    """decoders.hpp:37-38 / decoders.cpp:72-121: rows `known` of the result
    equal R, the others solve L_aa S_a = -L_ab R (batched Jacobi PCG)."""
    if L.rows() != L.cols():
        raise ValueError("graph upsample: square Laplacian required")
    kn = np.ascontiguousarray(known, np.int64).ravel()
    r = _In(R, N.F64)
    rr = r.shape[1] if len(r.shape) == 2 else 1
    if r.shape[0] != kn.size:
        raise ValueError("graph upsample: known set and R row count differ")
    S, sp = _out(_is_cuda(R), _torch_device(R), (L.rows(), rr), N.F64)
    N.check(N.lib().cpcag_cuda_graph_upsample(_ctx(ctx), L.handle, kn.ctypes.data if kn.size else None, kn.size,
                                              r.ptr, rr, float(pcg_tol), int(pcg_max_iter), sp))
    return S


@dataclass
class LowRankFactors:  # decoders.hpp:26-32
    U: object
    sigma: np.ndarray
    V: object
    k: int = 0
    scale_applied: bool = False


@dataclass
class ApproxDecodeResult:  # decoders.hpp:64-67
    X: object
    factors: LowRankFactors


def approx_decode(Xt, plan: SamplingPlan, Lr: SparseMatrix, Lc: SparseMatrix, cfg: DecoderConfig = DecoderConfig(),
                  precision=None, ctx=None) -> ApproxDecodeResult:
    """decoders.hpp:69-72 / decoders.cpp:188-225 (Algorithm 2)."""
    prec = _precision(Xt, precision)
    xt = _In(Xt, prec)
    if tuple(xt.shape) != (plan.rho_r(), plan.rho_c()):
        raise ValueError("approximate decoder: Xt does not match plan")
    om_r = np.ascontiguousarray(plan.omega_r, np.int64)
    om_c = np.ascontiguousarray(plan.omega_c, np.int64)
    cuda = _is_cuda(Xt)
    X, xp = _out(cuda, _torch_device(Xt), (plan.p, plan.n), prec)
    kcap = max(1, min(plan.rho_r(), plan.rho_c()))
    U = np.empty((plan.p, kcap), np.float64, order="F")
    V = np.empty((plan.n, kcap), np.float64, order="F")
    s = np.empty(kcap, np.float64)
    k = N.i64()
    c = cfg.approx_c()
    N.check(N.lib().cpcag_cuda_approx_decode(_ctx(ctx), prec, xt.ptr, plan.rho_r(), plan.rho_c(),
                                             om_r.ctypes.data if om_r.size else None,
                                             om_c.ctypes.data if om_c.size else None, plan.p, plan.n, Lr.handle,
                                             Lc.handle, C.byref(c), xp, U.ctypes.data, s.ctypes.data,
                                             V.ctypes.data, kcap, C.byref(k)))
    kk = int(k.value)
    f = LowRankFactors(np.asfortranarray(U.ravel(order="F")[: plan.p * kk].reshape((plan.p, kk), order="F")),
                       s[:kk].copy(),
                       np.asfortranarray(V.ravel(order="F")[: plan.n * kk].reshape((plan.n, kk), order="F")), kk,
                       True)
    return ApproxDecodeResult(X, f)


# ------------------------------------------------------------------ pipeline
STAGES = ("graphs", "plan", "subsample", "kron", "solve", "decode")


@dataclass
class PipelineConfig:  # pipeline.hpp:36-63
    knn: int = 10
    laplacian: str = "combinatorial"
    sigma2: float = 0.0
    a: int = 1
    b: int = 1
    rho_r_override: int = 0
    rho_c_override: int = 0
    kron_pcg_tol: float = 1e-11
    frpcag: FrpcagConfig = field(default_factory=FrpcagConfig)
    decoder: DecoderConfig = field(default_factory=DecoderConfig)
    lambda_k1_r: float = 0.0  # <= 0: computed on the device as the reference does (pipeline.cpp:343-349)
    lambda_k1_c: float = 0.0
    seed: int = 0
    task: str = "lowrank"     # Task (pipeline.hpp:18): "lowrank" | "cluster" | "both"
    n_clusters: int = 0       # 0: max(1, detected rank) (pipeline.cpp:374)
    kmeans_restarts: int = 10

    def c(self) -> N.PipelineConfigC:
        return N.PipelineConfigC(int(self.knn), _kind(self.laplacian), float(self.sigma2), int(self.a),
                                 int(self.b), int(self.rho_r_override), int(self.rho_c_override),
                                 float(self.kron_pcg_tol), self.frpcag.c(), self.decoder.c(),
                                 float(self.lambda_k1_r), float(self.lambda_k1_c),
                                 int(self.seed) & (2**64 - 1), _variant(self.decoder.variant),
                                 self.decoder.approx_c(), _task(self.task), int(self.n_clusters),
                                 int(self.kmeans_restarts))


def _task(t) -> int:
    table = {"lowrank": 0, "cluster": 1, "both": 2}
    if t not in table:
        raise ValueError(f"unknown task {t!r}")
    return table[t]


def _variant(v) -> int:
    table = {"ideal": N.DECODER_IDEAL, "alternate": N.DECODER_ALTERNATE, "approx": N.DECODER_APPROX}
    if v in table:
        return table[v]
    if v in table.values():
        return int(v)
    raise ValueError(f"unknown decoder variant {v!r}")


@dataclass
class PipelineReport:  # pipeline.hpp:73-94 (subset)
    p: int
    n: int
    rho_r: int
    rho_c: int
    trace: SolveTrace
    plan: SamplingPlan
    Xt: object
    X: object
    decoder_converged: bool
    decoder_iterations: int
    stages: dict
    detected_rank: int = 0
    factors: Optional[LowRankFactors] = None  # approximate decoder only
    has_factors: bool = False
    lambda_k1: tuple = (0.0, 0.0)  # gaps the alternate decoder used (rows, columns)
    labels: Optional[np.ndarray] = None  # decoded cluster labels (cluster/both tasks, pipeline.hpp:89)

    def stage_ms(self, name: str) -> float:
        return self.stages.get(name, 0.0)


def run_pipeline(Y, cfg: PipelineConfig, W_r: Optional[SparseMatrix] = None,
                 W_c: Optional[SparseMatrix] = None, precision=None, ctx=None, out=None) -> PipelineReport:
    """pipeline.hpp:100 / pipeline.cpp:228-350 on a resident data matrix Y (p x n).

    out: optional (Xt, X) column-major buffers to write the results into (for
    host inputs, e.g. views of pinned memory reused across calls, so the
    device->host copies are direct DMA); by default they are allocated."""
    prec = _precision(Y, precision)
    y = _In(Y, prec)
    p, n = y.shape
    rho_r = cfg.rho_r_override if cfg.rho_r_override > 0 else -(-p // max(cfg.b, 1))
    rho_c = cfg.rho_c_override if cfg.rho_c_override > 0 else -(-n // max(cfg.a, 1))
    rho_r, rho_c = min(rho_r, p), min(rho_c, n)
    cuda = _is_cuda(Y)
    if out is not None:
        xt, xtp = _given_out(out[0], (rho_r, rho_c), prec, "out[0] (Xt)")
        x, xp = _given_out(out[1], (p, n), prec, "out[1] (X)")
    else:
        xt, xtp = _out(cuda, _torch_device(Y), (rho_r, rho_c), prec)
        x, xp = _out(cuda, _torch_device(Y), (p, n), prec) if cfg.task != "cluster" else (None, None)
    om_r = np.empty(max(rho_r, 1), np.int64)
    om_c = np.empty(max(rho_c, 1), np.int64)
    obj = np.zeros(max(int(cfg.frpcag.max_iter), 1))
    rep = N.PipelineReportC()
    c = cfg.c()
    kcap = max(1, min(rho_r, rho_c)) if _variant(cfg.decoder.variant) == N.DECODER_APPROX else 0
    fU = np.empty((p, kcap), np.float64, order="F")
    fV = np.empty((n, kcap), np.float64, order="F")
    fs = np.empty(max(kcap, 1), np.float64)
    labels = np.empty(n, np.int32) if cfg.task in ("cluster", "both") else None
    fac = N.PipelineFactorsC(fU.ctypes.data if kcap else None, fs.ctypes.data if kcap else None,
                             fV.ctypes.data if kcap else None, kcap,
                             labels.ctypes.data if labels is not None else None)
    N.check(N.lib().cpcag_cuda_run_pipeline(_ctx(ctx), prec, y.ptr, p, n, W_r.handle if W_r else None,
                                            W_c.handle if W_c else None, C.byref(c), xtp, xp,
                                            om_r.ctypes.data, om_c.ctypes.data, obj.ctypes.data,
                                            C.byref(rep), C.byref(fac)))
    it = int(rep.trace.iterations)
    trace = SolveTrace(list(obj[:it]), it, bool(rep.trace.converged), float(rep.trace.final_rel_change),
                       float(rep.trace.step))
    plan = SamplingPlan(om_r[:rep.rho_r].copy(), om_c[:rep.rho_c].copy(), p, n, seed=cfg.seed)
    stages = {name: float(rep.stage_ms[k]) for k, name in enumerate(STAGES)}
    if labels is not None:
        stages["cluster"] = float(rep.cluster_ms)
    factors = None
    if rep.has_factors:
        k = int(rep.factors_k)
        factors = LowRankFactors(np.asfortranarray(fU[:, :k]), fs[:k].copy(), np.asfortranarray(fV[:, :k]), k, True)
    return PipelineReport(int(rep.p), int(rep.n), int(rep.rho_r), int(rep.rho_c), trace, plan, xt, x,
                          bool(rep.decoder_converged), int(rep.decoder_iterations), stages,
                          int(rep.detected_rank), factors, bool(rep.has_factors),
                          (float(rep.lambda_k1_r), float(rep.lambda_k1_c)), labels)


# ------------------------------------------------------------------ I/O (io.hpp:14-44)
def glr1_info(path: str):
    """(kind, dims) of a GLR1 file: kind 1 dense (rows, cols), 2 CSR (rows,
    cols, nnz), 3 factors (p, n, k, scale flag)."""
    kind = N.i64()
    dims = (N.i64 * 4)()
    N.check(N.lib().cpcag_glr1_info(os.fsencode(path), C.byref(kind), dims))
    nd = {1: 2, 2: 3, 3: 4}[int(kind.value)]
    return int(kind.value), tuple(int(dims[i]) for i in range(nd))


def load_matrix(path: str, format: str = "glr1", precision=None, device=None, ctx=None):
    """io.cpp:88-149.  glr1: streamed through pinned buffers into a
    column-major CUDA tensor (device given, default "cuda") or a numpy array
    (device="cpu"); fp32 destinations are narrowed on the device.  csv:
    "rows,cols" header then one line per row (host text, as the reference)."""
    prec = N.F64 if precision in (None, "f64", N.F64, np.float64) else N.F32
    if format == "csv":
        return _load_csv(path, prec)
    if format != "glr1":
        raise ValueError("load_matrix: format must be 'glr1' or 'csv'")
    kind, dims = glr1_info(path)
    if kind != 1:
        raise RuntimeError(f"{path}: not a dense-matrix block")
    rows, cols = dims
    dev = "cuda" if device is None else device
    out, op = _out(str(dev) != "cpu", dev if str(dev) != "cpu" else None, (rows, cols), prec)
    N.check(N.lib().cpcag_cuda_load_matrix_glr1(_ctx(ctx), os.fsencode(path), prec, op, rows, cols))
    return out


def save_matrix(M, path: str, format: str = "glr1", precision=None, ctx=None):
    """io.cpp:88-117 (fp64 on disk; fp32 device data is widened on the device)."""
    if format == "csv":
        a = M.detach().cpu().numpy() if _is_torch(M) else np.asarray(M)
        _save_csv(np.asarray(a, np.float64), path)
        return
    if format != "glr1":
        raise ValueError("save_matrix: format must be 'glr1' or 'csv'")
    prec = _precision(M, precision)
    m = _In(M, prec)
    if len(m.shape) != 2:
        raise ValueError("save_matrix: M must be a matrix")
    N.check(N.lib().cpcag_cuda_save_matrix_glr1(_ctx(ctx), os.fsencode(path), prec, m.ptr, m.shape[0], m.shape[1]))


def load_sparse(path: str, ctx=None) -> "SparseMatrix":
    """io.cpp:164-188: CSR block -> device SparseMatrix."""
    h = N.vp()
    N.check(N.lib().cpcag_cuda_load_sparse_glr1(_ctx(ctx), os.fsencode(path), C.byref(h)))
    return SparseMatrix(h, ctx)


def save_sparse(A: "SparseMatrix", path: str, ctx=None):
    """io.cpp:151-162."""
    N.check(N.lib().cpcag_cuda_save_sparse_glr1(_ctx(ctx), A.handle, os.fsencode(path)))


def save_factors(f: LowRankFactors, path: str, ctx=None):
    """io.cpp:200-211."""
    U = np.asfortranarray(f.U, np.float64)
    V = np.asfortranarray(f.V, np.float64)
    s = np.ascontiguousarray(f.sigma, np.float64)
    N.check(N.lib().cpcag_cuda_save_factors_glr1(_ctx(ctx), os.fsencode(path), U.shape[0], V.shape[0], int(f.k),
                                                 int(bool(f.scale_applied)), U.ctypes.data, s.ctypes.data,
                                                 V.ctypes.data))


def load_factors(path: str, ctx=None) -> LowRankFactors:
    """io.cpp:213-230."""
    kind, dims = glr1_info(path)
    if kind != 3:
        raise RuntimeError(f"{path}: not a factors block")
    p, n, k, _ = dims
    U = np.empty((p, k), np.float64, order="F")
    V = np.empty((n, k), np.float64, order="F")
    s = np.empty(k, np.float64)
    sc = C.c_int()
    N.check(N.lib().cpcag_cuda_load_factors_glr1(_ctx(ctx), os.fsencode(path), p, n, k, C.byref(sc),
                                                 U.ctypes.data, s.ctypes.data, V.ctypes.data))
    return LowRankFactors(U, s, V, k, bool(sc.value))


def _save_csv(a: np.ndarray, path: str):
    with open(path, "w") as f:
        f.write(f"{a.shape[0]},{a.shape[1]}\n")
        for row in a:
            f.write(",".join(_g17(x) for x in row) + "\n")


def _g17(x: float) -> str:
    return "%.17g" % x


def _load_csv(path: str, prec: int):
    """io.cpp:119-149 with its error texts."""
    try:
        f = open(path)
    except OSError:
        raise RuntimeError(f"{path}: cannot open for reading")
    with f:
        lines = f.read().split("\n")
    if not lines or lines[0] == "":
        raise RuntimeError(f"{path}: empty file")
    head = lines[0].split(",")
    if len(head) < 2:
        raise RuntimeError(f"{path}: malformed dimension header at line 1")
    rows, cols = int(_num(head[0], path, 1)), int(_num(head[1], path, 1))
    if rows < 0 or cols < 0:
        raise RuntimeError(f"{path}: negative dimensions in header")
    a = np.empty((rows, cols), np.float64, order="F")
    for i in range(rows):
        if i + 1 >= len(lines):
            raise RuntimeError(f"{path}: missing row {i + 1}")
        tok = lines[i + 1].split(",") if lines[i + 1] != "" else []
        if len(tok) < cols:
            raise RuntimeError(f"{path}: row {i + 1} has fewer than {cols} columns")
        if len(tok) > cols:
            raise RuntimeError(f"{path}: row {i + 1} has more than {cols} columns (dimension header mismatch)")
        for j in range(cols):
            a[i, j] = _num(tok[j], path, i + 2)
    return a if prec == N.F64 else a.astype(np.float32, order="F")


def _num(tok: str, path: str, line: int) -> float:
    try:
        if tok.strip() != tok or tok == "":
            raise ValueError
        return float(tok)
    except ValueError:
        raise RuntimeError(f"{path}: malformed number '{tok}' at line {line}")


def plan_to_json(plan: SamplingPlan) -> str:
    """io.cpp:232-243: nlohmann::json dump(2) of {seed, p, n, omega_r,
    omega_c, delta, epsilon} (object keys in sorted order, as nlohmann's
    std::map-backed objects print them)."""
    import json

    d = {"seed": int(plan.seed), "p": int(plan.p), "n": int(plan.n),
         "omega_r": [int(x) for x in plan.omega_r], "omega_c": [int(x) for x in plan.omega_c],
         "delta": float(plan.delta), "epsilon": float(plan.epsilon)}
    return json.dumps(d, indent=2, sort_keys=True)


def plan_from_json(text: str) -> SamplingPlan:
    """io.cpp:245-263 (index ranges validated)."""
    import json

    j = json.loads(text)
    plan = SamplingPlan(np.asarray(j["omega_r"], np.int64), np.asarray(j["omega_c"], np.int64), int(j["p"]),
                        int(j["n"]), float(j["delta"]), float(j["epsilon"]), int(j["seed"]))
    if np.any(plan.omega_r < 0) or np.any(plan.omega_r >= plan.p):
        raise RuntimeError("plan: omega_r index out of range")
    if np.any(plan.omega_c < 0) or np.any(plan.omega_c >= plan.n):
        raise RuntimeError("plan: omega_c index out of range")
    return plan


def save_plan(plan: SamplingPlan, path: str):
    with open(path, "w") as f:
        f.write(plan_to_json(plan) + "\n")


def load_plan(path: str) -> SamplingPlan:
    with open(path) as f:
        return plan_from_json(f.read())


# ------------------------------------------------------------------ clustering (clustering.hpp)
@dataclass
class ClusterLabels:  # clustering.hpp:13-21
    assignments: np.ndarray
    k: int = 0

    def size(self) -> int:
        return len(self.assignments)

    def indicator(self) -> np.ndarray:
        C = np.zeros((self.size(), self.k))
        C[np.arange(self.size()), self.assignments] = 1.0
        return C

    @staticmethod
    def from_assignments(assignments, k: int) -> "ClusterLabels":
        a = np.asarray(assignments, np.int32)
        if k < 1:
            raise ValueError("labels: k must be >= 1")
        if np.any(a < 0) or np.any(a >= k):
            raise ValueError("labels: assignment out of range")
        return ClusterLabels(a, int(k))


def kmeans(X, k: int, restarts: int = 10, seed: int = 0, max_iter: int = 100, precision=None,
           ctx=None) -> ClusterLabels:
    """clustering.hpp:26-29: k-means++ / Lloyd on the columns of X, on the device."""
    prec = _precision(X, precision)
    x = _In(X, prec)
    if len(x.shape) != 2:
        raise ValueError("kmeans: X must be a matrix")
    rows, n = x.shape
    a = np.empty(max(n, 1), np.int32)
    w = N.dbl()
    N.check(N.lib().cpcag_cuda_kmeans(_ctx(ctx), prec, x.ptr, rows, n, int(k), int(restarts), int(seed) & (2**64 - 1),
                                      int(max_iter), a.ctypes.data, C.byref(w)))
    return ClusterLabels(a[:n].copy(), int(k))


def decode_labels(sampled: ClusterLabels, plan: SamplingPlan, Lc: "SparseMatrix", pcg_tol: float = 1e-10,
                  pcg_max_iter: int = 5000, ctx=None) -> ClusterLabels:
    """clustering.hpp:31-35 / clustering.cpp:139-160 on the device."""
    if sampled.size() != plan.rho_c():
        raise ValueError("decode_labels: sampled labels do not match plan")
    if Lc.rows() != plan.n:
        raise ValueError("decode_labels: column Laplacian does not match plan")
    lab = np.ascontiguousarray(sampled.assignments, np.int32)
    om = np.ascontiguousarray(plan.omega_c, np.int64)
    out = np.empty(max(plan.n, 1), np.int32)
    N.check(N.lib().cpcag_cuda_decode_labels(_ctx(ctx), lab.ctypes.data, len(lab), int(sampled.k), om.ctypes.data,
                                             int(plan.n), Lc.handle, float(pcg_tol), int(pcg_max_iter),
                                             out.ctypes.data))
    return ClusterLabels(out[:plan.n].copy(), int(sampled.k))


def clustering_error(pred: ClusterLabels, truth: ClusterLabels) -> float:
    """clustering.hpp:37-39 / clustering.cpp:220-238."""
    if pred.size() != truth.size():
        raise ValueError("clustering error: label vectors differ in length")
    p = np.ascontiguousarray(pred.assignments, np.int32)
    t = np.ascontiguousarray(truth.assignments, np.int32)
    out = N.dbl()
    N.check(N.lib().cpcag_clustering_error(p.ctypes.data, t.ctypes.data, len(p), int(pred.k), int(truth.k),
                                           C.byref(out)))
    return float(out.value)


def save_labels_csv(labels, path: str):
    """io.cpp:268-273: "index,label" header, one line per item."""
    with open(path, "w") as f:
        f.write("index,label\n")
        for i, v in enumerate(np.asarray(labels).tolist()):
            f.write(f"{i},{int(v)}\n")


def load_labels_csv(path: str) -> np.ndarray:
    """io.cpp:275-290."""
    try:
        f = open(path)
    except OSError:
        raise RuntimeError(f"{path}: cannot open for reading")
    with f:
        lines = f.read().split("\n")
    if not lines or lines[0] == "":
        raise RuntimeError(f"{path}: empty file")
    out = []
    for no, line in enumerate(lines[1:], start=2):
        if line == "":
            continue
        if "," not in line:
            raise RuntimeError(f"{path}: missing comma at line {no}")
        out.append(int(_num(line.split(",", 1)[1], path, no)))
    return np.asarray(out, np.int32)


def report_to_json(rep: "PipelineReport", cfg: "PipelineConfig", include_timings: bool = True) -> str:
    """pipeline.cpp:393-415 for the fields this mirror models (the config
    subset of PipelineConfig, sizes, detected rank, the FISTA trace and the
    stage timings)."""
    import dataclasses
    import json

    def conf(c):
        d = dataclasses.asdict(c)
        return json.loads(json.dumps(d, default=str))

    j = {"config": conf(cfg), "p": rep.p, "n": rep.n, "rho_r": rep.rho_r, "rho_c": rep.rho_c, "seed": int(cfg.seed),
         "detected_rank": rep.detected_rank,
         "solve": {"iterations": rep.trace.iterations, "converged": bool(rep.trace.converged),
                   "final_rel_change": rep.trace.final_rel_change, "step": rep.trace.step,
                   "objective": [float(x) for x in rep.trace.objective]}}
    if include_timings:
        j["timings_ms"] = {k: float(v) for k, v in rep.stages.items()}
    return json.dumps(j, indent=2, sort_keys=True)


def emit_report(rep: "PipelineReport", cfg: "PipelineConfig", out_dir: str, ctx=None):
    """pipeline.cpp:417-439: report.json, plan.json, solution_compressed.glr1,
    decoded.glr1 + decoded.csv (when decoded), factors.glr1 (approximate
    decoder), labels.csv (clustering tasks), objective.csv.  Device results
    are written straight from HBM (GLR1 through pinned buffers)."""
    os.makedirs(out_dir, exist_ok=True)
    with open(os.path.join(out_dir, "report.json"), "w") as f:
        f.write(report_to_json(rep, cfg, True) + "\n")
    save_plan(rep.plan, os.path.join(out_dir, "plan.json"))
    save_matrix(rep.Xt, os.path.join(out_dir, "solution_compressed.glr1"), ctx=ctx)
    if rep.X is not None:
        save_matrix(rep.X, os.path.join(out_dir, "decoded.glr1"), ctx=ctx)
        save_matrix(rep.X, os.path.join(out_dir, "decoded.csv"), format="csv")
    if rep.has_factors and rep.factors is not None:
        save_factors(rep.factors, os.path.join(out_dir, "factors.glr1"), ctx=ctx)
    if rep.labels is not None:
        save_labels_csv(rep.labels, os.path.join(out_dir, "labels.csv"))
    with open(os.path.join(out_dir, "objective.csv"), "w") as f:
        f.write("iteration,objective\n")
        for i, v in enumerate(rep.trace.objective):
            f.write(f"{i + 1},{_g17(float(v))}\n")
