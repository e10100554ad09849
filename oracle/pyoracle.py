"""ctypes binding of the CPU oracle (oracle/_build/libcpcag_oracle.so).

TEST INFRASTRUCTURE ONLY.  The oracle is the checker for the CUDA product
path: only tests/, ``__graft_entry__.smoke()`` and bench.py's
``cpu_baseline`` / ``--impl reference`` legs may import this module.  The
product package (paper_1602_02070_b200) never imports it.

Every function restates a reference routine (see oracle/cpcag_oracle.cpp for
the file:line each follows) and raises the reference's exception type with
the reference's message.
"""
from __future__ import annotations

import ctypes as C
import math
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "_build", "libcpcag_oracle.so")
_lib = None

i64 = C.c_int64
dp = C.POINTER(C.c_double)
ip = C.POINTER(C.c_int64)
vp = C.c_void_p


class FrpcagCfg(C.Structure):
    _fields_ = [
        ("gamma_r", C.c_double),
        ("gamma_c", C.c_double),
        ("loss_l2", C.c_int),
        ("tol", C.c_double),
        ("max_iter", C.c_int64),
        ("step", C.c_double),
    ]


def build() -> str:
    """Compile the oracle (make in oracle/); returns the .so path."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = C.CDLL(_LIB_PATH)
        L.ora_last_error.restype = C.c_char_p
        L.ora_csr_rows.restype = i64
        L.ora_csr_cols.restype = i64
        L.ora_csr_nnz.restype = i64
        L.ora_rng_mix.restype = C.c_uint64
        L.ora_rng_mix.argtypes = [C.c_uint64]
        L.ora_rng_derive_seed.restype = C.c_uint64
        L.ora_rng_derive_seed.argtypes = [C.c_uint64, C.c_uint64]
        L.ora_rng_u64.argtypes = [C.c_uint64, i64, C.POINTER(C.c_uint64)]
        L.ora_rng_gaussian.argtypes = [C.c_uint64, i64, dp]
        L.ora_power_iteration_norm.argtypes = [vp, C.c_double, C.c_uint64, i64, dp]
        L.ora_draw_plan.argtypes = [i64, i64, i64, i64, C.c_uint64, ip, ip]
        L.ora_kmeans.argtypes = [dp, i64, i64, i64, i64, C.c_uint64, i64, C.POINTER(C.c_int), dp]
        L.ora_clustering_error.argtypes = [C.POINTER(C.c_int), C.POINTER(C.c_int), i64, i64, dp]
        _lib = L
    return _lib


def _check(rc: int) -> None:
    if rc == 0:
        return
    msg = lib().ora_last_error().decode()
    if rc == 1:
        raise ValueError(msg)
    if rc == 3:
        raise IndexError(msg)
    raise RuntimeError(msg)


def _d(a: np.ndarray):
    return a.ctypes.data_as(dp)


def _i(a: np.ndarray):
    return a.ctypes.data_as(ip)


def _f64(a) -> np.ndarray:
    return np.asfortranarray(np.asarray(a, dtype=np.float64))


def _idx(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.int64))


def set_threads(n: int) -> None:
    lib().ora_set_threads(int(n))


def get_threads() -> int:
    return int(lib().ora_get_threads())


class Csr:
    """Owning handle of an oracle CSR matrix (sparse.hpp:18-66 layout)."""

    def __init__(self, handle):
        self._h = handle if isinstance(handle, vp) else vp(handle)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value and _lib is not None:
            _lib.ora_csr_free(h)
            self._h = None

    @property
    def handle(self):
        return self._h

    @property
    def rows(self) -> int:
        return int(lib().ora_csr_rows(self._h))

    @property
    def cols(self) -> int:
        return int(lib().ora_csr_cols(self._h))

    @property
    def nnz(self) -> int:
        return int(lib().ora_csr_nnz(self._h))

    def arrays(self):
        rp = np.empty(self.rows + 1, np.int64)
        ci = np.empty(self.nnz, np.int64)
        v = np.empty(self.nnz, np.float64)
        lib().ora_csr_export(self._h, _i(rp), _i(ci), _d(v))
        return rp, ci, v

    def to_dense(self) -> np.ndarray:
        rp, ci, v = self.arrays()
        D = np.zeros((self.rows, self.cols))
        for r in range(self.rows):
            D[r, ci[rp[r]:rp[r + 1]]] = v[rp[r]:rp[r + 1]]
        return D

    def to_scipy(self):
        import scipy.sparse as sp

        rp, ci, v = self.arrays()
        return sp.csr_matrix((v, ci, rp), shape=(self.rows, self.cols))

    @staticmethod
    def from_triplets(rows, cols, ti, tj, tv, drop_below=0.0) -> "Csr":
        ti, tj, tv = _idx(ti), _idx(tj), np.ascontiguousarray(tv, np.float64)
        out = vp()
        _check(lib().ora_csr_from_triplets(i64(rows), i64(cols), i64(len(tv)), _i(ti), _i(tj),
                                           _d(tv), C.c_double(drop_below), C.byref(out)))
        return Csr(out)

    @staticmethod
    def from_csr(rows, cols, rp, ci, v) -> "Csr":
        rp, ci, v = _idx(rp), _idx(ci), np.ascontiguousarray(v, np.float64)
        out = vp()
        _check(lib().ora_csr_from_csr(i64(rows), i64(cols), _i(rp), _i(ci), _d(v), C.byref(out)))
        return Csr(out)

    @staticmethod
    def from_dense(D, drop_below=0.0) -> "Csr":
        D = _f64(D)
        out = vp()
        _check(lib().ora_csr_from_dense(_d(D), i64(D.shape[0]), i64(D.shape[1]),
                                        C.c_double(drop_below), C.byref(out)))
        return Csr(out)

    @staticmethod
    def from_scipy(S) -> "Csr":
        S = S.tocsr()
        S.sort_indices()
        return Csr.from_csr(S.shape[0], S.shape[1], S.indptr, S.indices, S.data)

    def submatrix(self, rows, cols) -> "Csr":
        rows, cols = _idx(rows), _idx(cols)
        out = vp()
        _check(lib().ora_csr_submatrix(self._h, _i(rows), i64(len(rows)), _i(cols),
                                       i64(len(cols)), C.byref(out)))
        return Csr(out)

    def row_sums(self) -> np.ndarray:
        out = np.empty(self.rows)
        lib().ora_csr_row_sums(self._h, _d(out))
        return out

    def components(self):
        lab = np.empty(self.rows, np.int64)
        nc = i64()
        _check(lib().ora_csr_components(self._h, _i(lab), C.byref(nc)))
        return lab, int(nc.value)

    def spmv(self, x) -> np.ndarray:
        x = np.ascontiguousarray(x, np.float64)
        y = np.empty(self.rows)
        _check(lib().ora_spmv(self._h, _d(x), i64(len(x)), _d(y)))
        return y

    def multiply(self, X) -> np.ndarray:
        X = _f64(X)
        if X.ndim == 1:
            return self.spmv(X)
        Y = np.empty((self.rows, X.shape[1]), order="F")
        _check(lib().ora_spmm_left(self._h, _d(X), i64(X.shape[0]), i64(X.shape[1]), _d(Y)))
        return Y

    def right_multiply(self, X) -> np.ndarray:
        X = _f64(X)
        Y = np.empty((X.shape[0], self.cols), order="F")
        _check(lib().ora_spmm_right(self._h, _d(X), i64(X.shape[0]), i64(X.shape[1]), _d(Y)))
        return Y


# ----------------------------------------------------------------- RNG
def rng_mix(z: int) -> int:
    return int(lib().ora_rng_mix(C.c_uint64(z & 0xFFFFFFFFFFFFFFFF)))


def rng_derive_seed(seed: int, stream: int) -> int:
    return int(lib().ora_rng_derive_seed(C.c_uint64(seed), C.c_uint64(stream)))


def rng_u64(seed: int, count: int) -> np.ndarray:
    out = np.empty(count, np.uint64)
    lib().ora_rng_u64(C.c_uint64(seed), i64(count), out.ctypes.data_as(C.POINTER(C.c_uint64)))
    return out


def rng_gaussian(seed: int, count: int) -> np.ndarray:
    out = np.empty(count)
    lib().ora_rng_gaussian(C.c_uint64(seed), i64(count), _d(out))
    return out


def gaussian_matrix(rows: int, cols: int, seed: int) -> np.ndarray:
    """oracles.hpp:26-32: CounterRng(mix(seed)), column-major fill."""
    v = rng_gaussian(rng_mix(seed), rows * cols)
    return v.reshape((rows, cols), order="F")


# ----------------------------------------------------------------- solvers
@dataclass
class PcgResult:
    iterations: int
    converged: bool
    relative_residual: float


def pcg_solve(A: Csr, b, x=None, tol=1e-10, max_iter=5000, jacobi=True):
    b = np.ascontiguousarray(b, np.float64)
    x = np.zeros_like(b) if x is None else np.ascontiguousarray(x, np.float64).copy()
    it, cv, rr = i64(), C.c_int(), C.c_double()
    _check(lib().ora_pcg_solve(A.handle, _d(b), _d(x), i64(len(b)), C.c_double(tol),
                               i64(max_iter), C.c_int(1 if jacobi else 0), C.byref(it),
                               C.byref(cv), C.byref(rr)))
    return x, PcgResult(int(it.value), bool(cv.value), float(rr.value))


def power_iteration_norm(A: Csr, tol=1e-9, seed=0, max_iter=50000) -> float:
    out = C.c_double()
    _check(lib().ora_power_iteration_norm(A.handle, C.c_double(tol), C.c_uint64(seed),
                                          i64(max_iter), C.byref(out)))
    return float(out.value)


# ----------------------------------------------------------------- graphs
@dataclass
class GraphModel:
    n_nodes: int
    K: int
    sigma2: float
    adjacency: Csr
    degrees: np.ndarray
    laplacian: Csr
    normalized: bool = False


def build_knn_graph(X, axis_rows: bool, K: int, normalized=False, sigma2_override=0.0):
    X = _f64(X)
    n = X.shape[0] if axis_rows else X.shape[1]
    W, L = vp(), vp()
    deg = np.empty(max(n, 0))
    s2 = C.c_double()
    _check(lib().ora_knn_graph(_d(X), i64(X.shape[0]), i64(X.shape[1]), C.c_int(int(axis_rows)),
                               i64(K), C.c_int(int(normalized)), C.c_double(sigma2_override),
                               C.byref(W), C.byref(L), _d(deg), C.byref(s2)))
    return GraphModel(n, K, float(s2.value), Csr(W), deg, Csr(L), normalized)


def knn_neighbors(X, axis_rows: bool, K: int):
    X = _f64(X)
    n = X.shape[0] if axis_rows else X.shape[1]
    nbr = np.empty((n, K), np.int64)
    d2 = np.empty((n, K))
    _check(lib().ora_knn_neighbors(_d(X), i64(X.shape[0]), i64(X.shape[1]),
                                   C.c_int(int(axis_rows)), i64(K), _i(nbr), _d(d2)))
    return nbr, d2


def knn_rows(X, axis_rows: bool, K: int, rows):
    """Exact kNN lists (graph.cpp:86-105) of the query points `rows` only."""
    X = _f64(X)
    rows = _idx(rows)
    nbr = np.empty((len(rows), K), np.int64)
    d2 = np.empty((len(rows), K))
    _check(lib().ora_knn_rows(_d(X), i64(X.shape[0]), i64(X.shape[1]), C.c_int(int(axis_rows)), i64(K),
                              _i(rows), i64(len(rows)), _i(nbr), _d(d2)))
    return nbr, d2


def graph_from_adjacency(W: Csr, normalized=False) -> GraphModel:
    L = vp()
    deg = np.empty(W.rows)
    _check(lib().ora_graph_from_adjacency(W.handle, C.c_int(int(normalized)), C.byref(L), _d(deg)))
    return GraphModel(W.rows, 0, 0.0, W, deg, Csr(L), normalized)


def kron_reduce(L: Csr, keep, pcg_tol=1e-12, prune_tol=1e-12) -> Csr:
    keep = _idx(keep)
    out = vp()
    _check(lib().ora_kron_reduce(L.handle, _i(keep), i64(len(keep)), C.c_double(pcg_tol),
                                 C.c_double(prune_tol), C.byref(out)))
    return Csr(out)


# ----------------------------------------------------------------- sampling
@dataclass
class SamplingPlan:
    omega_r: np.ndarray
    omega_c: np.ndarray
    p: int
    n: int
    delta: float = 0.0
    epsilon: float = 0.0
    seed: int = 0

    @property
    def rho_r(self):
        return len(self.omega_r)

    @property
    def rho_c(self):
        return len(self.omega_c)

    def norm_const(self):
        return (float(self.n) * float(self.p)) / (float(self.rho_r) * float(self.rho_c))


def draw_plan(p, n, rho_r, rho_c, delta=0.0, epsilon=0.0, seed=0) -> SamplingPlan:
    om_r = np.empty(max(rho_r, 0), np.int64)
    om_c = np.empty(max(rho_c, 0), np.int64)
    _check(lib().ora_draw_plan(i64(p), i64(n), i64(rho_r), i64(rho_c), C.c_uint64(seed),
                               _i(om_r), _i(om_c)))
    return SamplingPlan(om_r, om_c, p, n, delta, epsilon, seed)


def subsample(Y, plan: SamplingPlan) -> np.ndarray:
    Y = _f64(Y)
    if Y.shape != (plan.p, plan.n):
        raise ValueError("subsample: plan does not match matrix dimensions")
    out = np.empty((plan.rho_r, plan.rho_c), order="F")
    _check(lib().ora_subsample(_d(Y), i64(plan.p), i64(plan.n), _i(_idx(plan.omega_r)),
                               i64(plan.rho_r), _i(_idx(plan.omega_c)), i64(plan.rho_c), _d(out)))
    return out


# ----------------------------------------------------------------- FRPCAG
@dataclass
class FrpcagConfig:
    gamma_r: float = 1.0
    gamma_c: float = 1.0
    loss: str = "l1"
    tol: float = 1e-10
    max_iter: int = 500
    step: float = 0.0

    def c(self) -> FrpcagCfg:
        return FrpcagCfg(self.gamma_r, self.gamma_c, 1 if self.loss == "l2" else 0, self.tol,
                         self.max_iter, self.step)


@dataclass
class SolveTrace:
    objective: list = field(default_factory=list)
    iterations: int = 0
    converged: bool = False
    final_rel_change: float = 0.0
    step: float = 0.0


def objective(X, Y, Lr: Csr, Lc: Csr, cfg: FrpcagConfig) -> float:
    X, Y = _f64(X), _f64(Y)
    if X.shape != Y.shape:
        raise ValueError("frpcag: X and Y dimensions differ")
    out = C.c_double()
    c = cfg.c()
    _check(lib().ora_objective(_d(X), _d(Y), i64(X.shape[0]), i64(X.shape[1]), Lr.handle,
                               Lc.handle, C.byref(c), C.byref(out)))
    return float(out.value)


def prox_l1(Z, Y, lam) -> np.ndarray:
    Z, Y = _f64(Z), _f64(Y)
    if Z.shape != Y.shape:
        raise ValueError("prox: Z and Y dimensions differ")
    out = np.empty_like(Z, order="F")
    _check(lib().ora_prox_l1(_d(Z), _d(Y), i64(Z.size), C.c_double(lam), _d(out)))
    return out


def prox_l2(Z, Y, lam) -> np.ndarray:
    Z, Y = _f64(Z), _f64(Y)
    if Z.shape != Y.shape:
        raise ValueError("prox: Z and Y dimensions differ")
    out = np.empty_like(Z, order="F")
    _check(lib().ora_prox_l2(_d(Z), _d(Y), i64(Z.size), C.c_double(lam), _d(out)))
    return out


def grad_g(Z, Lr: Csr, Lc: Csr, cfg: FrpcagConfig) -> np.ndarray:
    Z = _f64(Z)
    G = np.empty_like(Z, order="F")
    c = cfg.c()
    _check(lib().ora_grad_g(_d(Z), i64(Z.shape[0]), i64(Z.shape[1]), Lr.handle, Lc.handle,
                            C.byref(c), _d(G)))
    return G


def fista_solve(Y, Lr: Csr, Lc: Csr, cfg: FrpcagConfig):
    Y = _f64(Y)
    X = np.empty_like(Y, order="F")
    obj = np.zeros(max(cfg.max_iter, 1))
    it, cv, frc, st = i64(), C.c_int(), C.c_double(), C.c_double()
    c = cfg.c()
    _check(lib().ora_fista_solve(_d(Y), i64(Y.shape[0]), i64(Y.shape[1]), Lr.handle, Lc.handle,
                                 C.byref(c), _d(X), _d(obj), C.byref(it), C.byref(cv),
                                 C.byref(frc), C.byref(st)))
    n = int(it.value)
    return X, SolveTrace(list(obj[:n]), n, bool(cv.value), float(frc.value), float(st.value))


# ----------------------------------------------------------------- decoder
@dataclass
class AlternateDecodeResult:
    X: np.ndarray
    converged: bool
    iterations: int


def alternate_decode(Xt, plan: SamplingPlan, Lr: Csr, Lc: Csr, lambda_k1_r: float,
                     lambda_k1_c: float, gamma=1.0, pcg_tol=1e-10, pcg_max_iter=5000):
    Xt = _f64(Xt)
    X = np.empty((plan.p, plan.n), order="F")
    cv, it = C.c_int(), i64()
    if Xt.shape != (plan.rho_r, plan.rho_c):
        raise ValueError("alternate decoder: Xt does not match plan")
    _check(lib().ora_alternate_decode(_d(Xt), i64(plan.rho_r), i64(plan.rho_c),
                                      _i(_idx(plan.omega_r)), _i(_idx(plan.omega_c)),
                                      i64(plan.p), i64(plan.n), Lr.handle, Lc.handle,
                                      C.c_double(lambda_k1_r), C.c_double(lambda_k1_c),
                                      C.c_double(gamma), C.c_double(pcg_tol), i64(pcg_max_iter),
                                      _d(X), C.byref(cv), C.byref(it)))
    return AlternateDecodeResult(X, bool(cv.value), int(it.value))


def decoder_apply(X, plan: SamplingPlan, Lr: Csr, Lc: Csr, gbar_r: float, gbar_c: float):
    X = _f64(X)
    out = np.empty_like(X, order="F")
    _check(lib().ora_decoder_apply(_d(X), i64(plan.p), i64(plan.n), _i(_idx(plan.omega_r)),
                                   i64(plan.rho_r), _i(_idx(plan.omega_c)), i64(plan.rho_c),
                                   Lr.handle, Lc.handle, C.c_double(gbar_r), C.c_double(gbar_c),
                                   _d(out)))
    return out


# ----------------------------------------------------------------- approximate decoder
def graph_upsample(L: Csr, known, R, pcg_tol=1e-10, pcg_max_iter=5000):
    """decoders.cpp:72-121 (restated in cpcag_oracle.cpp)."""
    known = _idx(known)
    R = _f64(np.asarray(R).reshape(len(known), -1) if np.ndim(R) == 1 else R)
    if R.shape[0] != len(known):
        raise ValueError("graph upsample: known set and R row count differ")
    r = R.shape[1]
    S = np.empty((L.rows, r), order="F")
    _check(lib().ora_graph_upsample(L.handle, _i(known), i64(len(known)), _d(R), i64(r), C.c_double(pcg_tol),
                                    i64(pcg_max_iter), _d(S)))
    return S


def thin_svd(A):
    """eigs.cpp:53-57.  The reference uses Eigen's JacobiSVD; Eigen is absent
    here, so LAPACK (numpy gesdd) stands in: both return the exact SVD to
    working precision, and every consumer below is invariant to the
    per-column sign choice (align_factor_signs, U S V^T)."""
    A = np.asarray(A, np.float64)
    if not np.all(np.isfinite(A)):
        raise ValueError("thin_svd: non-finite input")
    U, s, Vt = np.linalg.svd(A, full_matrices=False)
    return U, s, Vt.T


def detect_rank(sigma, threshold):
    """eigs.cpp:59-64."""
    if len(sigma) == 0 or not sigma[0] > 0.0:
        return 0
    k = 0
    while k < len(sigma) and sigma[k] / sigma[0] >= threshold:
        k += 1
    return k


@dataclass
class ApproxDecodeResult:
    X: np.ndarray
    U: np.ndarray
    sigma: np.ndarray
    V: np.ndarray
    k: int


def approx_decode(Xt, plan: SamplingPlan, Lr: Csr, Lc: Csr, delta_for_scaling=0.0, rank_threshold=0.1,
                  pcg_tol=1e-10, pcg_max_iter=5000) -> ApproxDecodeResult:
    """decoders.cpp:188-225 (Algorithm 2), loop for loop."""
    Xt = _f64(Xt)
    if Xt.shape != (plan.rho_r, plan.rho_c):
        raise ValueError("approximate decoder: Xt does not match plan")
    if Lr.rows != plan.p or Lc.rows != plan.n:
        raise ValueError("approximate decoder: Laplacians do not match plan")
    if not (0.0 < rank_threshold < 1.0):
        raise ValueError("approximate decoder: rank threshold must be in (0,1)")
    Ut, s, Vt = thin_svd(Xt)
    k = detect_rank(s, rank_threshold)
    if k == 0:
        raise RuntimeError("approximate decoder: no singular value above the rank threshold")
    U = graph_upsample(Lr, plan.omega_r, Ut[:, :k], pcg_tol, pcg_max_iter)
    V = graph_upsample(Lc, plan.omega_c, Vt[:, :k], pcg_tol, pcg_max_iter)
    for j in range(k):  # decoders.cpp:208-215
        nu = math.sqrt(float(np.sum(U[:, j] * U[:, j])))
        nv = math.sqrt(float(np.sum(V[:, j] * V[:, j])))
        if nu <= 1e-14 or nv <= 1e-14:
            raise RuntimeError(f"approximate decoder: zero column {j} after upsampling (rank overestimated)")
        U[:, j] /= nu
        V[:, j] /= nv
    for j in range(k):  # align_factor_signs, decoders.cpp:33-50 (first largest |U(i,j)|)
        arg, best = 0, -1.0
        for i in range(U.shape[0]):
            a = abs(U[i, j])
            if a > best:
                best, arg = a, i
        if U[arg, j] < 0.0:
            U[:, j] = -U[:, j]
            V[:, j] = -V[:, j]
    if not (0.0 <= delta_for_scaling < 1.0):
        raise ValueError("decoder: delta_for_scaling must be in [0,1)")
    norm_const = (float(plan.n) * float(plan.p)) / (float(plan.rho_r) * float(plan.rho_c))
    sigma = math.sqrt(norm_const / (1.0 - delta_for_scaling)) * s[:k]
    X = np.asfortranarray((U * sigma) @ V.T)
    return ApproxDecodeResult(X, U, sigma, V, k)


def sym_eig(L: Csr, k: int):
    """eigs.cpp:34-51: dense symmetrised eigendecomposition (numpy LAPACK
    stands in for Eigen's SelfAdjointEigenSolver), first k pairs, column
    signs fixed so the first entry above 1e-12 of the column peak is
    positive."""
    rp, ci, v = L.arrays()
    n = L.rows
    D = np.zeros((n, n))
    for r in range(n):
        D[r, ci[rp[r]:rp[r + 1]]] = v[rp[r]:rp[r + 1]]
    D = 0.5 * (D + D.T)
    w, E = np.linalg.eigh(D)
    E = E[:, :k].copy()
    for j in range(k):
        peak = np.abs(E[:, j]).max()
        if peak == 0.0:
            continue
        idx = np.nonzero(np.abs(E[:, j]) > 1e-12 * peak)[0][0]
        if E[idx, j] < 0:
            E[:, j] = -E[:, j]
    return w[:k].copy(), E


def spectral_gap(eigenvalues, k):
    """graph.cpp:237-249."""
    if k < 1 or len(eigenvalues) < k + 1:
        raise ValueError("spectral gap: need at least k+1 eigenvalues")
    lk = max(0.0, float(eigenvalues[k - 1]))
    lk1 = max(0.0, float(eigenvalues[k]))
    if lk1 <= 1e-14:
        raise RuntimeError("gap undefined: graph has > k components")
    return lk, lk1, lk / lk1


# ------------------------------------------------------------------ clustering (clustering.cpp)
def kmeans(X, k, restarts=10, seed=0, max_iter=100):
    """clustering.cpp:40-137 on the columns of X.  Returns (assignments, wcss)."""
    X = _f64(np.asarray(X).reshape(-1, 1) if np.ndim(X) == 1 else X)
    rows, n = X.shape
    a = np.empty(n, np.int32)
    w = C.c_double()
    _check(lib().ora_kmeans(_d(X), i64(rows), i64(n), i64(k), i64(restarts), C.c_uint64(int(seed) & (2**64 - 1)),
                            i64(max_iter), a.ctypes.data_as(C.POINTER(C.c_int)), C.byref(w)))
    return a, w.value


def decode_labels(sampled, k, plan, Lc: Csr, pcg_tol=1e-10, pcg_max_iter=5000):
    """clustering.cpp:139-160: upsample the sampled-column indicator over the
    column graph, then row-wise max pooling (ties keep the lowest column)."""
    sampled = np.asarray(sampled, np.int64)
    if len(sampled) != len(plan.omega_c):
        raise ValueError("decode_labels: sampled labels do not match plan")
    if Lc.rows != plan.n:
        raise ValueError("decode_labels: column Laplacian does not match plan")
    if k < 1 or np.any(sampled < 0) or np.any(sampled >= k):
        raise ValueError("labels: assignment out of range")
    Ct = np.zeros((len(sampled), k))
    Ct[np.arange(len(sampled)), sampled] = 1.0
    Cm = graph_upsample(Lc, plan.omega_c, Ct, pcg_tol, pcg_max_iter)
    return np.argmax(Cm, axis=1).astype(np.int32), Cm  # argmax: first maximum = strict '>' scan


def clustering_error(pred, truth, k):
    """clustering.cpp:222-238 (Hungarian max assignment on the k x k
    contingency matrix)."""
    pred = np.ascontiguousarray(pred, np.int32)
    truth = np.ascontiguousarray(truth, np.int32)
    if len(pred) != len(truth):
        raise ValueError("clustering error: label vectors differ in length")
    out = C.c_double()
    _check(lib().ora_clustering_error(pred.ctypes.data_as(C.POINTER(C.c_int)), truth.ctypes.data_as(C.POINTER(C.c_int)),
                                      i64(len(pred)), i64(k), C.byref(out)))
    return out.value
