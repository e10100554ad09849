"""Seeded synthetic inputs for the BASELINE.json configurations.

The reference measures nothing on public data for this path; the paper's
datasets (MNIST/USPS/ORL/videos) are not available, so these generators
stand in with the configs' shapes, ranks and corruption levels
(SURVEY.md Appendix A records each interpretation):

  config 0  200 x 300, rank 10 on two 3-D noisy-circle kNN graphs, 5 %
            additive outliers +-U(0, 5 max|X0|), a = b = 4.
  config 1  10 304 x 1 000 (112 x 92 pixels x samples), rank 10 on the
            8-neighbour pixel grid and a latent 1 000-node circle kNN graph,
            10 % additive outliers U(-255, 255), X0 scaled to max|X0| = 255,
            a = b = 10.
  (configs 0/1: the rank-k factors are graph-smooth bases -- low-pass
  filtered Gaussian vectors, smooth_basis -- so the data is the same bits on
  every machine; the spectral gaps are rounded to 10 digits.)
  config 3  decoder only: kNN graphs (K=10) over N(0, I_64) points, p = 4 096,
            n = 200 000, rank 20 low-pass basis, 1/8 x 1/8 sampling.

Generation uses numpy/scipy only (LAPACK only for eigenvalues); it is
harness code, never timed.
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np


def circle_points(n: int, rs: np.random.Generator, noise: float = 0.05) -> np.ndarray:
    th = rs.uniform(0.0, 2.0 * math.pi, n)
    pts = np.stack([np.cos(th), np.sin(th), np.zeros(n)])
    return pts + noise * rs.standard_normal((3, n))


def knn_laplacian_dense(pts: np.ndarray, K: int) -> np.ndarray:
    """Dense combinatorial Laplacian of the reference kNN rule (graph.cpp:47-135)
    for small generator graphs: union symmetrisation, sigma2 = mean of the
    per-point mean squared kNN distance, w = exp(-d2 / sigma2)."""
    P = pts.T
    if P.shape[1] <= 16:  # the generators' 3-D latent points: elementwise (no BLAS), the same bits everywhere
        g = np.zeros((P.shape[0], P.shape[0]))
        for d in range(P.shape[1]):
            g += P[:, d][:, None] * P[:, d][None, :]
    else:  # CPU-only fallback of _lambda_k1_of_knn
        g = P @ P.T
    sq = np.diag(g)
    d2 = np.maximum(0.0, sq[:, None] + sq[None, :] - 2.0 * g)
    n = d2.shape[0]
    np.fill_diagonal(d2, np.inf)
    idx = np.argsort(d2, axis=1, kind="stable")[:, :K]
    near = np.take_along_axis(d2, idx, axis=1)
    sigma2 = float(np.mean(near.mean(axis=1)))
    A = np.zeros((n, n), bool)
    A[np.repeat(np.arange(n), K), idx.ravel()] = True
    A |= A.T
    np.fill_diagonal(d2, 0.0)
    W = np.where(A, np.exp(-d2 / sigma2), 0.0)
    return np.diag(W.sum(axis=1)) - W


def grid_adjacency(h: int, w: int):
    """8-neighbour unit-weight pixel grid (scipy CSR), pixels column-major
    within the image like a vectorised face."""
    import scipy.sparse as sp

    rows, cols = [], []
    for dr, dc in [(0, 1), (1, -1), (1, 0), (1, 1)]:
        r = np.arange(h)[:, None]
        c = np.arange(w)[None, :]
        r2, c2 = r + dr, c + dc
        ok = (r2 >= 0) & (r2 < h) & (c2 >= 0) & (c2 < w)
        a = np.broadcast_to(r + c * h, ok.shape)[ok]
        b = np.broadcast_to(r2 + c2 * h, ok.shape)[ok]
        rows += [a, b]
        cols += [b, a]
    rows = np.concatenate(rows)
    cols = np.concatenate(cols)
    W = sp.csr_matrix((np.ones(rows.size), (rows, cols)), shape=(h * w, h * w))
    W.sum_duplicates()
    W.sort_indices()
    return W


def smooth_basis(L, k: int, rs: np.random.Generator, sweeps: int = 300) -> np.ndarray:
    """Orthonormal n x k basis of graph-smooth vectors: Gaussian vectors
    low-pass filtered by `sweeps` steps B <- B - L B / (2 max L_ii) (the
    Gershgorin bound of a Laplacian's spectrum), then modified Gram-Schmidt.
    Only sparse products and numpy's pairwise sums: the same bits on every
    machine, unlike LAPACK eigenvectors (arbitrary signs and rotations in
    degenerate eigenspaces, thread-count dependent)."""
    import scipy.sparse as sp

    L = sp.csr_matrix(L)
    s = 1.0 / (2.0 * float(L.diagonal().max()))
    B = rs.standard_normal((L.shape[0], k))
    for _ in range(sweeps):
        B = B - s * (L @ B)
    for j in range(k):
        for i in range(j):
            B[:, j] -= np.sum(B[:, i] * B[:, j]) * B[:, i]
        B[:, j] /= math.sqrt(np.sum(B[:, j] * B[:, j]))
    return B


def low_rank(U: np.ndarray, A: np.ndarray, V: np.ndarray) -> np.ndarray:
    """U A V^T as sums of outer products in a fixed order (elementwise numpy,
    no BLAS, so no FMA/blocking differences between machines)."""
    M = np.zeros((U.shape[0], A.shape[1]))
    for j in range(A.shape[0]):
        M += U[:, j][:, None] * A[j, :][None, :]
    X = np.zeros((U.shape[0], V.shape[0]), order="F")
    for j in range(A.shape[1]):
        X += M[:, j][:, None] * V[:, j][None, :]
    return X


def _round_sig(x: float, digits: int = 10) -> float:
    """Rounds a generator constant so every machine prints and uses the same value."""
    return float(f"{x:.{digits}g}")


def smallest_eigvecs_dense(L: np.ndarray, k: int):
    ev, V = np.linalg.eigh(0.5 * (L + L.T))
    return ev[:k], V[:, :k]


def smallest_eigvecs_sparse(L, k: int):
    import scipy.sparse.linalg as sla

    ev, V = sla.eigsh(L.tocsc(), k=k, sigma=-1e-3, which="LM")
    order = np.argsort(ev)
    return ev[order], V[:, order]


def add_outliers(X0: np.ndarray, frac: float, rs: np.random.Generator, amp: float | None = None,
                 symmetric_uniform: float | None = None) -> np.ndarray:
    Y = X0.copy()
    N = Y.size
    m = int(round(frac * N))
    pos = rs.choice(N, size=m, replace=False)
    if symmetric_uniform is not None:
        vals = rs.uniform(-symmetric_uniform, symmetric_uniform, m)
    else:
        vals = rs.choice([-1.0, 1.0], m) * rs.uniform(0.0, amp, m)
    Yf = Y.reshape(-1, order="F")
    Yf[pos] += vals
    return Yf.reshape(Y.shape, order="F")


@dataclass
class Workload:
    name: str
    Y: np.ndarray          # p x n, column-major
    X0: np.ndarray         # low-rank truth
    a: int
    b: int
    gamma: float           # gamma_r = gamma_c (gamma' = 1/lambda)
    fista_iters: int
    cg_iters: int
    cg_tol: float
    lambda_k1_r: float = 1.0
    lambda_k1_c: float = 1.0
    W_r: object = None     # optional row adjacency (scipy CSR)
    rank: int = 10


def config0(seed: int = 1602, small: bool = False) -> tuple[np.ndarray, np.ndarray]:
    """Config 0 data (Y, X0).  small=True shrinks to 60 x 80 for quick tests."""
    rs = np.random.default_rng(seed)
    p, n, k = (60, 80, 5) if small else (200, 300, 10)
    Lr = knn_laplacian_dense(circle_points(p, rs), 10)
    Lc = knn_laplacian_dense(circle_points(n, rs), 10)
    U = smooth_basis(Lr, k, rs)
    V = smooth_basis(Lc, k, rs)
    A = rs.standard_normal((k, k))
    X0 = np.asfortranarray(low_rank(U, A, V))
    Y = add_outliers(X0, 0.05, rs, amp=5.0 * np.abs(X0).max())
    return np.asfortranarray(Y), X0


def config0_workload(seed: int = 1602) -> Workload:
    Y, X0 = config0(seed)
    p, n = Y.shape
    lr = _lambda_k1_of_knn(Y, True, 10, 10)
    lc = _lambda_k1_of_knn(Y, False, 10, 10)
    return Workload("cfg0 CPCA 200x300 fp64", Y, X0, 4, 4, math.sqrt(max(p, n)), 200, 100, 1e-8, lr, lc)


def _lambda_k1_of_knn(Y, axis_rows, K, k):
    """lambda_{k+1} of the kNN Laplacian of Y's rows or columns (the decoder's
    spectral gap, pipeline.cpp:343-349).  The graph comes from the library's
    build_knn_graph when a GPU is present: its canonical fp64 distances are
    the same on every machine, so near-tie neighbour choices (and with them
    lambda) no longer depend on the host BLAS (round 1 saw 0.063-0.10 for
    config 1 across boxes).  Without a GPU (CPU-only tests) the numpy Gram
    form is used."""
    try:
        import torch

        have_gpu = torch.cuda.is_available()
    except ImportError:
        have_gpu = False
    if have_gpu:
        from . import cpcag as P

        g = P.build_knn_graph(np.asfortranarray(Y, dtype=np.float64), "rows" if axis_rows else "cols", K)
        L = g.laplacian.to_dense()
    else:
        pts = Y if axis_rows else Y.T
        L = knn_laplacian_dense(np.ascontiguousarray(pts.T), K)
    ev = np.linalg.eigvalsh(0.5 * (L + L.T))
    return _round_sig(max(ev[k], 1e-12))


def config1(seed: int = 1603) -> Workload:
    """Config 1: face-image-sized CPCA (10 304 x 1 000)."""
    rs = np.random.default_rng(seed)
    h, w, n, k = 112, 92, 1000, 10
    Wr = grid_adjacency(h, w)
    deg = np.asarray(Wr.sum(axis=1)).ravel()
    import scipy.sparse as sp

    Lr = sp.diags(deg) - Wr
    ev_r, _ = smallest_eigvecs_sparse(Lr, k + 1)  # lambda_{k+1} only (eigenvalues are well defined)
    U = smooth_basis(Lr, k, rs)
    Lc_lat = knn_laplacian_dense(circle_points(n, rs), 10)
    V = smooth_basis(Lc_lat, k, rs)
    A = rs.standard_normal((k, k))
    X0 = low_rank(U, A, V)
    X0 *= 255.0 / np.abs(X0).max()
    Y = add_outliers(np.asfortranarray(X0), 0.10, rs, symmetric_uniform=255.0)
    p = h * w
    lc = _lambda_k1_of_knn(Y, False, 10, k)
    return Workload("cfg1 CPCA 10304x1000 fp32", np.asfortranarray(Y), np.asfortranarray(X0), 10, 10,
                    math.sqrt(max(p, n)), 300, 200, 1e-8, _round_sig(float(ev_r[k])), lc, Wr, k)


def config2_points(seed: int = 1604, n: int = 100_000, d: int = 512, clusters: int = 20) -> np.ndarray:
    """Config 2: n points in R^d (columns of a d x n fp32 matrix), a 50/50
    mixture of N(0, I) background and `clusters` Gaussian clusters (centres
    N(0, 4 I), std 0.5).  The mixture weight is an assumption."""
    rs = np.random.default_rng(seed)
    X = rs.standard_normal((d, n), dtype=np.float32)
    m = n // 2
    centres = (2.0 * rs.standard_normal((d, clusters))).astype(np.float32)
    lab = rs.integers(0, clusters, m)
    X[:, :m] = centres[:, lab] + 0.5 * rs.standard_normal((d, m), dtype=np.float32)
    return np.asfortranarray(X)


def config3_points(seed: int = 1605, p: int = 4096, n: int = 200_000, dim: int = 64):
    """Config 3: row points (p x dim) and column points (n x dim), N(0, I)."""
    rs = np.random.default_rng(seed)
    return (rs.standard_normal((dim, p), dtype=np.float32), rs.standard_normal((dim, n), dtype=np.float32))


def config3_rhs(P, Lr, Lc, plan, ctx, rank: int = 20, sweeps: int = 20, seed: int = 1606):
    """Config 3's right-hand side: X0 = B_r A B_c^T with B the
    orthonormalised low-pass filtered Gaussian bases (`sweeps` Jacobi sweeps
    B <- B - L B / ||L|| through the library's fp64 SpMM) and A ~ N(0, 1),
    sampled on the plan: Xt = X0(omega_r, omega_c), fp64 column-major on the
    device.  Harness code (torch on the device for the QR), never timed."""
    import torch

    rs = np.random.default_rng(seed)

    def lowpass(L, m):
        nrm = P.power_iteration_norm(L, 1e-7, 42, ctx=ctx)
        B = torch.tensor(rs.standard_normal((m, rank)), device="cuda")
        for _ in range(sweeps):
            B = B - L.multiply(B) / nrm
        return torch.linalg.qr(B)[0]

    Br, Bc = lowpass(Lr, plan.p), lowpass(Lc, plan.n)
    A = torch.tensor(rs.standard_normal((rank, rank)), device="cuda")
    Xt = Br[torch.tensor(plan.omega_r, device="cuda")] @ A @ Bc[torch.tensor(plan.omega_c, device="cuda")].T
    return Xt.t().contiguous().t()
