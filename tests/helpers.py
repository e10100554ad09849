"""Shared seeded problem generators for the parity tests (CPU side uses the
oracle; nothing here touches the product path)."""
import numpy as np

from oracle import pyoracle as O


def random_laplacian(n, edge_prob, seed, connect=True):
    """Laplacian of oracles.hpp:129-142-style random weighted graph."""
    rs = np.random.default_rng(seed)
    ti, tj, tv = [], [], []
    for i in range(n):
        js = np.nonzero(rs.random(n - i - 1) < edge_prob)[0] + i + 1
        if connect and i + 1 < n and (i + 1) not in js:
            js = np.append(js, i + 1)
        for j in js:
            w = 0.05 + 0.95 * rs.random()
            ti += [i, j]
            tj += [j, i]
            tv += [w, w]
    W = O.Csr.from_triplets(n, n, ti, tj, tv)
    g = O.graph_from_adjacency(W)
    return g.laplacian


def knn_laplacian(n, dim, K, seed):
    pts = np.random.default_rng(seed).standard_normal((dim, n))
    return O.build_knn_graph(pts, False, K).laplacian


def to_device(ctx, oc):
    """Upload an oracle CSR to a device SparseMatrix."""
    from paper_1602_02070_b200 import SparseMatrix

    rp, ci, v = oc.arrays()
    return SparseMatrix.from_csr(oc.rows, oc.cols, rp, ci, v, ctx=ctx)


def rel(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    d = np.linalg.norm(b)
    return np.linalg.norm(a - b) / (d if d > 0 else 1.0)
