"""Pins the oracle's graph_upsample / approx_decode (decoders.cpp:72-121,
188-225) against SPEC.md's known answers and properties.  The reference
ships no unit test for these functions, so the pins are:
  * harmonic interpolation (0, ?, 2) -> 1 to 1e-10;
  * KKT identity L_aa S_a + L_ab R = 0 (residual <= tol);
  * SPEC.md:578 / Lemma 1 -- the closed form S_a = -L_aa^{-1} L_ab R
    (dense LAPACK solve, not the iterative path under test);
  * singular-value transfer: on zero-gap noiseless data the
    decoded X equals the ground truth, sigma_i(X) = sqrt(np/(rho_r rho_c))
    sigma~_i;
  * the error texts of decoders.cpp:17-25, 84-94, 115-117, 196-199, 210-212.
CPU only.
"""
import math

import numpy as np
import pytest

from oracle import pyoracle as O


def path_laplacian(n):
    ti, tj, tv = [], [], []
    for i in range(n - 1):
        ti += [i, i + 1]
        tj += [i + 1, i]
        tv += [1.0, 1.0]
    return O.graph_from_adjacency(O.Csr.from_triplets(n, n, ti, tj, tv)).laplacian


def blocks_laplacian(sizes, seed):
    """Disjoint union of random connected weighted graphs (one per block)."""
    rs = np.random.default_rng(seed)
    n = sum(sizes)
    ti, tj, tv = [], [], []
    o = 0
    for s in sizes:
        for i in range(s - 1):  # a path keeps the block connected
            w = 0.5 + rs.random()
            ti += [o + i, o + i + 1]
            tj += [o + i + 1, o + i]
            tv += [w, w]
        for _ in range(2 * s):
            a, b = rs.integers(0, s, 2)
            if a != b and abs(int(a) - int(b)) > 1:
                w = 0.5 + rs.random()
                ti += [o + a, o + b]
                tj += [o + b, o + a]
                tv += [w, w]
        o += s
    W = O.Csr.from_triplets(n, n, ti, tj, tv)  # duplicates are summed: still symmetric
    return O.graph_from_adjacency(W).laplacian


def dense(L):
    rp, ci, v = L.arrays()
    D = np.zeros((L.rows, L.cols))
    for r in range(L.rows):
        D[r, ci[rp[r]:rp[r + 1]]] = v[rp[r]:rp[r + 1]]
    return D


def test_harmonic_interpolation_spec_example():
    # path 0-1-2, known values 0 and 2 -> the middle node is 1.
    S = O.graph_upsample(path_laplacian(3), [0, 2], np.array([[0.0], [2.0]]))
    assert abs(S[1, 0] - 1.0) <= 1e-10 and S[0, 0] == 0.0 and S[2, 0] == 2.0


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_upsample_matches_closed_form_and_kkt(seed):
    rs = np.random.default_rng(seed)
    n = 60
    L = blocks_laplacian([n], seed)
    known = rs.permutation(n)[:17]
    R = rs.standard_normal((17, 3))
    S = O.graph_upsample(L, known, R, 1e-12)
    D = dense(L)
    unk = np.setdiff1d(np.arange(n), known)
    Sa = -np.linalg.solve(D[np.ix_(unk, unk)], D[np.ix_(unk, known)] @ R)  # Lemma 1
    assert np.array_equal(S[known], R)
    assert np.abs(S[unk] - Sa).max() <= 1e-9 * max(1.0, np.abs(Sa).max())
    kkt = D[np.ix_(unk, unk)] @ S[unk] + D[np.ix_(unk, known)] @ R
    assert np.linalg.norm(kkt) <= 1e-9 * np.linalg.norm(D[np.ix_(unk, known)] @ R)


def test_upsample_errors():
    L = blocks_laplacian([5, 6], 4)
    R = np.ones((2, 1))
    with pytest.raises(RuntimeError, match="graph upsample: connected component containing node 5 has no sampled node"):
        O.graph_upsample(L, [0, 1], R)
    with pytest.raises(ValueError, match="graph upsample: duplicate index"):
        O.graph_upsample(L, [0, 0], R)
    with pytest.raises(ValueError, match="graph upsample: index out of range"):
        O.graph_upsample(L, [0, 11], R)
    with pytest.raises(ValueError, match="known set and R row count differ"):
        O.graph_upsample(L, [0, 5, 6], R)
    with pytest.raises(RuntimeError, match=r"graph upsample: interior solve did not converge \(column 0\)"):
        O.graph_upsample(blocks_laplacian([40], 5), [0], np.ones((1, 1)) * 3.0, 1e-14, 1)


def zero_gap_case(p=120, n=200, kr=4, kc=5, per_r=6, per_c=8, seed=7):
    """Rows / columns in kr / kc equal blocks (disconnected graphs: the first
    k Laplacian eigenvalues are 0, a zero spectral gap).  X0 is rank
    min(kr, kc), piecewise constant on the blocks; each block is sampled
    with the same count, so upsampling is exact and the norms transfer."""
    rs = np.random.default_rng(seed)
    Lr = blocks_laplacian([p // kr] * kr, seed)
    Lc = blocks_laplacian([n // kc] * kc, seed + 1)
    A = rs.standard_normal((kr, kc))
    X0 = np.kron(A, np.ones((p // kr, n // kc)))
    om_r = np.concatenate([b * (p // kr) + rs.permutation(p // kr)[:per_r] for b in range(kr)])
    om_c = np.concatenate([b * (n // kc) + rs.permutation(n // kc)[:per_c] for b in range(kc)])
    om_r, om_c = rs.permutation(om_r), rs.permutation(om_c)
    plan = O.SamplingPlan(om_r.astype(np.int64), om_c.astype(np.int64), p, n)
    return Lr, Lc, plan, X0


def test_approx_decode_exact_recovery_and_sigma_transfer():
    Lr, Lc, plan, X0 = zero_gap_case()
    Xt = X0[np.ix_(plan.omega_r, plan.omega_c)]
    res = O.approx_decode(Xt, plan, Lr, Lc, rank_threshold=1e-6, pcg_tol=1e-12)
    assert res.k == np.linalg.matrix_rank(X0)
    assert np.linalg.norm(res.X - X0) <= 1e-9 * np.linalg.norm(X0)
    s_dec = np.linalg.svd(res.X, compute_uv=False)[:res.k]
    s_t = np.linalg.svd(Xt, compute_uv=False)[:res.k]
    scale = math.sqrt(plan.p * plan.n / (plan.rho_r * plan.rho_c))
    assert np.allclose(s_dec, scale * s_t, rtol=1e-6)
    # unit columns, largest-magnitude entry of each U column positive
    assert np.allclose(np.linalg.norm(res.U, axis=0), 1.0)
    assert np.all(res.U[np.argmax(np.abs(res.U), axis=0), np.arange(res.k)] > 0)


def test_approx_decode_errors():
    Lr, Lc, plan, X0 = zero_gap_case()
    Xt = X0[np.ix_(plan.omega_r, plan.omega_c)]
    with pytest.raises(ValueError, match="rank threshold must be in"):
        O.approx_decode(Xt, plan, Lr, Lc, rank_threshold=1.0)
    with pytest.raises(ValueError, match="Xt does not match plan"):
        O.approx_decode(Xt[:, 1:], plan, Lr, Lc)
    with pytest.raises(RuntimeError, match="no singular value above the rank threshold"):
        O.approx_decode(np.zeros_like(Xt), plan, Lr, Lc)
    with pytest.raises(ValueError, match="delta_for_scaling must be in"):
        O.approx_decode(Xt, plan, Lr, Lc, delta_for_scaling=1.0)
    with pytest.raises(ValueError, match="non-finite input"):
        O.approx_decode(np.full_like(Xt, np.nan), plan, Lr, Lc)
