"""GPU parity of thin_svd, graph_upsample and approx_decode (approx.cu,
kron.cu) against the oracle (decoders.cpp:72-121, 188-225; eigs.cpp:53-64).

Bars: singular values 1e-12 relative, singular vectors up to sign; fp64
upsampling / decoder outputs 1e-9 relative (only PCG reduction order
differs); fp32 X within the north_star 1e-4 relative Frobenius error.
"""
import numpy as np
import pytest

from helpers import knn_laplacian, rel, to_device
from oracle import pyoracle as O
from test_oracle_approx import blocks_laplacian, zero_gap_case

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    import paper_1602_02070_b200 as P

    return P


@pytest.fixture(scope="module")
def ctx(P):
    return P.Context(0)


@pytest.mark.parametrize("shape", [(103, 40), (40, 103), (25, 25)])
def test_thin_svd_matches_lapack(P, ctx, shape):
    A = np.random.default_rng(shape[0]).standard_normal(shape)
    r = P.thin_svd(A, ctx=ctx)
    U, s, V = O.thin_svd(A)
    assert np.allclose(r.sigma, s, rtol=1e-12, atol=0)
    sign = np.sign(np.sum(r.U * U, axis=0))
    assert np.allclose(r.U * sign, U, atol=1e-10)
    assert np.allclose(r.V * sign, V, atol=1e-10)
    assert np.allclose((r.U * r.sigma) @ r.V.T, A, atol=1e-11)


def test_thin_svd_non_finite(P, ctx):
    A = np.ones((4, 3))
    A[2, 1] = np.inf
    with pytest.raises(ValueError, match="thin_svd: non-finite input"):
        P.thin_svd(A, ctx=ctx)


@pytest.mark.parametrize("n,m,r", [(300, 41, 3), (1000, 100, 10), (64, 64, 2)])
def test_graph_upsample_matches_oracle(P, ctx, n, m, r):
    L = knn_laplacian(n, 3, 10, n + m)
    rs = np.random.default_rng(m)
    known = rs.permutation(n)[:m]  # draw order (not sorted): exercises the L_ab row re-sort
    R = rs.standard_normal((m, r))
    S = P.graph_upsample(to_device(ctx, L), known, R, 1e-12, ctx=ctx)
    So = O.graph_upsample(L, known, R, 1e-12)
    assert np.array_equal(S[known], R)
    assert rel(S, So) <= 1e-9


def test_graph_upsample_device_arrays(P, ctx):
    import torch

    L = knn_laplacian(200, 3, 10, 5)
    known = np.random.default_rng(1).permutation(200)[:30]
    R = np.random.default_rng(2).standard_normal((30, 4))
    S = P.graph_upsample(to_device(ctx, L), known, torch.tensor(R, device="cuda"), 1e-12, ctx=ctx)
    assert S.is_cuda
    assert rel(S.cpu().numpy(), O.graph_upsample(L, known, R, 1e-12)) <= 1e-9


def test_graph_upsample_errors(P, ctx):
    Lb = blocks_laplacian([5, 6], 4)
    L = to_device(ctx, Lb)
    R = np.ones((2, 1))
    with pytest.raises(RuntimeError, match="graph upsample: connected component containing node 5 has no sampled node"):
        P.graph_upsample(L, [0, 1], R, ctx=ctx)
    with pytest.raises(ValueError, match="graph upsample: duplicate index"):
        P.graph_upsample(L, [0, 0], R, ctx=ctx)
    with pytest.raises(ValueError, match="graph upsample: index out of range"):
        P.graph_upsample(L, [0, 11], R, ctx=ctx)
    with pytest.raises(ValueError, match="known set and R row count differ"):
        P.graph_upsample(L, [0, 5, 6], R, ctx=ctx)
    L40 = to_device(ctx, blocks_laplacian([40], 5))
    with pytest.raises(RuntimeError, match=r"graph upsample: interior solve did not converge \(column 0\)"):
        P.graph_upsample(L40, [0], np.ones((1, 1)) * 3.0, 1e-14, 1, ctx=ctx)


def _decoder_case(p=300, n=240, rr=75, rc=60, seed=11):
    Lr, Lc = knn_laplacian(p, 3, 10, seed), knn_laplacian(n, 3, 10, seed + 1)
    plan = O.draw_plan(p, n, rr, rc, seed=seed)
    rs = np.random.default_rng(seed)
    Xt = rs.standard_normal((rr, 4)) @ np.diag([10.0, 5.0, 2.0, 1.5]) @ rs.standard_normal((4, rc))
    Xt += 0.01 * rs.standard_normal((rr, rc))
    return Lr, Lc, plan, Xt


def test_approx_decode_fp64_matches_oracle(P, ctx):
    Lr, Lc, plan_o, Xt = _decoder_case()
    plan = P.SamplingPlan(plan_o.omega_r, plan_o.omega_c, plan_o.p, plan_o.n)
    cfg = P.DecoderConfig(pcg_tol=1e-12, rank_threshold=0.1)
    res = P.approx_decode(Xt, plan, to_device(ctx, Lr), to_device(ctx, Lc), cfg, ctx=ctx)
    ro = O.approx_decode(Xt, plan_o, Lr, Lc, rank_threshold=0.1, pcg_tol=1e-12)
    assert res.factors.k == ro.k == 4
    assert rel(res.X, ro.X) <= 1e-9
    assert rel(res.factors.U, ro.U) <= 1e-9 and rel(res.factors.V, ro.V) <= 1e-9
    assert np.allclose(res.factors.sigma, ro.sigma, rtol=1e-12)


def test_approx_decode_fp32_and_device(P, ctx):
    import torch

    Lr, Lc, plan_o, Xt = _decoder_case(seed=12)
    plan = P.SamplingPlan(plan_o.omega_r, plan_o.omega_c, plan_o.p, plan_o.n)
    xd = torch.tensor(Xt.astype(np.float32), device="cuda")
    res = P.approx_decode(xd, plan, to_device(ctx, Lr), to_device(ctx, Lc), P.DecoderConfig(pcg_tol=1e-10),
                          ctx=ctx)
    ro = O.approx_decode(Xt.astype(np.float32).astype(np.float64), plan_o, Lr, Lc, pcg_tol=1e-10)
    assert res.X.is_cuda and res.X.dtype == torch.float32
    assert rel(res.X.cpu().numpy(), ro.X) <= 1e-4


def test_approx_decode_exact_recovery(P, ctx):
    Lr, Lc, plan_o, X0 = zero_gap_case()
    Xt = X0[np.ix_(plan_o.omega_r, plan_o.omega_c)]
    plan = P.SamplingPlan(plan_o.omega_r, plan_o.omega_c, plan_o.p, plan_o.n)
    res = P.approx_decode(Xt, plan, to_device(ctx, Lr), to_device(ctx, Lc),
                          P.DecoderConfig(pcg_tol=1e-12, rank_threshold=1e-6), ctx=ctx)
    assert res.factors.k == np.linalg.matrix_rank(X0)
    assert rel(res.X, X0) <= 1e-9


def test_approx_decode_errors(P, ctx):
    Lr, Lc, plan_o, Xt = _decoder_case()
    plan = P.SamplingPlan(plan_o.omega_r, plan_o.omega_c, plan_o.p, plan_o.n)
    dLr, dLc = to_device(ctx, Lr), to_device(ctx, Lc)
    with pytest.raises(ValueError, match="rank threshold must be in"):
        P.approx_decode(Xt, plan, dLr, dLc, P.DecoderConfig(rank_threshold=0.0), ctx=ctx)
    with pytest.raises(ValueError, match="Laplacians do not match plan"):
        P.approx_decode(Xt, plan, dLc, dLr, ctx=ctx)
    with pytest.raises(ValueError, match="Xt does not match plan"):
        P.approx_decode(Xt[:, 1:], plan, dLr, dLc, ctx=ctx)
    with pytest.raises(RuntimeError, match="no singular value above the rank threshold"):
        P.approx_decode(np.zeros_like(Xt), plan, dLr, dLc, ctx=ctx)
    with pytest.raises(ValueError, match="delta_for_scaling must be in"):
        P.approx_decode(Xt, plan, dLr, dLc, P.DecoderConfig(delta_for_scaling=1.5), ctx=ctx)


# ------------------------------------------------------------------ sym_eig / spectral gap (eigs.cpp:34-51)
@pytest.mark.parametrize("n,k", [(60, 5), (257, 11)])
def test_sym_eig_matches_lapack(P, ctx, n, k):
    L = knn_laplacian(n, 3, 10, n)
    ep = P.sym_eig(to_device(ctx, L), k, ctx=ctx)
    w, E = O.sym_eig(L, k)
    assert np.allclose(ep.eigenvalues, w, rtol=1e-10, atol=1e-12)
    # same sign rule; vectors of simple eigenvalues agree
    assert np.abs(ep.eigenvectors - E).max() <= 1e-8


def test_spectral_gap_and_errors(P, ctx):
    L = knn_laplacian(80, 3, 10, 9)
    ep = P.sym_eig(to_device(ctx, L), 4, vectors=False, ctx=ctx)
    g = P.spectral_gap(ep, 3)
    lk, lk1, ratio = O.spectral_gap(O.sym_eig(L, 4)[0], 3)
    assert g.k == 3 and abs(g.lambda_k1 - lk1) <= 1e-10 * lk1 and abs(g.ratio - ratio) <= 1e-9
    with pytest.raises(ValueError, match="order k out of range"):
        P.sym_eig(to_device(ctx, L), 81, ctx=ctx)
    two = blocks_laplacian([10, 12], 3)
    with pytest.raises(RuntimeError, match="gap undefined: graph has > k components"):
        P.spectral_gap(P.sym_eig(to_device(ctx, two), 2, vectors=False, ctx=ctx), 1)


def test_pipeline_computes_gaps_like_the_reference(P, ctx):
    """lambda_k1 <= 0: run_pipeline computes the gaps (pipeline.cpp:343-349)."""
    import math

    from paper_1602_02070_b200.workloads import config0

    Y, _ = config0(seed=1602, small=True)
    p, n = Y.shape
    g = math.sqrt(max(p, n))
    cfg = P.PipelineConfig(knn=10, a=4, b=4, frpcag=P.FrpcagConfig(gamma_r=g, gamma_c=g, tol=1e-300, max_iter=40),
                           decoder=P.DecoderConfig(1.0, 1e-8, 100, variant="alternate"), seed=1602)
    rep = P.run_pipeline(Y, cfg, ctx=ctx)
    k = max(1, rep.detected_rank)
    gr = O.build_knn_graph(Y, True, 10)
    gc = O.build_knn_graph(Y, False, 10)
    lr = O.spectral_gap(O.sym_eig(gr.laplacian, k + 1)[0], k)[1]
    lc = O.spectral_gap(O.sym_eig(gc.laplacian, k + 1)[0], k)[1]
    assert abs(rep.lambda_k1[0] - lr) <= 1e-10 * lr and abs(rep.lambda_k1[1] - lc) <= 1e-10 * lc


# ------------------------------------------------------------------ Lanczos spectral gap (large graphs)
@pytest.mark.parametrize("n,dim,k", [(400, 3, 6), (3000, 8, 21)])
def test_lanczos_smallest_eigenvalues_match_lapack(P, ctx, n, dim, k):
    """sym_eigvals_lanczos vs the dense oracle (numpy LAPACK) on kNN
    Laplacians small enough for the dense solver."""
    L = knn_laplacian(n, dim, 10, 7 + n)
    ev, steps = P.sym_eigvals_lanczos(to_device(ctx, L), k, tol=1e-10, ctx=ctx)
    w = np.linalg.eigvalsh(0.5 * (L.to_dense() + L.to_dense().T))[:k]
    assert steps >= k
    assert np.allclose(ev, w, rtol=1e-8, atol=1e-9 * np.abs(w).max())
    # deterministic for a seed
    ev2, steps2 = P.sym_eigvals_lanczos(to_device(ctx, L), k, tol=1e-10, ctx=ctx)
    assert steps2 == steps and np.array_equal(ev, ev2)


def test_lanczos_errors_and_components(P, ctx):
    L = knn_laplacian(50, 3, 10, 3)
    with pytest.raises(ValueError, match="order k out of range"):
        P.sym_eigvals_lanczos(to_device(ctx, L), 51, ctx=ctx)
    two = blocks_laplacian([30, 40], 3)
    ev, _ = P.sym_eigvals_lanczos(to_device(ctx, two), 3, ctx=ctx)
    # two components: a double zero eigenvalue, then the smaller Fiedler value
    assert abs(ev[0]) <= 1e-9 and abs(ev[1]) <= 1e-9 and ev[2] > 1e-6
    with pytest.raises(RuntimeError, match="not converged after"):
        P.sym_eigvals_lanczos(to_device(ctx, knn_laplacian(3000, 8, 10, 5)), 21, tol=1e-14, max_iter=40, ctx=ctx)


def test_pipeline_gaps_by_lanczos_match_dense(P, ctx, monkeypatch):
    """CPCAG_GAP_LANCZOS=1 forces the Lanczos gap inside run_pipeline; it
    agrees with the dense path (which the previous test pins to the oracle)."""
    import math

    from paper_1602_02070_b200.workloads import config0

    Y, _ = config0(seed=1602, small=True)
    p, n = Y.shape
    g = math.sqrt(max(p, n))
    cfg = P.PipelineConfig(knn=10, a=4, b=4, frpcag=P.FrpcagConfig(gamma_r=g, gamma_c=g, tol=1e-300, max_iter=40),
                           decoder=P.DecoderConfig(1.0, 1e-8, 100, variant="alternate"), seed=1602)
    dense = P.run_pipeline(Y, cfg, ctx=ctx)
    monkeypatch.setenv("CPCAG_GAP_LANCZOS", "1")
    lz = P.run_pipeline(Y, cfg, ctx=ctx)
    for a, b in zip(lz.lambda_k1, dense.lambda_k1):
        assert abs(a - b) <= 1e-8 * b
    assert rel(lz.X, dense.X) <= 1e-8
