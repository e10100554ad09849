"""GPU parity for the graph stages: kNN graph (neighbour sets and CSR
structure bit-exact; values to 1 ulp of exp), graph_from_adjacency,
Kron reduction (values <= 1e-9 of ||L~||, reference known answers), the
Jacobi PCG (reference known answers) and the end-to-end pipeline."""
import math

import numpy as np
import pytest

from helpers import knn_laplacian, random_laplacian, rel, to_device
from oracle import pyoracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    import paper_1602_02070_b200 as P

    return P


@pytest.fixture(scope="module")
def ctx(P):
    return P.Context(0)


def csr_equal_structure(a, b):
    rp1, ci1, v1 = a.arrays()
    rp2, ci2, v2 = b.arrays()
    return np.array_equal(rp1, rp2) and np.array_equal(ci1, ci2), v1, v2


# ------------------------------------------------------------------ kNN
@pytest.mark.parametrize("shape,K,axis,seed", [
    ((5, 40), 3, "cols", 1), ((12, 300), 10, "cols", 2), ((300, 7), 10, "rows", 3),
    ((64, 1000), 10, "cols", 4), ((3, 130), 1, "cols", 5), ((40, 257), 17, "cols", 6),
])
def test_knn_neighbours_bit_exact(P, ctx, shape, K, axis, seed):
    X = np.random.default_rng(seed).standard_normal(shape)
    nbr, d2 = P.knn(X, axis, K, ctx=ctx)
    nbr_o, d2_o = O.knn_neighbors(X, axis == "rows", K)
    assert np.array_equal(nbr, nbr_o)
    assert np.array_equal(d2, d2_o)


def test_knn_ties_and_duplicates(P, ctx):
    # test_graph.cpp:77-86: equidistant candidates break toward the lower index.
    X = np.array([[0.0, 1.0, 0.0, 5.0], [0.0, 0.0, 1.0, 5.0]])
    g = P.build_knn_graph(X, "cols", 1, ctx=ctx)
    W = g.adjacency.to_dense()
    assert W[1, 3] > 0.0 and W[2, 3] == 0.0
    # Integer lattice points: many exact ties at every distance.
    rs = np.random.default_rng(7)
    L = rs.integers(0, 4, size=(3, 200)).astype(np.float64)
    L[:, 50:60] = L[:, 0:10]  # coincident points
    nbr, d2 = P.knn(L, "cols", 8, ctx=ctx)
    nbr_o, d2_o = O.knn_neighbors(L, False, 8)
    assert np.array_equal(nbr, nbr_o) and np.array_equal(d2, d2_o)


def test_knn_graph_matches_oracle_structure_and_values(P, ctx):
    rs = np.random.default_rng(11)
    centres = rs.standard_normal((16, 5)) * 2.0
    X = centres[:, rs.integers(0, 5, 600)] + 0.5 * rs.standard_normal((16, 600))
    for kind in ("combinatorial", "normalized"):
        g = P.build_knn_graph(X, "cols", 10, kind=kind, ctx=ctx)
        go = O.build_knn_graph(X, False, 10, normalized=(kind == "normalized"))
        assert g.sigma2 == go.sigma2
        same, v1, v2 = csr_equal_structure(g.adjacency, go.adjacency)
        assert same
        assert np.max(np.abs(v1 - v2) / v2) <= 4e-16
        same, v1, v2 = csr_equal_structure(g.laplacian, go.laplacian)
        assert same
        assert np.max(np.abs(v1 - v2)) <= 1e-14 * np.max(np.abs(v2))
        assert np.max(np.abs(g.degrees - go.degrees) / go.degrees) <= 1e-14


def test_knn_graph_fp32_input_and_known_answers(P, ctx):
    # test_graph.cpp:60-75
    g = P.build_knn_graph(np.array([[0.0, 1.0, 10.0]]), "cols", 1, ctx=ctx)
    s2 = (1.0 + 1.0 + 81.0) / 3.0
    assert g.sigma2 == pytest.approx(s2, rel=1e-15)
    W = g.adjacency.to_dense()
    assert W[0, 1] == pytest.approx(math.exp(-1.0 / s2), rel=1e-15)
    assert W[1, 2] == pytest.approx(math.exp(-81.0 / s2), rel=1e-15)
    assert W[0, 2] == 0.0 and g.adjacency.nonzeros() == 4
    # test_graph.cpp:51-58
    g2 = P.build_knn_graph(np.array([[1.0, 1.0], [2.0, 2.0]]), "cols", 1, ctx=ctx)
    assert g2.adjacency.to_dense()[0, 1] == 1.0
    # fp32 input: distances of the fp32 values, computed in fp64.
    X = np.random.default_rng(3).standard_normal((30, 200)).astype(np.float32)
    n1, _ = P.knn(X, "cols", 10, ctx=ctx)
    n2, _ = O.knn_neighbors(X.astype(np.float64), False, 10)
    assert np.array_equal(n1, n2)
    # override
    assert P.build_knn_graph(X, "cols", 3, sigma2_override=2.5, ctx=ctx).sigma2 == 2.5


def test_knn_errors(P, ctx):
    # test_graph.cpp:95-103
    with pytest.raises(ValueError, match="at least K\\+1 points"):
        P.build_knn_graph(np.array([[0.0, 1.0, 2.0]]), "cols", 3, ctx=ctx)
    with pytest.raises(ValueError, match=r"fewer distinct points \(1\) than K \(2\)"):
        P.build_knn_graph(np.array([[2.0, 2.0, 2.0, 2.0]]), "cols", 2, ctx=ctx)
    with pytest.raises(ValueError, match="K must be >= 1"):
        P.build_knn_graph(np.array([[0.0, 1.0, 2.0]]), "cols", 0, ctx=ctx)


def test_rows_axis_equals_cols_axis_on_transpose(P, ctx):
    # test_graph.cpp:88-93
    X = O.gaussian_matrix(6, 12, 17)
    a = P.build_knn_graph(X, "rows", 2, ctx=ctx)
    b = P.build_knn_graph(np.asfortranarray(X.T), "cols", 2, ctx=ctx)
    assert np.array_equal(a.adjacency.to_dense(), b.adjacency.to_dense())


# ------------------------------------------------------------------ adjacency
def test_graph_from_adjacency(P, ctx):
    Lo = random_laplacian(50, 0.1, 3)
    rp, ci, v = Lo.arrays()
    D = Lo.to_dense()
    Wd = -D.copy()
    np.fill_diagonal(Wd, 0.0)
    W = P.SparseMatrix.from_dense(Wd, ctx=ctx)
    for kind in ("combinatorial", "normalized"):
        g = P.graph_from_adjacency(W, kind, ctx=ctx)
        go = O.graph_from_adjacency(O.Csr.from_dense(Wd), normalized=(kind == "normalized"))
        same, v1, v2 = csr_equal_structure(g.laplacian, go.laplacian)
        assert same and np.array_equal(v1, v2)
        assert np.array_equal(g.degrees, go.degrees)
    bad = Wd.copy()
    bad[0, 1] += 0.5
    with pytest.raises(ValueError, match="symmetric"):
        P.graph_from_adjacency(P.SparseMatrix.from_dense(bad, ctx=ctx), ctx=ctx)
    diag = Wd.copy()
    diag[3, 3] = 1.0
    with pytest.raises(ValueError, match="zero diagonal"):
        P.graph_from_adjacency(P.SparseMatrix.from_dense(diag, ctx=ctx), ctx=ctx)
    neg = Wd.copy()
    neg[0, 1] = neg[1, 0] = -0.25
    with pytest.raises(ValueError, match="nonnegative"):
        P.graph_from_adjacency(P.SparseMatrix.from_dense(neg, ctx=ctx), ctx=ctx)


# ------------------------------------------------------------------ PCG
def test_pcg_known_answers(P, ctx):
    # test_numeric.cpp:110-177
    eye = P.SparseMatrix.from_triplets(4, 4, range(4), range(4), [1.0] * 4, ctx=ctx)
    b = O.gaussian_matrix(4, 1, 31)[:, 0]
    x, r = P.pcg_solve(eye, b, ctx=ctx)
    assert r.converged and r.iterations == 1 and np.linalg.norm(x - b) <= 1e-12 * np.linalg.norm(b)
    A = P.SparseMatrix.from_triplets(3, 3, [0, 1, 2], [0, 1, 2], [1.0, 2.0, 4.0], ctx=ctx)
    x, r = P.pcg_solve(A, [1.0, 2.0, 4.0], ctx=ctx)
    assert r.converged and np.abs(x - 1.0).max() <= 1e-12
    for seed in range(5):
        G = O.gaussian_matrix(12, 12, 100 + seed)
        S = G @ G.T + 0.5 * np.eye(12)
        b = O.gaussian_matrix(12, 1, 200 + seed)[:, 0]
        x, r = P.pcg_solve(P.SparseMatrix.from_dense(S, ctx=ctx), b, opt=P.PcgOptions(tol=1e-9), ctx=ctx)
        assert r.converged and np.linalg.norm(S @ x - b) <= 1e-9 * np.linalg.norm(b) * 1.0000001
    zero = P.SparseMatrix.from_triplets(2, 2, [], [], [], ctx=ctx)
    with pytest.raises(RuntimeError, match="iteration 0"):
        P.pcg_solve(zero, [1.0, 1.0], jacobi=False, ctx=ctx)
    x, r = P.pcg_solve(eye, np.zeros(4), ctx=ctx)
    assert r.converged and r.iterations == 0 and np.linalg.norm(x) == 0.0


def test_pcg_matches_oracle_iterates(P, ctx):
    L = knn_laplacian(400, 3, 8, 9)
    rp, ci, v = L.arrays()
    Ld = L.to_dense() + 0.01 * np.eye(400)
    A_o = O.Csr.from_dense(Ld)
    b = np.random.default_rng(1).standard_normal(400)
    x, r = P.pcg_solve(to_device(ctx, A_o), b, opt=P.PcgOptions(tol=1e-10, max_iter=1000), ctx=ctx)
    xo, ro = O.pcg_solve(A_o, b, tol=1e-10, max_iter=1000)
    assert abs(r.iterations - ro.iterations) <= 1 and r.converged == ro.converged
    assert rel(x, xo) <= 1e-9


# ------------------------------------------------------------------ Kron
def test_kron_known_answers(P, ctx):
    path = P.SparseMatrix.from_triplets(3, 3, [0, 0, 1, 1, 1, 2, 2], [0, 1, 0, 1, 2, 1, 2],
                                        [1.0, -1.0, -1.0, 2.0, -1.0, -1.0, 1.0], ctx=ctx)
    assert np.array_equal(P.kron_reduce(path, [0, 1, 2], ctx=ctx).to_dense(), path.to_dense())
    R = P.kron_reduce(path, [0, 2], ctx=ctx)
    assert np.abs(R.to_dense() - np.array([[0.5, -0.5], [-0.5, 0.5]])).max() <= 1e-12
    L2 = P.SparseMatrix.from_triplets(4, 4, [0, 0, 1, 1, 2, 2, 3, 3], [0, 1, 0, 1, 2, 3, 2, 3],
                                      [1.0, -1.0, -1.0, 1.0, 2.0, -2.0, -2.0, 2.0], ctx=ctx)
    R2 = P.kron_reduce(L2, [0, 2], ctx=ctx)
    assert R2.nonzeros() == 0 and R2.rows() == 2
    U = P.SparseMatrix.from_triplets(4, 4, [0, 0, 1, 1, 2, 2, 3, 3], [0, 1, 0, 1, 2, 3, 2, 3],
                                     [1.0, -1.0, -1.0, 1.0, 1.0, -1.0, -1.0, 1.0], ctx=ctx)
    with pytest.raises(RuntimeError, match="connected component containing node 2 has no kept node"):
        P.kron_reduce(U, [0, 1], ctx=ctx)
    with pytest.raises(ValueError, match="duplicate index"):
        P.kron_reduce(path, [0, 0], ctx=ctx)
    with pytest.raises(ValueError, match="index out of range"):
        P.kron_reduce(path, [5], ctx=ctx)


@pytest.mark.parametrize("n,keep_frac,seed", [(60, 0.3, 1), (400, 0.1, 2), (1000, 0.1, 3)])
def test_kron_matches_oracle(P, ctx, n, keep_frac, seed):
    L = knn_laplacian(n, 4, 10, seed)
    keep = O.draw_plan(n, 1, max(2, int(keep_frac * n)), 1, seed=seed).omega_r
    R = P.kron_reduce(to_device(ctx, L), keep, 1e-11, 1e-12, ctx=ctx)
    Ro = O.kron_reduce(L, keep, 1e-11, 1e-12)
    Rd, Rod = R.to_dense(), Ro.to_dense()
    assert np.abs(Rd - Rod).max() <= 1e-9 * np.abs(Rod).max()
    assert np.array_equal(Rd, Rd.T)


def test_kron_grid_graph(P, ctx):
    # 8-neighbour pixel grid (the config-1 row graph), 10% kept.
    h, w = 30, 24
    ti, tj = [], []
    for r in range(h):
        for c in range(w):
            for dr, dc in [(0, 1), (1, -1), (1, 0), (1, 1)]:
                r2, c2 = r + dr, c + dc
                if 0 <= r2 < h and 0 <= c2 < w:
                    a, b = r * w + c, r2 * w + c2
                    ti += [a, b]
                    tj += [b, a]
    Wo = O.Csr.from_triplets(h * w, h * w, ti, tj, [1.0] * len(ti))
    Lo = O.graph_from_adjacency(Wo).laplacian
    keep = O.draw_plan(h * w, 1, 72, 1, seed=4).omega_r
    R = P.kron_reduce(to_device(ctx, Lo), keep, 1e-11, 1e-12, ctx=ctx)
    Ro = O.kron_reduce(Lo, keep, 1e-11, 1e-12)
    assert np.abs(R.to_dense() - Ro.to_dense()).max() <= 1e-9 * np.abs(Ro.to_dense()).max()


def _stencil_laplacian(h, w, offsets, weighted=False):
    ti, tj, tv = [], [], []
    rs = np.random.default_rng(h * w)
    for r in range(h):
        for c in range(w):
            for dr, dc in offsets:
                r2, c2 = r + dr, c + dc
                if 0 <= r2 < h and 0 <= c2 < w:
                    a, b = r * w + c, r2 * w + c2
                    x = {False: 1.0, "fp32": 1.0 + 2.0 ** -12, True: None}[weighted]
                    x = float(rs.uniform(0.5, 2.0)) if x is None else x
                    ti += [a, b]
                    tj += [b, a]
                    tv += [x, x]
    return O.graph_from_adjacency(O.Csr.from_triplets(h * w, h * w, ti, tj, tv)).laplacian


@pytest.mark.parametrize("shape,offsets,keep,weighted", [
    ((41, 37), [(0, 1), (1, -1), (1, 0), (1, 1)], 150, False),                # CSR staged in shared memory
    ((33, 29), [(0, 1), (0, 2), (1, -1), (1, 0), (1, 1), (2, 0)], 90, False),  # rows of <= 13 entries
    ((95, 90), [(0, 1), (1, -1), (1, 0), (1, 1)], 700, False),                # ELL from L2, (fp16, u16) words
    ((95, 90), [(0, 1), (1, -1), (1, 0), (1, 1)], 700, "fp32"),               # ELL from L2, (fp32, int) words
    ((95, 90), [(0, 1), (1, -1), (1, 0), (1, 1)], 700, True),                 # ELL from L2, fp64 values
])
def test_kron_shared_memory_pcg(P, ctx, shape, offsets, keep, weighted):
    """Interiors whose PCG vectors fit one CTA's shared memory run one
    right-hand side per CTA (pcg_smem_k): the operator staged in shared
    memory when it fits, else ELL from L2 (packed (fp16, u16) or (fp32,
    int32) words when every value is exact in that format); same
    recurrence, <= 1e-9."""
    Lo = _stencil_laplacian(*shape, offsets, weighted)
    n = shape[0] * shape[1]
    kp = O.draw_plan(n, 1, keep, 1, seed=7).omega_r
    R = P.kron_reduce(to_device(ctx, Lo), kp, 1e-11, 1e-12, ctx=ctx)
    Ro = O.kron_reduce(Lo, kp, 1e-11, 1e-12)
    assert np.abs(R.to_dense() - Ro.to_dense()).max() <= 1e-9 * np.abs(Ro.to_dense()).max()


def test_kron_config1_rows_matches_oracle(P, ctx):
    """Config 1's row reduction at full size: the 112 x 92 pixel grid,
    1 031 kept pixels, 9 273 interior nodes per PCG (graph.cpp:170-235)."""
    from paper_1602_02070_b200 import workloads

    W = workloads.grid_adjacency(112, 92)
    Lo = O.graph_from_adjacency(O.Csr.from_scipy(W)).laplacian
    kp = O.draw_plan(112 * 92, 1000, 1031, 100, seed=1603).omega_r
    R = P.kron_reduce(to_device(ctx, Lo), kp, 1e-11, 1e-12, ctx=ctx)
    Ro = O.kron_reduce(Lo, kp, 1e-11, 1e-12)
    Rd, Rod = R.to_dense(), Ro.to_dense()
    assert np.abs(Rd - Rod).max() <= 1e-9 * np.abs(Rod).max()
    assert np.array_equal(Rd, Rd.T)


# ------------------------------------------------------------------ pipeline
def test_pipeline_small_matches_oracle_stages(P, ctx):
    from paper_1602_02070_b200.workloads import config0

    Y, truth = config0(seed=1602, small=True)
    p, n = Y.shape
    cfg = P.PipelineConfig(knn=10, a=4, b=4, frpcag=P.FrpcagConfig(gamma_r=math.sqrt(max(p, n)),
                           gamma_c=math.sqrt(max(p, n)), tol=1e-300, max_iter=60),
                           decoder=P.DecoderConfig(1.0, 1e-8, 100, variant="alternate"), lambda_k1_r=0.5, lambda_k1_c=0.5, seed=1602)
    rep = P.run_pipeline(Y, cfg, ctx=ctx)
    # oracle stages
    gr = O.build_knn_graph(Y, True, 10)
    gc = O.build_knn_graph(Y, False, 10)
    plan = O.draw_plan(p, n, -(-p // 4), -(-n // 4), seed=1602)
    assert np.array_equal(rep.plan.omega_r, plan.omega_r) and np.array_equal(rep.plan.omega_c, plan.omega_c)
    Yt = O.subsample(Y, plan)
    Lr_t = O.kron_reduce(gr.laplacian, plan.omega_r, 1e-11)
    Lc_t = O.kron_reduce(gc.laplacian, plan.omega_c, 1e-11)
    Xt, tr = O.fista_solve(Yt, Lr_t, Lc_t, O.FrpcagConfig(math.sqrt(max(p, n)), math.sqrt(max(p, n)), "l1", 1e-300, 60))
    assert rep.trace.iterations == 60
    assert rel(rep.Xt, Xt) <= 1e-7
    dec = O.alternate_decode(Xt, plan, gr.laplacian, gc.laplacian, 0.5, 0.5, 1.0, 1e-8, 100)
    assert rel(rep.X, dec.X) <= 1e-7
    assert abs(rep.decoder_iterations - dec.iterations) <= 1
    # caller-provided (pinned) result buffers: same results, written in place
    import torch

    Xh = torch.empty((n, p), dtype=torch.float64, pin_memory=True).numpy().T
    Xth = torch.empty((rep.rho_c, rep.rho_r), dtype=torch.float64, pin_memory=True).numpy().T
    rep2 = P.run_pipeline(Y, cfg, ctx=ctx, out=(Xth, Xh))
    assert rep2.X is Xh and rep2.Xt is Xth
    assert np.array_equal(rep2.X, rep.X) and np.array_equal(rep2.Xt, rep.Xt)
    with pytest.raises(ValueError, match="out\\[1\\] \\(X\\): expected"):
        P.run_pipeline(Y, cfg, ctx=ctx, out=(Xth, np.empty((p, n))))
    assert all(rep.stages[s] > 0 for s in ("graphs", "kron", "solve", "decode"))


def test_pipeline_approx_decoder_matches_oracle(P, ctx):
    """The reference default decoder (pipeline.cpp:361-367) and the detected
    rank (pipeline.cpp:319-320) through run_pipeline."""
    from paper_1602_02070_b200.workloads import config0

    Y, truth = config0(seed=1602, small=True)
    p, n = Y.shape
    g = math.sqrt(max(p, n))
    cfg = P.PipelineConfig(knn=10, a=4, b=4, frpcag=P.FrpcagConfig(gamma_r=g, gamma_c=g, tol=1e-300, max_iter=60),
                           decoder=P.DecoderConfig(pcg_tol=1e-12, variant="approx", rank_threshold=0.1), seed=1602)
    rep = P.run_pipeline(Y, cfg, ctx=ctx)
    gr = O.build_knn_graph(Y, True, 10)
    gc = O.build_knn_graph(Y, False, 10)
    plan = O.draw_plan(p, n, -(-p // 4), -(-n // 4), seed=1602)
    Yt = O.subsample(Y, plan)
    Lr_t = O.kron_reduce(gr.laplacian, plan.omega_r, 1e-11)
    Lc_t = O.kron_reduce(gc.laplacian, plan.omega_c, 1e-11)
    Xt, _ = O.fista_solve(Yt, Lr_t, Lc_t, O.FrpcagConfig(g, g, "l1", 1e-300, 60))
    assert rep.detected_rank == O.detect_rank(O.thin_svd(Xt)[1], 0.1)
    dec = O.approx_decode(Xt, plan, gr.laplacian, gc.laplacian, rank_threshold=0.1, pcg_tol=1e-12)
    assert rep.has_factors and rep.factors.k == dec.k
    assert rel(rep.X, dec.X) <= 1e-6
    assert rel(rep.factors.U, dec.U) <= 1e-6 and np.allclose(rep.factors.sigma, dec.sigma, rtol=1e-7)


@pytest.mark.parametrize("a,b", [(4, 4), (2, 2)])
def test_pipeline_detected_rank_beside_the_decoder(P, ctx, a, b):
    """With the alternate decoder, both spectral gaps given and no clustering,
    the detected rank (pipeline.cpp:319-321) runs on the side stream beside
    the decode (Gram + one-CTA Jacobi eigenvalues when min(rho_r, rho_c) <=
    110; a = b = 2 gives 30 x 40, a = b = 4 gives 15 x 20) and must equal the
    oracle's SVD-based rank."""
    from paper_1602_02070_b200.workloads import config0

    Y, _ = config0(seed=1602, small=True)
    p, n = Y.shape
    g = math.sqrt(max(p, n))
    cfg = P.PipelineConfig(knn=10, a=a, b=b, frpcag=P.FrpcagConfig(gamma_r=g, gamma_c=g, tol=1e-300, max_iter=60),
                           decoder=P.DecoderConfig(pcg_tol=1e-10, pcg_max_iter=300, variant="alternate",
                                                   rank_threshold=0.05),
                           lambda_k1_r=0.05, lambda_k1_c=0.07, seed=1602)
    rep = P.run_pipeline(Y, cfg, ctx=ctx)
    gr = O.build_knn_graph(Y, True, 10)
    gc = O.build_knn_graph(Y, False, 10)
    plan = O.draw_plan(p, n, -(-p // b), -(-n // a), seed=1602)
    Lr_t = O.kron_reduce(gr.laplacian, plan.omega_r, 1e-11)
    Lc_t = O.kron_reduce(gc.laplacian, plan.omega_c, 1e-11)
    Xt, _ = O.fista_solve(O.subsample(Y, plan), Lr_t, Lc_t, O.FrpcagConfig(g, g, "l1", 1e-300, 60))
    sv = O.thin_svd(Xt)[1]
    assert rep.detected_rank == O.detect_rank(sv, 0.05)
    dec = O.alternate_decode(Xt, plan, gr.laplacian, gc.laplacian, 0.05, 0.07, 1.0, 1e-10, 300)
    assert rel(rep.X, dec.X) <= 1e-8


def test_pipeline_stage_error_is_tagged(P, ctx):
    Y = np.random.default_rng(0).standard_normal((20, 30))
    cfg = P.PipelineConfig(knn=50, a=2, b=2)
    with pytest.raises(RuntimeError, match="stage graphs: knn graph: need at least K\\+1 points"):
        P.run_pipeline(Y, cfg, ctx=ctx)


# ------------------------------------------------------------------ tensor-core Gram
@pytest.mark.parametrize("n,d", [(128, 32), (300, 70), (517, 512)])
def test_gram_tf32x3_tensor_cores(P, ctx, n, d):
    """tcgen05 kind::tf32 3xTF32 Gram: error within the filter's bound."""
    import ctypes

    from paper_1602_02070_b200 import _native as N

    X = np.random.default_rng(n + d).standard_normal((n, d))
    G = np.empty((n, n), np.float32)
    Xc = np.ascontiguousarray(X)
    N.check(N.lib().cpcag_cuda_gram_tf32x3(ctx.handle, Xc.ctypes.data, n, d, G.ctypes.data))
    ref = X @ X.T
    nrm = np.linalg.norm(X, axis=1)
    bound = (d * 2.0 ** -23 + 2.0 ** -19) * np.outer(nrm, nrm)
    err = np.abs(G.astype(np.float64) - ref)
    assert np.all(err <= bound), float((err / bound).max())
    # and far better than plain TF32 would be
    assert err.max() <= 1e-4 * np.abs(ref).max()


@pytest.mark.parametrize("n,d,K", [(4500, 64, 10), (5000, 16, 12), (4200, 200, 10)])
def test_knn_tensor_core_filter_bit_exact(P, ctx, n, d, K, monkeypatch):
    """3xTF32 tcgen05 filter + certified fp64 re-rank: neighbour sets and
    distances bit-identical to the oracle's canonical fp64 search."""
    monkeypatch.setenv("CPCAG_KNN", "tc")
    rs = np.random.default_rng(n + d)
    centres = rs.standard_normal((d, 8)) * 2.0
    X = centres[:, rs.integers(0, 8, n)] + 0.5 * rs.standard_normal((d, n))
    X[:, 100:110] = X[:, 0:10]  # coincident points
    nbr, d2 = P.knn(X, "cols", K, ctx=ctx)
    nbr_o, d2_o = O.knn_neighbors(X, False, K)
    assert np.array_equal(nbr, nbr_o)
    assert np.array_equal(d2, d2_o)
