"""Parity at the BASELINE configurations' full sizes, through checks whose
cost does not grow with the whole problem (the oracle cannot run the full
problems in test time):

  cfg2  kNN graph of 100 000 x 512 points: the device neighbour lists of a
        random sample of points are bit-exact against the oracle's exact
        per-point selection (graph.cpp:86-105) over all 100 000 candidates;
        every list is sorted by (d2, j) and excludes the point; W is
        symmetric and the Laplacian rows sum to zero.
  cfg3  decoder operator 4096 x 200 000 (band apply, the path the size
        selects): one fp64 apply is bit-exact on sampled columns against
        the reference's per-entry arithmetic (decoders.cpp:160-170),
        emulated in Python floats (IEEE binary64, same operation order).
  cfg1  the whole pipeline at 10 304 x 1 000 with reduced iteration counts
        (FISTA 20, decoder 20) against the oracle's stage-by-stage fp64
        composite: fp32 X within the north_star 1e-4.
"""
import math

import numpy as np
import pytest

from helpers import rel
from oracle import pyoracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    import paper_1602_02070_b200 as P

    return P


@pytest.fixture(scope="module")
def ctx(P):
    return P.Context(0)


def test_cfg2_knn_full_size_sampled_rows_bit_exact(P, ctx):
    import torch

    from paper_1602_02070_b200 import workloads

    X = workloads.config2_points()  # d x n fp32
    d, n = X.shape
    Xd = torch.tensor(np.ascontiguousarray(X.T), device="cuda").t()
    nbr, d2 = P.knn(Xd, "cols", 10, ctx=ctx)
    rows = np.random.default_rng(7).choice(n, 48, replace=False)
    onbr, od2 = O.knn_rows(X.astype(np.float64), False, 10, rows)
    assert np.array_equal(nbr[rows], onbr)
    assert np.array_equal(d2[rows], od2)
    # size-independent properties over every point
    assert np.all((d2[:, 1:] > d2[:, :-1]) | ((d2[:, 1:] == d2[:, :-1]) & (nbr[:, 1:] > nbr[:, :-1])))
    assert not np.any(nbr == np.arange(n)[:, None])
    g = P.build_knn_graph(Xd, "cols", 10, ctx=ctx)
    W = g.adjacency.to_scipy()
    assert abs(W - W.T).max() == 0.0
    Ls = g.laplacian.to_scipy()
    assert np.abs(np.asarray(Ls.sum(axis=1)).ravel()).max() <= 1e-12 * max(1.0, np.abs(g.degrees).max())


def _apply_entry(rp_r, ci_r, v_r, rp_c, ci_c, v_c, Pm, rsel, csel, gr, gc, i, c):
    """decoders.cpp:160-170 for one entry, binary64 in the reference order."""
    x1 = 0.0
    for k in range(rp_c[c], rp_c[c + 1]):
        x1 = x1 + v_c[k] * Pm[i, ci_c[k]]
    x2 = 0.0
    for k in range(rp_r[i], rp_r[i + 1]):
        x2 = x2 + v_r[k] * Pm[ci_r[k], c]
    out = gc * x1 + gr * x2
    if rsel[i] and csel[c]:
        out = out + Pm[i, c]
    return out


def test_cfg3_apply_full_size_sampled_columns_bit_exact(P, ctx):
    """One fp64 application of the decoder operator at the full cfg3 size
    (4096 x 200 000: the lc pass with the band resident in L2, the lr pass
    over degree-sorted kNN rows) on sampled entries against the reference's
    per-entry arithmetic (decoders.cpp:160-170) in Python binary64."""
    import torch

    from paper_1602_02070_b200 import workloads

    Pr, Pc = workloads.config3_points()
    p, n = Pr.shape[1], Pc.shape[1]
    gr_ = P.build_knn_graph(torch.tensor(np.ascontiguousarray(Pr.T), device="cuda").t(), "cols", 10, ctx=ctx)
    gc_ = P.build_knn_graph(torch.tensor(np.ascontiguousarray(Pc.T), device="cuda").t(), "cols", 10, ctx=ctx)
    plan = P.draw_plan(p, n, p // 8, n // 8, seed=1607)
    gr, gc = 1.0 / 0.37, 1.0 / 0.53
    gen = torch.Generator(device="cuda").manual_seed(5)
    Pt = torch.randn(n, p, dtype=torch.float64, device="cuda", generator=gen).t()
    AP, dot = P.decoder_apply(Pt, plan, gr_.laplacian, gc_.laplacian, gr, gc, ctx=ctx)
    torch.cuda.synchronize()
    cols = np.random.default_rng(3).choice(n, 6, replace=False)
    rp_c, ci_c, v_c = gc_.laplacian.arrays()
    rp_r, ci_r, v_r = gr_.laplacian.arrays()
    need = sorted(set(int(j) for c in cols for j in ci_c[rp_c[c]:rp_c[c + 1]]) | set(int(c) for c in cols))
    Pm = np.zeros((p, n))
    for j in need:
        Pm[:, j] = Pt[:, j].cpu().numpy()
    rsel = np.zeros(p, bool)
    rsel[np.asarray(plan.omega_r)] = True
    csel = np.zeros(n, bool)
    csel[np.asarray(plan.omega_c)] = True
    rows = np.random.default_rng(4).choice(p, 64, replace=False)
    for c in cols:
        got = AP[:, int(c)].cpu().numpy()
        for i in rows:
            want = _apply_entry(rp_r, ci_r, v_r, rp_c, ci_c, v_c, Pm, rsel, csel, gr, gc, int(i), int(c))
            assert got[i] == want, (i, c)
    # size-independent: <P, AP> equals the sum of the stored products
    assert abs(dot - float((Pt * AP).sum())) <= 1e-9 * abs(dot)
    # repeat with a fresh output: the stream ordering holds across calls
    AP2, _ = P.decoder_apply(Pt, plan, gr_.laplacian, gc_.laplacian, gr, gc, ctx=ctx)
    torch.cuda.synchronize()
    assert torch.equal(AP2, AP)


def test_cfg1_pipeline_full_size_reduced_iterations(P, ctx):
    import torch

    from paper_1602_02070_b200 import workloads

    wl = workloads.config1()
    p, n = wl.Y.shape
    its = 20
    cfg = P.PipelineConfig(knn=10, a=wl.a, b=wl.b, kron_pcg_tol=1e-11,
                           frpcag=P.FrpcagConfig(gamma_r=wl.gamma, gamma_c=wl.gamma, loss="l1", tol=1e-300,
                                                 max_iter=its),
                           decoder=P.DecoderConfig(1.0, 1e-30, its, variant="alternate"),
                           lambda_k1_r=wl.lambda_k1_r, lambda_k1_c=wl.lambda_k1_c, seed=1603)
    Yd = torch.tensor(np.ascontiguousarray(wl.Y.T), dtype=torch.float32, device="cuda").t()
    Wr = P.SparseMatrix.from_scipy(wl.W_r, ctx=ctx)
    rep = P.run_pipeline(Yd, cfg, W_r=Wr, ctx=ctx)
    # oracle composite, stage by stage (pipeline.cpp:273-350), fp64
    Y = wl.Y.astype(np.float32).astype(np.float64)
    gr = O.graph_from_adjacency(O.Csr.from_scipy(wl.W_r))
    gc = O.build_knn_graph(Y, False, 10)
    plan = O.draw_plan(p, n, -(-p // wl.b), -(-n // wl.a), seed=1603)
    assert np.array_equal(rep.plan.omega_r, plan.omega_r) and np.array_equal(rep.plan.omega_c, plan.omega_c)
    Yt = O.subsample(Y, plan)
    Lr_t = O.kron_reduce(gr.laplacian, plan.omega_r, 1e-11)
    Lc_t = O.kron_reduce(gc.laplacian, plan.omega_c, 1e-11)
    Xt, _ = O.fista_solve(Yt, Lr_t, Lc_t, O.FrpcagConfig(wl.gamma, wl.gamma, "l1", 1e-300, its))
    assert rel(rep.Xt.cpu().numpy(), Xt) <= 1e-4
    dec = O.alternate_decode(Xt, plan, gr.laplacian, gc.laplacian, wl.lambda_k1_r, wl.lambda_k1_c, 1.0, 1e-30, its)
    assert rel(rep.X.cpu().numpy(), dec.X) <= 1e-4
    assert math.isfinite(rep.trace.objective[-1])


def test_cfg3_sharded_emulated_matches_single_gpu(P, ctx):
    """The device-resident sharded decoder at the full cfg3 size with four
    ranks emulated on one GPU (halo exchange as device copies, all-reduced
    dots), 4 CG iterations: equal to the one-GPU decoder's result up to the
    dots' summation order."""
    import torch

    from paper_1602_02070_b200 import workloads
    from paper_1602_02070_b200.sharded import alternate_decode_sharded_emulated

    Pr, Pc = workloads.config3_points()
    p, n = Pr.shape[1], Pc.shape[1]
    gr_ = P.build_knn_graph(torch.tensor(np.ascontiguousarray(Pr.T), device="cuda").t(), "cols", 10, ctx=ctx)
    gc_ = P.build_knn_graph(torch.tensor(np.ascontiguousarray(Pc.T), device="cuda").t(), "cols", 10, ctx=ctx)
    plan = P.draw_plan(p, n, p // 8, n // 8, seed=1607)
    gen = torch.Generator(device="cuda").manual_seed(9)
    Xt = torch.randn(len(plan.omega_c), len(plan.omega_r), device="cuda", generator=gen).t()
    its = 4
    g1 = P.SpectralGap(lambda_k1=1.0)
    cfg = P.DecoderConfig(1.0, 1e-30, its)
    sh, st = alternate_decode_sharded_emulated(Xt, plan, gr_.laplacian, gc_.laplacian, g1, g1, cfg, 4, ctx=ctx)
    assert sh.iterations == its
    assert 0 < st.halo_cols <= n - n // 4
    Xs = sh.X.cpu().numpy().astype(np.float64)
    del sh
    one = P.alternate_decode(Xt, plan, gr_.laplacian, gc_.laplacian, g1, g1, cfg, ctx=ctx)
    assert one.iterations == its
    assert rel(Xs, one.X.cpu().numpy().astype(np.float64)) <= 1e-6


def test_knn_second_tensor_core_pass_equals_exact_path(P, ctx, monkeypatch, capfd):
    """Points the 32-candidate filter cannot certify go through a second
    tensor-core pass with 64-candidate lists (knn.cu); its lists must equal
    the exact fp64 path's (CPCAG_KNN_PASS2=0 sends them all there)."""
    import re

    import torch

    from paper_1602_02070_b200 import workloads

    X = workloads.config2_points()  # 100 000 x 512: ~2.3 % of the points need the second pass
    d, n = X.shape
    Xd = torch.tensor(np.ascontiguousarray(X.T), device="cuda").t()
    monkeypatch.setenv("CPCAG_TRACE", "1")
    capfd.readouterr()
    nbr, d2 = P.knn(Xd, "cols", 10, ctx=ctx)
    err = capfd.readouterr().err
    m = re.search(r"\[knn\] (\d+) points, (\d+) certified by the tensor-core filter \((\d+) left by pass 1\), "
                  r"(\d+) exact fallback rows", err)
    assert m, err[-2000:]
    left1, rest = int(m.group(3)), int(m.group(4))
    assert left1 > 0 and rest < left1  # pass 2 certified some points
    monkeypatch.setenv("CPCAG_KNN_PASS2", "0")
    nbr0, d20 = P.knn(Xd, "cols", 10, ctx=ctx)
    assert np.array_equal(nbr, nbr0) and np.array_equal(d2, d20)
    rows = np.random.default_rng(11).choice(n, 24, replace=False)
    onbr, od2 = O.knn_rows(X.astype(np.float64), False, 10, rows)
    assert np.array_equal(nbr[rows], onbr) and np.array_equal(d2[rows], od2)


def test_cfg1_pipeline_full_iterations_within_north_star(P, ctx):
    """The headline configuration end to end at its full iteration counts
    (FISTA 300, CG 200; fp32 on the device, every decoder vector fp32 -- the
    path bench.py times for config 1) against the fp64 oracle composite:
    relative Frobenius error of Xt and X <= 1e-4 (north_star).  ~1 min of
    oracle time on the box's cores."""
    import torch

    from paper_1602_02070_b200 import workloads

    wl = workloads.config1()
    p, n = wl.Y.shape
    cfg = P.PipelineConfig(knn=10, a=wl.a, b=wl.b, kron_pcg_tol=1e-11,
                           frpcag=P.FrpcagConfig(gamma_r=wl.gamma, gamma_c=wl.gamma, loss="l1", tol=1e-300,
                                                 max_iter=wl.fista_iters),
                           decoder=P.DecoderConfig(1.0, 1e-30, wl.cg_iters, variant="alternate",
                                                   krylov_precision="fp32"),
                           lambda_k1_r=wl.lambda_k1_r, lambda_k1_c=wl.lambda_k1_c, seed=1603)
    Yd = torch.tensor(np.ascontiguousarray(wl.Y.T), dtype=torch.float32, device="cuda").t()
    rep = P.run_pipeline(Yd, cfg, W_r=P.SparseMatrix.from_scipy(wl.W_r, ctx=ctx), ctx=ctx)
    assert rep.trace.iterations == 300 and rep.decoder_iterations == 200
    Y = wl.Y.astype(np.float32).astype(np.float64)
    gr = O.graph_from_adjacency(O.Csr.from_scipy(wl.W_r))
    gc = O.build_knn_graph(Y, False, 10)
    plan = O.draw_plan(p, n, -(-p // wl.b), -(-n // wl.a), seed=1603)
    Xt, tr = O.fista_solve(O.subsample(Y, plan), O.kron_reduce(gr.laplacian, plan.omega_r, 1e-11),
                           O.kron_reduce(gc.laplacian, plan.omega_c, 1e-11),
                           O.FrpcagConfig(wl.gamma, wl.gamma, "l1", 1e-300, 300))
    assert rel(rep.Xt.cpu().numpy(), Xt) <= 1e-4
    assert np.allclose(rep.trace.objective, tr.objective, rtol=1e-4)
    dec = O.alternate_decode(Xt, plan, gr.laplacian, gc.laplacian, wl.lambda_k1_r, wl.lambda_k1_c, 1.0, 1e-30, 200)
    assert rel(rep.X.cpu().numpy(), dec.X) <= 1e-4


def _cfg3_problem(P, ctx, n=None):
    """The bench's config-3 decoder problem: kNN graphs over
    N(0, I_64) points, rank-20 low-pass right-hand side sampled 1/8 x 1/8.
    n: a reduced column count (the same generator, fewer column points)."""
    import torch

    from paper_1602_02070_b200 import workloads

    Pr, Pc = workloads.config3_points() if n is None else workloads.config3_points(n=n)
    p, n = Pr.shape[1], Pc.shape[1]
    gr = P.build_knn_graph(torch.tensor(np.ascontiguousarray(Pr.T), device="cuda").t(), "cols", 10, ctx=ctx)
    gc = P.build_knn_graph(torch.tensor(np.ascontiguousarray(Pc.T), device="cuda").t(), "cols", 10, ctx=ctx)
    plan = P.draw_plan(p, n, p // 8, n // 8, seed=1607)
    Xt = workloads.config3_rhs(P, gr.laplacian, gc.laplacian, plan, ctx)
    return gr, gc, plan, Xt


def test_cfg3_decoder_fp32_within_north_star_of_fp64(P, ctx):
    """Config 3 at full size (4096 x 200 000, 100 CG iterations): the fp32
    decoder as the bench runs it (fp32 X, fp64 Krylov vectors) within the
    north_star 1e-4 of the fp64 decoder, which matches the oracle to 1e-9
    wherever the oracle runs (test below at n = 20 000).  Every-vector-fp32
    CG drifts 7-8e-4 here (tools/cfg3_precision.py), which is why the fp32
    path keeps R, P and AP in fp64."""
    import torch

    ctx.reserve(48 << 30)
    gr, gc, plan, Xt = _cfg3_problem(P, ctx)
    g1 = P.SpectralGap(lambda_k1=1.0)
    dcfg = P.DecoderConfig(1.0, 1e-30, 100)
    X64 = P.alternate_decode(Xt, plan, gr.laplacian, gc.laplacian, g1, g1, dcfg, ctx=ctx).X
    X32 = P.alternate_decode(Xt.float().t().contiguous().t(), plan, gr.laplacian, gc.laplacian, g1, g1, dcfg,
                             ctx=ctx).X
    assert X32.dtype == torch.float32
    d = torch.linalg.norm(X32.double() - X64) / torch.linalg.norm(X64)
    assert float(d) <= 1e-4, float(d)


def test_cfg3_shaped_decoder_matches_oracle(P, ctx):
    """A config-3-shaped case the oracle finishes in about a minute (p = 4096,
    n = 20 000, gamma-bar = 1, 1/8 x 1/8 sampling, 100 iterations): the fp32
    decoder (the bench's path) within the north_star 1e-4 of the oracle
    (decoders.cpp:145-186).  fp64 against fp64: 100 unconverged iterations of
    this system amplify the dot products' last-ulp summation order (the
    oracle sums sequentially, the device in a fixed tree) to ~2.5e-7 (two fp64
    implementations at full config 3: 1.5e-6, tools/cfg3_precision.py), so the
    fp64 bar is 1e-6; each single apply is bit-exact (test above)."""
    gr, gc, plan, Xt = _cfg3_problem(P, ctx, n=20_000)
    g1 = P.SpectralGap(lambda_k1=1.0)
    dcfg = P.DecoderConfig(1.0, 1e-30, 100)
    X64 = P.alternate_decode(Xt, plan, gr.laplacian, gc.laplacian, g1, g1, dcfg, ctx=ctx).X.cpu().numpy()
    X32 = P.alternate_decode(Xt.float().t().contiguous().t(), plan, gr.laplacian, gc.laplacian, g1, g1, dcfg,
                             ctx=ctx).X.cpu().numpy()
    Lr = O.Csr.from_csr(*gr.laplacian.shape, *gr.laplacian.arrays())
    Lc = O.Csr.from_csr(*gc.laplacian.shape, *gc.laplacian.arrays())
    oplan = O.SamplingPlan(np.asarray(plan.omega_r), np.asarray(plan.omega_c), plan.p, plan.n)
    ro = O.alternate_decode(Xt.cpu().numpy(), oplan, Lr, Lc, 1.0, 1.0, 1.0, 1e-30, 100)
    assert rel(X64, ro.X) <= 1e-6
    X32o = O.alternate_decode(Xt.float().double().cpu().numpy(), oplan, Lr, Lc, 1.0, 1.0, 1.0, 1e-30, 100)
    assert rel(X32, X32o.X) <= 1e-4


def test_cfg0_full_size_pipeline_matches_oracle(P, ctx):
    """BASELINE config 0 at its stated size (200 x 300 fp64; K = 10 row and
    column graphs, a = b = 4, FISTA 200 iterations, CG max 100 at tol 1e-8):
    every stage of run_pipeline against the oracle composite
    (pipeline.cpp:273-350) -- plan bit-exact, Xt and X within 1e-9."""
    from paper_1602_02070_b200 import workloads

    wl = workloads.config0_workload()
    Y = wl.Y
    p, n = Y.shape
    g = wl.gamma
    cfg = P.PipelineConfig(knn=10, a=wl.a, b=wl.b, kron_pcg_tol=1e-11,
                           frpcag=P.FrpcagConfig(gamma_r=g, gamma_c=g, loss="l1", tol=1e-300, max_iter=200),
                           decoder=P.DecoderConfig(1.0, 1e-8, 100, variant="alternate"),
                           lambda_k1_r=wl.lambda_k1_r, lambda_k1_c=wl.lambda_k1_c, seed=1602)
    rep = P.run_pipeline(Y, cfg, ctx=ctx)
    gr, gc = O.build_knn_graph(Y, True, 10), O.build_knn_graph(Y, False, 10)
    plan = O.draw_plan(p, n, -(-p // wl.b), -(-n // wl.a), seed=1602)
    assert np.array_equal(rep.plan.omega_r, plan.omega_r) and np.array_equal(rep.plan.omega_c, plan.omega_c)
    Xt, tr = O.fista_solve(O.subsample(Y, plan), O.kron_reduce(gr.laplacian, plan.omega_r, 1e-11),
                           O.kron_reduce(gc.laplacian, plan.omega_c, 1e-11),
                           O.FrpcagConfig(g, g, "l1", 1e-300, 200))
    assert rep.trace.iterations == tr.iterations == 200
    assert rel(rep.Xt, Xt) <= 1e-9
    assert np.allclose(rep.trace.objective, tr.objective, rtol=1e-9)
    dec = O.alternate_decode(Xt, plan, gr.laplacian, gc.laplacian, wl.lambda_k1_r, wl.lambda_k1_c, 1.0, 1e-8, 100)
    assert abs(rep.decoder_iterations - dec.iterations) <= 1
    assert rel(rep.X, dec.X) <= 1e-9


def test_cfg2_knn_full_size_matches_oracle_fixture(P, ctx):
    """Config 2 (100 000 x 512, K = 10) in full: every neighbour list, its
    canonical fp64 squared distances and the CSR structure of W equal the
    oracle's exact result, pinned by SHA-256 in tests/golden/cfg2_knn_sha256.json
    (written by tests/golden/make_cfg2_fixture.py; graph.cpp:86-133)."""
    import hashlib
    import json
    import os

    import torch

    from paper_1602_02070_b200 import workloads

    fx = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "cfg2_knn_sha256.json")))
    sha = lambda a: hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()
    X = workloads.config2_points()
    Xd = torch.tensor(np.ascontiguousarray(X.T), device="cuda").t()
    nbr, d2 = P.knn(Xd, "cols", 10, ctx=ctx)
    for i, row in fx["sample_rows"].items():
        assert list(nbr[int(i)]) == row, i
    assert sha(nbr.astype(np.int64)) == fx["nbr_int64_sha256"]
    assert sha(d2.astype(np.float64)) == fx["d2_float64_sha256"]
    g = P.build_knn_graph(Xd, "cols", 10, ctx=ctx)
    rp, ci, _ = g.adjacency.arrays()
    assert len(ci) == fx["W_nnz"]
    assert sha(np.asarray(rp, np.int64)) == fx["W_row_ptr_int64_sha256"]
    assert sha(np.asarray(ci, np.int64)) == fx["W_col_idx_int64_sha256"]
