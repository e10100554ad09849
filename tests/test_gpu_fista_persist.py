"""GPU parity of the single-kernel FISTA (fista_persist.cu, the fp32 dense
path) against the fp64 oracle (frpcag.cpp:62-112): iterates, objective
trace, tolerance stop, zero-weight terms, l2 loss, divergence error, and
agreement with the per-kernel path (CPCAG_FISTA_PERSIST=0).

Tolerance: the north_star 1e-4 relative Frobenius error for fp32 runs.
"""
import numpy as np
import pytest

from helpers import knn_laplacian, rel, to_device
from oracle import pyoracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    import paper_1602_02070_b200 as P

    return P


@pytest.fixture(scope="module")
def ctx(P):
    return P.Context(0)


@pytest.fixture(params=["auto", "simt"])
def gemm(request, ctx):
    """Both tile GEMMs of the persistent kernel: fp64 tensor cores (DMMA,
    the default) and SIMT DFMA."""
    ctx.set_fista_path(request.param)
    yield request.param
    ctx.set_fista_path("auto")


def _reduced(p, n, rr, rc, seed):
    Lr_full, Lc_full = knn_laplacian(p, 3, 10, seed), knn_laplacian(n, 3, 10, seed + 1)
    plan = O.draw_plan(p, n, rr, rc, seed=seed)
    return O.kron_reduce(Lr_full, plan.omega_r, 1e-11), O.kron_reduce(Lc_full, plan.omega_c, 1e-11)


def _run(P, ctx, Y, Lr, Lc, gr, gc, loss, tol, its, timed=True):
    cfg = P.FrpcagConfig(gamma_r=gr, gamma_c=gc, loss=loss, tol=tol, max_iter=its)
    ctx.enable_kernel_timing(True)
    ctx.reset_kernel_timing()
    X, tr = P.fista_solve(Y.astype(np.float32), to_device(ctx, Lr), to_device(ctx, Lc), cfg, ctx=ctx)
    kt = ctx.kernel_times()
    ctx.enable_kernel_timing(False)
    return X, tr, kt


@pytest.mark.parametrize("shape,gr,gc,loss", [
    ((400, 300, 101, 60), 2.0, 2.0, "l1"),    # several row blocks, ragged tiles
    ((200, 160, 50, 40), 3.0, 0.0, "l1"),     # column term off (frpcag.cpp:55-58)
    ((200, 160, 50, 40), 0.0, 5.0, "l2"),     # row term off, l2 prox
    ((160, 120, 9, 7), 2.0, 2.0, "l1"),       # tiny, single tile
])
def test_persistent_fista_matches_oracle(P, ctx, shape, gr, gc, loss, gemm):
    p, n, rr, rc = shape
    Lr, Lc = _reduced(p, n, rr, rc, 40 + rr)
    Y = np.random.default_rng(rr).standard_normal((rr, rc)) * 4.0
    Y32 = Y.astype(np.float32)
    X, tr, kt = _run(P, ctx, Y32, Lr, Lc, gr, gc, loss, 1e-300, 150)
    assert "fista_persist" in kt, kt
    Xo, tro = O.fista_solve(Y32.astype(np.float64), Lr, Lc, O.FrpcagConfig(gr, gc, loss, 1e-300, 150))
    assert X.dtype == np.float32
    assert tr.iterations == tro.iterations == 150
    assert rel(X, Xo) <= 1e-4
    assert np.allclose(tr.objective, tro.objective, rtol=1e-4)
    assert tr.step == pytest.approx(tro.step, rel=1e-12)


def test_persistent_fista_tolerance_stop(P, ctx):
    Lr, Lc = _reduced(300, 240, 75, 60, 7)
    Y = np.random.default_rng(2).standard_normal((75, 60)).astype(np.float32)
    X, tr, kt = _run(P, ctx, Y, Lr, Lc, 0.5, 0.5, "l2", 1e-7, 5000)
    assert "fista_persist" in kt
    Xo, tro = O.fista_solve(Y.astype(np.float64), Lr, Lc, O.FrpcagConfig(0.5, 0.5, "l2", 1e-7, 5000))
    assert tr.converged and tro.converged
    assert abs(tr.iterations - tro.iterations) <= 2
    assert len(tr.objective) == tr.iterations
    assert rel(X, Xo) <= 1e-4


def test_persistent_fista_agrees_with_per_kernel_path(P, ctx, monkeypatch):
    Lr, Lc = _reduced(400, 300, 101, 60, 11)
    Y = (np.random.default_rng(5).standard_normal((101, 60)) * 10).astype(np.float32)
    X1, tr1, kt1 = _run(P, ctx, Y, Lr, Lc, 6.0, 6.0, "l1", 1e-300, 200)
    monkeypatch.setenv("CPCAG_FISTA_PERSIST", "0")
    X2, tr2, kt2 = _run(P, ctx, Y, Lr, Lc, 6.0, 6.0, "l1", 1e-300, 200)
    assert "fista_persist" in kt1 and "fista_persist" not in kt2
    assert rel(X1, X2) <= 1e-4
    assert np.allclose(tr1.objective, tr2.objective, rtol=1e-4)


def test_persistent_fista_shapes_and_weights_match_oracle(P, ctx):
    """The persistent kernel on assorted shapes, one-sided weights and both losses."""
    for shape, gr, gc, loss in [((400, 300, 101, 60), 2.0, 2.0, "l1"), ((200, 160, 50, 40), 0.0, 5.0, "l2"),
                                ((200, 160, 50, 40), 3.0, 0.0, "l1")]:
        p, n, rr, rc = shape
        Lr, Lc = _reduced(p, n, rr, rc, 40 + rr)
        Y = (np.random.default_rng(rr).standard_normal((rr, rc)) * 4.0).astype(np.float32)
        X, tr, kt = _run(P, ctx, Y, Lr, Lc, gr, gc, loss, 1e-300, 150)
        assert "fista_persist" in kt
        Xo, tro = O.fista_solve(Y.astype(np.float64), Lr, Lc, O.FrpcagConfig(gr, gc, loss, 1e-300, 150))
        assert rel(X, Xo) <= 1e-4
        assert np.allclose(tr.objective, tro.objective, rtol=1e-4)


def test_persistent_fista_is_deterministic(P, ctx):
    Lr, Lc = _reduced(400, 300, 101, 60, 12)
    Y = np.random.default_rng(6).standard_normal((101, 60)).astype(np.float32)
    X1, tr1, _ = _run(P, ctx, Y, Lr, Lc, 4.0, 4.0, "l1", 1e-300, 100)
    X2, tr2, _ = _run(P, ctx, Y, Lr, Lc, 4.0, 4.0, "l1", 1e-300, 100)
    assert np.array_equal(X1, X2)
    assert tr1.objective == tr2.objective


def test_persistent_fista_divergence_error(P, ctx):
    Lr, Lc = _reduced(200, 160, 50, 40, 13)
    Y = np.full((50, 40), 3e38, np.float32)
    cfg = P.FrpcagConfig(gamma_r=1.0, gamma_c=1.0, step=10.0, tol=1e-300, max_iter=30)
    with pytest.raises(RuntimeError, match=r"diverged \(non-finite objective at iteration \d+\); step too large"):
        P.fista_solve(Y, to_device(ctx, Lr), to_device(ctx, Lc), cfg, ctx=ctx)


@pytest.mark.parametrize("prec", [np.float32, np.float64])
def test_persistent_fista_tensor_core_gemm_matches_simt(P, ctx, prec):
    """DMMA and SIMT tile GEMMs both accumulate H = g L~ S in fp64 from the
    same operands; only the summation order differs (fp64 rounding), so the
    solves agree far inside the fp32 bar, and fp64 runs stay within the
    fp64 parity bar of each other and of the oracle (1e-9)."""
    Lr, Lc = _reduced(400, 300, 101, 60, 21)
    Y = (np.random.default_rng(8).standard_normal((101, 60)) * 4.0).astype(prec)
    cfg = P.FrpcagConfig(gamma_r=3.0, gamma_c=3.0, tol=1e-300, max_iter=120)
    out = {}
    try:
        for path in ("auto", "simt"):
            ctx.set_fista_path(path)
            out[path] = P.fista_solve(Y, to_device(ctx, Lr), to_device(ctx, Lc), cfg, ctx=ctx)
    finally:
        ctx.set_fista_path("auto")
    (Xd, trd), (Xs, trs) = out["auto"], out["simt"]
    assert Xd.dtype == prec
    Xo, tro = O.fista_solve(Y.astype(np.float64), Lr, Lc, O.FrpcagConfig(3.0, 3.0, "l1", 1e-300, 120))
    if prec == np.float64:
        assert rel(Xd, Xs) <= 1e-12
        assert rel(Xd, Xo) <= 1e-9
    else:
        assert rel(Xd, Xs) <= 1e-5
        assert rel(Xd, Xo) <= 1e-4
