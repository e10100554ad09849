"""GPU parity: SpMM/SpMV, power iteration, sampling, FRPCAG operators, FISTA
and the alternate decoder through the C-ABI, against the CPU oracle.

Tolerances: fp64 SpMM/SpMV/gather are bit-exact (same per-entry operation
order); fp64 solvers within 1e-9 relative (only full-array reduction order
differs); fp32 device runs within the north_star 1e-4 relative Frobenius
error of the fp64 oracle.
"""
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


def test_spmm_left_right_fp64_bit_exact(P, ctx):
    L = knn_laplacian(300, 5, 10, 3)
    A = to_device(ctx, L)
    X = np.random.default_rng(0).standard_normal((300, 17))
    assert np.array_equal(A.multiply(X), L.multiply(X))
    Xr = np.random.default_rng(1).standard_normal((23, 300))
    assert np.array_equal(A.right_multiply(Xr), L.right_multiply(Xr))
    x = X[:, 0].copy()
    assert np.array_equal(A.multiply(x), L.spmv(x))


def test_spmm_nonsymmetric_uses_transpose_order(P, ctx):
    rs = np.random.default_rng(5)
    D = rs.standard_normal((40, 30)) * (rs.random((40, 30)) < 0.2)
    L = O.Csr.from_dense(D)
    A = to_device(ctx, L)
    X = rs.standard_normal((11, 40))
    assert np.array_equal(A.right_multiply(X), L.right_multiply(X))
    X2 = rs.standard_normal((30, 4))
    assert np.array_equal(A.multiply(X2), L.multiply(X2))
    assert not A.is_symmetric()


def test_spmm_fp32_and_device_tensors(P, ctx):
    import torch

    L = random_laplacian(200, 0.05, 7)
    A = to_device(ctx, L)
    X = np.random.default_rng(2).standard_normal((200, 9))
    Xd = torch.tensor(X, dtype=torch.float32, device="cuda")
    Y = A.multiply(Xd)
    assert Y.is_cuda and Y.dtype == torch.float32
    assert rel(Y.cpu().numpy(), L.multiply(X)) <= 1e-6


def test_spmm_dimension_mismatch(P, ctx):
    A = to_device(ctx, random_laplacian(10, 0.3, 1))
    with pytest.raises(ValueError, match="dimension mismatch"):
        A.multiply(np.zeros((9, 2)))
    with pytest.raises(ValueError, match="dimension mismatch"):
        A.multiply(np.zeros(4))


def test_power_iteration_known_answers(P, ctx):
    # test_numeric.cpp:179-199
    A = P.SparseMatrix.from_triplets(3, 3, [0, 1, 2], [0, 1, 2], [1.0, 5.0, 3.0], ctx=ctx)
    assert P.power_iteration_norm(A, 1e-12, 3, ctx=ctx) == pytest.approx(5.0, rel=1e-9)
    ti, tj, tv = [], [], []
    for i in range(4):
        for j in range(4):
            ti.append(i), tj.append(j), tv.append(3.0 if i == j else -1.0)
    K4 = P.SparseMatrix.from_triplets(4, 4, ti, tj, tv, ctx=ctx)
    assert P.power_iteration_norm(K4, 1e-12, 5, ctx=ctx) == pytest.approx(4.0, rel=1e-9)
    Z = P.SparseMatrix.from_triplets(4, 4, [], [], [], ctx=ctx)
    assert P.power_iteration_norm(Z, 1e-10, 9, ctx=ctx) == 0.0


def test_power_iteration_matches_oracle(P, ctx):
    # 50, 700: one CTA; 3000: cooperative grid, v in shared memory;
    # 20000: cooperative grid, v renormalised in global memory
    for seed, n in [(1, 50), (2, 700), (3, 3000), (4, 20000)]:
        L = knn_laplacian(n, 4, 8, seed)
        got = P.power_iteration_norm(to_device(ctx, L), 1e-7, 42, ctx=ctx)
        want = O.power_iteration_norm(L, 1e-7, 42)
        assert got == pytest.approx(want, rel=1e-6)


def test_power_iteration_several_products_per_barrier(P, ctx):
    # operators whose rows of A A (and A A A) fit a CTA's shared memory iterate
    # two or three times per grid barrier (w_m = A^m v): same estimates and stop
    # iteration as solvers.cpp:43-51, also against the one-product kernel
    rs = np.random.default_rng(17)
    W = np.abs(rs.standard_normal((900, 900))) * (rs.random((900, 900)) < 0.6)
    W = np.triu(W, 1)
    W = W + W.T
    Ld = np.diag(W.sum(1)) - W  # dense-ish Laplacian, the shape of a Kron-reduced graph
    ii, jj = np.nonzero(Ld)
    # 900 rows: 7 rows of A^2 and A^3 per CTA fit; 1400 rows: only A^2's 10 rows do
    cases = [(O.Csr.from_triplets(900, 900, ii, jj, Ld[ii, jj]), "triple"), (knn_laplacian(1400, 4, 8, 5), "double")]
    for L, auto in cases:
        A = to_device(ctx, L)
        want = O.power_iteration_norm(L, 1e-7, 42)
        got = {}
        try:
            for path, ran in (("auto", auto), ("double", "double"), ("single", "single")):
                ctx.set_power_path(path)
                got[path] = P.power_iteration_norm(A, 1e-7, 42, ctx=ctx)
                assert ctx.last_power_path() == ran
                assert got[path] == pytest.approx(want, rel=1e-9)
                # iteration caps of every residue stop where the reference stops
                for cap in (1, 2, 3, 4, 5, 6, 7):
                    g = P.power_iteration_norm(A, 1e-30, 42, cap, ctx=ctx)
                    w = O.power_iteration_norm(L, 1e-30, 42, cap)
                    assert g == pytest.approx(w, rel=1e-9)
        finally:
            ctx.set_power_path("auto")
        assert got["auto"] == pytest.approx(got["single"], rel=1e-12)
        assert got["double"] == pytest.approx(got["single"], rel=1e-12)


def test_plan_and_subsample_bit_exact(P, ctx):
    plan = P.draw_plan(1000, 777, 101, 93, seed=1602)
    plan_o = O.draw_plan(1000, 777, 101, 93, seed=1602)
    assert np.array_equal(plan.omega_r, plan_o.omega_r)
    assert np.array_equal(plan.omega_c, plan_o.omega_c)
    Y = np.random.default_rng(3).standard_normal((1000, 777))
    assert np.array_equal(P.subsample(Y, plan, ctx=ctx), O.subsample(Y, plan_o))
    with pytest.raises(ValueError, match="does not match"):
        P.subsample(Y[:, :10], plan, ctx=ctx)


def test_prox_grad_objective_match_oracle(P, ctx):
    rs = np.random.default_rng(9)
    r, c = 37, 29
    Lr, Lc = random_laplacian(r, 0.2, 1), random_laplacian(c, 0.3, 2)
    dLr, dLc = to_device(ctx, Lr), to_device(ctx, Lc)
    Z, Y = rs.standard_normal((r, c)), rs.standard_normal((r, c))
    assert np.array_equal(P.prox_l1(Z, Y, 0.3, ctx=ctx), O.prox_l1(Z, Y, 0.3))
    assert np.array_equal(P.prox_l2(Z, Y, 0.3, ctx=ctx), O.prox_l2(Z, Y, 0.3))
    cfg = P.FrpcagConfig(gamma_r=1.5, gamma_c=0.7)
    ocfg = O.FrpcagConfig(gamma_r=1.5, gamma_c=0.7)
    assert np.array_equal(P.grad_g(Z, dLr, dLc, cfg, ctx=ctx), O.grad_g(Z, Lr, Lc, ocfg))
    assert P.objective(Z, Y, dLr, dLc, cfg, ctx=ctx) == pytest.approx(O.objective(Z, Y, Lr, Lc, ocfg), rel=1e-12)
    with pytest.raises(ValueError, match="negative threshold"):
        P.prox_l1(Z, Y, -1.0, ctx=ctx)


@pytest.mark.parametrize("loss", ["l1", "l2"])
def test_fista_fp64_matches_oracle(P, ctx, loss):
    rs = np.random.default_rng(11)
    r, c = 60, 45
    Lr, Lc = knn_laplacian(r, 3, 6, 4), knn_laplacian(c, 3, 6, 5)
    Y = rs.standard_normal((r, c))
    cfg = P.FrpcagConfig(gamma_r=3.0, gamma_c=2.0, loss=loss, tol=1e-300, max_iter=120)
    X, tr = P.fista_solve(Y, to_device(ctx, Lr), to_device(ctx, Lc), cfg, ctx=ctx)
    Xo, tro = O.fista_solve(Y, Lr, Lc, O.FrpcagConfig(3.0, 2.0, loss, 1e-300, 120))
    assert tr.iterations == tro.iterations == 120 and not tr.converged
    assert tr.step == pytest.approx(tro.step, rel=1e-6)
    assert rel(X, Xo) <= 1e-9
    assert np.allclose(tr.objective, tro.objective, rtol=1e-9)


def test_fista_stops_on_tolerance_like_oracle(P, ctx):
    rs = np.random.default_rng(12)
    Lr, Lc = knn_laplacian(30, 3, 5, 6), knn_laplacian(25, 3, 5, 7)
    Y = rs.standard_normal((30, 25))
    cfg = P.FrpcagConfig(gamma_r=0.5, gamma_c=0.5, loss="l2", tol=1e-8, max_iter=5000)
    X, tr = P.fista_solve(Y, to_device(ctx, Lr), to_device(ctx, Lc), cfg, ctx=ctx)
    Xo, tro = O.fista_solve(Y, Lr, Lc, O.FrpcagConfig(0.5, 0.5, "l2", 1e-8, 5000))
    assert tr.converged and tro.converged
    assert abs(tr.iterations - tro.iterations) <= 1
    assert rel(X, Xo) <= 1e-7


def test_fista_fp32_within_north_star_tolerance(P, ctx):
    rs = np.random.default_rng(13)
    Lr, Lc = knn_laplacian(120, 3, 8, 8), knn_laplacian(90, 3, 8, 9)
    Y = rs.standard_normal((120, 90))
    cfg = P.FrpcagConfig(gamma_r=2.0, gamma_c=2.0, tol=1e-300, max_iter=200)
    X, tr = P.fista_solve(Y.astype(np.float32), to_device(ctx, Lr), to_device(ctx, Lc), cfg, ctx=ctx)
    Xo, _ = O.fista_solve(Y.astype(np.float32).astype(np.float64), Lr, Lc,
                          O.FrpcagConfig(2.0, 2.0, "l1", 1e-300, 200))
    assert X.dtype == np.float32
    assert rel(X, Xo) <= 1e-4


def test_fista_errors(P, ctx):
    Lr, Lc = random_laplacian(6, 0.5, 1), random_laplacian(5, 0.5, 2)
    dLr, dLc = to_device(ctx, Lr), to_device(ctx, Lc)
    Y = np.ones((6, 5))
    with pytest.raises(ValueError, match="negative regularization"):
        P.fista_solve(Y, dLr, dLc, P.FrpcagConfig(gamma_r=-1.0), ctx=ctx)
    with pytest.raises(ValueError, match="column Laplacian"):
        P.fista_solve(Y, dLr, dLr, P.FrpcagConfig(), ctx=ctx)
    with pytest.raises(RuntimeError, match=r"diverged \(non-finite objective at iteration"):
        P.fista_solve(Y * 1e300, dLr, dLc, P.FrpcagConfig(step=10.0, tol=1e-300, max_iter=20), ctx=ctx)


def _decoder_case(p=150, n=120, rr=40, rc=30, seed=21):
    Lr, Lc = knn_laplacian(p, 3, 7, seed), knn_laplacian(n, 3, 7, seed + 1)
    plan = O.draw_plan(p, n, rr, rc, seed=seed)
    Xt = np.random.default_rng(seed).standard_normal((rr, rc))
    return Lr, Lc, plan, Xt


def _grid_laplacian(h, w):
    """Unit-weight 8-neighbour grid (pixel order column-major): a row graph
    with locality, so the lr pass splits into row ranges with windows."""
    from paper_1602_02070_b200 import workloads

    W = workloads.grid_adjacency(h, w)
    return O.graph_from_adjacency(O.Csr.from_scipy(W)).laplacian


# Shapes that take every path of the apply engine (decoder.cuh): the lc pass
# with the band in shared memory (n * 128 B <= 200 KB) or resident in L2;
# the lr pass as one range (kNN rows) or windowed row ranges (grid rows), in
# natural or degree-sorted row order (hub-heavy 24-d kNN rows).
DECODER_CASES = {
    "smem": lambda: (knn_laplacian(150, 3, 7, 21), knn_laplacian(120, 3, 7, 22), 150, 120, 40, 30),
    "l2": lambda: (knn_laplacian(70, 3, 7, 31), knn_laplacian(2100, 3, 7, 32), 70, 2100, 20, 300),
    "grid": lambda: (_grid_laplacian(48, 40), knn_laplacian(90, 3, 7, 42), 48 * 40, 90, 480, 25),
    "hubs": lambda: (knn_laplacian(600, 24, 10, 51), knn_laplacian(80, 3, 7, 52), 600, 80, 150, 20),
}


def _case_by_name(name, seed=7):
    Lr, Lc, p, n, rr, rc = DECODER_CASES[name]()
    plan = O.draw_plan(p, n, rr, rc, seed=seed)
    Xt = np.random.default_rng(seed).standard_normal((rr, rc))
    return Lr, Lc, plan, Xt


@pytest.fixture(params=["fused", "split", "slab"])
def path(request, ctx):
    """Every operator path (fused one-pass / two-pass band + row groups /
    32-row slab for fp32 iterates; fp64 iterates fall back from "slab" to
    the two passes)."""
    ctx.set_apply_path(request.param)
    yield request.param
    ctx.set_apply_path("auto")


@pytest.mark.parametrize("case", sorted(DECODER_CASES))
def test_decoder_apply_fp64_bit_exact(P, ctx, case, path):
    """One application of the operator (decoders.cpp:160-170) through the
    two passes equals the oracle's reference-order loop bit for bit."""
    Lr, Lc, plan_o, _ = _case_by_name(case)
    plan = P.SamplingPlan(plan_o.omega_r, plan_o.omega_c, plan_o.p, plan_o.n)
    X = np.asfortranarray(np.random.default_rng(3).standard_normal((plan.p, plan.n)))
    AP, dot = P.decoder_apply(X, plan, to_device(ctx, Lr), to_device(ctx, Lc), 1 / 0.3, 1 / 0.4, ctx=ctx)
    want = O.decoder_apply(X, plan_o, Lr, Lc, 1 / 0.3, 1 / 0.4)
    assert np.array_equal(AP, want)
    assert abs(dot - float(np.sum(X * want))) <= 1e-12 * abs(dot)


def _star_laplacian(n, hub_deg, seed):
    """kNN graph plus one hub joined to `hub_deg` nodes: a pull row longer
    than the slab pass's record ring holds at once."""
    import scipy.sparse as sp

    W = knn_laplacian(n, 3, 5, seed).to_scipy()
    W = -(W - sp.diags(W.diagonal()))
    hub = sp.coo_matrix((np.ones(hub_deg), (np.zeros(hub_deg, int), np.arange(1, hub_deg + 1))), shape=(n, n))
    W = (W + hub + hub.T).tocsr()
    return O.graph_from_adjacency(O.Csr.from_scipy(W)).laplacian


SLAB_CASES = {  # (operators, p, n, |omega_r|, |omega_c>), the path the slab request takes
    "knn_rows": (lambda: (knn_laplacian(96, 3, 7, 23), knn_laplacian(120, 3, 7, 24), 96, 120, 30, 30), "slab"),
    "grid": (DECODER_CASES["grid"], "slab"),  # 9-entry pixel stencil, +-w rows in the staged window
    "grid_ragged": (lambda: (_grid_laplacian(37, 28), knn_laplacian(300, 3, 10, 61), 37 * 28, 300, 110, 40), "slab"),
    "col_hubs": (lambda: (_grid_laplacian(20, 16), knn_laplacian(700, 24, 10, 71), 320, 700, 40, 90), "slab"),
    # a 231-entry pull row: its quad runs as several steps of the record ring
    "long_pull_row": (lambda: (_grid_laplacian(16, 12), _star_laplacian(400, 230, 81), 192, 400, 30, 50), "slab"),
    # fallbacks to the fused pass: p not a multiple of 4; row windows wider
    # than 32 chunks (random rows over p = 600)
    "p_odd": (DECODER_CASES["smem"], "fused"),
    "wide_rows": (lambda: (knn_laplacian(600, 3, 7, 91), knn_laplacian(80, 3, 7, 92), 600, 80, 150, 20), "fused"),
}


@pytest.mark.parametrize("case", sorted(SLAB_CASES))
def test_decoder_apply_fp32_slab_equals_fused(P, ctx, case):
    """fp32 iterates: the slab pass (shared-memory slab of 32 rows x all
    columns, L_c records streamed through warp rings) accumulates every
    entry in the same CSR order as the fused pass -- bit-identical -- and
    sits within fp32 rounding of the fp64 oracle (decoders.cpp:160-170)."""
    make, want_path = SLAB_CASES[case]
    Lr, Lc, p, n, rr, rc = make()
    plan_o = O.draw_plan(p, n, rr, rc, seed=5)
    plan = P.SamplingPlan(plan_o.omega_r, plan_o.omega_c, plan_o.p, plan_o.n)
    X = np.asfortranarray(np.random.default_rng(4).standard_normal((p, n)).astype(np.float32))
    dLr, dLc = to_device(ctx, Lr), to_device(ctx, Lc)
    out = {}
    try:
        for path in ("slab", "fused"):
            ctx.set_apply_path(path)
            out[path] = P.decoder_apply(X, plan, dLr, dLc, 1 / 0.3, 1 / 0.4, ctx=ctx)
            assert ctx.last_apply_path() == (want_path if path == "slab" else "fused")
    finally:
        ctx.set_apply_path("auto")
    (As, ds), (Af, df) = out["slab"], out["fused"]
    assert As.dtype == np.float32
    assert np.array_equal(As, Af)
    assert abs(ds - df) <= 1e-12 * abs(df)  # fp64 partial sums over different CTA grids
    want = O.decoder_apply(X.astype(np.float64), plan_o, Lr, Lc, 1 / 0.3, 1 / 0.4)
    assert rel(As, want) <= 1e-6
    assert abs(ds - float(np.sum(X.astype(np.float64) * want))) <= 1e-5 * abs(ds)


@pytest.mark.parametrize("case", sorted(DECODER_CASES))
def test_alternate_decode_fp64_matches_oracle(P, ctx, case, path):
    Lr, Lc, plan_o, Xt = _case_by_name(case)
    plan = P.SamplingPlan(plan_o.omega_r, plan_o.omega_c, plan_o.p, plan_o.n)
    res = P.alternate_decode(Xt, plan, to_device(ctx, Lr), to_device(ctx, Lc), P.SpectralGap(lambda_k1=0.3),
                             P.SpectralGap(lambda_k1=0.4), P.DecoderConfig(1.0, 1e-10, 4000), ctx=ctx)
    ro = O.alternate_decode(Xt, plan_o, Lr, Lc, 0.3, 0.4, 1.0, 1e-10, 4000)
    assert res.converged and ro.converged  # converged: the dots' summation order does not matter
    assert abs(res.iterations - ro.iterations) <= 1
    assert rel(res.X, ro.X) <= 1e-9


@pytest.mark.parametrize("krylov", ["fp64", "fp32"])
@pytest.mark.parametrize("case", sorted(DECODER_CASES))
def test_alternate_decode_fixed_iterations_fp32(P, ctx, case, krylov, path):
    """fp32 data: fp32 X with fp64 Krylov vectors (default) or every vector
    fp32, 100 iterations, against the fp64 oracle on the fp32-rounded input
    (fp64 Krylov: only X's and the operator values' fp32 rounding remain,
    ~1e-6; the north_star bar is 1e-4)."""
    Lr, Lc, plan_o, Xt = _case_by_name(case)
    plan = P.SamplingPlan(plan_o.omega_r, plan_o.omega_c, plan_o.p, plan_o.n)
    Xt32 = Xt.astype(np.float32)
    res = P.alternate_decode(Xt32, plan, to_device(ctx, Lr), to_device(ctx, Lc), P.SpectralGap(lambda_k1=1.0),
                             P.SpectralGap(lambda_k1=1.0),
                             P.DecoderConfig(1.0, 1e-30, 100, krylov_precision=krylov), ctx=ctx)
    ro = O.alternate_decode(Xt32.astype(np.float64), plan_o, Lr, Lc, 1.0, 1.0, 1.0, 1e-30, 100)
    assert res.X.dtype == np.float32
    assert res.iterations == ro.iterations == 100
    assert rel(res.X, ro.X) <= (1e-5 if krylov == "fp64" else 1e-4)


def test_alternate_decode_max_iter_zero_returns_zero(P, ctx):
    """pcg_core's loop `while (it < max_iter)` runs no iteration for
    max_iter <= 0: X stays 0 (solvers.hpp:52)."""
    Lr, Lc, plan_o, Xt = _decoder_case(40, 30, 10, 8, 5)
    plan = P.SamplingPlan(plan_o.omega_r, plan_o.omega_c, plan_o.p, plan_o.n)
    g = P.SpectralGap(lambda_k1=1.0)
    for mi in (0, -3):
        res = P.alternate_decode(Xt, plan, to_device(ctx, Lr), to_device(ctx, Lc), g, g,
                                 P.DecoderConfig(1.0, 1e-10, mi), ctx=ctx)
        ro = O.alternate_decode(Xt, plan_o, Lr, Lc, 1.0, 1.0, 1.0, 1e-10, mi)
        assert res.iterations == ro.iterations == 0
        assert np.all(res.X == 0) and res.converged == ro.converged


def test_alternate_decode_zero_rhs_and_validation(P, ctx):
    Lr, Lc, plan_o, Xt = _decoder_case(20, 15, 5, 4, 3)
    plan = P.SamplingPlan(plan_o.omega_r, plan_o.omega_c, plan_o.p, plan_o.n)
    dLr, dLc = to_device(ctx, Lr), to_device(ctx, Lc)
    g = P.SpectralGap(lambda_k1=1.0)
    res = P.alternate_decode(np.zeros_like(Xt), plan, dLr, dLc, g, g, ctx=ctx)
    assert res.converged and res.iterations == 0 and np.all(res.X == 0)
    with pytest.raises(ValueError, match="gamma must be positive"):
        P.alternate_decode(Xt, plan, dLr, dLc, g, g, P.DecoderConfig(gamma=0.0), ctx=ctx)
    with pytest.raises(ValueError, match="Laplacians do not match"):
        P.alternate_decode(Xt, plan, dLc, dLc, g, g, ctx=ctx)
    with pytest.raises(ValueError, match="Xt does not match"):
        P.alternate_decode(Xt[:, :2], plan, dLr, dLc, g, g, ctx=ctx)


def test_decoder_breakdown_names_iteration(P, ctx):
    # A zero operator (no graph, no samples on the support) breaks down at 0:
    # mask empty rows/cols are impossible with a plan, so use negative weights.
    p, n = 6, 5
    Lr = P.SparseMatrix.from_triplets(p, p, range(p), range(p), [-1.0] * p, ctx=ctx)
    Lc = P.SparseMatrix.from_triplets(n, n, range(n), range(n), [-1.0] * n, ctx=ctx)
    plan = P.draw_plan(p, n, 2, 2, seed=1)
    g = P.SpectralGap(lambda_k1=1.0)
    with pytest.raises(RuntimeError, match="pcg: breakdown .* at iteration 0"):
        P.alternate_decode(np.ones((2, 2)), plan, Lr, Lc, g, g, ctx=ctx)


def test_launches_are_counted(P, ctx):
    ctx.reset_launch_count()
    L = random_laplacian(50, 0.1, 3)
    to_device(ctx, L).multiply(np.ones((50, 3)))
    assert ctx.launch_count >= 1


@pytest.mark.parametrize("prec", ["f64", "f32"])
def test_fista_dense_operator_path(P, ctx, prec):
    """Kron-reduced Laplacians are near dense: the dense tiled-GEMM path."""
    Lr_full, Lc_full = knn_laplacian(300, 3, 10, 31), knn_laplacian(240, 3, 10, 32)
    plan = O.draw_plan(300, 240, 75, 60, seed=5)
    Lr, Lc = O.kron_reduce(Lr_full, plan.omega_r, 1e-11), O.kron_reduce(Lc_full, plan.omega_c, 1e-11)
    assert Lr.nnz >= 0.25 * 75 * 75 and Lc.nnz >= 0.25 * 60 * 60
    Y = np.random.default_rng(4).standard_normal((75, 60)) * 3.0
    dt = np.float64 if prec == "f64" else np.float32
    cfg = P.FrpcagConfig(gamma_r=8.0, gamma_c=8.0, tol=1e-300, max_iter=150)
    X, tr = P.fista_solve(Y.astype(dt), to_device(ctx, Lr), to_device(ctx, Lc), cfg, ctx=ctx)
    Xo, tro = O.fista_solve(Y.astype(dt).astype(np.float64), Lr, Lc, O.FrpcagConfig(8.0, 8.0, "l1", 1e-300, 150))
    assert rel(X, Xo) <= (1e-9 if prec == "f64" else 1e-4)
    assert np.allclose(tr.objective, tro.objective, rtol=1e-9 if prec == "f64" else 1e-4)


def test_context_stream_follows_torch_default_stream(P):
    """torch's default stream (handle 0) maps to cudaStreamLegacy, not to the
    C-ABI's NULL = "own stream"."""
    import torch

    from paper_1602_02070_b200 import _native as N

    c = P.Context(0)
    c.set_stream(torch.cuda.current_stream().cuda_stream)
    assert N.lib().cpcag_ctx_stream(c.handle) == P.cpcag.CUDA_STREAM_LEGACY
    s = torch.cuda.Stream()
    c.set_stream(s.cuda_stream)
    assert N.lib().cpcag_ctx_stream(c.handle) == s.cuda_stream
    c.set_stream(None)
    own = N.lib().cpcag_ctx_stream(c.handle)
    assert own not in (None, 0, P.cpcag.CUDA_STREAM_LEGACY)
