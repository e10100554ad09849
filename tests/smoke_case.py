"""The smoke() case: one small CPCA run on cuda:0 checked against the oracle."""
import numpy as np

from oracle import pyoracle as O


def run_smoke():
    import paper_1602_02070_b200 as P
    from helpers import knn_laplacian, rel, to_device

    ctx = P.Context(0)
    p, n = 60, 80
    rs = np.random.default_rng(1602)
    Y = rs.standard_normal((p, n))
    Lr_o = knn_laplacian(p, 3, 6, 1)
    Lc_o = knn_laplacian(n, 3, 6, 2)
    plan = P.draw_plan(p, n, 20, 25, seed=1602)
    plan_o = O.draw_plan(p, n, 20, 25, seed=1602)
    assert np.array_equal(plan.omega_r, plan_o.omega_r) and np.array_equal(plan.omega_c, plan_o.omega_c)
    Yt = P.subsample(Y, plan, ctx=ctx)
    assert np.array_equal(Yt, O.subsample(Y, plan_o))
    Lr_t = O.kron_reduce(Lr_o, plan_o.omega_r, 1e-11)
    Lc_t = O.kron_reduce(Lc_o, plan_o.omega_c, 1e-11)
    cfg = P.FrpcagConfig(gamma_r=2.0, gamma_c=2.0, tol=1e-300, max_iter=40)
    Xt, tr = P.fista_solve(Yt, to_device(ctx, Lr_t), to_device(ctx, Lc_t), cfg, ctx=ctx)
    Xt_o, tr_o = O.fista_solve(Yt, Lr_t, Lc_t, O.FrpcagConfig(2.0, 2.0, "l1", 1e-300, 40))
    assert tr.iterations == tr_o.iterations == 40
    assert rel(Xt, Xt_o) <= 1e-8, rel(Xt, Xt_o)
    res = P.alternate_decode(Xt, plan, to_device(ctx, Lr_o), to_device(ctx, Lc_o),
                             P.SpectralGap(lambda_k1=0.5), P.SpectralGap(lambda_k1=0.7),
                             P.DecoderConfig(1.0, 1e-8, 100), ctx=ctx)
    res_o = O.alternate_decode(Xt_o, plan_o, Lr_o, Lc_o, 0.5, 0.7, 1.0, 1e-8, 100)
    assert abs(res.iterations - res_o.iterations) <= 1
    assert rel(res.X, res_o.X) <= 1e-8, rel(res.X, res_o.X)
    assert ctx.launch_count > 0
