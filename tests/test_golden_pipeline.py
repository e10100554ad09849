"""The committed golden fixture tests/golden/cpca_small.npz (every stage of a
small CPCA run, written by the oracle restatement with
tests/golden/make_pipeline_fixture.py): the oracle must reproduce it bit for
bit (CPU), and the device path must match it (GPU: plan, gathers and CSR
structure bit-exact, weights to 1e-14, solver outputs within the fp64 bars
of DESIGN.md §2)."""
import os
import sys

import numpy as np
import pytest

from helpers import rel

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
sys.path.insert(0, GOLD)


@pytest.fixture(scope="module")
def gold():
    return dict(np.load(os.path.join(GOLD, "cpca_small.npz")))


def test_oracle_reproduces_the_fixture(gold):
    from make_pipeline_fixture import stages

    now = stages(gold["Y"])
    assert set(now) == set(gold)
    for k, v in gold.items():
        assert np.array_equal(np.asarray(now[k]), v), k


@pytest.mark.gpu
def test_device_stages_match_the_fixture(gold):
    import paper_1602_02070_b200 as P

    ctx = P.Context(0)
    Y = gold["Y"]
    p, n = Y.shape
    gr = P.build_knn_graph(Y, "rows", 10, ctx=ctx)
    gc = P.build_knn_graph(Y, "cols", 10, ctx=ctx)
    for g, name in ((gr, "Lr"), (gc, "Lc")):
        rp, ci, v = g.laplacian.arrays()
        # structure bit-exact; weights exp(-d2 / sigma2) to the last ulps (CUDA
        # vs glibc exp), as test_gpu_graph.py
        assert np.array_equal(rp, gold[name + "_rp"]) and np.array_equal(ci, gold[name + "_ci"])
        assert np.abs(v - gold[name + "_v"]).max() <= 1e-14 * np.abs(gold[name + "_v"]).max(), name
    assert gr.sigma2 == pytest.approx(float(gold["sigma2_r"]), rel=1e-15)
    assert gc.sigma2 == pytest.approx(float(gold["sigma2_c"]), rel=1e-15)
    plan = P.draw_plan(p, n, 15, 20, seed=1602)
    assert np.array_equal(plan.omega_r, gold["omega_r"]) and np.array_equal(plan.omega_c, gold["omega_c"])
    Yt = P.subsample(Y, plan, ctx=ctx)
    assert np.array_equal(Yt, gold["Yt"])
    Lrt = P.kron_reduce(gr.laplacian, plan.omega_r, 1e-11, ctx=ctx)
    Lct = P.kron_reduce(gc.laplacian, plan.omega_c, 1e-11, ctx=ctx)
    for L, name in ((Lrt, "Lrt"), (Lct, "Lct")):
        rp, ci, v = L.arrays()
        assert np.array_equal(rp, gold[name + "_rp"]) and np.array_equal(ci, gold[name + "_ci"])
        assert np.abs(v - gold[name + "_v"]).max() <= 1e-9 * np.abs(gold[name + "_v"]).max()
    g = float(np.sqrt(max(p, n)))
    Xt, tr = P.fista_solve(Yt, Lrt, Lct, P.FrpcagConfig(gamma_r=g, gamma_c=g, tol=1e-300, max_iter=60), ctx=ctx)
    assert tr.iterations == 60 and abs(tr.step - gold["step"]) <= 1e-12 * gold["step"]
    assert rel(Xt, gold["Xt"]) <= 1e-9
    # the device Kron operators agree with the oracle's to the PCG tolerance
    # (~1e-10 relative), which the penalty terms carry into the objective
    assert np.allclose(tr.objective, gold["objective"], rtol=1e-8)
    res = P.alternate_decode(gold["Xt"], plan, gr.laplacian, gc.laplacian, P.SpectralGap(lambda_k1=0.05),
                             P.SpectralGap(lambda_k1=0.07), P.DecoderConfig(1.0, 1e-10, 300), ctx=ctx)
    assert abs(res.iterations - int(gold["dec_iters"])) <= 1
    assert rel(res.X, gold["X"]) <= 1e-9


@pytest.mark.gpu
def test_device_pipeline_matches_the_fixture(gold):
    """run_pipeline (device resident, fp64) from Y to X."""
    import paper_1602_02070_b200 as P

    Y = gold["Y"]
    p, n = Y.shape
    g = float(np.sqrt(max(p, n)))
    cfg = P.PipelineConfig(knn=10, a=4, b=4, kron_pcg_tol=1e-11,
                           frpcag=P.FrpcagConfig(gamma_r=g, gamma_c=g, loss="l1", tol=1e-300, max_iter=60),
                           decoder=P.DecoderConfig(gamma=1.0, pcg_tol=1e-10, pcg_max_iter=300, variant="alternate"),
                           lambda_k1_r=0.05, lambda_k1_c=0.07, seed=1602)
    rep = P.run_pipeline(Y, cfg, ctx=P.Context(0))
    assert np.array_equal(rep.plan.omega_r, gold["omega_r"]) and np.array_equal(rep.plan.omega_c, gold["omega_c"])
    assert rel(rep.Xt, gold["Xt"]) <= 1e-9
    assert rel(rep.X, gold["X"]) <= 1e-8
