"""Writes tests/golden/cpca_small.npz: every stage of a small CPCA run
(config-0 style, 60 x 80, fp64) computed by the oracle restatement of the
reference (oracle/cpcag_oracle.cpp, pipeline.cpp:273-350 stage order), so
the oracle itself is pinned by a committed fixture and the device path is
checked against the same bytes.  Run from the repo root:
    python tests/golden/make_pipeline_fixture.py"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle import pyoracle as O  # noqa: E402
from paper_1602_02070_b200.workloads import config0  # noqa: E402


def stages(Y=None):
    """Every stage from Y (default: the config-0 generator's 60 x 80 input;
    the committed fixture keeps its own Y, so it does not depend on the
    generator)."""
    if Y is None:
        Y, _ = config0(seed=1602, small=True)  # 60 x 80, rank 5 on circle-manifold kNN graphs + 5 % outliers
    p, n = Y.shape
    gr = O.build_knn_graph(Y, True, 10)
    gc = O.build_knn_graph(Y, False, 10)
    plan = O.draw_plan(p, n, 15, 20, seed=1602)
    Yt = O.subsample(Y, plan)
    Lrt = O.kron_reduce(gr.laplacian, plan.omega_r, 1e-11)
    Lct = O.kron_reduce(gc.laplacian, plan.omega_c, 1e-11)
    g = float(np.sqrt(max(p, n)))
    Xt, tr = O.fista_solve(Yt, Lrt, Lct, O.FrpcagConfig(g, g, "l1", 1e-300, 60))
    dec = O.alternate_decode(Xt, plan, gr.laplacian, gc.laplacian, 0.05, 0.07, 1.0, 1e-10, 300)
    out = dict(Y=Y, omega_r=plan.omega_r, omega_c=plan.omega_c, Yt=Yt, sigma2_r=gr.sigma2, sigma2_c=gc.sigma2,
               Xt=Xt, objective=np.asarray(tr.objective), step=tr.step, X=dec.X, dec_iters=dec.iterations)
    for name, L in (("Lr", gr.laplacian), ("Lc", gc.laplacian), ("Lrt", Lrt), ("Lct", Lct)):
        rp, ci, v = L.arrays()
        out[name + "_rp"], out[name + "_ci"], out[name + "_v"] = rp, ci, v
    return out


if __name__ == "__main__":
    np.savez_compressed(os.path.join(os.path.dirname(os.path.abspath(__file__)), "cpca_small.npz"), **stages())
