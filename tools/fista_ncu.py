"""One cfg1-sized fp32 dense FISTA solve (1031 x 100, 300 iterations) for ncu:
launch 1 is a 1-iteration warm-up, launch 2 the measured solve."""
import os, sys
import numpy as np
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, root); sys.path.insert(0, os.path.join(root, "tests"))
from helpers import knn_laplacian, to_device
from oracle import pyoracle as O
import paper_1602_02070_b200 as P

ctx = P.Context(0)
Lr_full, Lc_full = knn_laplacian(4000, 3, 10, 3), knn_laplacian(1000, 3, 10, 4)
plan = O.draw_plan(4000, 1000, 1031, 100, seed=3)
Lr, Lc = O.kron_reduce(Lr_full, plan.omega_r, 1e-11), O.kron_reduce(Lc_full, plan.omega_c, 1e-11)
dLr, dLc = to_device(ctx, Lr), to_device(ctx, Lc)
Y = (np.random.default_rng(0).standard_normal((1031, 100)) * 50).astype(
    np.float64 if os.environ.get("DT") == "f64" else np.float32)
for its in (1, int(os.environ.get("ITS", "300"))):
    cfg = P.FrpcagConfig(gamma_r=101.5, gamma_c=101.5, loss="l1", tol=1e-300, max_iter=its)
    X, tr = P.fista_solve(Y, dLr, dLc, cfg, ctx=ctx)
print("ok", tr.iterations)
