"""Timing of the column-sharded FISTA (emulated ranks on one GPU) beside the
one-GPU fista_solve at the config-1 compressed size (1031 x 100, 300 it)."""
import sys
import time

import numpy as np

sys.path.insert(0, "tests")
sys.path.insert(0, ".")
import paper_1602_02070_b200 as P
from helpers import knn_laplacian, rel, to_device
from paper_1602_02070_b200.sharded import fista_solve_sharded_emulated

ctx = P.Context(0)
r, c = 1031, 100
Lr, Lc = knn_laplacian(r, 3, 8, 1), knn_laplacian(c, 3, 8, 2)
dLr, dLc = to_device(ctx, Lr), to_device(ctx, Lc)
Y = np.random.default_rng(0).standard_normal((r, c)).astype(np.float32)
cfg = P.FrpcagConfig(gamma_r=2.0, gamma_c=2.0, tol=1e-300, max_iter=300, step=0.01)


def timed(f, n=3):
    f()
    t = []
    for _ in range(n):
        t0 = time.perf_counter()
        out = f()
        t.append(time.perf_counter() - t0)
    return min(t) * 1e3, out


ms1, (X1, _) = timed(lambda: P.fista_solve(Y, dLr, dLc, cfg, ctx=ctx))
print(f"one-GPU fista_solve: {ms1:.2f} ms")
for G in (1, 2, 4, 8):
    ms, (X, tr) = timed(lambda: fista_solve_sharded_emulated(Y, dLr, dLc, cfg, G, ctx=ctx))
    print(f"sharded emulated G={G}: {ms:.2f} ms (all ranks serialised on one GPU), rel vs one-GPU {rel(X, X1):.2e}, it {tr.iterations}")
