"""FISTA diagnostics: persistent vs per-kernel path (error vs oracle, time)."""
import os, sys, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
from helpers import knn_laplacian, rel, to_device
from oracle import pyoracle as O
import paper_1602_02070_b200 as P

ctx = P.Context(0)

def reduced(p, n, rr, rc, seed, K=10):
    Lr_full, Lc_full = knn_laplacian(p, 3, K, seed), knn_laplacian(n, 3, K, seed + 1)
    plan = O.draw_plan(p, n, rr, rc, seed=seed)
    return O.kron_reduce(Lr_full, plan.omega_r, 1e-11), O.kron_reduce(Lc_full, plan.omega_c, 1e-11)

def run(Y, dLr, dLc, g, its, persist):
    os.environ["CPCAG_FISTA_PERSIST"] = "1" if persist else "0"
    cfg = P.FrpcagConfig(gamma_r=g, gamma_c=g, loss="l1", tol=1e-300, max_iter=its)
    P.fista_solve(Y, dLr, dLc, cfg, ctx=ctx)
    ctx.enable_kernel_timing(True); ctx.reset_kernel_timing()
    t = time.perf_counter()
    X, tr = P.fista_solve(Y, dLr, dLc, cfg, ctx=ctx)
    t = time.perf_counter() - t
    kt = ctx.kernel_times(); ctx.enable_kernel_timing(False)
    return X, tr, t, kt

for (p, n, rr, rc, g, its) in [(400, 300, 101, 60, 8.0, 150), (300, 240, 75, 60, 8.0, 150)]:
    Lr, Lc = reduced(p, n, rr, rc, 40 + rr)
    Y = (np.random.default_rng(rr).standard_normal((rr, rc)) * 4.0).astype(np.float32)
    Xo, tro = O.fista_solve(Y.astype(np.float64), Lr, Lc, O.FrpcagConfig(g, g, "l1", 1e-300, its))
    dLr, dLc = to_device(ctx, Lr), to_device(ctx, Lc)
    for persist in (1, 0):
        X, tr, t, kt = run(Y, dLr, dLc, g, its, persist)
        print(f"shape {rr}x{rc} persist={persist} rel={rel(X, Xo):.3e} objrel={abs(tr.objective[-1]-tro.objective[-1])/abs(tro.objective[-1]):.2e} wall={t*1e3:.2f}ms {kt}")
    # fp64 Y through the oracle but with fp32-rounded operators: noise floor
# cfg1-sized timing: dense 1031 x 100
rs = np.random.default_rng(0)
from paper_1602_02070_b200 import workloads
for its in (1, 10, 300):
    for persist in (1, 0):
        Lr, Lc = reduced(4000, 1000, 1031, 100, 3, K=10) if its == 1 and persist == 1 else (Lr, Lc)
        dLr, dLc = to_device(ctx, Lr), to_device(ctx, Lc)
        Y = (rs.standard_normal((1031, 100)) * 50).astype(np.float32)
        X, tr, t, kt = run(Y, dLr, dLc, 101.5, its, persist)
        print(f"1031x100 nnz {Lr.nnz},{Lc.nnz} its={its} persist={persist} wall={t*1e3:.2f}ms {kt}")
