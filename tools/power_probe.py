"""Times the two FRPCAG power iterations of config 1 (frpcag.cpp:72-73) alone
and as the concurrent pair (diagnostic)."""
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1602_02070_b200 as P  # noqa: E402
from paper_1602_02070_b200 import workloads  # noqa: E402

ctx = P.Context(0)
stream = torch.cuda.current_stream()
ctx.set_stream(stream.cuda_stream)
wl = workloads.config1()
Y = torch.tensor(np.ascontiguousarray(wl.Y.T), dtype=torch.float32, device="cuda").t()
gc = P.build_knn_graph(Y, "cols", 10, ctx=ctx)
gr = P.graph_from_adjacency(P.SparseMatrix.from_scipy(wl.W_r, ctx=ctx), ctx=ctx)
p, n = wl.Y.shape
plan = P.draw_plan(p, n, -(-p // 10), -(-n // 10), seed=1603)
Lr = P.kron_reduce(gr.laplacian, plan.omega_r, 1e-11, ctx=ctx)
Lc = P.kron_reduce(gc.laplacian, plan.omega_c, 1e-11, ctx=ctx)
print("Lr", Lr.rows(), Lr.nonzeros(), "Lc", Lc.rows(), Lc.nonzeros())


def t(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        r = fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps * 1e3, r


for name, L in [("Lr", Lr), ("Lc", Lc)]:
    ms, est = t(lambda: P.power_iteration_norm(L, 1e-7, 42, ctx=ctx))
    print(f"power {name}: {ms:.2f} ms est {est:.12g}")
Yt = P.subsample(Y, plan, ctx=ctx)
cfg = P.FrpcagConfig(gamma_r=wl.gamma, gamma_c=wl.gamma, loss="l1", tol=1e-300, max_iter=1)
ms, _ = t(lambda: P.fista_solve(Yt, Lr, Lc, cfg, ctx=ctx))
print(f"fista 1 iteration incl. both norms: {ms:.2f} ms")
