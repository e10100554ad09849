"""A few decoder iterations of config 1 or 3 (for ncu captures)."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1602_02070_b200 as P  # noqa: E402
from paper_1602_02070_b200 import workloads  # noqa: E402

cfgname, kp, its = sys.argv[1], sys.argv[2], int(sys.argv[3])
ctx = P.Context(0)
ctx.set_stream(torch.cuda.current_stream().cuda_stream)
if cfgname == "cfg1":
    wl = workloads.config1()
    Y = torch.tensor(np.ascontiguousarray(wl.Y.T), dtype=torch.float32, device="cuda").t()
    gc = P.build_knn_graph(Y, "cols", 10, ctx=ctx)
    gr = P.graph_from_adjacency(P.SparseMatrix.from_scipy(wl.W_r, ctx=ctx), ctx=ctx)
    p, n = wl.Y.shape
    plan = P.draw_plan(p, n, -(-p // 10), -(-n // 10), seed=1603)
    Xt = P.subsample(Y, plan, ctx=ctx)
else:
    Pr, Pc = workloads.config3_points()
    p, n = Pr.shape[1], Pc.shape[1]
    gr = P.build_knn_graph(torch.tensor(np.ascontiguousarray(Pr.T), device="cuda").t(), "cols", 10, ctx=ctx)
    gc = P.build_knn_graph(torch.tensor(np.ascontiguousarray(Pc.T), device="cuda").t(), "cols", 10, ctx=ctx)
    plan = P.draw_plan(p, n, p // 8, n // 8, seed=1607)
    Xt = workloads.config3_rhs(P, gr.laplacian, gc.laplacian, plan, ctx).float().t().contiguous().t()
g1 = P.SpectralGap(lambda_k1=1.0)
r = P.alternate_decode(Xt, plan, gr.laplacian, gc.laplacian, g1, g1, P.DecoderConfig(1.0, 1e-30, its, krylov_precision=kp),
                       ctx=ctx)
torch.cuda.synchronize()
print("ok", r.iterations)
