"""Debug: determinism + sampled-entry check of the column-block apply at cfg3 size."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1602_02070_b200 as P
from paper_1602_02070_b200 import _native as N, workloads
from paper_1602_02070_b200.sharded import CudaBlockBackend

prec = sys.argv[1]
Pr, Pc = workloads.config3_points()
p, n = Pr.shape[1], Pc.shape[1]
ctx = P.Context(0)
ctx.set_stream(torch.cuda.current_stream().cuda_stream)
gr = P.build_knn_graph(torch.tensor(np.ascontiguousarray(Pr.T), device="cuda").t(), "cols", 10, ctx=ctx)
gc = P.build_knn_graph(torch.tensor(np.ascontiguousarray(Pc.T), device="cuda").t(), "cols", 10, ctx=ctx)
plan = P.draw_plan(p, n, p // 8, n // 8, seed=1607)
dt = torch.float32 if prec == "f32" else torch.float64
be = CudaBlockBackend(ctx, N.F32 if prec == "f32" else N.F64, plan, gr.laplacian, gc.laplacian, 1.0, 1.0, 0, n)
g = torch.Generator(device="cuda").manual_seed(3)
Pv = torch.randn(p * n, device="cuda", generator=g, dtype=dt)
rp, ci, v = gc.laplacian.arrays(); rpr, cir, vr = gr.laplacian.arrays()
rs = np.zeros(p, bool); rs[np.asarray(plan.omega_r)] = True
cs = np.zeros(n, bool); cs[np.asarray(plan.omega_c)] = True
rng = np.random.default_rng(1)
ent = [(int(i), int(c)) for i, c in zip(rng.integers(0, p, 300), rng.integers(0, n, 300))]
deg = np.diff(rpr)
hub = np.argsort(-deg)[:5]
ent += [(int(i), int(c)) for i in hub for c in rng.integers(0, n, 20)]
M = Pv.view(n, p)
outs = []
for k in range(3):
    AP = torch.zeros(p * n, device="cuda", dtype=dt)
    cv = be.apply(Pv, AP)
    torch.cuda.synchronize()
    outs.append(AP)
    print("call", k, "curv", cv, "dot", float((Pv.double() * AP.double()).sum()))
print("equal 0-1", torch.equal(outs[0], outs[1]), "1-2", torch.equal(outs[1], outs[2]))
d = (outs[0] != outs[1]).nonzero().flatten()
print("diff entries", int(d.numel()), "rows", torch.unique(d % p)[:10].tolist())
print("max deg_r", int(deg.max()), "hubs", hub.tolist(), deg[hub].tolist())
worst = 0.0
badl = []
for (i, c) in ent:
    x1 = sum(float(v[t]) * float(M[int(ci[t]), i]) for t in range(rp[c], rp[c + 1]))
    x2 = sum(float(vr[t]) * float(M[c, int(cir[t])]) for t in range(rpr[i], rpr[i + 1]))
    want = x1 + x2 + (float(M[c, i]) if rs[i] and cs[c] else 0.0)
    for k in range(3):
        got = float(outs[k][c * p + i])
        e = abs(got - want) / (abs(want) + 1e-3)
        if e > 1e-4:
            badl.append((k, i, c, got, want, int(deg[i])))
        worst = max(worst, e)
print("sampled worst rel", worst, "bad", len(badl), badl[:6])
