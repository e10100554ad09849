"""Config-3 decoder: fp32 vs fp64 vs a mixed-precision CG (fp32 operator
applies through the block C-ABI, fp64 iterates and recurrences in torch).
Prints the relative Frobenius distance of each to the fp64 decoder."""
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1602_02070_b200 as P  # noqa: E402
from paper_1602_02070_b200 import _native as N  # noqa: E402
from paper_1602_02070_b200 import workloads  # noqa: E402
from paper_1602_02070_b200.sharded import CudaBlockBackend  # noqa: E402

its = int(os.environ.get("ITS", "100"))
ctx = P.Context(0)
ctx.set_stream(torch.cuda.current_stream().cuda_stream)
ctx.reserve(48 << 30)
Pr, Pc = workloads.config3_points()
p, n = Pr.shape[1], Pc.shape[1]
gr = P.build_knn_graph(torch.tensor(np.ascontiguousarray(Pr.T), device="cuda").t(), "cols", 10, ctx=ctx)
gc = P.build_knn_graph(torch.tensor(np.ascontiguousarray(Pc.T), device="cuda").t(), "cols", 10, ctx=ctx)
plan = P.draw_plan(p, n, p // 8, n // 8, seed=1607)
rs = np.random.default_rng(1606)


def lowpass(L, m, k=20, sweeps=20):
    nrm = P.power_iteration_norm(L, 1e-7, 42, ctx=ctx)
    B = torch.tensor(rs.standard_normal((m, k)), device="cuda")
    for _ in range(sweeps):
        B = B - L.multiply(B) / nrm
    return torch.linalg.qr(B)[0]


Br, Bc = lowpass(gr.laplacian, p), lowpass(gc.laplacian, n)
A = torch.tensor(rs.standard_normal((20, 20)), device="cuda")
Xt = (Br[torch.tensor(plan.omega_r, device="cuda")] @ A @ Bc[torch.tensor(plan.omega_c, device="cuda")].T)
Xt64 = Xt.t().contiguous().t()
g1 = P.SpectralGap(lambda_k1=1.0)
dcfg = P.DecoderConfig(1.0, 1e-30, its)
X64 = P.alternate_decode(Xt64, plan, gr.laplacian, gc.laplacian, g1, g1, dcfg, ctx=ctx).X
X32 = P.alternate_decode(Xt64.float().t().contiguous().t(), plan, gr.laplacian, gc.laplacian, g1, g1, dcfg, ctx=ctx).X
rel = lambda a, b: float(torch.linalg.norm(a.double() - b) / torch.linalg.norm(b))
print(f"fp32 decoder vs fp64: {rel(X32, X64):.3e}", flush=True)

# mixed: fp32 applies (block backend), fp64 vectors
be32 = CudaBlockBackend(ctx, N.F32, plan, gr.laplacian, gc.laplacian, 1.0, 1.0, 0, n)
be64 = CudaBlockBackend(ctx, N.F64, plan, gr.laplacian, gc.laplacian, 1.0, 1.0, 0, n)
B = torch.zeros(p * n, dtype=torch.float64, device="cuda")
bb = be64.rhs(Xt64, B)
X = torch.zeros_like(B)
R = B.clone()
Pv = R.clone()
AP32 = torch.zeros(p * n, dtype=torch.float32, device="cuda")
rho = float(R @ R)
t = time.time()
for it in range(its):
    P32 = Pv.float()
    be32.apply(P32, AP32)
    AP = AP32.double()
    curv = float(Pv @ AP)
    alpha = rho / curv
    X += alpha * Pv
    R -= alpha * AP
    rho_n = float(R @ R)
    Pv = R + (rho_n / rho) * Pv
    rho = rho_n
torch.cuda.synchronize()
Xm = X.view(n, p).t()
print(f"mixed (fp32 apply, fp64 vectors) vs fp64: {rel(Xm, X64):.3e}  ({time.time() - t:.1f}s)", flush=True)
be32.close()
be64.close()
