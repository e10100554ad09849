"""Config-4 feasibility probe (diagnostic): the 10^6 x 64 kNN graph through
the tensor-core path, and a few decoder iterations at 4096 x 10^6."""
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
ctx.set_stream(torch.cuda.current_stream().cuda_stream)
Pr, Pc = workloads.config3_points(n=1_000_000)
t0 = time.time()
gr = P.build_knn_graph(torch.tensor(np.ascontiguousarray(Pr.T), device="cuda").t(), "cols", 10, ctx=ctx)
torch.cuda.synchronize()
print(f"row graph {time.time() - t0:.2f}s", flush=True)
ctx.reset_kernel_timing()
ctx.enable_kernel_timing(True)
t0 = time.time()
gc = P.build_knn_graph(torch.tensor(np.ascontiguousarray(Pc.T), device="cuda").t(), "cols", 10, ctx=ctx)
torch.cuda.synchronize()
ctx.enable_kernel_timing(False)
print(f"column graph 1e6 x 64: {time.time() - t0:.2f}s nnz {gc.laplacian.nonzeros()} kernels {ctx.kernel_times()}",
      flush=True)
plan = P.draw_plan(4096, 1_000_000, 1024, 50_000, seed=1608)
t0 = time.time()
Lk = P.kron_reduce(gc.laplacian, plan.omega_c[:256], 1e-11, ctx=ctx)
torch.cuda.synchronize()
print(f"kron 256 of 50000 kept nodes: {time.time() - t0:.2f}s", flush=True)
Xt = workloads.config3_rhs(P, gr.laplacian, gc.laplacian, P.draw_plan(4096, 1_000_000, 1024, 50_000, seed=1608), ctx)
Xt = Xt.float().t().contiguous().t()
g1 = P.SpectralGap(lambda_k1=1.0)
for kp in ("fp32", "fp64"):
    torch.cuda.synchronize()
    t0 = time.time()
    r = P.alternate_decode(Xt, plan, gr.laplacian, gc.laplacian, g1, g1, P.DecoderConfig(1.0, 1e-30, 5, krylov_precision=kp),
                           ctx=ctx)
    torch.cuda.synchronize()
    print(f"decoder 4096 x 1e6, 5 iterations, krylov {kp}: {time.time() - t0:.2f}s", flush=True)
    del r
    torch.cuda.empty_cache()
print(f"max memory allocated by torch {torch.cuda.max_memory_allocated() / 1e9:.1f} GB")
