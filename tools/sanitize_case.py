"""Small cases covering every kernel family for compute-sanitizer runs
(memcheck / racecheck / synccheck / initcheck): the smoke pipeline (kNN,
Kron, fp64 FISTA, decoder), the fp32 persistent FISTA, the decoder's fused
and two-pass operators (band in shared memory and in L2, register row groups
with lockstep stripes), the emulated 3-rank sharded decoder, and the
tensor-core kNN filter (n >= 4096)."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import paper_1602_02070_b200 as P  # noqa: E402
from helpers import knn_laplacian, to_device  # noqa: E402
from oracle import pyoracle as O  # noqa: E402
from paper_1602_02070_b200.sharded import alternate_decode_sharded_emulated  # noqa: E402
from smoke_case import run_smoke  # noqa: E402

run_smoke()
ctx = P.Context(0)
# decoder: both operator paths, fp64 and fp32 data
for path in ("fused", "split"):
    ctx.set_apply_path(path)
    for (p, n, seed) in ((150, 120, 3), (64, 1700, 4)):
        Lr, Lc = knn_laplacian(p, 24, 10, seed), knn_laplacian(n, 3, 7, seed + 1)
        plan = O.draw_plan(p, n, p // 4, n // 4, seed=seed)
        Xt = np.random.default_rng(seed).standard_normal((p // 4, n // 4))
        pl = P.SamplingPlan(plan.omega_r, plan.omega_c, plan.p, plan.n)
        g = P.SpectralGap(lambda_k1=0.5)
        for dt in (np.float64, np.float32):
            P.alternate_decode(Xt.astype(dt), pl, to_device(ctx, Lr), to_device(ctx, Lc), g, g,
                               P.DecoderConfig(1.0, 1e-12, 12), ctx=ctx)
ctx.set_apply_path("auto")
# sharded (3 ranks emulated, uneven blocks)
Lr, Lc = knn_laplacian(90, 3, 6, 9), knn_laplacian(70, 3, 6, 10)
plan = O.draw_plan(90, 70, 20, 15, seed=9)
pl = P.SamplingPlan(plan.omega_r, plan.omega_c, plan.p, plan.n)
g = P.SpectralGap(lambda_k1=0.5)
alternate_decode_sharded_emulated(np.ones((20, 15)), pl, to_device(ctx, Lr), to_device(ctx, Lc), g, g,
                                  P.DecoderConfig(1.0, 1e-12, 10), 3, bounds=np.array([0, 5, 40, 70]), ctx=ctx)
# fp32 FISTA (persistent kernel)
from paper_1602_02070_b200 import workloads  # noqa: E402

Y = np.random.default_rng(2).standard_normal((100, 60)).astype(np.float32)
Lrt = O.kron_reduce(knn_laplacian(400, 3, 8, 5), list(range(0, 400, 4)), 1e-11)
Lct = O.kron_reduce(knn_laplacian(300, 3, 8, 6), list(range(0, 300, 5)), 1e-11)
P.fista_solve(Y, to_device(ctx, Lrt), to_device(ctx, Lct), P.FrpcagConfig(tol=1e-300, max_iter=20), ctx=ctx)
# tensor-core kNN filter
X = workloads.config2_points(n=4608, d=64)
P.knn(X, "cols", 10, ctx=ctx)
print("sanitize case: ok")
