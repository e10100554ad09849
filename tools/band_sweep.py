"""Sweep the band-apply variants (CPCAG_BAND_V, CPCAG_BAND_NT, CPCAG_BAND_RB)
on the config-3 decoder operator (4096 x 200000 fp32): per-kernel device
times over a short fixed-iteration decode, and the max difference of X
against the first variant."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1602_02070_b200 as P  # noqa: E402
from paper_1602_02070_b200 import workloads  # noqa: E402

iters = int(os.environ.get("SWEEP_ITERS", "20"))
Pr, Pc = workloads.config3_points()
p, n = Pr.shape[1], Pc.shape[1]
ctx = P.Context(0)
ctx.set_stream(torch.cuda.current_stream().cuda_stream)
gr = P.build_knn_graph(torch.tensor(np.ascontiguousarray(Pr.T), device="cuda").t(), "cols", 10, ctx=ctx)
gc = P.build_knn_graph(torch.tensor(np.ascontiguousarray(Pc.T), device="cuda").t(), "cols", 10, ctx=ctx)
plan = P.draw_plan(p, n, p // 8, n // 8, seed=1607)
rs = np.random.default_rng(3)
Xt = torch.tensor(rs.standard_normal((p // 8, n // 8)), dtype=torch.float32, device="cuda").t().contiguous().t()
g1 = P.SpectralGap(lambda_k1=1.0)
variants = [v.split(",") for v in sys.argv[1:]] or [["1", "1024", "32", "1"]]
ref = None
for v, nt, rb, perm in variants:
    os.environ["CPCAG_BAND_V"], os.environ["CPCAG_BAND_NT"], os.environ["CPCAG_BAND_RB"] = v, nt, rb
    os.environ["CPCAG_BAND_PERM"] = perm
    ctx.enable_kernel_timing(True)
    ctx.reset_kernel_timing()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    res = P.alternate_decode(Xt, plan, gr.laplacian, gc.laplacian, g1, g1, P.DecoderConfig(1.0, 1e-30, iters), ctx=ctx)
    torch.cuda.synchronize()
    wall = (time.perf_counter() - t0) * 1e3
    kt = ctx.kernel_times()
    ctx.enable_kernel_timing(False)
    X = torch.as_tensor(res.X).float().cpu() if not isinstance(res.X, np.ndarray) else torch.from_numpy(res.X)
    if ref is None:
        ref = X
    d = float((X - ref).abs().max()) / float(ref.abs().max())
    real = res.iterations + 1  # launches that did work (the rest exit on the done flag)
    ks = "  ".join(f"{k}={t / real:.3f}ms" for k, (c, t) in sorted(kt.items()) if k.startswith("cg_apply"))
    print(f"V={v} NT={nt} RB={rb} perm={perm}: wall {wall:8.1f} ms  {ks}  reldiff {d:.2e}", flush=True)
