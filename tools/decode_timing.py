"""Decoder timing on the GPU (diagnostic): cfg3 (4096 x 200000, 100 CG
iterations) and the cfg1 decoder (10304 x 1000, 200 iterations) per precision
mode, with the per-kernel device time split (live CUDA events)."""
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
ctx.reserve(60 << 30)
which = sys.argv[1:] or ["cfg3", "cfg1"]


def timed(fn, reps=2):
    fn()
    torch.cuda.synchronize()
    ctx.reset_kernel_timing()
    ctx.enable_kernel_timing(True)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(stream)
    for _ in range(reps):
        r = fn()
    b.record(stream)
    torch.cuda.synchronize()
    ctx.enable_kernel_timing(False)
    kt = ctx.kernel_times()
    return a.elapsed_time(b) / reps, {k: (v[0] // reps, round(v[1] / reps, 3)) for k, v in kt.items()}, r


if "cfg3" in which:
    Pr, Pc = workloads.config3_points()
    p, n = Pr.shape[1], Pc.shape[1]
    gr = P.build_knn_graph(torch.tensor(np.ascontiguousarray(Pr.T), device="cuda").t(), "cols", 10, ctx=ctx)
    gc = P.build_knn_graph(torch.tensor(np.ascontiguousarray(Pc.T), device="cuda").t(), "cols", 10, ctx=ctx)
    plan = P.draw_plan(p, n, p // 8, n // 8, seed=1607)
    Xt = workloads.config3_rhs(P, gr.laplacian, gc.laplacian, plan, ctx)
    g1 = P.SpectralGap(lambda_k1=1.0)
    out = {}
    variants = [("f32/krylov64", Xt.float().t().contiguous().t(), "fp64"),
                ("f32/krylov32", Xt.float().t().contiguous().t(), "fp32"),
                ("f64", Xt, "fp64")]
    only = os.environ.get("VARIANTS")
    if only:
        variants = [v for v in variants if v[0] in only.split(",")]
    for name, xt, kp in variants:
        cfg = P.DecoderConfig(1.0, 1e-30, 100, krylov_precision=kp)
        ms, kt, r = timed(lambda: P.alternate_decode(xt, plan, gr.laplacian, gc.laplacian, g1, g1, cfg, ctx=ctx))
        out[name] = r.X.double()
        print(f"cfg3 {name}: {ms:.1f} ms ({ms / 100:.2f} ms/it) kernels {kt}", flush=True)
        del r
    for k in ("f32/krylov64", "f32/krylov32"):
        if k not in out or "f64" not in out:
            continue
        d = float(torch.linalg.norm(out[k] - out["f64"]) / torch.linalg.norm(out["f64"]))
        print(f"cfg3 {k} vs f64: {d:.3e}", flush=True)
    del out, gr, gc, Xt
    torch.cuda.empty_cache()

if "cfg1" in which:
    wl = workloads.config1()
    Y = torch.tensor(np.ascontiguousarray(wl.Y.T), dtype=torch.float32, device="cuda").t()
    gc = P.build_knn_graph(Y, "cols", 10, ctx=ctx)
    Wr = P.SparseMatrix.from_scipy(wl.W_r, ctx=ctx)
    gr = P.graph_from_adjacency(Wr, ctx=ctx)
    p, n = wl.Y.shape
    plan = P.draw_plan(p, n, -(-p // 10), -(-n // 10), seed=1603)
    Xt = P.subsample(Y, plan, ctx=ctx)
    paths = os.environ.get("PATHS", "auto").split(",")
    for kp in ("fp64", "fp32"):
        for path in paths:
            ctx.set_apply_path(path)
            cfg = P.DecoderConfig(1.0, 1e-30, 200, krylov_precision=kp)
            ms, kt, r = timed(lambda: P.alternate_decode(Xt, plan, gr.laplacian, gc.laplacian,
                                                         P.SpectralGap(lambda_k1=wl.lambda_k1_r),
                                                         P.SpectralGap(lambda_k1=wl.lambda_k1_c), cfg, ctx=ctx), reps=5)
            print(f"cfg1 decode krylov {kp} path {path} ({ctx.last_apply_path()}): {ms:.2f} ms kernels {kt}",
                  flush=True)
    ctx.set_apply_path("auto")
