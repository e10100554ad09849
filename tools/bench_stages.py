"""Micro-benchmark of the config-1 decoder (apply variants) and FISTA on the
device, with per-kernel event timing.  Usage: python tools/bench_stages.py"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np
import torch

import paper_1602_02070_b200 as P
from bench import make_workload, pipeline_config


def timed(ctx, fn, reps=3):
    fn()
    torch.cuda.synchronize()
    ctx.reset_kernel_timing()
    ctx.kernel_timing_filter(None)
    ctx.enable_kernel_timing(True)
    t0 = time.perf_counter()
    for _ in range(reps):
        out = fn()
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    ctx.enable_kernel_timing(False)
    kt = ctx.kernel_times()
    return out, (t1 - t0) / reps * 1e3, {k: (n // reps, ms / reps) for k, (n, ms) in kt.items()}


def main():
    wl = make_workload()
    ctx = P.Context(0)
    ctx.set_stream(torch.cuda.current_stream().cuda_stream)
    Yd = torch.tensor(np.ascontiguousarray(wl.Y.T), dtype=torch.float32, device="cuda").t()
    Wr = P.SparseMatrix.from_scipy(wl.W_r, ctx=ctx)
    cfg = pipeline_config(P, wl)
    rep = P.run_pipeline(Yd, cfg, W_r=Wr, ctx=ctx)
    gr = P.graph_from_adjacency(Wr, ctx=ctx)
    gc = P.build_knn_graph(Yd, "cols", 10, ctx=ctx)
    plan = rep.plan
    dcfg = P.DecoderConfig(1.0, 1e-30, 200)
    ref = None
    for variant in ["fast2", "fast3"]:
        os.environ["CPCAG_APPLY"] = variant
        res, wall, kt = timed(ctx, lambda: P.alternate_decode(rep.Xt, plan, gr.laplacian, gc.laplacian,
                                                               P.SpectralGap(lambda_k1=wl.lambda_k1_r),
                                                               P.SpectralGap(lambda_k1=wl.lambda_k1_c), dcfg, ctx=ctx))
        X = res.X.cpu().numpy()
        if ref is None:
            ref = X
        diff = float(np.abs(X - ref).max())
        print(f"decode[{variant:6s}] wall {wall:8.2f} ms  iters {res.iterations}  maxdiff vs staged {diff:.3e}  "
              + "  ".join(f"{k}={v[1]:.2f}ms/{v[0]}" for k, v in kt.items()), flush=True)
    os.environ.pop("CPCAG_APPLY", None)
    Lrt = P.kron_reduce(gr.laplacian, plan.omega_r, 1e-11, ctx=ctx)
    Lct = P.kron_reduce(gc.laplacian, plan.omega_c, 1e-11, ctx=ctx)
    Yt = P.subsample(Yd, plan, ctx=ctx)
    fcfg = P.FrpcagConfig(wl.gamma, wl.gamma, "l1", 1e-300, 300)
    _, wall, kt = timed(ctx, lambda: P.fista_solve(Yt, Lrt, Lct, fcfg, ctx=ctx))
    print(f"fista wall {wall:8.2f} ms  " + "  ".join(f"{k}={v[1]:.2f}ms/{v[0]}" for k, v in kt.items()), flush=True)
    for nt, sl in []:
        os.environ["CPCAG_PCG_NT"] = nt
        if sl != "0":
            os.environ["CPCAG_KRON_SLICE"] = sl
        else:
            os.environ.pop("CPCAG_KRON_SLICE", None)
        _, wall, kt = timed(ctx, lambda: P.kron_reduce(gr.laplacian, plan.omega_r, 1e-11, ctx=ctx), reps=2)
        print(f"kron(rows, NT={nt}, slice={sl}) wall {wall:8.2f} ms  " + "  ".join(f"{k}={v[1]:.2f}ms/{v[0]}" for k, v in kt.items()),
              flush=True)
    os.environ.pop("CPCAG_PCG_NT", None)


if __name__ == "__main__":
    main()
