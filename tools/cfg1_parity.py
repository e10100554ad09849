"""Config-1 parity diagnostics at the full iteration counts: the fp32 device
stages against the fp64 oracle composite (relative Frobenius errors), FISTA
through each device path and the decoder on the oracle's Xt."""
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from helpers import rel, to_device  # noqa: E402
from oracle import pyoracle as O  # noqa: E402

import paper_1602_02070_b200 as P  # noqa: E402
from paper_1602_02070_b200 import workloads  # noqa: E402

wl = workloads.config1()
p, n = wl.Y.shape
ctx = P.Context(0)
Y = wl.Y.astype(np.float32).astype(np.float64)
t0 = time.time()
gr = O.graph_from_adjacency(O.Csr.from_scipy(wl.W_r))
gc = O.build_knn_graph(Y, False, 10)
plan = O.draw_plan(p, n, -(-p // wl.b), -(-n // wl.a), seed=1603)
Yt = O.subsample(Y, plan)
Lrt = O.kron_reduce(gr.laplacian, plan.omega_r, 1e-11)
Lct = O.kron_reduce(gc.laplacian, plan.omega_c, 1e-11)
its = int(os.environ.get("ITS", "300"))
Xt, tr = O.fista_solve(Yt, Lrt, Lct, O.FrpcagConfig(wl.gamma, wl.gamma, "l1", 1e-300, its))
print(f"oracle FISTA done {time.time() - t0:.1f}s", flush=True)
dLr, dLc = to_device(ctx, Lrt), to_device(ctx, Lct)
for mode in ["persist", "perkernel"]:
    os.environ["CPCAG_FISTA_PERSIST"] = "1" if mode == "persist" else "0"
    for prec in (np.float32, np.float64):
        X, trd = P.fista_solve(Yt.astype(prec), dLr, dLc, P.FrpcagConfig(gamma_r=wl.gamma, gamma_c=wl.gamma, tol=1e-300,
                                                                      max_iter=its), ctx=ctx)
        print(f"FISTA {mode} {np.dtype(prec).name}: rel {rel(X, Xt):.3e}", flush=True)
os.environ["CPCAG_FISTA_PERSIST"] = "1"
cg = int(os.environ.get("CG", "200"))
dec = O.alternate_decode(Xt, plan, gr.laplacian, gc.laplacian, wl.lambda_k1_r, wl.lambda_k1_c, 1.0, 1e-30, cg)
print(f"oracle decoder done {time.time() - t0:.1f}s", flush=True)
pl = P.SamplingPlan(plan.omega_r, plan.omega_c, p, n)
for prec in (np.float32, np.float64):
    r = P.alternate_decode(Xt.astype(prec), pl, to_device(ctx, gr.laplacian), to_device(ctx, gc.laplacian),
                           P.SpectralGap(lambda_k1=wl.lambda_k1_r), P.SpectralGap(lambda_k1=wl.lambda_k1_c),
                           P.DecoderConfig(1.0, 1e-30, cg), ctx=ctx)
    print(f"decoder {np.dtype(prec).name} on the oracle's Xt: rel {rel(r.X, dec.X):.3e}", flush=True)
