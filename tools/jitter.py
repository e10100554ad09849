"""Per-call wall time of repeated kron_reduce / alternate_decode calls on the
config-1 operators (diagnoses run-to-run jitter)."""
import gc
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1602_02070_b200 as P  # noqa: E402
from bench import make_workload, pipeline_config  # noqa: E402

if os.environ.get("JIT_NOGC"):
    gc.disable()
wl = make_workload()
ctx = P.Context(0)
if os.environ.get("JIT_RESERVE"):
    ctx.reserve(int(float(os.environ["JIT_RESERVE"]) * 2**30))
ctx.set_stream(torch.cuda.current_stream().cuda_stream)
Yd = torch.tensor(np.ascontiguousarray(wl.Y.T), dtype=torch.float32, device="cuda").t()
Wr = P.SparseMatrix.from_scipy(wl.W_r, ctx=ctx)
cfg = pipeline_config(P, wl)
rep = P.run_pipeline(Yd, cfg, W_r=Wr, ctx=ctx)
gr = P.graph_from_adjacency(Wr, ctx=ctx)
ts = []
for _ in range(int(os.environ.get("JIT_N", "30"))):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    P.kron_reduce(gr.laplacian, rep.plan.omega_r, 1e-11, ctx=ctx)
    torch.cuda.synchronize()
    ts.append((time.perf_counter() - t0) * 1e3)
print("kron ms", [round(t, 1) for t in ts], flush=True)

flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
for use_flush in ((False,) if os.environ.get("JIT_ONE") else (False, True)):
    ts, st = [], []
    for _ in range(int(os.environ.get("JIT_N", "20"))):
        if use_flush:
            flush.zero_()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r = P.run_pipeline(Yd, cfg, W_r=Wr, ctx=ctx)
        torch.cuda.synchronize()
        ts.append((time.perf_counter() - t0) * 1e3)
        st.append({k: round(v) for k, v in r.stages.items() if v > 1})
    print(f"pipeline flush={use_flush} ms", [round(t, 1) for t in ts], flush=True)
    worst = int(np.argmax(ts))
    print("  worst stages", st[worst], "median stages", st[len(st) // 2], flush=True)
