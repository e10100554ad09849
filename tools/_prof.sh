CPCAG_TRACE=1 python - <<'PY' 2>&1 | tail -40
import os, sys, time
sys.path.insert(0, '.')
import numpy as np, torch
import paper_1602_02070_b200 as P
from bench import make_workload, pipeline_config
wl = make_workload()
ctx = P.Context(0)
Yd = torch.tensor(np.ascontiguousarray(wl.Y.T), dtype=torch.float32, device="cuda").t()
Wr = P.SparseMatrix.from_scipy(wl.W_r, ctx=ctx)
gr = P.graph_from_adjacency(Wr, ctx=ctx)
plan = P.draw_plan(10304, 1000, 1031, 100, seed=1603)
for k in range(3):
    t = time.perf_counter(); R = P.kron_reduce(gr.laplacian, plan.omega_r, 1e-11, ctx=ctx); print("kron wall", (time.perf_counter()-t)*1e3, "ms", file=sys.stderr)
PY
