"""Runs the config-1 pipeline N times with CPCAG_TRACE marks and prints the
slowest regions (diagnostic for step-time outliers)."""
import os
import re
import subprocess
import sys

if os.environ.get("STALL_CHILD"):
    ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, ROOT)
    import numpy as np
    import torch

    import paper_1602_02070_b200 as P
    from bench import make_workload, pipeline_config

    wl = make_workload()
    ctx = P.Context(0)
    stream = torch.cuda.current_stream()
    ctx.set_stream(stream.cuda_stream)
    ctx.reserve(8 << 30)
    Yd = torch.tensor(np.ascontiguousarray(wl.Y.T), dtype=torch.float32, device="cuda").t()
    Wr = P.SparseMatrix.from_scipy(wl.W_r, ctx=ctx)
    cfg = pipeline_config(P, wl, "fp32")
    import time
    for k in range(int(os.environ.get("N", "12"))):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        print(f"=== run {k}", file=sys.stderr, flush=True)
        P.run_pipeline(Yd, cfg, W_r=Wr, ctx=ctx)
        torch.cuda.synchronize()
        print(f"=== run {k} wall {(time.perf_counter() - t0) * 1e3:.2f} ms", file=sys.stderr, flush=True)
else:
    env = dict(os.environ, STALL_CHILD="1", CPCAG_TRACE="1")
    out = subprocess.run([sys.executable, __file__], env=env, capture_output=True, text=True).stderr
    runs, cur = [], None
    for ln in out.splitlines():
        m = re.match(r"=== run (\d+) wall ([\d.]+)", ln)
        if m:
            runs.append((float(m.group(2)), cur))
            cur = None
        elif ln.startswith("=== run"):
            cur = []
        elif cur is not None and "[cpcag trace]" in ln:
            cur.append(ln)
    for wall, lines in runs:
        print(f"run wall {wall:.2f} ms")
    wall, lines = max(runs[1:], key=lambda r: r[0])
    print("slowest run", wall)
    for ln in lines:
        print("  ", ln)
    print(out[-2000:] if not runs else "")
