"""One config-1 CPCA step between cudaProfilerStart/Stop, for ncu
(`ncu --profile-from-start off ...`).  Warm-up runs happen before the
profiled range so only the steady-state launches are captured."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np
import torch

import paper_1602_02070_b200 as P
from bench import make_workload, pipeline_config


def main():
    fp64 = "--fp64" in sys.argv
    wl = make_workload()
    ctx = P.Context(0)
    stream = torch.cuda.current_stream()
    ctx.set_stream(stream.cuda_stream)
    tdt = torch.float64 if fp64 else torch.float32
    Yd = torch.tensor(np.ascontiguousarray(wl.Y.T), dtype=tdt, device="cuda").t()
    Wr = P.SparseMatrix.from_scipy(wl.W_r, ctx=ctx)
    cfg = pipeline_config(P, wl, "fp64" if fp64 else "fp32")  # the bench step's decoder precision
    P.run_pipeline(Yd, cfg, W_r=Wr, ctx=ctx)
    torch.cuda.synchronize()
    torch.cuda.profiler.start()
    rep = P.run_pipeline(Yd, cfg, W_r=Wr, ctx=ctx)
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
    print("profiled step:", {k: round(v, 3) for k, v in rep.stages.items()}, "launches", ctx.launch_count)


if __name__ == "__main__":
    main()
