"""bench.py's multi-GPU blocks (sharded cfg3 decoder, sharded cfg1 FRPCAG)
exercised at world size 1 over NCCL -- one GPU is all this pool grants."""
import json
import os
import sys

sys.path.insert(0, ".")
os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
os.environ.setdefault("MASTER_PORT", "29533")
import numpy as np
import torch
import torch.distributed as dist

import bench
import paper_1602_02070_b200 as P

torch.cuda.set_device(0)
dist.init_process_group("nccl", rank=0, world_size=1)
wl = bench.make_workload()
ctx = P.Context(0)
ctx.set_stream(torch.cuda.current_stream().cuda_stream)
ctx.reserve(8 << 30)
Yd = torch.tensor(np.ascontiguousarray(wl.Y.T), dtype=torch.float32, device="cuda").t()
Wr_dev = P.SparseMatrix.from_scipy(wl.W_r, ctx=ctx)
cfg = bench.pipeline_config(P, wl)
gc = P.build_knn_graph(Yd, "cols", 10, ctx=ctx)
rep = P.run_pipeline(Yd, cfg, W_r=Wr_dev, ctx=ctx)
blk = bench.frpcag_sharded_block(P, ctx, torch, dist, wl, Yd, Wr_dev, gc, rep.plan, cfg, 0, 1)
blk["pipeline_solve_ms_one_gpu"] = rep.solve_ms if hasattr(rep, "solve_ms") else None
print(json.dumps(blk))
dist.destroy_process_group()
