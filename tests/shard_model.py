"""Host model of the column-sharded decoder's distributed algorithm (test
infrastructure): the CG of decoders.cpp:145-186 over column blocks, with the
halo exchange planned by the library's host code (sharded.HaloPlan ->
cpcag_halo_plan) and torch.distributed collectives.  tests/test_sharded.py
runs it over gloo (world 2 and 3) with a NumPy block backend against the
oracle; the device implementation of the same algorithm is
cpcag_cuda_alternate_decode_sharded (csrc/sharded.cu)."""
from __future__ import annotations

import math
from dataclasses import dataclass
from typing import Optional

import numpy as np

from paper_1602_02070_b200.sharded import HaloPlan, column_blocks


class TorchCollectives:
    """all-gather / all-to-all / all-reduce on torch.distributed (NCCL for
    CUDA tensors)."""

    def __init__(self, group=None):
        import torch.distributed as dist

        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)

    def all_gather_blocks(self, full_padded, block_padded):
        """full_padded: 1-D tensor of world * len(block_padded) elements."""
        if self.dist.get_backend(self.group) == "nccl":
            self.dist.all_gather_into_tensor(full_padded, block_padded, group=self.group)
        else:
            parts = list(full_padded.chunk(self.world))
            self.dist.all_gather(parts, block_padded, group=self.group)

    def exchange_halo(self, full_padded, block_padded, halo: HaloPlan, p: int, c0: int, nloc: int):
        """full_padded[:, c0:c0+nloc] = this block; full_padded[:, halo] =
        the columns other ranks own, received with one all-to-all (uneven
        splits); columns nobody needs are left stale (never read)."""
        import torch

        send_idx = torch.as_tensor(np.concatenate(halo.send), dtype=torch.int64, device=block_padded.device)
        recv_idx = torch.as_tensor(np.concatenate(halo.recv), dtype=torch.int64, device=block_padded.device)
        Pv = block_padded[: p * nloc].view(nloc, p)  # column-major p x nloc
        Pf = full_padded.view(-1, p)
        Pf[c0:c0 + nloc] = Pv
        sendbuf = Pv.index_select(0, send_idx).reshape(-1)
        in_split = [len(x) * p for x in halo.send]
        out_split = [len(x) * p for x in halo.recv]
        recvbuf = full_padded.new_empty(sum(out_split))
        self.dist.all_to_all_single(recvbuf, sendbuf, out_split, in_split, group=self.group)
        if recv_idx.numel():
            Pf.index_copy_(0, recv_idx, recvbuf.view(-1, p))

    def allreduce_sum(self, value: float, like) -> float:
        import torch

        t = torch.tensor([value], dtype=torch.float64, device=like.device)
        self.dist.all_reduce(t, group=self.group)
        return float(t.item())


@dataclass
class ShardedResult:
    X_block: object      # p x (c1 - c0) solution block of this rank
    c0: int
    c1: int
    converged: bool
    iterations: int


def alternate_decode_sharded(Xt, plan, backend, coll, zeros, tol=1e-10, max_iter=5000,
                             halo: Optional[HaloPlan] = None) -> ShardedResult:
    """The CG of decoders.cpp:145-186 over column blocks.

    backend: local primitives (rhs/apply/residual/update) of this rank's block.
    coll:    rank/world + all_gather_blocks + allreduce_sum (+ exchange_halo
             when a HaloPlan is given: only the halo columns move).
    zeros:   allocator zeros(count) -> 1-D array/tensor on the backend's device.
    Blocks are p x w with w = ceil(n / world) columns (zero-padded).
    """
    p, n = plan.p, plan.n
    w, blocks = column_blocks(n, coll.world)
    c0, c1 = blocks[coll.rank]
    nloc = c1 - c0
    B = zeros(p * w)
    X = zeros(p * w)
    R = zeros(p * w)
    P = zeros(p * w)
    AP = zeros(p * w)
    Pfull = zeros(p * w * coll.world)
    view = lambda a: a[: p * nloc]
    bb = coll.allreduce_sum(backend.rhs(Xt, view(B)), B)
    norm_b = math.sqrt(bb)
    if norm_b == 0.0:  # solvers.hpp:38-42
        return ShardedResult(view(X), c0, c1, True, 0)
    target = tol * norm_b
    R[:] = B  # r = b - A x with x = 0
    P[:] = R  # z = r
    rho = bb
    it = 0
    while it < max_iter:
        if math.sqrt(rho) <= target:
            break
        if halo is not None:
            coll.exchange_halo(Pfull, P, halo, p, c0, nloc)
        else:
            coll.all_gather_blocks(Pfull, P)
        curv = coll.allreduce_sum(backend.apply(Pfull, view(AP)), AP)
        if not math.isfinite(curv) or curv <= 0.0:
            raise RuntimeError(f"pcg: breakdown (nonpositive curvature) at iteration {it}")
        alpha = rho / curv
        rho_next = coll.allreduce_sum(backend.residual(alpha, view(R), view(AP)), R)
        beta = rho_next / rho
        backend.update(alpha, beta, view(X), view(P), view(R))
        rho = rho_next
        it += 1
    # true residual (solvers.hpp:69-72)
    coll.all_gather_blocks(Pfull, X)
    backend.apply(Pfull, view(AP))
    E = B.clone() if hasattr(B, "clone") else B.copy()
    rt = coll.allreduce_sum(backend.residual(1.0, view(E), view(AP)), E)
    rel = math.sqrt(rt) / norm_b
    return ShardedResult(view(X), c0, c1, rel <= tol, it)
