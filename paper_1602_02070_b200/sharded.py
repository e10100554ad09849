"""Column-sharded alternate decoder across the GPUs of one node.

X (p x n) is split into contiguous column blocks, one per rank.  Per CG
iteration (the reference recurrence of detail::pcg_core, solvers.hpp:33-74,
identity preconditioner):

  1. exchange the halo: the X·L_c term of block g needs the columns of P
     that L_c's rows in the block reference outside it.  With a `HaloPlan`
     every rank sends exactly the columns each other rank needs (one NCCL
     all-to-all with uneven splits over NVLink) and receives only its own
     halo; without one, the blocks are all-gathered (for kNN graphs over
     high-dimensional points the halo is 82-100 % of the remote columns,
     SURVEY §8(e), so the two move similar bytes there);
  2. AP_g = (γ̄_c P L_c + γ̄_r L_r P + M∘P)(:, block g) on the local GPU;
     L_r·P is block-local;
  3. all-reduce ⟨P_g, AP_g⟩ -> α;  R_g -= α AP_g;  all-reduce ‖R_g‖² -> β;
  4. X_g += α P_g;  P_g = R_g + β P_g.

The local work runs in libcpcag_cuda.so (`CudaBlockBackend`, the
cpcag_cuda_decoder_block_* / cpcag_cuda_cg_* entry points); the
communication is torch.distributed (`TorchCollectives`).  Both are plain
objects handed to `alternate_decode_sharded`, which holds only the
algorithm, so the distributed logic is testable on CPU (gloo) with a test
double standing in for the GPU backend.
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass
from typing import Optional

import numpy as np

from . import _native as N


def column_blocks(n: int, world: int):
    """Equal-width blocks (the last one may be short or empty) so all-gather
    buffers have one size: block g is [g * w, min(n, (g + 1) * w))."""
    w = -(-n // world) if world > 0 else n
    return w, [(min(n, g * w), min(n, (g + 1) * w)) for g in range(world)]


class HaloPlan:
    """Which columns of P each rank sends to / receives from every other rank
    for the X·L_c term (the pull over L_c's rows c of the block: L_c is a
    symmetric Laplacian).  Built identically on every rank from L_c's CSR
    structure (host arrays), O(nnz)."""

    def __init__(self, rp, ci, n, world, rank):
        rp = np.asarray(rp, np.int64)
        ci = np.asarray(ci, np.int64)
        w, blocks = column_blocks(n, world)
        self.w, self.world, self.rank = w, world, rank
        need = []
        for r in range(world):
            c0, c1 = blocks[r]
            cols = ci[rp[c0]:rp[c1]]
            need.append(np.unique(cols[(cols < c0) | (cols >= c1)]))
        c0 = blocks[rank][0]
        # send[d]: local indices (in this rank's block) of the columns rank d needs
        self.send = [need[d][need[d] // w == rank] - c0 if d != rank else np.zeros(0, np.int64)
                     for d in range(world)]
        # recv[s]: global indices of the columns this rank receives from rank s
        self.recv = [need[rank][need[rank] // w == s] if s != rank else np.zeros(0, np.int64) for s in range(world)]
        self.halo_cols = int(sum(len(x) for x in self.recv))
        self.remote_cols = int(n - (blocks[rank][1] - blocks[rank][0]))
        self._dev = {}

    def device_index(self, device):
        import torch

        key = str(device)
        if key not in self._dev:
            self._dev[key] = (torch.as_tensor(np.concatenate(self.send) if self.send else np.zeros(0, np.int64),
                                              dtype=torch.int64, device=device),
                              torch.as_tensor(np.concatenate(self.recv) if self.recv else np.zeros(0, np.int64),
                                              dtype=torch.int64, device=device))
        return self._dev[key]


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
        send_idx, recv_idx = halo.device_index(block_padded.device)
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


class CudaBlockBackend:
    """GPU-local primitives through the C-ABI (device tensors, column-major)."""

    def __init__(self, ctx, precision, plan, Lr, Lc, gbar_r, gbar_c, c0, c1, stream=None):
        import torch

        # The collectives (NCCL) and the tensor copies run on torch's stream;
        # the block kernels must be ordered with them.
        ctx.set_stream(stream if stream is not None else torch.cuda.current_stream().cuda_stream)
        self.ctx = ctx
        self._graphs = (Lr, Lc)  # the block keeps raw CSR handles: hold the owners
        self.prec = precision
        self.p, self.n = plan.p, plan.n
        self.c0, self.c1 = c0, c1
        om_r = np.ascontiguousarray(plan.omega_r, np.int64)
        om_c = np.ascontiguousarray(plan.omega_c, np.int64)
        h = N.vp()
        N.check(N.lib().cpcag_cuda_decoder_block_create(
            ctx.handle, precision, self.p, self.n, c0, c1, Lr.handle, Lc.handle, om_r.ctypes.data, len(om_r),
            om_c.ctypes.data, len(om_c), float(gbar_r), float(gbar_c), C.byref(h)))
        self.h = h

    def close(self):
        if self.h is not None and self.h.value:
            N.lib().cpcag_cuda_decoder_block_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def rhs(self, Xt, B) -> float:
        out = N.dbl()
        N.check(N.lib().cpcag_cuda_decoder_block_rhs(self.h, Xt.data_ptr(), B.data_ptr(), C.byref(out)))
        return float(out.value)

    def apply(self, P_full, AP) -> float:
        out = N.dbl()
        N.check(N.lib().cpcag_cuda_decoder_block_apply(self.h, P_full.data_ptr(), AP.data_ptr(), C.byref(out)))
        return float(out.value)

    def residual(self, alpha, R, AP) -> float:
        out = N.dbl()
        N.check(N.lib().cpcag_cuda_cg_residual(self.ctx.handle, self.prec, R.numel(), float(alpha), R.data_ptr(),
                                               AP.data_ptr(), C.byref(out)))
        return float(out.value)

    def update(self, alpha, beta, X, P, R):
        N.check(N.lib().cpcag_cuda_cg_update(self.ctx.handle, self.prec, X.numel(), float(alpha), float(beta),
                                             X.data_ptr(), P.data_ptr(), R.data_ptr()))


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
