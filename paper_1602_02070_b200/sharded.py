"""Column-sharded alternate decoder across the GPUs of one node.

X (p x n) is split into contiguous column blocks, one per rank (one process
per GPU).  The whole CG loop runs inside libcpcag_cuda.so
(`cpcag_cuda_alternate_decode_sharded`, csrc/sharded.cu): per iteration the
halo columns of the search direction move by one grouped NCCL send/recv
(overlapped with the block-local L_r pass), the CG dot products are
all-reduced on device scalars, and the host only polls the done flag once
per 32 iterations.  This module holds the Python side of that C-ABI:

  * `column_blocks` / `bounds_of`: the partition;
  * `HaloPlan`: the library's host-side halo plan (`cpcag_halo_plan`), i.e.
    which columns each rank sends and receives -- no device needed, so it is
    covered by CPU tests (gloo, world 2 and 3, tests/test_sharded.py);
  * `ShardComm`: the library's NCCL communicator, bootstrapped over
    torch.distributed (rank 0's ncclUniqueId is broadcast);
  * `alternate_decode_sharded`: this rank's block of the solution;
  * `alternate_decode_sharded_emulated`: all ranks in one process on one GPU
    (device copies for the exchange), for tests of the multi-rank logic;
  * `fista_solve_sharded` / `fista_solve_sharded_emulated`: FRPCAG's FISTA on
    column blocks of the compressed matrix (S blocks all-gathered, the five
    objective / stopping scalars all-reduced on the device).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _native as N


def column_blocks(n: int, world: int):
    """Equal-width blocks (the last one may be short or empty): block g is
    [g * w, min(n, (g + 1) * w))."""
    w = -(-n // world) if world > 0 else n
    return w, [(min(n, g * w), min(n, (g + 1) * w)) for g in range(world)]


def bounds_of(n: int, world: int) -> np.ndarray:
    """Block boundaries (world + 1 ascending entries, 0 ... n)."""
    _, blocks = column_blocks(n, world)
    return np.array([b[0] for b in blocks] + [n], dtype=np.int64)


class HaloPlan:
    """Which columns of P rank `rank` receives from / sends to every other
    rank for the X L_c term (the library's host code, csrc/sharded.cu
    make_halo_plan).  recv[s]: global column ids received from rank s
    (ascending); send[d]: local ids (column - bounds[rank]) sent to rank d."""

    def __init__(self, rp, ci, n, world, rank, bounds=None):
        rp = np.ascontiguousarray(rp, np.int64)
        ci = np.ascontiguousarray(ci, np.int64)
        bd = np.ascontiguousarray(bounds_of(n, world) if bounds is None else bounds, np.int64)
        rc = np.zeros(world, np.int64)
        sc = np.zeros(world, np.int64)
        nb = int(bd[rank + 1] - bd[rank])
        recv = np.zeros(max(n, 1), np.int64)
        send = np.zeros(max(nb * world, 1), np.int64)
        N.check(N.lib().cpcag_halo_plan(rp.ctypes.data, ci.ctypes.data, int(n), bd.ctypes.data, int(world),
                                        int(rank), rc.ctypes.data, sc.ctypes.data, recv.ctypes.data,
                                        send.ctypes.data))
        ro = np.concatenate([[0], np.cumsum(rc)])
        so = np.concatenate([[0], np.cumsum(sc)])
        self.world, self.rank, self.bounds = world, rank, bd
        self.recv = [recv[ro[s]:ro[s + 1]].copy() for s in range(world)]
        self.send = [send[so[d]:so[d + 1]].copy() for d in range(world)]
        self.halo_cols = int(rc.sum())
        self.send_cols = int(sc.sum())
        self.remote_cols = int(n - nb)


class ShardComm:
    """The library's NCCL communicator for this process's rank.  The unique
    id is created on rank 0 and broadcast over torch.distributed (any
    backend); every rank then joins with ncclCommInitRank."""

    def __init__(self, ctx, group=None):
        import torch.distributed as dist

        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        buf = (C.c_char * 128)()
        if self.rank == 0:
            N.check(N.lib().cpcag_cuda_comm_unique_id(buf))
        obj = [bytes(buf)]
        dist.broadcast_object_list(obj, src=dist.get_global_rank(group, 0) if group is not None else 0, group=group)
        idb = (C.c_char * 128).from_buffer_copy(obj[0])
        h = N.vp()
        N.check(N.lib().cpcag_cuda_comm_create(ctx.handle, idb, self.world, self.rank, C.byref(h)))
        self.h = h
        self.ctx = ctx

    def close(self):
        if getattr(self, "h", None) is not None and self.h.value:
            N.lib().cpcag_cuda_comm_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


@dataclass
class ShardStats:
    halo_cols: int
    send_cols: int
    bytes_per_iteration: float
    exchange_ms: float


@dataclass
class ShardedResult:
    X_block: object      # p x (c1 - c0) solution block of this rank
    c0: int
    c1: int
    converged: bool
    iterations: int
    stats: ShardStats


def _stats(s) -> ShardStats:
    return ShardStats(int(s.halo_cols), int(s.send_cols), float(s.bytes_per_iteration), float(s.exchange_ms))


def alternate_decode_sharded(Xt, plan, Lr, Lc, gap_r, gap_c, cfg, comm: ShardComm, bounds=None, precision=None,
                             measure_exchange=False, out=None, ctx=None) -> ShardedResult:
    """decoders.cpp:145-186 for this rank's column block.  Xt, plan, Lr and
    Lc are the same on every rank; `out` (optional) receives the p x nb
    block."""
    from .cpcag import _ctx, _In, _is_cuda, _out, _precision, _torch_device, _given_out

    prec = _precision(Xt, precision)
    xt = _In(Xt, prec)
    if tuple(xt.shape) != (plan.rho_r(), plan.rho_c()):
        raise ValueError("alternate decoder: Xt does not match plan")
    bd = np.ascontiguousarray(bounds_of(plan.n, comm.world) if bounds is None else bounds, np.int64)
    c0, c1 = int(bd[comm.rank]), int(bd[comm.rank + 1])
    om_r = np.ascontiguousarray(plan.omega_r, np.int64)
    om_c = np.ascontiguousarray(plan.omega_c, np.int64)
    if out is None:
        res, op = _out(_is_cuda(Xt), _torch_device(Xt), (plan.p, c1 - c0), prec)
    else:
        res, op = _given_out(out, (plan.p, c1 - c0), prec, "out")
    st = N.ShardStatsC(0, 0, 0.0, 0.0, 1 if measure_exchange else 0)
    cv, it = C.c_int(), N.i64()
    dc = cfg.c()
    N.check(N.lib().cpcag_cuda_alternate_decode_sharded(
        _ctx(ctx), comm.h, prec, xt.ptr, plan.rho_r(), plan.rho_c(), om_r.ctypes.data if om_r.size else None,
        om_c.ctypes.data if om_c.size else None, plan.p, plan.n, Lr.handle, Lc.handle, float(gap_r.lambda_k1),
        float(gap_c.lambda_k1), C.byref(dc), bd.ctypes.data, op, C.byref(cv), C.byref(it), C.byref(st)))
    return ShardedResult(res, c0, c1, bool(cv.value), int(it.value), _stats(st))


def alternate_decode_sharded_emulated(Xt, plan, Lr, Lc, gap_r, gap_c, cfg, nranks: int, bounds=None,
                                      precision=None, ctx=None):
    """All `nranks` ranks of the sharded decoder in this process on one GPU
    (tests).  Returns (AlternateDecodeResult, rank-0 ShardStats)."""
    from .cpcag import AlternateDecodeResult, _ctx, _In, _is_cuda, _out, _precision, _torch_device

    prec = _precision(Xt, precision)
    xt = _In(Xt, prec)
    bd = np.ascontiguousarray(bounds_of(plan.n, nranks) if bounds is None else bounds, np.int64)
    om_r = np.ascontiguousarray(plan.omega_r, np.int64)
    om_c = np.ascontiguousarray(plan.omega_c, np.int64)
    res, op = _out(_is_cuda(Xt), _torch_device(Xt), (plan.p, plan.n), prec)
    st = N.ShardStatsC(0, 0, 0.0, 0.0, 0)
    cv, it = C.c_int(), N.i64()
    dc = cfg.c()
    N.check(N.lib().cpcag_cuda_alternate_decode_sharded_emulated(
        _ctx(ctx), int(nranks), prec, xt.ptr, plan.rho_r(), plan.rho_c(), om_r.ctypes.data if om_r.size else None,
        om_c.ctypes.data if om_c.size else None, plan.p, plan.n, Lr.handle, Lc.handle, float(gap_r.lambda_k1),
        float(gap_c.lambda_k1), C.byref(dc), bd.ctypes.data, op, C.byref(cv), C.byref(it), C.byref(st)))
    return AlternateDecodeResult(res, bool(cv.value), int(it.value)), _stats(st)


@dataclass
class ShardedFistaResult:
    X_block: object      # rows x (c1 - c0) block of this rank
    c0: int
    c1: int
    trace: object        # SolveTrace, identical on every rank


def fista_solve_sharded(Y, Lr, Lc, cfg, comm: ShardComm, bounds=None, precision=None, ctx=None) -> ShardedFistaResult:
    """frpcag.cpp:62-112 for this rank's column block of the compressed
    matrix.  Y, Lr, Lc and cfg are the same on every rank."""
    from .cpcag import SolveTrace, _ctx, _In, _is_cuda, _out, _precision, _torch_device

    prec = _precision(Y, precision)
    y = _In(Y, prec)
    if len(y.shape) != 2:
        raise ValueError("fista: Y must be a matrix")
    rows, cols = y.shape
    bd = np.ascontiguousarray(bounds_of(cols, comm.world) if bounds is None else bounds, np.int64)
    if bd.size != comm.world + 1:
        raise ValueError("sharded fista: bounds must hold world + 1 entries")
    c0, c1 = int(bd[comm.rank]), int(bd[comm.rank + 1])
    out, op = _out(_is_cuda(Y), _torch_device(Y), (rows, max(c1 - c0, 0)), prec)
    obj = np.zeros(max(int(cfg.max_iter), 1))
    tr = N.SolveTraceC()
    c = cfg.c()
    N.check(N.lib().cpcag_cuda_fista_sharded(_ctx(ctx), comm.h, prec, y.ptr, rows, cols, Lr.handle, Lc.handle,
                                             C.byref(c), bd.ctypes.data, op, obj.ctypes.data, C.byref(tr)))
    n = int(tr.iterations)
    return ShardedFistaResult(out, c0, c1, SolveTrace(list(obj[:n]), n, bool(tr.converged),
                                                      float(tr.final_rel_change), float(tr.step)))


def fista_solve_sharded_emulated(Y, Lr, Lc, cfg, nranks: int, bounds=None, precision=None, ctx=None):
    """All `nranks` ranks of the sharded FISTA in this process on one GPU
    (tests).  Returns (X, SolveTrace) like fista_solve."""
    from .cpcag import SolveTrace, _ctx, _In, _is_cuda, _out, _precision, _torch_device

    prec = _precision(Y, precision)
    y = _In(Y, prec)
    if len(y.shape) != 2:
        raise ValueError("fista: Y must be a matrix")
    rows, cols = y.shape
    bd = np.ascontiguousarray(bounds_of(cols, nranks) if bounds is None else bounds, np.int64)
    if bd.size != nranks + 1:
        raise ValueError("sharded fista: bounds must hold world + 1 entries")
    out, op = _out(_is_cuda(Y), _torch_device(Y), (rows, cols), prec)
    obj = np.zeros(max(int(cfg.max_iter), 1))
    tr = N.SolveTraceC()
    c = cfg.c()
    N.check(N.lib().cpcag_cuda_fista_sharded_emulated(_ctx(ctx), int(nranks), prec, y.ptr, rows, cols, Lr.handle,
                                                      Lc.handle, C.byref(c), bd.ctypes.data, op, obj.ctypes.data,
                                                      C.byref(tr)))
    n = int(tr.iterations)
    return out, SolveTrace(list(obj[:n]), n, bool(tr.converged), float(tr.final_rel_change), float(tr.step))
