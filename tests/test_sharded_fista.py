"""Column-sharded FRPCAG solve ("FISTA scalars all-reduced, X~
all-gathered"; frpcag.cpp:62-112).

CPU: the distributed algorithm (blocks of S all-gathered, five scalars
all-reduced, Z_next formed locally) as a NumPy model over gloo with world
size 2 and 3 against the single-process oracle.
GPU: the device implementation (csrc/sharded.cu) -- 1, 2, 3 and 8 emulated
ranks on one GPU, ragged and empty blocks, and the NCCL driver at world size
1 -- against the oracle and the one-GPU fista_solve."""
import socket

import numpy as np
import pytest

from helpers import knn_laplacian, rel, to_device
from oracle import pyoracle as O


def _case(r=60, c=45, seed=11):
    Lr, Lc = knn_laplacian(r, 3, 6, seed), knn_laplacian(c, 3, 6, seed + 1)
    Y = np.random.default_rng(seed).standard_normal((r, c))
    return Lr, Lc, Y


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _dense(L):
    rp, ci, v = L.arrays()
    D = np.zeros((L.rows, L.rows))
    for i in range(L.rows):
        D[i, ci[rp[i]:rp[i + 1]]] = v[rp[i]:rp[i + 1]]
    return D


def _fista_block_model(Y, Dr, Dc, gr, gc, loss, tol, max_iter, step, c0, c1, allgather, allreduce):
    """One rank of the sharded FISTA (the steps of csrc/sharded.cu's
    fista_sharded_nccl in NumPy)."""
    Z = Y.copy()
    Sp = Y.copy()
    S = Y.copy()
    t = 1.0
    objective, converged, frc = [], False, 0.0
    for _ in range(max_iter):
        G = 2.0 * gc * (Z @ Dc[:, c0:c1]) + 2.0 * gr * (Dr @ Z[:, c0:c1])
        T = Z[:, c0:c1] - step * G
        Yb = Y[:, c0:c1]
        if loss == "l2":
            Sb = (T + 2.0 * step * Yb) / (1.0 + 2.0 * step)
        else:
            D = T - Yb
            Sb = Yb + np.sign(D) * np.maximum(np.abs(D) - step, 0.0)
        S = allgather(Sb)
        tn = 0.5 * (1.0 + np.sqrt(1.0 + 4.0 * t * t))
        coef = (t - 1.0) / tn
        E = Yb - Sb
        Znb = Sb + coef * (Sb - Sp[:, c0:c1])
        sc = np.array([np.sum(E * E) if loss == "l2" else np.sum(np.abs(E)),
                       np.sum((S @ Dc[:, c0:c1]) * Sb), np.sum((Dr @ Sb) * Sb),
                       np.sum(Z[:, c0:c1] ** 2), np.sum((Znb - Z[:, c0:c1]) ** 2)])
        sc = allreduce(sc)
        objective.append(sc[0] + gc * sc[1] + gr * sc[2])
        frc = sc[4] / sc[3] if sc[3] > 0 else sc[4]
        if sc[4] < tol * sc[3]:
            converged = True
            break
        Z = S + coef * (S - Sp)
        Sp = S
        t = tn
    return S[:, c0:c1], objective, converged, frc


def _gloo_worker(rank, world, port, out, loss, tol):
    import torch
    import torch.distributed as dist

    from paper_1602_02070_b200.sharded import bounds_of

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    Lr, Lc, Y = _case()
    bd = bounds_of(Y.shape[1], world)
    c0, c1 = int(bd[rank]), int(bd[rank + 1])
    w = int(np.max(np.diff(bd)))

    def allgather(Sb):
        pad = torch.zeros(Y.shape[0] * w, dtype=torch.float64)
        pad[: Sb.size] = torch.from_numpy(np.asfortranarray(Sb).reshape(-1, order="F"))
        parts = [torch.zeros_like(pad) for _ in range(world)]
        dist.all_gather(parts, pad)
        S = np.empty_like(Y)
        for g in range(world):
            nb = int(bd[g + 1] - bd[g])
            S[:, bd[g]:bd[g + 1]] = parts[g][: Y.shape[0] * nb].numpy().reshape((Y.shape[0], nb), order="F")
        return S

    def allreduce(v):
        tv = torch.from_numpy(v.copy())
        dist.all_reduce(tv)
        return tv.numpy()

    step = O.fista_solve(Y, Lr, Lc, O.FrpcagConfig(3.0, 2.0, loss, 1e-300, 1))[1].step
    Xb, obj, conv, frc = _fista_block_model(Y, _dense(Lr), _dense(Lc), 3.0, 2.0, loss, tol, 120, step, c0, c1,
                                            allgather, allreduce)
    out[rank] = (c0, c1, Xb.copy(), obj, conv)
    dist.destroy_process_group()


@pytest.mark.parametrize("world,loss,tol", [(2, "l1", 1e-300), (3, "l2", 1e-6)])
def test_sharded_fista_algorithm_gloo_matches_oracle(world, loss, tol):
    import torch.multiprocessing as mp

    port = _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    ctx = mp.get_context("spawn")
    procs = [ctx.Process(target=_gloo_worker, args=(r, world, port, out, loss, tol)) for r in range(world)]
    for pr in procs:
        pr.start()
    for pr in procs:
        pr.join(120)
        assert pr.exitcode == 0
    Lr, Lc, Y = _case()
    Xo, tro = O.fista_solve(Y, Lr, Lc, O.FrpcagConfig(3.0, 2.0, loss, tol, 120))
    X = np.zeros_like(Y)
    for r in range(world):
        c0, c1, blk, obj, conv = out[r]
        X[:, c0:c1] = blk
        assert len(obj) == tro.iterations and conv == tro.converged  # every rank stops at the same iteration
        assert np.allclose(obj, tro.objective, rtol=1e-9)
    assert rel(X, Xo) <= 1e-9


@pytest.mark.gpu
@pytest.mark.parametrize("loss", ["l1", "l2"])
@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_sharded_fista_emulated_ranks_match_oracle(world, loss):
    import paper_1602_02070_b200 as P
    from paper_1602_02070_b200.sharded import fista_solve_sharded_emulated

    ctx = P.Context(0)
    Lr, Lc, Y = _case()
    cfg = P.FrpcagConfig(gamma_r=3.0, gamma_c=2.0, loss=loss, tol=1e-300, max_iter=120)
    dLr, dLc = to_device(ctx, Lr), to_device(ctx, Lc)
    X, tr = fista_solve_sharded_emulated(Y, dLr, dLc, cfg, world, ctx=ctx)
    Xo, tro = O.fista_solve(Y, Lr, Lc, O.FrpcagConfig(3.0, 2.0, loss, 1e-300, 120))
    assert tr.iterations == tro.iterations == 120 and not tr.converged
    assert tr.step == pytest.approx(tro.step, rel=1e-6)
    assert rel(X, Xo) <= 1e-9
    assert np.allclose(tr.objective, tro.objective, rtol=1e-9)
    # the block formulas are the one-GPU CSR path's: same S at every iteration
    X1, tr1 = P.fista_solve(Y, dLr, dLc, cfg, ctx=ctx)
    assert rel(X, X1) <= 1e-12 and np.allclose(tr.objective, tr1.objective, rtol=1e-12)


@pytest.mark.gpu
def test_sharded_fista_emulated_ragged_blocks_tolerance_stop_and_fp32():
    import paper_1602_02070_b200 as P
    from paper_1602_02070_b200.sharded import fista_solve_sharded_emulated

    ctx = P.Context(0)
    Lr, Lc = knn_laplacian(30, 3, 5, 6), knn_laplacian(25, 3, 5, 7)
    Y = np.random.default_rng(12).standard_normal((30, 25))
    dLr, dLc = to_device(ctx, Lr), to_device(ctx, Lc)
    cfg = P.FrpcagConfig(gamma_r=0.5, gamma_c=0.5, loss="l2", tol=1e-8, max_iter=5000)
    bd = np.array([0, 4, 4, 19, 25])  # rank 1 owns no column
    X, tr = fista_solve_sharded_emulated(Y, dLr, dLc, cfg, 4, bounds=bd, ctx=ctx)
    Xo, tro = O.fista_solve(Y, Lr, Lc, O.FrpcagConfig(0.5, 0.5, "l2", 1e-8, 5000))
    assert tr.converged and tro.converged
    assert abs(tr.iterations - tro.iterations) <= 1
    assert rel(X, Xo) <= 1e-7
    # fp32 data within north_star's 1e-4 of the fp64 oracle
    cfg32 = P.FrpcagConfig(gamma_r=2.0, gamma_c=2.0, tol=1e-300, max_iter=200)
    Y32 = Y.astype(np.float32)
    X32, _ = fista_solve_sharded_emulated(Y32, dLr, dLc, cfg32, 3, ctx=ctx)
    Xo32, _ = O.fista_solve(Y32.astype(np.float64), Lr, Lc, O.FrpcagConfig(2.0, 2.0, "l1", 1e-300, 200))
    assert X32.dtype == np.float32 and rel(X32, Xo32) <= 1e-4


@pytest.mark.gpu
def test_sharded_fista_errors():
    import paper_1602_02070_b200 as P
    from paper_1602_02070_b200.sharded import fista_solve_sharded_emulated

    ctx = P.Context(0)
    Lr, Lc = knn_laplacian(12, 3, 4, 1), knn_laplacian(10, 3, 4, 2)
    dLr, dLc = to_device(ctx, Lr), to_device(ctx, Lc)
    Y = np.ones((12, 10))
    with pytest.raises(ValueError, match="negative regularization"):
        fista_solve_sharded_emulated(Y, dLr, dLc, P.FrpcagConfig(gamma_r=-1.0), 2, ctx=ctx)
    with pytest.raises(ValueError, match="max_iter must be >= 1"):
        fista_solve_sharded_emulated(Y, dLr, dLc, P.FrpcagConfig(max_iter=0), 2, ctx=ctx)
    with pytest.raises(ValueError, match="bounds must run from 0 to cols"):
        fista_solve_sharded_emulated(Y, dLr, dLc, P.FrpcagConfig(), 2, bounds=np.array([0, 5, 9]), ctx=ctx)
    with pytest.raises(ValueError, match="bounds must ascend"):
        fista_solve_sharded_emulated(Y, dLr, dLc, P.FrpcagConfig(), 2, bounds=np.array([0, 11, 10]), ctx=ctx)
    with pytest.raises(RuntimeError, match="diverged"):
        fista_solve_sharded_emulated(Y * 1e300, dLr, dLc, P.FrpcagConfig(step=10.0, tol=1e-300, max_iter=20), 2,
                                     ctx=ctx)


@pytest.mark.gpu
@pytest.mark.parametrize("prec", ["f64", "f32"])
@pytest.mark.parametrize("world", [1, 3])
def test_sharded_fista_dense_operator_path(world, prec):
    """Kron-reduced (near dense) Laplacians: the block kernels' tiled dense
    form, 32-column tiles that straddle ragged block ends."""
    import paper_1602_02070_b200 as P
    from paper_1602_02070_b200.sharded import fista_solve_sharded_emulated

    ctx = P.Context(0)
    Lr_full, Lc_full = knn_laplacian(300, 3, 10, 31), knn_laplacian(240, 3, 10, 32)
    plan = O.draw_plan(300, 240, 75, 60, seed=5)
    Lr, Lc = O.kron_reduce(Lr_full, plan.omega_r, 1e-11), O.kron_reduce(Lc_full, plan.omega_c, 1e-11)
    assert Lr.nnz >= 0.25 * 75 * 75 and Lc.nnz >= 0.25 * 60 * 60
    dt = np.float64 if prec == "f64" else np.float32
    Y = (np.random.default_rng(4).standard_normal((75, 60)) * 3.0).astype(dt)
    cfg = P.FrpcagConfig(gamma_r=8.0, gamma_c=8.0, tol=1e-300, max_iter=150)
    bd = np.array([0, 60]) if world == 1 else np.array([0, 7, 41, 60])
    dLr, dLc = to_device(ctx, Lr), to_device(ctx, Lc)
    X, tr = fista_solve_sharded_emulated(Y, dLr, dLc, cfg, world, bounds=bd, ctx=ctx)
    Xo, tro = O.fista_solve(Y.astype(np.float64), Lr, Lc, O.FrpcagConfig(8.0, 8.0, "l1", 1e-300, 150))
    assert tr.iterations == 150
    assert rel(X, Xo) <= (1e-9 if prec == "f64" else 1e-4)
    assert np.allclose(tr.objective, tro.objective, rtol=1e-9 if prec == "f64" else 1e-4)
    X1, _ = P.fista_solve(Y, dLr, dLc, cfg, ctx=ctx)  # the one-GPU (persistent) solve sums in another order
    assert rel(X, X1) <= (1e-8 if prec == "f64" else 1e-4)


def _nccl_worker(port, out):
    import torch
    import torch.distributed as dist

    import paper_1602_02070_b200 as P
    from paper_1602_02070_b200.sharded import ShardComm, fista_solve_sharded

    torch.cuda.set_device(0)
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1)
    Lr, Lc, Y = _case()
    ctx = P.Context(0)
    comm = ShardComm(ctx)
    Yd = torch.tensor(np.asfortranarray(Y).T.copy(), device="cuda").t()
    cfg = P.FrpcagConfig(gamma_r=3.0, gamma_c=2.0, loss="l1", tol=1e-300, max_iter=120)
    res = fista_solve_sharded(Yd, to_device(ctx, Lr), to_device(ctx, Lc), cfg, comm, ctx=ctx)
    torch.cuda.synchronize()
    out["r"] = (res.X_block.cpu().numpy().copy(), res.c0, res.c1, res.trace.iterations, list(res.trace.objective))
    comm.close()
    dist.destroy_process_group()


@pytest.mark.gpu
def test_sharded_fista_nccl_world1_matches_oracle():
    import torch.multiprocessing as mp

    port = _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    pr = mp.get_context("spawn").Process(target=_nccl_worker, args=(port, out))
    pr.start()
    pr.join(300)
    assert pr.exitcode == 0
    Lr, Lc, Y = _case()
    Xo, tro = O.fista_solve(Y, Lr, Lc, O.FrpcagConfig(3.0, 2.0, "l1", 1e-300, 120))
    blk, c0, c1, it, obj = out["r"]
    assert (c0, c1, it) == (0, Y.shape[1], 120)
    assert rel(blk, Xo) <= 1e-9 and np.allclose(obj, tro.objective, rtol=1e-9)
