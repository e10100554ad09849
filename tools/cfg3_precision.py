"""Config-3 decoder precision study (diagnostic tool, not a test).

Runs 100 CG iterations of the alternate decoder system (decoders.cpp:145-186)
at 4096 x 200000 in several precision variants and prints each one's relative
Frobenius distance to the fp64 library decoder:

  lib32        the library's fp32 decoder
  t64          independent torch/cuSPARSE fp64 CG (sanity: should be ~1e-12)
  t32          torch fp32 CG, fp32 Laplacian values, fp64 dots
  t64_L32      fp64 CG on the fp32-rounded Laplacian (operator rounding only)
  t32_Lsum     fp32 CG, off-diagonals rounded to fp32 and the diagonal their
               exact row sum (a Laplacian of the rounded graph)
  t32_op64     fp32 iterates, operator applied in fp64 (P widened, fp64 L)
"""
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1602_02070_b200 as P  # noqa: E402
from paper_1602_02070_b200 import workloads  # noqa: E402

its = int(os.environ.get("ITS", "100"))
ctx = P.Context(0)
ctx.set_stream(torch.cuda.current_stream().cuda_stream)
ctx.reserve(40 << 30)
Pr, Pc = workloads.config3_points()
p, n = Pr.shape[1], Pc.shape[1]
gr = P.build_knn_graph(torch.tensor(np.ascontiguousarray(Pr.T), device="cuda").t(), "cols", 10, ctx=ctx)
gc = P.build_knn_graph(torch.tensor(np.ascontiguousarray(Pc.T), device="cuda").t(), "cols", 10, ctx=ctx)
plan = P.draw_plan(p, n, p // 8, n // 8, seed=1607)
rs = np.random.default_rng(1606)


def lowpass(L, m, k=20, sweeps=20):
    nrm = P.power_iteration_norm(L, 1e-7, 42, ctx=ctx)
    B = torch.tensor(rs.standard_normal((m, k)), device="cuda")
    for _ in range(sweeps):
        B = B - L.multiply(B) / nrm
    return torch.linalg.qr(B)[0]


Br, Bc = lowpass(gr.laplacian, p), lowpass(gc.laplacian, n)
A = torch.tensor(rs.standard_normal((20, 20)), device="cuda")
om_r = torch.tensor(plan.omega_r, device="cuda")
om_c = torch.tensor(plan.omega_c, device="cuda")
Xt = (Br[om_r] @ A @ Bc[om_c].T)
Xt64 = Xt.t().contiguous().t()
del Br, Bc
g1 = P.SpectralGap(lambda_k1=1.0)
dcfg = P.DecoderConfig(1.0, 1e-30, its)
t0 = time.time()
X64 = P.alternate_decode(Xt64, plan, gr.laplacian, gc.laplacian, g1, g1, dcfg, ctx=ctx).X
X64T = X64.t().contiguous()  # n x p
del X64
nrm = float(torch.linalg.norm(X64T))
print(f"lib64 {time.time() - t0:.1f}s |X| {nrm:.4e}", flush=True)
torch.cuda.empty_cache()


def csr_torch(L, dt, mode="plain"):
    if dt == torch.float32 and mode == "plain":
        return csr_torch(L, torch.float64, "round")
    rp, ci, v = L.arrays()
    rp = np.asarray(rp, np.int64)
    ci = np.asarray(ci, np.int64)
    v = np.asarray(v, np.float64).copy()
    if mode == "round":
        v = v.astype(np.float32).astype(np.float64)
    elif mode == "sum":
        rows = np.repeat(np.arange(len(rp) - 1), np.diff(rp))
        off = rows != ci
        v[off] = v[off].astype(np.float32).astype(np.float64)
        s = np.zeros(len(rp) - 1)
        np.add.at(s, rows[off], v[off])
        v[~off] = -s[rows[~off]]
    m = len(rp) - 1
    return torch.sparse_csr_tensor(torch.tensor(rp, device="cuda"), torch.tensor(ci, device="cuda"),
                                   torch.tensor(v, device="cuda", dtype=dt), size=(m, m))


rsel = torch.zeros(p, dtype=torch.bool, device="cuda")
rsel[om_r] = True
csel = torch.zeros(n, dtype=torch.bool, device="cuda")
csel[om_c] = True
# right-hand side b = scatter(Xt) in PT (n x p) layout
B64 = torch.zeros(n, p, dtype=torch.float64, device="cuda")
B64[om_c[:, None], om_r[None, :]] = Xt64.t()
MT = (csel[:, None] & rsel[None, :])


def cg(dt, Lr, Lc, op_dt=None, xdt=None, rdt=None, apdt=None, replace=0):
    """CG with per-vector storage precisions: dt = P, xdt = X, rdt = R,
    apdt = stored AP (defaults: dt); op_dt = operator arithmetic."""
    op_dt = op_dt or dt
    xdt, rdt, apdt = xdt or dt, rdt or dt, apdt or dt

    def apply(PT):
        Q = PT.to(op_dt)
        return torch.sparse.mm(Lc, Q) + torch.sparse.mm(Lr, Q.t()).t() + Q * MT

    X = torch.zeros(n, p, dtype=xdt, device="cuda")
    R = B64.to(rdt).clone()
    Pv = R.to(dt).clone()
    rho = float((R.double() ** 2).sum())
    hist = []
    for k in range(its):
        AP = apply(Pv).to(apdt)
        curv = float((Pv.double() * AP.double()).sum())
        al = rho / curv
        X = (X.double() + al * Pv.double()).to(xdt)
        R = (R.double() - al * AP.double()).to(rdt)
        if replace and k % replace == replace - 1:
            R = (B64 - apply(X.to(op_dt)).double()).to(rdt)
        rn = float((R.double() ** 2).sum())
        Pv = (R.double() + (rn / rho) * Pv.double()).to(dt)
        rho = rn
        if k % 10 == 9:
            hist.append((k, rho, curv))
    print("   hist " + " ".join(f"{k}:{r:.3e}" for k, r, c in hist), flush=True)
    return X


f32, f64 = torch.float32, torch.float64
for name, L_dt, kw in [("m8 P64 X32 R32 AP32, op64", f64, dict(dt=f64, xdt=f32, rdt=f32, apdt=f32, op_dt=f64)),
                       ("m9 P64 X64 R32 AP64, op64", f64, dict(dt=f64, xdt=f64, rdt=f32, apdt=f64, op_dt=f64)),
                       ("m10 P64 X32 R64 AP64, op64", f64, dict(dt=f64, xdt=f32, rdt=f64, apdt=f64, op_dt=f64)),
                       ("m11 P64 X64 R64 AP32, op64", f64, dict(dt=f64, xdt=f64, rdt=f64, apdt=f32, op_dt=f64)),
                       ("m12 all fp64, fp32-rounded operator values", f32, dict(dt=f64, op_dt=f64)),
                       ("m13 P64 X32 R64 AP32, op64", f64, dict(dt=f64, xdt=f32, rdt=f64, apdt=f32, op_dt=f64))]:
    t0 = time.time()
    Lr, Lc = csr_torch(gr.laplacian, L_dt), csr_torch(gc.laplacian, L_dt)
    X = cg(Lr=Lr, Lc=Lc, **kw)
    d = float(torch.linalg.norm(X.double() - X64T)) / nrm
    print(f"{name} vs lib64: {d:.3e} ({time.time() - t0:.1f}s)", flush=True)
    del X, Lr, Lc
    torch.cuda.empty_cache()
