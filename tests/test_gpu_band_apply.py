"""GPU parity of the band decoder apply (decoder.cu, BandApply): the two-sweep
A(P) = gc P L_c + gr L_r P + M o P used when the iterate does not fit in L2.

It is selected automatically only for large problems (cfg3), so these tests
force it with CPCAG_APPLY=band on small seeded cases and check
  * one apply through the decoder-block C-ABI is bit-exact in fp64 against
    the oracle's decoder_apply (decoders.cpp:160-170 per-entry order), for
    every band height (RPL 1/2/4), both row-record widths (16/32 bytes), a
    column block that starts mid-matrix, and ragged sizes;
  * full alternate decodes with the band apply match the oracle
    (fp64 1e-9, fp32 1e-4 relative Frobenius, the north_star bar).
"""
import numpy as np
import pytest

from helpers import knn_laplacian, rel, to_device
from oracle import pyoracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    import paper_1602_02070_b200 as P

    return P


@pytest.fixture(scope="module")
def ctx(P):
    return P.Context(0)


@pytest.fixture
def band(monkeypatch):
    monkeypatch.setenv("CPCAG_APPLY", "band")


def _apply_case(p, n, seed, dim=4):
    Lr = knn_laplacian(p, dim, 10, seed)
    Lc = knn_laplacian(n, dim, 10, seed + 1)
    plan = O.draw_plan(p, n, max(1, p // 4), max(1, n // 5), seed=seed)
    Pm = np.random.default_rng(seed).standard_normal((p, n))
    return Lr, Lc, plan, Pm


@pytest.mark.parametrize("p,n,c0,c1", [
    (20, 37, 0, 37),      # RPL 1 (one 32-row band, 12 idle lanes)
    (40, 131, 0, 131),    # RPL 2
    (333, 517, 0, 517),   # RPL 4, ragged bands and column groups
    (333, 517, 129, 300),  # a column block starting mid-matrix
    (7000, 23, 0, 23),    # 16-byte row records (p * 32 B > 200 KB)
])
def test_band_apply_fp64_bit_exact(P, ctx, band, p, n, c0, c1):
    import torch

    from paper_1602_02070_b200 import _native as N
    from paper_1602_02070_b200.sharded import CudaBlockBackend

    Lr, Lc, plan_o, Pm = _apply_case(p, n, 11 + p)
    plan = P.SamplingPlan(plan_o.omega_r, plan_o.omega_c, plan_o.p, plan_o.n)
    gr, gc = 1.0 / 0.3, 1.0 / 0.7
    be = CudaBlockBackend(ctx, N.F64, plan, to_device(ctx, Lr), to_device(ctx, Lc), gr, gc, c0, c1)
    Pflat = torch.tensor(np.asfortranarray(Pm).ravel(order="F"), dtype=torch.float64, device="cuda")
    AP = torch.zeros(p * (c1 - c0), dtype=torch.float64, device="cuda")
    dot = be.apply(Pflat, AP)
    torch.cuda.synchronize()
    got = AP.cpu().numpy().reshape((p, c1 - c0), order="F")
    want = O.decoder_apply(Pm, plan_o, Lr, Lc, gr, gc)[:, c0:c1]
    assert np.array_equal(got, want)
    ref_dot = float(np.sum(Pm[:, c0:c1] * want))
    assert dot == pytest.approx(ref_dot, rel=1e-12)
    be.close()


@pytest.mark.parametrize("perm", ["1", "0"])
def test_band_decode_fp64_matches_oracle(P, ctx, band, monkeypatch, perm):
    # perm 1: iterates stored in descending-L_r-degree row order (the default)
    monkeypatch.setenv("CPCAG_BAND_PERM", perm)
    Lr, Lc, plan_o, _ = _apply_case(150, 210, 3)
    Xt = np.random.default_rng(4).standard_normal((plan_o.rho_r, plan_o.rho_c))
    plan = P.SamplingPlan(plan_o.omega_r, plan_o.omega_c, plan_o.p, plan_o.n)
    res = P.alternate_decode(Xt, plan, to_device(ctx, Lr), to_device(ctx, Lc), P.SpectralGap(lambda_k1=0.3),
                             P.SpectralGap(lambda_k1=0.4), P.DecoderConfig(1.0, 1e-10, 400), ctx=ctx)
    ro = O.alternate_decode(Xt, plan_o, Lr, Lc, 0.3, 0.4, 1.0, 1e-10, 400)
    assert res.converged == ro.converged
    assert abs(res.iterations - ro.iterations) <= 1
    assert rel(res.X, ro.X) <= 1e-9


def test_band_decode_fp32_fixed_iterations(P, ctx, band):
    Lr, Lc, plan_o, _ = _apply_case(400, 300, 23)
    Xt = np.random.default_rng(5).standard_normal((plan_o.rho_r, plan_o.rho_c)).astype(np.float32)
    plan = P.SamplingPlan(plan_o.omega_r, plan_o.omega_c, plan_o.p, plan_o.n)
    res = P.alternate_decode(Xt, plan, to_device(ctx, Lr), to_device(ctx, Lc), P.SpectralGap(lambda_k1=1.0),
                             P.SpectralGap(lambda_k1=1.0), P.DecoderConfig(1.0, 1e-8, 100), ctx=ctx)
    ro = O.alternate_decode(Xt.astype(np.float64), plan_o, Lr, Lc, 1.0, 1.0, 1.0, 1e-8, 100)
    assert res.iterations == ro.iterations
    assert rel(res.X, ro.X) <= 1e-4


def test_band_kernels_are_the_ones_launched(P, ctx, band):
    Lr, Lc, plan_o, _ = _apply_case(64, 90, 8)
    Xt = np.random.default_rng(6).standard_normal((plan_o.rho_r, plan_o.rho_c))
    plan = P.SamplingPlan(plan_o.omega_r, plan_o.omega_c, plan_o.p, plan_o.n)
    ctx.enable_kernel_timing(True)
    ctx.reset_kernel_timing()
    P.alternate_decode(Xt, plan, to_device(ctx, Lr), to_device(ctx, Lc), P.SpectralGap(lambda_k1=1.0),
                       P.SpectralGap(lambda_k1=1.0), P.DecoderConfig(1.0, 1e-10, 20), ctx=ctx)
    names = set(ctx.kernel_times())
    ctx.enable_kernel_timing(False)
    assert {"cg_apply_band", "cg_apply_col"} <= names


@pytest.mark.parametrize("split", ["8", "64"])
def test_band_decode_fp32_split_rows_deterministic(P, ctx, band, monkeypatch, split):
    # split 8 cuts most rows into chunks (partial sums combined in chunk order)
    monkeypatch.setenv("CPCAG_BAND_SPLIT", split)
    Lr, Lc, plan_o, _ = _apply_case(333, 260, 29, dim=3)
    Xt = np.random.default_rng(7).standard_normal((plan_o.rho_r, plan_o.rho_c)).astype(np.float32)
    plan = P.SamplingPlan(plan_o.omega_r, plan_o.omega_c, plan_o.p, plan_o.n)
    dLr, dLc = to_device(ctx, Lr), to_device(ctx, Lc)
    g = P.SpectralGap(lambda_k1=1.0)
    cfg = P.DecoderConfig(1.0, 1e-8, 60)
    r1 = P.alternate_decode(Xt, plan, dLr, dLc, g, g, cfg, ctx=ctx)
    r2 = P.alternate_decode(Xt, plan, dLr, dLc, g, g, cfg, ctx=ctx)
    assert np.array_equal(r1.X, r2.X)  # fixed warp assignment: deterministic dots
    ro = O.alternate_decode(Xt.astype(np.float64), plan_o, Lr, Lc, 1.0, 1.0, 1.0, 1e-8, 60)
    assert r1.iterations == ro.iterations
    assert rel(r1.X, ro.X) <= 1e-4
