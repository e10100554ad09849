"""GLR1 device-direct I/O (paper_1602_02070_b200/csrc/io.cu) against the
fixtures of tests/golden/ and the numpy restatement oracle/glr1.py:
bit-exact fp64 round trips, fp32 narrowing/widening on
the device, multi-chunk streaming, CSR canonicalisation like
SparseMatrix::from_triplets (sparse.cpp:10-46), and the reference's error
texts (io.cpp:22-75, 164-176)."""
import os

import numpy as np
import pytest

from oracle import glr1

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


@pytest.fixture(scope="module")
def P():
    import paper_1602_02070_b200 as P

    return P


@pytest.fixture(scope="module")
def ctx(P):
    return P.Context(0)


def _g(name):
    return os.path.join(GOLD, name)


def test_dense_fixture_to_device_and_back(P, ctx, tmp_path):
    import torch

    _, M = glr1.read(open(_g("dense_3x4.glr1"), "rb").read())
    d = P.load_matrix(_g("dense_3x4.glr1"), ctx=ctx)
    assert d.is_cuda and d.dtype == torch.float64 and d.t().is_contiguous()
    assert np.array_equal(d.cpu().numpy(), M) and np.signbit(d.cpu().numpy()[1, 1])
    f = str(tmp_path / "d.glr1")
    P.save_matrix(d, f, ctx=ctx)
    assert open(f, "rb").read() == open(_g("dense_3x4.glr1"), "rb").read()
    h = P.load_matrix(_g("dense_3x4.glr1"), device="cpu", ctx=ctx)
    assert isinstance(h, np.ndarray) and np.array_equal(h, M)


@pytest.mark.parametrize("shape", [(4100, 1100), (1, 1), (0, 5)])
def test_dense_streaming_fp64_and_fp32(P, ctx, tmp_path, shape):
    """4100 x 1100 doubles span two 32 MB staging chunks."""
    import torch

    M = np.random.default_rng(sum(shape)).standard_normal(shape)
    f = str(tmp_path / "m.glr1")
    open(f, "wb").write(glr1.dense_bytes(M))
    d64 = P.load_matrix(f, ctx=ctx)
    assert np.array_equal(d64.cpu().numpy(), M)
    d32 = P.load_matrix(f, precision="f32", ctx=ctx)
    assert d32.dtype == torch.float32 and np.array_equal(d32.cpu().numpy(), M.astype(np.float32))
    g = str(tmp_path / "w.glr1")
    P.save_matrix(d32, g, ctx=ctx)  # widened on the device
    _, back = glr1.read(open(g, "rb").read())
    assert np.array_equal(back, M.astype(np.float32).astype(np.float64))
    P.save_matrix(d64, g, ctx=ctx)
    assert open(g, "rb").read() == open(f, "rb").read()


def test_dense_errors(P, ctx, tmp_path):
    f = str(tmp_path / "bad.glr1")
    open(f, "wb").write(b"GLR2" + bytes(24))
    with pytest.raises(RuntimeError, match=r"not a GLR1 container \(bad magic\)"):
        P.load_matrix(f, ctx=ctx)
    with pytest.raises(RuntimeError, match="not a dense-matrix block"):
        P.load_matrix(_g("csr_path5.glr1"), ctx=ctx)
    data = glr1.dense_bytes(np.ones((10, 10)))
    open(f, "wb").write(data[:-8])
    with pytest.raises(RuntimeError, match="truncated data section"):
        P.load_matrix(f, ctx=ctx)
    with pytest.raises(RuntimeError, match="cannot open for reading"):
        P.load_matrix(str(tmp_path / "none.glr1"), ctx=ctx)


def test_sparse_fixture_round_trip(P, ctx, tmp_path):
    A = P.load_sparse(_g("csr_path5.glr1"), ctx=ctx)
    assert (A.rows(), A.cols(), A.nonzeros()) == (5, 5, 13)
    y = A.multiply(np.ones((5, 1)))
    assert np.array_equal(np.asarray(y).ravel(), np.zeros(5))
    f = str(tmp_path / "a.glr1")
    P.save_sparse(A, f, ctx=ctx)
    assert open(f, "rb").read() == open(_g("csr_path5.glr1"), "rb").read()


def test_sparse_noncanonical_rebuilt_like_from_triplets(P, ctx, tmp_path):
    A = P.load_sparse(_g("csr_noncanonical.glr1"), ctx=ctx)
    f = str(tmp_path / "c.glr1")
    P.save_sparse(A, f, ctx=ctx)
    _, (r, c, rp, ci, v) = glr1.read(open(f, "rb").read())
    # row 0: (2, 1) + (0, 2) + (2, .5) -> (0, 2), (2, 1.5); row 1 drops the
    # explicit zero; row 2's duplicates cancel and are dropped
    assert (r, c) == (3, 4) and list(rp) == [0, 2, 3, 3] and list(ci) == [0, 2, 3] and list(v) == [2.0, 1.5, 4.0]
    bad = str(tmp_path / "bad.glr1")
    open(bad, "wb").write(glr1.csr_bytes(2, 2, [0, 2, 1], [0, 1, 0], [1.0, 2.0, 3.0]))
    with pytest.raises(RuntimeError, match="inconsistent row pointers"):
        P.load_sparse(bad, ctx=ctx)
    open(bad, "wb").write(glr1.csr_bytes(3, 2, [0, 3, 1, 3], [0, 1, 0], [1.0, 2.0, 3.0]))
    with pytest.raises(RuntimeError, match="row pointers not monotone"):
        P.load_sparse(bad, ctx=ctx)


def test_factors_round_trip(P, ctx, tmp_path):
    f = P.load_factors(_g("factors_4x3_k2.glr1"), ctx=ctx)
    UV = np.load(_g("factors_4x3_k2_UV.npy"))
    assert f.k == 2 and f.scale_applied and np.array_equal(np.concatenate([f.U, f.V]), UV)
    g = str(tmp_path / "f.glr1")
    P.save_factors(f, g, ctx=ctx)
    assert open(g, "rb").read() == open(_g("factors_4x3_k2.glr1"), "rb").read()


def test_emit_report_artifacts(P, ctx, tmp_path):
    """pipeline.cpp:417-439: the artifact set of a run, written from HBM."""
    import json

    from paper_1602_02070_b200.workloads import config0

    Y, _ = config0(seed=1602, small=True)
    cfg = P.PipelineConfig(knn=10, a=4, b=4, frpcag=P.FrpcagConfig(gamma_r=9.0, gamma_c=9.0, tol=1e-300, max_iter=20),
                           decoder=P.DecoderConfig(1.0, 1e-8, 100, variant="alternate"), lambda_k1_r=0.05,
                           lambda_k1_c=0.07, seed=1602, task="both", n_clusters=2, kmeans_restarts=2)
    rep = P.run_pipeline(Y, cfg, ctx=ctx)
    out = str(tmp_path / "run")
    P.emit_report(rep, cfg, out, ctx=ctx)
    names = sorted(os.listdir(out))
    assert names == ["decoded.csv", "decoded.glr1", "labels.csv", "objective.csv", "plan.json", "report.json",
                     "solution_compressed.glr1"]
    j = json.load(open(os.path.join(out, "report.json")))
    assert j["solve"]["iterations"] == 20 and len(j["solve"]["objective"]) == 20 and "timings_ms" in j
    _, X = glr1.read(open(os.path.join(out, "decoded.glr1"), "rb").read())
    assert np.array_equal(X, rep.X)
    assert np.array_equal(P.load_labels_csv(os.path.join(out, "labels.csv")), rep.labels)
    assert list(P.load_plan(os.path.join(out, "plan.json")).omega_c) == list(rep.plan.omega_c)
    assert open(os.path.join(out, "objective.csv")).readline() == "iteration,objective\n"
