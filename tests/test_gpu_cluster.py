"""GPU parity of the clustering path (cluster.cu) against the oracle
restatement of clustering.cpp:40-238: kmeans assignments bit-identical
(sequential distance sums, in-order centroid sums, device counter RNG),
decode_labels equal to the oracle's upsample + max pooling, the SPEC.md
examples, and the reference's error texts."""
import numpy as np
import pytest

from helpers import knn_laplacian, to_device
from oracle import pyoracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    import paper_1602_02070_b200 as P

    return P


@pytest.fixture(scope="module")
def ctx(P):
    return P.Context(0)


def _blobs(rows, per, k, seed, spread=0.6):
    rs = np.random.default_rng(seed)
    centres = rs.standard_normal((rows, k)) * 3.0
    X = np.concatenate([centres[:, [c]] + spread * rs.standard_normal((rows, per)) for c in range(k)], axis=1)
    return X[:, rs.permutation(X.shape[1])]


@pytest.mark.parametrize("rows,per,k,restarts,seed", [(5, 40, 3, 4, 0), (20, 60, 7, 3, 11), (1031, 10, 10, 10, 1603),
                                                      (3, 30, 12, 2, 5)])
def test_kmeans_bit_identical_to_oracle(P, ctx, rows, per, k, restarts, seed):
    X = _blobs(rows, per, min(k, 6), seed)
    lab = P.kmeans(X, k, restarts=restarts, seed=seed, ctx=ctx)
    a, w = O.kmeans(X, k, restarts=restarts, seed=seed)
    assert lab.k == k and np.array_equal(lab.assignments, a)


def test_kmeans_fp32_input_and_spec_examples(P, ctx):
    rs = np.random.default_rng(3)
    X = rs.standard_normal((4, 50)).astype(np.float32)
    lab = P.kmeans(X, 3, restarts=2, seed=1, ctx=ctx)
    assert np.array_equal(lab.assignments, O.kmeans(X.astype(np.float64), 3, 2, 1)[0])
    assert np.all(P.kmeans(X, 1, ctx=ctx).assignments == 0)
    Y = np.concatenate([rs.standard_normal((3, 20)) * 0.1, rs.standard_normal((3, 25)) * 0.1 + 40], axis=1)
    a = P.kmeans(Y, 2, restarts=3, seed=2, ctx=ctx).assignments
    assert len(set(a[:20])) == 1 and len(set(a[20:])) == 1 and a[0] != a[20]
    with pytest.raises(ValueError, match="more clusters than points"):
        P.kmeans(X, 51, ctx=ctx)
    with pytest.raises(ValueError, match="restarts must be >= 1"):
        P.kmeans(X, 2, restarts=0, ctx=ctx)


def test_kmeans_empty_cluster_reseed_matches_oracle(P, ctx):
    """Many duplicate points and k close to the number of distinct points:
    Lloyd empties clusters, re-seeded from the farthest point."""
    rs = np.random.default_rng(8)
    base = rs.standard_normal((2, 6))
    X = base[:, rs.integers(0, 6, 80)] + 1e-9 * rs.standard_normal((2, 80))
    for seed in range(6):
        lab = P.kmeans(X, 9, restarts=2, seed=seed, ctx=ctx)
        assert np.array_equal(lab.assignments, O.kmeans(X, 9, 2, seed)[0])


def test_decode_labels_matches_oracle(P, ctx):
    n, k = 600, 4
    Lc = knn_laplacian(n, 3, 10, 21)
    plan_o = O.draw_plan(50, n, 10, 60, seed=4)
    sampled = np.random.default_rng(2).integers(0, k, 60)
    lab_o, _ = O.decode_labels(sampled, k, plan_o, Lc, 1e-10, 5000)
    plan = P.SamplingPlan(plan_o.omega_r, plan_o.omega_c, plan_o.p, plan_o.n)
    lab = P.decode_labels(P.ClusterLabels.from_assignments(sampled, k), plan, to_device(ctx, Lc), ctx=ctx)
    assert np.array_equal(lab.assignments, lab_o)
    # sampled columns keep their labels (upsampling interpolates)
    assert np.array_equal(lab.assignments[plan_o.omega_c], sampled)
    with pytest.raises(ValueError, match="sampled labels do not match plan"):
        P.decode_labels(P.ClusterLabels.from_assignments(sampled[:-1], k), plan, to_device(ctx, Lc), ctx=ctx)


def test_decode_labels_component_example_and_clustering_error(P, ctx):
    from test_oracle_approx import blocks_laplacian

    L = blocks_laplacian([8, 11, 6], 3)
    plan = P.SamplingPlan(np.arange(3), np.array([2, 12, 21]), 3, 25)
    lab = P.decode_labels(P.ClusterLabels.from_assignments([0, 1, 2], 3), plan, to_device(ctx, L), ctx=ctx)
    assert list(lab.assignments) == [0] * 8 + [1] * 11 + [2] * 6
    t = P.ClusterLabels.from_assignments([0, 0, 1, 1], 2)
    assert P.clustering_error(P.ClusterLabels.from_assignments([1, 1, 1, 1], 2), t) == 0.5
    assert P.clustering_error(P.ClusterLabels.from_assignments([1, 1, 0, 0], 2), t) == 0.0
    rs = np.random.default_rng(1)
    for _ in range(10):
        p, q = rs.integers(0, 5, 40), rs.integers(0, 5, 40)
        assert P.clustering_error(P.ClusterLabels(p, 5), P.ClusterLabels(q, 5)) == O.clustering_error(p, q, 5)
    with pytest.raises(ValueError, match="cluster counts differ"):
        P.clustering_error(P.ClusterLabels(np.zeros(4, np.int32), 2), P.ClusterLabels(np.zeros(4, np.int32), 3))


@pytest.mark.parametrize("task", ["cluster", "both"])
def test_pipeline_cluster_task_matches_oracle(P, ctx, task):
    """run_pipeline with the clustering task (pipeline.cpp:371-388): k-means on
    Xt (seed mix(seed ^ "kmean")) then decode_labels over the column graph."""
    rs = np.random.default_rng(31)
    p, n, k = 40, 90, 3
    centres = rs.standard_normal((p, k)) * 4.0
    truth = np.repeat(np.arange(k), n // k)
    Y = np.asfortranarray(centres[:, truth] + 0.3 * rs.standard_normal((p, n)))
    g = float(np.sqrt(max(p, n)))
    cfg = P.PipelineConfig(knn=10, a=3, b=2, kron_pcg_tol=1e-11,
                           frpcag=P.FrpcagConfig(gamma_r=g, gamma_c=g, loss="l1", tol=1e-300, max_iter=50),
                           decoder=P.DecoderConfig(gamma=1.0, pcg_tol=1e-10, pcg_max_iter=500, variant="alternate"),
                           lambda_k1_r=0.1, lambda_k1_c=0.1, seed=77, task=task, n_clusters=k, kmeans_restarts=4)
    rep = P.run_pipeline(Y, cfg, ctx=ctx)
    assert rep.labels is not None and rep.labels.shape == (n,)
    assert (rep.X is None) == (task == "cluster")
    # oracle composite
    gr, gc = O.build_knn_graph(Y, True, 10), O.build_knn_graph(Y, False, 10)
    plan = O.draw_plan(p, n, -(-p // 2), -(-n // 3), seed=77)
    assert np.array_equal(rep.plan.omega_c, plan.omega_c)
    Xt, _ = O.fista_solve(O.subsample(Y, plan), O.kron_reduce(gr.laplacian, plan.omega_r, 1e-11),
                          O.kron_reduce(gc.laplacian, plan.omega_c, 1e-11), O.FrpcagConfig(g, g, "l1", 1e-300, 50))
    a, _ = O.kmeans(Xt, k, 4, O.rng_mix(77 ^ 0x6B6D65616E))
    lab, _ = O.decode_labels(a, k, plan, gc.laplacian, 1e-10, 500)
    assert np.array_equal(rep.labels, lab)
    assert O.clustering_error(rep.labels, truth, k) <= 0.05
