"""The clustering restatement (oracle, clustering.cpp:40-238) against the
SPEC.md examples of the clustering module and a brute-force
permutation oracle for clustering_error."""
import itertools

import numpy as np
import pytest

from oracle import pyoracle as O


def test_kmeans_spec_examples():
    rs = np.random.default_rng(0)
    X = rs.standard_normal((3, 40))
    a, _ = O.kmeans(X, 1, restarts=3, seed=5)
    assert np.all(a == 0)  # k = 1 -> one cluster
    # two well-separated clouds -> the construction's partition
    Y = np.concatenate([rs.standard_normal((4, 30)) * 0.1, rs.standard_normal((4, 25)) * 0.1 + 50.0], axis=1)
    a, _ = O.kmeans(Y, 2, restarts=5, seed=1)
    assert len(set(a[:30])) == 1 and len(set(a[30:])) == 1 and a[0] != a[30]
    # duplicate points are co-assigned
    Z = np.concatenate([X, X[:, :7]], axis=1)
    a, _ = O.kmeans(Z, 4, restarts=4, seed=2)
    assert np.array_equal(a[:7], a[40:])
    # deterministic given seed
    assert np.array_equal(O.kmeans(X, 3, 4, 9)[0], O.kmeans(X, 3, 4, 9)[0])


def test_kmeans_errors():
    X = np.ones((2, 3))
    with pytest.raises(ValueError, match="k must be >= 1"):
        O.kmeans(X, 0)
    with pytest.raises(ValueError, match="more clusters than points"):
        O.kmeans(X, 4)
    with pytest.raises(ValueError, match="restarts must be >= 1"):
        O.kmeans(X, 2, restarts=0)


def test_clustering_error_spec_and_brute_force():
    assert O.clustering_error([1, 1, 1, 1], [0, 0, 1, 1], 2) == 0.5
    assert O.clustering_error([2, 2, 0, 1], [0, 0, 1, 2], 3) == 0.0
    rs = np.random.default_rng(4)
    for _ in range(20):
        k, n = 4, 30
        p, t = rs.integers(0, k, n), rs.integers(0, k, n)
        best = max(sum(perm[p[i]] == t[i] for i in range(n)) for perm in itertools.permutations(range(k)))
        assert O.clustering_error(p, t, k) == pytest.approx(1 - best / n, abs=1e-15)


def test_decode_labels_component_example():
    """k-component graph, one sampled node per component labelled by its
    component -> decoded labels = component membership."""
    from test_oracle_approx import blocks_laplacian

    L = blocks_laplacian([8, 11, 6], 3)
    plan = O.draw_plan(25, 25, 25, 25, seed=0)
    keep = np.array([2, 12, 21])
    plan.omega_c = keep
    lab, C = O.decode_labels([0, 1, 2], 3, plan, L)
    assert list(lab) == [0] * 8 + [1] * 11 + [2] * 6
    assert np.allclose(C.sum(axis=1), 1.0)
