"""Pins the CPU oracle against the reference's own known answers.

Each test transcribes a case of proj/tests/test_numeric.cpp,
proj/tests/test_graph.cpp or a SPEC.md example (file:line cited), with the
reference's tolerance.  The dense oracles of proj/tests/oracles.hpp are
restated with numpy/LAPACK (never through the sparse/iterative paths under
test).  These run on CPU only.
"""
import math

import numpy as np
import pytest

from oracle import pyoracle as O


def path3():
    # test_numeric.cpp:16-25
    return O.Csr.from_triplets(3, 3, [0, 0, 1, 1, 1, 2, 2], [0, 1, 0, 1, 2, 1, 2],
                               [1.0, -1.0, -1.0, 2.0, -1.0, -1.0, 1.0])


def complete4():
    # test_numeric.cpp:27-35
    ti, tj, tv = [], [], []
    for i in range(4):
        ti.append(i), tj.append(i), tv.append(3.0)
        for j in range(4):
            if i != j:
                ti.append(i), tj.append(j), tv.append(-1.0)
    return O.Csr.from_triplets(4, 4, ti, tj, tv)


def random_graph_adjacency(n, edge_prob, seed, connect=True):
    """oracles.hpp:129-142 restated on the oracle RNG stream."""
    s = O.rng_mix(seed ^ 0x6772617068)
    u = iter(O.rng_u64(s, 4 * n * n + 16))

    def nd():
        return float(int(next(u)) >> 11) * 2.0 ** -53

    ti, tj, tv = [], [], []
    for i in range(n):
        for j in range(i + 1, n):
            chain = connect and j == i + 1
            if not chain and nd() >= edge_prob:
                continue
            w = 0.05 + 0.95 * nd()
            ti += [i, j]
            tj += [j, i]
            tv += [w, w]
    return O.Csr.from_triplets(n, n, ti, tj, tv)


def dense_laplacian(W: O.Csr):
    Wd = W.to_dense()
    return np.diag(Wd.sum(axis=1)) - Wd


def dense_kron(L, keep):
    """oracles.hpp:52-60 (LDLT Schur complement), numpy solve."""
    n = L.shape[0]
    keep = list(keep)
    inter = [i for i in range(n) if i not in set(keep)]
    Lbb = L[np.ix_(keep, keep)]
    if not inter:
        return Lbb
    Laa = L[np.ix_(inter, inter)]
    Lab = L[np.ix_(inter, keep)]
    Lba = L[np.ix_(keep, inter)]
    return Lbb - Lba @ np.linalg.solve(Laa, Lab)


# ------------------------------------------------------------------ CSR
def test_csr_merges_duplicates_and_drops_zeros():
    # test_numeric.cpp:39-50
    A = O.Csr.from_triplets(2, 3, [0, 0, 1, 1, 1], [2, 2, 0, 1, 1], [1.0, 2.0, 5.0, -5.0, 5.0])
    assert A.nnz == 2
    D = A.to_dense()
    assert D[0, 2] == 3.0 and D[1, 0] == 5.0 and D[1, 1] == 0.0
    rp, ci, _ = A.arrays()
    assert np.all(np.diff(rp) >= 0)


def test_csr_round_trip_against_dense_accumulation():
    # test_numeric.cpp:52-65 (40 random triplets with duplicates, <= 1e-15)
    rs = np.random.default_rng(7)
    ti = rs.integers(0, 6, 40)
    tj = rs.integers(0, 5, 40)
    tv = rs.standard_normal(40)
    dense = np.zeros((6, 5))
    for i, j, v in zip(ti, tj, tv):
        dense[i, j] += v
    A = O.Csr.from_triplets(6, 5, ti, tj, tv)
    assert np.abs(A.to_dense() - dense).max() <= 1e-15


def test_triplet_validation():
    with pytest.raises(ValueError, match="index out of range"):
        O.Csr.from_triplets(2, 2, [2], [0], [1.0])
    with pytest.raises(ValueError, match="non-finite"):
        O.Csr.from_triplets(2, 2, [0], [0], [np.inf])


def test_spmv_identity_and_zero():
    # test_numeric.cpp:67-74 / SPEC.md:42-43
    x = np.array([1.0, 2.0, 3.0])
    eye = O.Csr.from_triplets(3, 3, [0, 1, 2], [0, 1, 2], [1.0, 1.0, 1.0])
    assert np.array_equal(eye.spmv(x), x)
    zero = O.Csr.from_triplets(3, 3, [], [], [])
    assert np.linalg.norm(zero.spmv(x)) == 0.0


def test_spmv_spmm_match_dense_product():
    # test_numeric.cpp:76-85 (<= 1e-14)
    D = O.gaussian_matrix(5, 5, 11)
    A = O.Csr.from_dense(D)
    x = O.gaussian_matrix(5, 1, 12)[:, 0]
    assert np.abs(A.spmv(x) - D @ x).max() <= 1e-14
    X = O.gaussian_matrix(5, 3, 13)
    assert np.abs(A.multiply(X) - D @ X).max() <= 1e-14
    assert np.abs(A.right_multiply(X.T) - X.T @ D).max() <= 1e-14


def test_spmv_dimension_mismatch_throws():
    # test_numeric.cpp:87-90
    eye = O.Csr.from_triplets(3, 3, [0, 1, 2], [0, 1, 2], [1.0, 1.0, 1.0])
    with pytest.raises(ValueError, match="dimension mismatch"):
        eye.spmv(np.zeros(4))


def test_submatrix_is_pure_gather():
    # test_numeric.cpp:92-98
    D = O.gaussian_matrix(6, 6, 21)
    A = O.Csr.from_dense(D)
    rows, cols = [4, 0, 2], [1, 5]
    assert np.array_equal(A.submatrix(rows, cols).to_dense(), D[np.ix_(rows, cols)])


def test_connected_components_two_blocks():
    # test_numeric.cpp:100-108
    W = O.Csr.from_triplets(5, 5, [0, 1, 1, 2, 3, 4], [1, 0, 2, 1, 4, 3], [1.0] * 6)
    lab, nc = W.components()
    assert nc == 2
    assert list(lab) == [0, 0, 0, 1, 1]


# ------------------------------------------------------------------ PCG
def test_pcg_identity_one_iteration():
    # test_numeric.cpp:110-118
    eye = O.Csr.from_triplets(4, 4, range(4), range(4), [1.0] * 4)
    b = O.gaussian_matrix(4, 1, 31)[:, 0]
    x, r = O.pcg_solve(eye, b)
    assert r.converged and r.iterations == 1
    assert np.linalg.norm(x - b) <= 1e-12 * np.linalg.norm(b)


def test_pcg_diagonal_solve():
    # test_numeric.cpp:120-129 / SPEC.md:52
    A = O.Csr.from_triplets(3, 3, [0, 1, 2], [0, 1, 2], [1.0, 2.0, 4.0])
    x, r = O.pcg_solve(A, [1.0, 2.0, 4.0])
    assert r.converged
    assert np.abs(x - 1.0).max() <= 1e-12


def test_pcg_grounded_path_block_matches_dense_lu():
    # test_numeric.cpp:131-145
    L = path3().to_dense()
    Ab = L[np.ix_([1, 2], [1, 2])]
    A = O.Csr.from_dense(Ab)
    b = O.gaussian_matrix(2, 1, 32)[:, 0]
    x, r = O.pcg_solve(A, b, tol=1e-12)
    assert r.converged
    assert np.abs(x - np.linalg.solve(Ab, b)).max() <= 1e-10


def test_pcg_residual_contract_random_spd():
    # test_numeric.cpp:147-160
    for seed in range(5):
        G = O.gaussian_matrix(12, 12, 100 + seed)
        S = G @ G.T + 0.5 * np.eye(12)
        A = O.Csr.from_dense(S)
        b = O.gaussian_matrix(12, 1, 200 + seed)[:, 0]
        x, r = O.pcg_solve(A, b, tol=1e-9)
        assert r.converged
        assert np.linalg.norm(S @ x - b) <= 1e-9 * np.linalg.norm(b) * 1.0000001


def test_pcg_breakdown_names_iteration():
    # test_numeric.cpp:162-169
    zero = O.Csr.from_triplets(2, 2, [], [], [])
    with pytest.raises(RuntimeError, match="iteration 0"):
        O.pcg_solve(zero, [1.0, 1.0], jacobi=False)


def test_pcg_zero_rhs():
    # test_numeric.cpp:171-177
    eye = O.Csr.from_triplets(3, 3, range(3), range(3), [1.0] * 3)
    x, r = O.pcg_solve(eye, np.zeros(3))
    assert r.converged and r.iterations == 0 and np.linalg.norm(x) == 0.0


# ------------------------------------------------------------------ power iteration
def test_power_iteration_diagonal():
    # test_numeric.cpp:179-183 / SPEC.md:60
    A = O.Csr.from_triplets(3, 3, [0, 1, 2], [0, 1, 2], [1.0, 5.0, 3.0])
    assert O.power_iteration_norm(A, 1e-12, 3) == pytest.approx(5.0, rel=1e-9)


def test_power_iteration_complete_graph():
    # test_numeric.cpp:185-189 / SPEC.md:61
    assert O.power_iteration_norm(complete4(), 1e-12, 5) == pytest.approx(4.0, rel=1e-9)


def test_power_iteration_zero_matrix():
    # test_numeric.cpp:191-193
    assert O.power_iteration_norm(O.Csr.from_triplets(4, 4, [], [], []), 1e-10, 9) == 0.0


def test_power_iteration_deterministic():
    # test_numeric.cpp:195-199
    G = O.gaussian_matrix(8, 8, 41)
    A = O.Csr.from_dense(G + G.T)
    assert O.power_iteration_norm(A, 1e-10, 7) == O.power_iteration_norm(A, 1e-10, 7)


# ------------------------------------------------------------------ RNG
def test_counter_rng_is_splitmix64():
    # rng.hpp:15-24: the i-th output is mix(seed + golden * i), i from 1.
    seed = 1602
    out = O.rng_u64(seed, 4)
    golden = 0x632BE59BD9B4E019
    for i, v in enumerate(out, start=1):
        assert int(v) == O.rng_mix((seed + golden * i) & 0xFFFFFFFFFFFFFFFF)
    # Known-answer of the SplitMix64 finaliser (Steele et al.) at 0.
    assert O.rng_mix(0) == 0xE220A8397B1DCDAF


# ------------------------------------------------------------------ kNN graph
def check_graph_invariants(g):
    # test_graph.cpp:35-47
    W = g.adjacency.to_dense()
    assert np.array_equal(W, W.T)
    assert np.all(np.diag(W) == 0.0)
    _, _, v = g.adjacency.arrays()
    assert np.all(v > 0.0) and np.all(v <= 1.0)
    assert np.array_equal(g.degrees, g.adjacency.row_sums())
    if not g.normalized:
        assert np.abs(g.laplacian.row_sums()).max() <= 1e-12
    assert np.linalg.eigvalsh(g.laplacian.to_dense())[0] >= -1e-10


def test_knn_coincident_points_weight_one():
    # test_graph.cpp:51-58 / SPEC.md:131
    X = np.array([[1.0, 1.0], [2.0, 2.0]])
    g = O.build_knn_graph(X, False, 1)
    W = g.adjacency.to_dense()
    assert W[0, 1] == 1.0 and W[1, 0] == 1.0
    check_graph_invariants(g)


def test_knn_collinear_points_exhaustive_kernel():
    # test_graph.cpp:60-75 / SPEC.md:132
    X = np.array([[0.0, 1.0, 10.0]])
    g = O.build_knn_graph(X, False, 1)
    s2 = (1.0 + 1.0 + 81.0) / 3.0
    assert g.sigma2 == pytest.approx(s2, rel=1e-15)
    W = g.adjacency.to_dense()
    assert W[0, 1] == pytest.approx(math.exp(-1.0 / s2), rel=1e-15)
    assert W[1, 2] == pytest.approx(math.exp(-81.0 / s2), rel=1e-15)
    assert W[0, 2] == 0.0
    assert g.adjacency.nnz == 4
    check_graph_invariants(g)


def test_knn_ties_break_toward_lower_index():
    # test_graph.cpp:77-86
    X = np.array([[0.0, 1.0, 0.0, 5.0], [0.0, 0.0, 1.0, 5.0]])
    W = O.build_knn_graph(X, False, 1).adjacency.to_dense()
    assert W[1, 3] > 0.0
    assert W[2, 3] == 0.0


def test_knn_rows_axis_equals_cols_axis_on_transpose():
    # test_graph.cpp:88-93
    X = O.gaussian_matrix(6, 12, 17)
    a = O.build_knn_graph(X, True, 2)
    b = O.build_knn_graph(X.T, False, 2)
    assert np.array_equal(a.adjacency.to_dense(), b.adjacency.to_dense())


def test_knn_errors():
    # test_graph.cpp:95-103
    with pytest.raises(ValueError):
        O.build_knn_graph(np.array([[0.0, 1.0, 2.0]]), False, 3)
    with pytest.raises(ValueError, match="fewer distinct points"):
        O.build_knn_graph(np.array([[2.0, 2.0, 2.0, 2.0]]), False, 2)
    with pytest.raises(ValueError, match="K must be"):
        O.build_knn_graph(np.array([[0.0, 1.0, 2.0]]), False, 0)


def test_knn_normalized_laplacian_dense_formula():
    # test_graph.cpp:105-114
    X = O.gaussian_matrix(4, 10, 23)
    g = O.build_knn_graph(X, False, 3, normalized=True)
    W = g.adjacency.to_dense()
    deg = W.sum(axis=1)
    Dinv = np.diag(np.where(deg > 0, 1.0 / np.sqrt(deg), 0.0))
    Ln = Dinv @ (np.diag(deg) - W) @ Dinv
    assert np.abs(g.laplacian.to_dense() - Ln).max() <= 1e-14


def test_knn_sigma2_positive_and_override():
    # test_graph.cpp:116-122
    X = O.gaussian_matrix(3, 8, 29)
    assert O.build_knn_graph(X, False, 2).sigma2 > 0.0
    assert O.build_knn_graph(X, False, 2, sigma2_override=2.5).sigma2 == 2.5


def test_knn_exhaustive_neighbour_sets():
    """Brute-force oracle: sorted (d2, j) pairs per point."""
    X = O.gaussian_matrix(7, 40, 77)
    nbr, d2 = O.knn_neighbors(X, False, 5)
    P = X.T
    for i in range(40):
        cand = sorted((max(0.0, P[i] @ P[i] + P[j] @ P[j] - 2 * (P[i] @ P[j])), j)
                      for j in range(40) if j != i)
        assert [j for _, j in cand[:5]] == list(nbr[i])


# ------------------------------------------------------------------ Kron
def test_kron_keep_all_returns_l():
    # test_graph.cpp:171-175 / SPEC.md:149
    L = path3()
    R = O.kron_reduce(L, [0, 1, 2])
    assert np.array_equal(R.to_dense(), L.to_dense())


def test_kron_path_endpoints_series_resistors():
    # test_graph.cpp:177-182 / SPEC.md:150
    R = O.kron_reduce(path3(), [0, 2])
    assert np.abs(R.to_dense() - np.array([[0.5, -0.5], [-0.5, 0.5]])).max() <= 1e-12


def test_kron_disconnected_stays_disconnected():
    # test_graph.cpp:184-192 / SPEC.md:151
    L = O.Csr.from_triplets(4, 4, [0, 0, 1, 1, 2, 2, 3, 3], [0, 1, 0, 1, 2, 3, 2, 3],
                            [1.0, -1.0, -1.0, 1.0, 2.0, -2.0, -2.0, 2.0])
    R = O.kron_reduce(L, [0, 2])
    assert R.nnz == 0 and R.rows == 2


def test_kron_matches_dense_schur_on_random_graphs():
    # test_graph.cpp:194-213 (<= 1e-10, Laplacian structure survives)
    for seed in range(8):
        n = 10 + 5 * seed
        W = random_graph_adjacency(n, 0.15, 1000 + seed)
        Ld = dense_laplacian(W)
        u = O.rng_u64(O.rng_mix(seed), n)
        keep = [i for i in range(n) if (float(int(u[i]) >> 11) * 2.0 ** -53) < 0.4 or i == 0]
        R = O.kron_reduce(O.Csr.from_dense(Ld), keep)
        Rd = R.to_dense()
        assert np.abs(Rd - dense_kron(Ld, keep)).max() <= 1e-10
        assert np.abs(Rd - Rd.T).max() <= 1e-12
        assert np.abs(R.row_sums()).max() <= 1e-9
        assert np.linalg.eigvalsh(Rd)[0] >= -1e-10


def test_kron_component_count_preserved():
    # test_graph.cpp:215-234
    ti, tj, tv = [], [], []
    for (i, j, w) in [(0, 1, 1.0), (1, 2, 1.0), (3, 4, 1.0)]:
        ti += [i, j, i, j]
        tj += [j, i, i, j]
        tv += [-w, -w, w, w]
    L = O.Csr.from_triplets(5, 5, ti, tj, tv)
    R = O.kron_reduce(L, [0, 2, 3, 4])
    ev = np.linalg.eigvalsh(R.to_dense())
    assert int(np.sum(np.abs(ev) <= 1e-10)) == 2


def test_kron_ungrounded_component_error():
    # test_graph.cpp:236-242
    L = O.Csr.from_triplets(4, 4, [0, 0, 1, 1, 2, 2, 3, 3], [0, 1, 0, 1, 2, 3, 2, 3],
                            [1.0, -1.0, -1.0, 1.0, 1.0, -1.0, -1.0, 1.0])
    with pytest.raises(RuntimeError, match="node 2"):
        O.kron_reduce(L, [0, 1])


# ------------------------------------------------------------------ sampling
def test_draw_plan_full_is_permutation():
    # SPEC.md:209
    plan = O.draw_plan(7, 9, 7, 9, seed=3)
    assert sorted(plan.omega_r) == list(range(7))
    assert sorted(plan.omega_c) == list(range(9))


def test_draw_plan_deterministic_and_uniform():
    # SPEC.md:210-211
    a = O.draw_plan(50, 80, 10, 20, seed=11)
    b = O.draw_plan(50, 80, 10, 20, seed=11)
    assert np.array_equal(a.omega_r, b.omega_r) and np.array_equal(a.omega_c, b.omega_c)
    counts = np.zeros(10)
    for s in range(10000):
        counts[O.draw_plan(10, 10, 1, 1, seed=s).omega_r[0]] += 1
    freq = counts / 10000
    assert np.all(freq >= 0.08) and np.all(freq <= 0.12)


def test_draw_plan_matches_fisher_yates_restatement():
    # sampling.cpp:35-64 restated in Python on the oracle's raw u64 stream.
    p, n, rr, rc, seed = 37, 53, 9, 14, 1602

    def shuffle(N, take, stream):
        s = O.rng_derive_seed(seed, stream)
        u = iter(O.rng_u64(s, 4 * take + 64))
        pool = list(range(N))
        for i in range(take):
            m = N - i
            lim = 0xFFFFFFFFFFFFFFFF - 0xFFFFFFFFFFFFFFFF % m
            v = int(next(u))
            while v >= lim:
                v = int(next(u))
            j = i + v % m
            pool[i], pool[j] = pool[j], pool[i]
        return pool[:take]

    plan = O.draw_plan(p, n, rr, rc, seed=seed)
    assert list(plan.omega_r) == shuffle(p, rr, 0x726F7773)
    assert list(plan.omega_c) == shuffle(n, rc, 0x636F6C73)


def test_draw_plan_errors():
    with pytest.raises(ValueError, match="rho_r out of range"):
        O.draw_plan(5, 5, 6, 1)
    with pytest.raises(ValueError, match="rho_c out of range"):
        O.draw_plan(5, 5, 1, 0)


def test_subsample_is_selection_product():
    # SPEC.md:218-220
    Y = O.gaussian_matrix(8, 11, 5)
    plan = O.draw_plan(8, 11, 3, 4, seed=9)
    Mr = np.zeros((3, 8))
    Mr[np.arange(3), plan.omega_r] = 1.0
    Mc = np.zeros((11, 4))
    Mc[plan.omega_c, np.arange(4)] = 1.0
    assert np.array_equal(O.subsample(Y, plan), Mr @ Y @ Mc)
    one = O.SamplingPlan(np.array([2]), np.array([7]), 8, 11)
    assert O.subsample(Y, one)[0, 0] == Y[2, 7]


# ------------------------------------------------------------------ FRPCAG
def test_prox_l1_examples():
    # SPEC.md:278-280
    assert O.prox_l1([[3.0]], [[0.0]], 1.0)[0, 0] == 2.0
    assert O.prox_l1([[-0.5]], [[0.0]], 1.0)[0, 0] == 0.0
    Z = O.gaussian_matrix(3, 4, 1)
    Y = O.gaussian_matrix(3, 4, 2)
    # Y + sign(Z-Y)|Z-Y| reproduces Z up to the rounding of Z-Y.
    assert np.abs(O.prox_l1(Z, Y, 0.0) - Z).max() <= 1e-15 * 4
    assert np.array_equal(O.prox_l1(Y, Y, 0.7), Y)


def small_problem(seed=3, r=6, c=5):
    Wr = random_graph_adjacency(r, 0.5, seed)
    Wc = random_graph_adjacency(c, 0.5, seed + 1)
    Lr = O.Csr.from_dense(dense_laplacian(Wr))
    Lc = O.Csr.from_dense(dense_laplacian(Wc))
    Y = O.gaussian_matrix(r, c, seed + 2)
    return Y, Lr, Lc


def test_objective_constants_and_dense_trace():
    # SPEC.md:269-271
    Y, Lr, Lc = small_problem()
    ones = np.ones_like(Y)
    cfg = O.FrpcagConfig(gamma_r=2.0, gamma_c=3.0)
    assert abs(O.objective(ones, ones, Lr, Lc, cfg)) <= 1e-12
    X = O.gaussian_matrix(6, 5, 99)
    Lrd, Lcd = Lr.to_dense(), Lc.to_dense()
    want = np.abs(Y - X).sum() + 3.0 * np.trace(X @ Lcd @ X.T) + 2.0 * np.trace(X.T @ Lrd @ X)
    assert O.objective(X, Y, Lr, Lc, cfg) == pytest.approx(want, rel=1e-12)
    cfg0 = O.FrpcagConfig(gamma_r=0.0, gamma_c=0.0)
    assert O.objective(X, Y, Lr, Lc, cfg0) == pytest.approx(np.abs(Y - X).sum(), rel=1e-14)


def test_grad_g_zero_on_constants_and_finite_differences():
    # SPEC.md:287-289
    Y, Lr, Lc = small_problem()
    cfg = O.FrpcagConfig(gamma_r=1.5, gamma_c=0.5, loss="l2")
    assert np.abs(O.grad_g(np.ones_like(Y), Lr, Lc, cfg)).max() <= 1e-12
    Z = O.gaussian_matrix(6, 5, 7)
    G = O.grad_g(Z, Lr, Lc, cfg)
    Lrd, Lcd = Lr.to_dense(), Lc.to_dense()

    def g(M):
        return 0.5 * np.trace(M @ Lcd @ M.T) + 1.5 * np.trace(M.T @ Lrd @ M)

    h = 1e-6
    num = np.zeros_like(Z)
    for i in range(6):
        for j in range(5):
            E = np.zeros_like(Z)
            E[i, j] = h
            num[i, j] = (g(Z + E) - g(Z - E)) / (2 * h)
    assert np.abs(G - num).max() <= 1e-5


def test_fista_zero_gamma_is_prox_fixed_point():
    # SPEC.md:296
    Y, Lr, Lc = small_problem()
    X, tr = O.fista_solve(Y, Lr, Lc, O.FrpcagConfig(gamma_r=0.0, gamma_c=0.0))
    assert np.array_equal(X, Y)
    assert tr.iterations == 1 and tr.converged


def test_fista_l2_matches_dense_quadratic_minimizer():
    # SPEC.md:297 / oracles.hpp:96-106 (normal equations of the vectorised problem)
    Y, Lr, Lc = small_problem(seed=5)
    cfg = O.FrpcagConfig(gamma_r=0.3, gamma_c=0.2, loss="l2", tol=1e-30, max_iter=4000)
    X, tr = O.fista_solve(Y, Lr, Lc, cfg)
    r, c = Y.shape
    Lrd, Lcd = Lr.to_dense(), Lc.to_dense()
    op = np.kron(np.eye(c), np.eye(r)) + 0.2 * np.kron(Lcd.T, np.eye(r)) + 0.3 * np.kron(np.eye(c), Lrd)
    want = np.linalg.solve(op, Y.reshape(-1, order="F")).reshape((r, c), order="F")
    assert np.linalg.norm(X - want) <= 1e-6 * np.linalg.norm(want)
    assert tr.objective[-1] <= tr.objective[0]


def test_fista_l1_objective_decreases_and_trace_fields():
    # SPEC.md:301 (final <= initial)
    Y, Lr, Lc = small_problem(seed=8, r=9, c=7)
    cfg = O.FrpcagConfig(gamma_r=1.0, gamma_c=1.0, tol=1e-300, max_iter=50)
    X, tr = O.fista_solve(Y, Lr, Lc, cfg)
    assert tr.iterations == 50 and not tr.converged and len(tr.objective) == 50
    assert tr.objective[-1] <= tr.objective[0]
    beta = 2 * O.power_iteration_norm(Lc, 1e-7, 42) + 2 * O.power_iteration_norm(Lr, 1e-7, 42)
    assert tr.step == 1.0 / beta


def test_fista_validation():
    Y, Lr, Lc = small_problem()
    with pytest.raises(ValueError, match="negative regularization"):
        O.fista_solve(Y, Lr, Lc, O.FrpcagConfig(gamma_r=-1.0))
    with pytest.raises(ValueError, match="tolerance must be positive"):
        O.fista_solve(Y, Lr, Lc, O.FrpcagConfig(tol=0.0))
    with pytest.raises(ValueError, match="column Laplacian"):
        O.fista_solve(Y, Lr, Lr, O.FrpcagConfig())
    with pytest.raises(RuntimeError, match="diverged"):
        O.fista_solve(Y * 1e300, Lr, Lc, O.FrpcagConfig(step=10.0, max_iter=20, tol=1e-300))


# ------------------------------------------------------------------ alternate decoder
def test_alternate_decoder_matches_dense_normal_equations():
    # SPEC.md:360 / oracles.hpp:109-125 (<= 1e-8)
    p, n = 9, 8
    Lr = O.Csr.from_dense(dense_laplacian(random_graph_adjacency(p, 0.4, 21)))
    Lc = O.Csr.from_dense(dense_laplacian(random_graph_adjacency(n, 0.4, 22)))
    plan = O.draw_plan(p, n, 4, 3, seed=5)
    Xt = O.gaussian_matrix(4, 3, 23)
    res = O.alternate_decode(Xt, plan, Lr, Lc, 2.0, 4.0, gamma=1.0, pcg_tol=1e-14,
                             pcg_max_iter=5000)
    gr, gc = 1.0 / 2.0, 1.0 / 4.0
    Mr = np.zeros((4, p))
    Mr[np.arange(4), plan.omega_r] = 1
    Mc = np.zeros((n, 3))
    Mc[plan.omega_c, np.arange(3)] = 1
    op = (np.kron((Mc @ Mc.T).T, Mr.T @ Mr) + gc * np.kron(Lc.to_dense().T, np.eye(p))
          + gr * np.kron(np.eye(n), Lr.to_dense()))
    rhs = (Mr.T @ Xt @ Mc.T).reshape(-1, order="F")
    want = np.linalg.solve(op, rhs).reshape((p, n), order="F")
    assert np.abs(res.X - want).max() <= 1e-8
    assert res.converged


def test_alternate_decoder_zero_data_and_validation():
    # SPEC.md:358
    p, n = 6, 5
    Lr = O.Csr.from_dense(dense_laplacian(random_graph_adjacency(p, 0.5, 1)))
    Lc = O.Csr.from_dense(dense_laplacian(random_graph_adjacency(n, 0.5, 2)))
    plan = O.draw_plan(p, n, 3, 2, seed=1)
    res = O.alternate_decode(np.zeros((3, 2)), plan, Lr, Lc, 1.0, 1.0)
    assert np.array_equal(res.X, np.zeros((p, n))) and res.converged and res.iterations == 0
    with pytest.raises(ValueError, match="gamma must be positive"):
        O.alternate_decode(np.ones((3, 2)), plan, Lr, Lc, 1.0, 1.0, gamma=0.0)
