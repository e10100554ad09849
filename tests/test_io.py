"""GLR1 container, CSV and plan JSON (io.cpp) -- host-side checks: the
numpy restatement (oracle/glr1.py) reproduces the committed fixtures, the
library's header parser reads them, and the mirror's CSV / plan-JSON
functions round-trip (binary bit-identical, CSV 17 digits,
header mismatch is an error)."""
import os

import numpy as np
import pytest

from oracle import glr1

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _bytes(name):
    return open(os.path.join(GOLD, name), "rb").read()


def test_oracle_reads_fixtures():
    k, M = glr1.read(_bytes("dense_3x4.glr1"))
    assert k == 1 and M.shape == (3, 4) and M[0, 3] == 1e-310 and np.signbit(M[1, 1])
    k, (r, c, rp, ci, v) = glr1.read(_bytes("csr_path5.glr1"))
    assert k == 2 and (r, c) == (5, 5) and rp[-1] == 13 and v.sum() == 0.0
    assert glr1.dense_bytes(M) == _bytes("dense_3x4.glr1")
    k, (U, s, V, sc) = glr1.read(_bytes("factors_4x3_k2.glr1"))
    UV = np.load(os.path.join(GOLD, "factors_4x3_k2_UV.npy"))
    assert k == 3 and sc and np.array_equal(np.concatenate([U, V]), UV) and list(s) == [3.5, 1.25]


def test_library_header_parser():
    from paper_1602_02070_b200 import glr1_info

    assert glr1_info(os.path.join(GOLD, "dense_3x4.glr1")) == (1, (3, 4))
    assert glr1_info(os.path.join(GOLD, "csr_path5.glr1")) == (2, (5, 5, 13))
    assert glr1_info(os.path.join(GOLD, "factors_4x3_k2.glr1")) == (3, (4, 3, 2, 1))
    with pytest.raises(RuntimeError, match="cannot open for reading"):
        glr1_info(os.path.join(GOLD, "missing.glr1"))
    with pytest.raises(RuntimeError, match=r"not a GLR1 container \(bad magic\)"):
        glr1_info(os.path.join(GOLD, "plan.json"))


def test_csv_round_trip_and_errors(tmp_path):
    import paper_1602_02070_b200 as P

    M = np.random.default_rng(3).standard_normal((5, 7)) * 1e3
    f = str(tmp_path / "m.csv")
    P.save_matrix(M, f, format="csv")
    assert open(f).readline() == "5,7\n"
    back = P.load_matrix(f, format="csv")
    assert np.array_equal(back, M)  # 17 significant digits round-trip doubles exactly
    open(f, "w").write("2,3\n1,2,3\n4,5\n")
    with pytest.raises(RuntimeError, match="row 2 has fewer than 3 columns"):
        P.load_matrix(f, format="csv")
    open(f, "w").write("1,2\n1,2,3\n")
    with pytest.raises(RuntimeError, match=r"more than 2 columns \(dimension header mismatch\)"):
        P.load_matrix(f, format="csv")
    open(f, "w").write("1,2\n1,x\n")
    with pytest.raises(RuntimeError, match="malformed number 'x' at line 2"):
        P.load_matrix(f, format="csv")


def test_plan_json_matches_fixture_and_round_trips(tmp_path):
    import paper_1602_02070_b200 as P

    plan = P.SamplingPlan(np.array([7, 2, 9]), np.array([0, 5]), 10, 8, 0.0, 0.25, 1603)
    assert P.plan_to_json(plan) + "\n" == open(os.path.join(GOLD, "plan.json")).read()
    back = P.load_plan(os.path.join(GOLD, "plan.json"))
    assert list(back.omega_r) == [7, 2, 9] and back.seed == 1603 and back.epsilon == 0.25
    f = str(tmp_path / "p.json")
    P.save_plan(P.draw_plan(100, 50, 10, 5, seed=9), f)
    again = P.load_plan(f)
    assert list(again.omega_r) == list(P.draw_plan(100, 50, 10, 5, seed=9).omega_r)
    bad = P.plan_to_json(plan).replace("9\n", "19\n")
    with pytest.raises(RuntimeError, match="omega_r index out of range"):
        P.plan_from_json(bad)
