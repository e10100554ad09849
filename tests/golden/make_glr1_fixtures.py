"""Writes the GLR1 / plan-JSON fixtures of tests/golden/ with the numpy
restatement of the reference container (oracle/glr1.py, io.cpp:16-263).
Run from the repo root: python tests/golden/make_glr1_fixtures.py"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle import glr1  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))
rs = np.random.default_rng(1602)
# dense 3 x 4 with exact binary fractions and one subnormal / negative zero
M = np.array([[1.0, -2.5, 0.125, 1e-310], [3.0, -0.0, 7.75, 1e300], [-1.5, 2.0**-20, 5.0, -6.25]])
open(os.path.join(OUT, "dense_3x4.glr1"), "wb").write(glr1.dense_bytes(M))
# CSR: 5-node path-graph Laplacian (canonical)
rp = [0, 2, 5, 8, 11, 13]
ci = [0, 1, 0, 1, 2, 1, 2, 3, 2, 3, 4, 3, 4]
v = [1.0, -1.0, -1.0, 2.0, -1.0, -1.0, 2.0, -1.0, -1.0, 2.0, -1.0, -1.0, 1.0]
open(os.path.join(OUT, "csr_path5.glr1"), "wb").write(glr1.csr_bytes(5, 5, rp, ci, v))
# CSR, non-canonical: unsorted row, a duplicate pair and an explicit zero
open(os.path.join(OUT, "csr_noncanonical.glr1"), "wb").write(
    glr1.csr_bytes(3, 4, [0, 3, 5, 7], [2, 0, 2, 1, 3, 0, 0], [1.0, 2.0, 0.5, 0.0, 4.0, 1.25, -1.25]))
# factors: p = 4, n = 3, k = 2
U = rs.standard_normal((4, 2))
V = rs.standard_normal((3, 2))
open(os.path.join(OUT, "factors_4x3_k2.glr1"), "wb").write(glr1.factors_bytes(U, [3.5, 1.25], V, True))
np.save(os.path.join(OUT, "factors_4x3_k2_UV.npy"), np.concatenate([U, V]))
# plan JSON as nlohmann::json::dump(2) prints it (sorted keys, io.cpp:232-243)
plan = {"seed": 1603, "p": 10, "n": 8, "omega_r": [7, 2, 9], "omega_c": [0, 5], "delta": 0.0, "epsilon": 0.25}
open(os.path.join(OUT, "plan.json"), "w").write(json.dumps(plan, indent=2, sort_keys=True) + "\n")
