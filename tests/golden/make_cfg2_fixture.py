"""Writes tests/golden/cfg2_knn_sha256.json: the oracle's exact kNN result on
the full config-2 input (100 000 x 512, K = 10; graph.cpp:86-133) as SHA-256
digests -- the neighbour index lists, their canonical fp64 squared
distances, and the CSR structure (row_ptr, col_idx) of the union-symmetrised
adjacency W (the Laplacian's structure is W's plus the diagonal) -- plus a
few rows in clear.  Run once (about 10 minutes on 8 cores):
    python tests/golden/make_cfg2_fixture.py
"""
import hashlib
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle import pyoracle as O  # noqa: E402
from paper_1602_02070_b200 import workloads  # noqa: E402


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def knn_structure(nbr: np.ndarray):
    """CSR structure of the union-symmetrised kNN adjacency (graph.cpp:108-133)."""
    n, K = nbr.shape
    rows = np.repeat(np.arange(n, dtype=np.int64), K)
    cols = nbr.reshape(-1).astype(np.int64)
    r = np.concatenate([rows, cols])
    c = np.concatenate([cols, rows])
    key = np.unique(r * n + c)
    rr, cc = key // n, key % n
    rp = np.zeros(n + 1, np.int64)
    np.add.at(rp, rr + 1, 1)
    return np.cumsum(rp), cc.astype(np.int64)


def main():
    X = workloads.config2_points()
    t0 = time.time()
    nbr, d2 = O.knn_neighbors(X.astype(np.float64), False, 10)
    rp, ci = knn_structure(nbr)
    sample = [0, 1, 2, 49_999, 50_000, 99_999]
    out = {
        "input": "workloads.config2_points() (100000 x 512 fp32, seed 1604), columns are points, K = 10",
        "oracle": "oracle/cpcag_oracle.cpp knn_select (graph.cpp:86-105), canonical fp64 distances",
        "nbr_int64_sha256": sha(nbr.astype(np.int64)),
        "d2_float64_sha256": sha(d2.astype(np.float64)),
        "W_row_ptr_int64_sha256": sha(rp),
        "W_col_idx_int64_sha256": sha(ci),
        "W_nnz": int(ci.size),
        "sample_rows": {str(i): [int(j) for j in nbr[i]] for i in sample},
        "oracle_seconds": round(time.time() - t0, 1),
    }
    with open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "cfg2_knn_sha256.json"), "w") as f:
        json.dump(out, f, indent=1)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
