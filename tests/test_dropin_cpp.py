"""The compiled cpcag:: C++ drop-in layer (cpp/: the reference's API over
the C-ABI).  CPU: the layer links and exports the reference's entry points.
GPU: cpp/tests/test_dropin.cpp runs the reference's known answers, exception
types and messages through it."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BUILD = os.path.join(ROOT, "cpp", "build")


def _build():
    subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "cpp")], check=True)


def test_dropin_layer_exports_reference_api():
    _build()
    syms = subprocess.run(["nm", "-D", "-C", os.path.join(BUILD, "libcpcag_b200.so")], check=True,
                          capture_output=True, text=True).stdout
    for name in ("cpcag::build_knn_graph(", "cpcag::kron_reduce(", "cpcag::fista_solve(", "cpcag::alternate_decode(",
                 "cpcag::SparseMatrix::multiply(", "cpcag::SparseMatrix::right_multiply(", "cpcag::draw_plan(",
                 "cpcag::subsample(", "cpcag::pcg_solve(", "cpcag::power_iteration_norm(", "cpcag::objective(",
                 "cpcag::prox_l1(", "cpcag::grad_g(", "cpcag::graph_from_adjacency("):
        assert name in syms, name


@pytest.mark.gpu
def test_dropin_cpp_known_answers():
    _build()
    r = subprocess.run([os.path.join(BUILD, "test_dropin")], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failed" in r.stdout
