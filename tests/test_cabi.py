"""CPU-side checks of the drop-in boundary: the C-ABI library loads, exports
every symbol include/cpcag_cuda.h declares, runs its host-only entry point
(draw_plan) bit-identically to the oracle, and fails loudly (no CPU
fallback) when no device is present."""
import ctypes
import os
import re

import numpy as np
import pytest

from oracle import pyoracle as O

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    names = set()
    for fn in os.listdir(os.path.join(ROOT, "include")):
        if not fn.endswith(".h"):
            continue
        text = open(os.path.join(ROOT, "include", fn)).read()
        text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
        for m in re.finditer(r"^[A-Za-z_][\w\s\*]*?\b(cpcag_\w+)\s*\(", text, flags=re.M):
            names.add(m.group(1))
    return names


def test_library_exports_every_declared_symbol():
    from paper_1602_02070_b200 import _native

    L = _native.lib()
    names = declared_symbols()
    assert len(names) >= 30
    for n in sorted(names):
        assert hasattr(L, n), n
        assert n in _native.SIGNATURES, n


def test_no_oracle_in_product_library():
    so = open(os.path.join(ROOT, "paper_1602_02070_b200", "lib", "libcpcag_cuda.so"), "rb").read()
    assert b"ora_" not in so  # every oracle export is ora_*: none may be linked into the product
    import subprocess
    dyn = subprocess.run(["nm", "-D", "--undefined-only", os.path.join(ROOT, "paper_1602_02070_b200", "lib",
                                                                      "libcpcag_cuda.so")],
                         capture_output=True, text=True, check=True).stdout
    assert "ora_" not in dyn and "cpcag_oracle" not in dyn
    src = os.path.join(ROOT, "paper_1602_02070_b200")
    for dirpath, _, files in os.walk(src):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".cpp", ".h")):
                t = open(os.path.join(dirpath, f)).read()
                assert "pyoracle" not in t and "cpcag_oracle" not in t, f


def test_draw_plan_host_entry_bit_exact():
    import paper_1602_02070_b200 as P

    for (p, n, rr, rc, seed) in [(200, 300, 50, 75, 1602), (10304, 1000, 1031, 100, 1603), (7, 9, 7, 9, 0)]:
        a = P.draw_plan(p, n, rr, rc, seed=seed)
        b = O.draw_plan(p, n, rr, rc, seed=seed)
        assert np.array_equal(a.omega_r, b.omega_r) and np.array_equal(a.omega_c, b.omega_c)
    with pytest.raises(ValueError, match=r"rho_r out of range \[1, 5\]"):
        P.draw_plan(5, 5, 6, 1)


def test_from_triplets_host_construction_semantics():
    """SparseMatrix.from_triplets' host-side merge/drop rules (sparse.cpp:10-46)."""
    from paper_1602_02070_b200 import cpcag

    with pytest.raises(ValueError, match="index out of range"):
        cpcag.SparseMatrix.from_triplets(2, 2, [2], [0], [1.0])
    with pytest.raises(ValueError, match="non-finite"):
        cpcag.SparseMatrix.from_triplets(2, 2, [0], [0], [np.nan])


@pytest.mark.skipif(os.environ.get("CUDA_VISIBLE_DEVICES", None) != "" and
                    os.path.exists("/dev/nvidia0"), reason="a GPU is present")
def test_fails_loudly_without_device():
    from paper_1602_02070_b200 import _native

    L = _native.lib()
    h = ctypes.c_void_p()
    rc = L.cpcag_ctx_create(0, ctypes.byref(h))
    assert rc == _native.ERR_CUDA
    assert L.cpcag_cuda_last_error()


def test_pipeline_out_buffer_validation():
    """run_pipeline(out=...) accepts Fortran-ordered arrays of the result
    shape and dtype, and rejects anything else before calling the library."""
    import numpy as np

    from paper_1602_02070_b200 import _native as N
    from paper_1602_02070_b200.cpcag import _given_out

    a = np.empty((5, 3), np.float32, order="F")
    arr, ptr = _given_out(a, (5, 3), N.F32, "X")
    assert arr is a and ptr == a.ctypes.data
    for bad in (np.empty((5, 3), np.float32), np.empty((5, 3), np.float64, order="F"),
                np.empty((3, 5), np.float32, order="F")):
        with pytest.raises(ValueError, match="X: expected a Fortran-ordered"):
            _given_out(bad, (5, 3), N.F32, "X")
