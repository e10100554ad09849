"""GLR1 container restated in numpy -- TEST INFRASTRUCTURE ONLY (the
checker for the device-direct loaders in paper_1602_02070_b200/csrc/io.cu;
never imported by the product).

Follows /root/reference/proj/core/src/io.cpp:
  magic "GLR1" + u64 kind (io.cpp:16-20, 70-75), little-endian u64 fields
  (io.cpp:39-51), raw fp64 arrays (io.cpp:53-63);
  dense   kind 1: rows, cols, data column-major           (io.cpp:88-96, 108-118)
  CSR     kind 2: rows, cols, nnz, row_ptr, col_idx (u64), values (io.cpp:151-162)
  factors kind 3: p, n, k, scale flag, U, sigma, V        (io.cpp:200-211)
"""
import struct

import numpy as np


def _hdr(kind):
    return b"GLR1" + struct.pack("<Q", kind)


def dense_bytes(M) -> bytes:
    M = np.asarray(M, np.float64)
    return _hdr(1) + struct.pack("<QQ", *M.shape) + np.asfortranarray(M).tobytes(order="F")


def csr_bytes(rows, cols, row_ptr, col_idx, values) -> bytes:
    rp = np.asarray(row_ptr, "<u8")
    ci = np.asarray(col_idx, "<u8")
    v = np.asarray(values, "<f8")
    return _hdr(2) + struct.pack("<QQQ", rows, cols, len(v)) + rp.tobytes() + ci.tobytes() + v.tobytes()


def factors_bytes(U, sigma, V, scale_applied) -> bytes:
    U = np.asfortranarray(U, np.float64)
    V = np.asfortranarray(V, np.float64)
    s = np.asarray(sigma, np.float64)
    return (_hdr(3) + struct.pack("<QQQQ", U.shape[0], V.shape[0], len(s), 1 if scale_applied else 0) +
            U.tobytes(order="F") + s.tobytes() + V.tobytes(order="F"))


def read(data: bytes):
    """-> (kind, payload) with payload a dense array, a (rows, cols, rp, ci, v)
    tuple or a (U, sigma, V, scale) tuple."""
    if data[:4] != b"GLR1":
        raise ValueError("not a GLR1 container (bad magic)")
    kind = struct.unpack_from("<Q", data, 4)[0]
    off = 12
    if kind == 1:
        r, c = struct.unpack_from("<QQ", data, off)
        off += 16
        return kind, np.frombuffer(data, "<f8", r * c, off).reshape((r, c), order="F")
    if kind == 2:
        r, c, nnz = struct.unpack_from("<QQQ", data, off)
        off += 24
        rp = np.frombuffer(data, "<u8", r + 1, off).astype(np.int64)
        off += 8 * (r + 1)
        ci = np.frombuffer(data, "<u8", nnz, off).astype(np.int64)
        off += 8 * nnz
        v = np.frombuffer(data, "<f8", nnz, off)
        return kind, (r, c, rp, ci, v)
    if kind == 3:
        p, n, k, sc = struct.unpack_from("<QQQQ", data, off)
        off += 32
        U = np.frombuffer(data, "<f8", p * k, off).reshape((p, k), order="F")
        off += 8 * p * k
        s = np.frombuffer(data, "<f8", k, off)
        off += 8 * k
        V = np.frombuffer(data, "<f8", n * k, off).reshape((n, k), order="F")
        return kind, (U, s, V, bool(sc))
    raise ValueError(f"unknown kind {kind}")
