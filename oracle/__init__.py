"""CPU oracle for the q4f16 dequantize+matmul path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this package.  The
product package (``paper_2311_02103_b200``) never imports it, and it imports
nothing from the product package: the two share no code.  The only module
both sides use is ``paper_2311_02103_b200.inputs`` (seeded input generators,
none of the method's arithmetic) -- and this package does not even import
that; callers pass arrays in.

The arithmetic lives in ``q4_oracle.c`` (plain C, fp64, see its header for
the definition and the PAPER.md passages it follows).  This file only builds
that C file with gcc and marshals numpy arrays through ctypes.

Public functions (all numpy in / numpy out):
    dequant(packed_w, scales, K, N)            -> uint16 fp16 bits [N, K]
    matmul_f64(x_bits, packed_w, scales, K, N) -> float64 r [n, N]
    matmul_cols_f64(x_bits, packed_w, scales, K, cols) -> float64 r [n, len(cols)]
    round_f16(r)                               -> uint16 fp16 bits, same shape
    f16_to_f64(bits)                           -> float64
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "q4_oracle.c")
_LIB = os.path.join(_HERE, "libq4oracle.so")
_lock = threading.Lock()
_lib = None

# -O2, no fast-math, no -march (portable soft-float fp16 conversions),
# no fp contraction (fp64 sums stay separate multiply then add).
CFLAGS = ["-O2", "-std=c11", "-fopenmp", "-ffp-contract=off", "-fno-fast-math",
          "-Wall", "-Wextra", "-shared", "-fPIC"]


def build(force: bool = False) -> str:
    """Compile q4_oracle.c into libq4oracle.so (in-tree) if missing or stale."""
    if (not force and os.path.exists(_LIB)
            and os.path.getmtime(_LIB) >= os.path.getmtime(_SRC)):
        return _LIB
    tmp = _LIB + f".tmp{os.getpid()}"
    subprocess.run(["gcc", *CFLAGS, "-o", tmp, _SRC], check=True)
    os.replace(tmp, _LIB)
    return _LIB


def _load():
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        build()
        lib = ctypes.CDLL(_LIB)
        P = ctypes.c_void_p
        I64 = ctypes.c_int64
        lib.q4o_dequant.argtypes = [P, P, I64, I64, P]
        lib.q4o_dequant.restype = ctypes.c_int
        lib.q4o_matmul_f64.argtypes = [P, I64, I64, I64, P, P, P, ctypes.c_int]
        lib.q4o_matmul_f64.restype = ctypes.c_int
        lib.q4o_matmul_cols_f64.argtypes = [P, I64, I64, P, P, P, I64, P, ctypes.c_int]
        lib.q4o_matmul_cols_f64.restype = ctypes.c_int
        lib.q4o_round_f16.argtypes = [P, I64, P]
        lib.q4o_round_f16.restype = None
        lib.q4o_f16_to_f64.argtypes = [P, I64, P]
        lib.q4o_f16_to_f64.restype = None
        lib.q4o_max_threads.argtypes = []
        lib.q4o_max_threads.restype = ctypes.c_int
        _lib = lib
        return lib


def _ptr(a: np.ndarray) -> int:
    return a.ctypes.data


def _c(a, dtype):
    a = np.ascontiguousarray(a)
    if a.dtype != dtype:
        raise TypeError(f"expected {dtype}, got {a.dtype}")
    return a


def max_threads() -> int:
    return int(_load().q4o_max_threads())


def dequant(packed_w: np.ndarray, scales: np.ndarray, K: int, N: int) -> np.ndarray:
    """W as fp16 bit patterns, layout [N][K] (column j of W is row j here)."""
    lib = _load()
    pw = _c(packed_w, np.uint32).reshape(-1)
    sc = _c(scales, np.uint16).reshape(-1)
    assert pw.size == N * K // 8 and sc.size == N * K // 32
    out = np.empty((N, K), dtype=np.uint16)
    rc = lib.q4o_dequant(_ptr(pw), _ptr(sc), K, N, _ptr(out))
    if rc != 0:
        raise ValueError(f"q4o_dequant rejected K={K} N={N}")
    return out


def matmul_f64(x_bits: np.ndarray, packed_w: np.ndarray, scales: np.ndarray,
               K: int, N: int, nthreads: int | None = None) -> np.ndarray:
    """r[i][j] = sum_k x[i][k] W(k,j) in fp64 (k ascending)."""
    lib = _load()
    x = _c(x_bits, np.uint16).reshape(-1, K)
    n = x.shape[0]
    pw = _c(packed_w, np.uint32).reshape(-1)
    sc = _c(scales, np.uint16).reshape(-1)
    assert pw.size == N * K // 8 and sc.size == N * K // 32
    r = np.empty((n, N), dtype=np.float64)
    nt = nthreads or max_threads()
    rc = lib.q4o_matmul_f64(_ptr(x), n, K, N, _ptr(pw), _ptr(sc), _ptr(r), nt)
    if rc != 0:
        raise ValueError("q4o_matmul_f64 rejected its arguments")
    return r


def matmul_cols_f64(x_bits: np.ndarray, packed_w: np.ndarray, scales: np.ndarray,
                    K: int, cols, nthreads: int | None = None) -> np.ndarray:
    """r[i][c] = sum_k x[i][k] W(k, cols[c]) in fp64, for sampled columns."""
    lib = _load()
    x = _c(x_bits, np.uint16).reshape(-1, K)
    n = x.shape[0]
    pw = _c(packed_w, np.uint32).reshape(-1)
    sc = _c(scales, np.uint16).reshape(-1)
    cols = np.ascontiguousarray(np.asarray(cols, dtype=np.int64))
    N = pw.size * 8 // K
    assert cols.size == 0 or (cols.min() >= 0 and cols.max() < N)
    r = np.empty((n, cols.size), dtype=np.float64)
    nt = nthreads or max_threads()
    rc = lib.q4o_matmul_cols_f64(_ptr(x), n, K, _ptr(pw), _ptr(sc), _ptr(cols),
                                 cols.size, _ptr(r), nt)
    if rc != 0:
        raise ValueError("q4o_matmul_cols_f64 rejected its arguments")
    return r


def round_f16(r: np.ndarray) -> np.ndarray:
    lib = _load()
    rr = _c(r, np.float64)
    out = np.empty(rr.shape, dtype=np.uint16)
    lib.q4o_round_f16(_ptr(rr), rr.size, _ptr(out))
    return out


def f16_to_f64(bits: np.ndarray) -> np.ndarray:
    lib = _load()
    b = _c(bits, np.uint16)
    out = np.empty(b.shape, dtype=np.float64)
    lib.q4o_f16_to_f64(_ptr(b), b.size, _ptr(out))
    return out
