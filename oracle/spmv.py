"""ctypes wrapper of oracle/bsr_spmv.c (TEST INFRASTRUCTURE).

Restates cutdg BlockSparseMatrix.matvec (blockmatrix.py:119-125) on
row-major BSR arrays; bit-identical to scipy csr_matvec on tocsr().
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "liboracle.so")
_lib = None


def build() -> str:
    src = os.path.join(HERE, "bsr_spmv.c")
    if not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(src):
        subprocess.run(["make", "-s", "-C", HERE], check=True)
    return LIB


def _load():
    global _lib
    if _lib is None:
        build()
        lib = C.CDLL(LIB)
        lib.oracle_bsr_spmv.restype = None
        lib.oracle_bsr_spmv.argtypes = [C.c_int64, C.c_int] + [C.c_void_p] * 5 + [C.c_int]
        lib.oracle_max_threads.restype = C.c_int
        _lib = lib
    return _lib


def max_threads() -> int:
    return int(_load().oracle_max_threads())


def bsr_spmv(row_ptr, col, val, x, nthreads: int = 1) -> np.ndarray:
    """y = M x for row-major BSR (row_ptr, col, val[nnzb, N, N])."""
    rp = np.ascontiguousarray(row_ptr, np.int64)
    cl = np.ascontiguousarray(col, np.int64)
    v = np.ascontiguousarray(val, np.float64)
    N = v.shape[1] if v.ndim == 3 else int(round((v.size // max(len(cl), 1)) ** 0.5))
    xx = np.ascontiguousarray(x, np.float64)
    nbr = len(rp) - 1
    y = np.empty(nbr * N)
    _load().oracle_bsr_spmv(nbr, N, rp.ctypes.data, cl.ctypes.data, v.ctypes.data,
                            xx.ctypes.data, y.ctypes.data, int(nthreads))
    return y
