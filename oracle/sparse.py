"""Tier S oracle: ctypes wrapper of oracle/csrc/sparse_oracle.c (TEST INFRASTRUCTURE ONLY)."""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "csrc", "sparse_oracle.c")
_LIB = os.path.join(_HERE, "csrc", "libsparse_oracle.so")
_lib = None

CFLAGS = ["-O3", "-march=x86-64-v3", "-fPIC", "-shared", "-std=c11"]


def build(force: bool = False) -> str:
    """Compile the oracle C (gcc).  Building the checker is not using it."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", *CFLAGS, "-o", _LIB, _SRC, "-lm"])
    return _LIB


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB)
        P = ctypes.c_void_p
        L.orc_nd_order.argtypes = [ctypes.c_int, P, P, ctypes.c_int, P]
        L.orc_nd_order.restype = ctypes.c_int
        L.orc_symbolic.argtypes = [ctypes.c_int, P, P, P, P, P, P]
        L.orc_symbolic.restype = ctypes.c_int64
        L.orc_cholesky.argtypes = [ctypes.c_int, P, P, P, P, P, P]
        L.orc_cholesky.restype = ctypes.c_int
        L.orc_lsolve.argtypes = [ctypes.c_int, P, P, P, P]
        L.orc_lsolve.restype = None
        L.orc_ltsolve.argtypes = [ctypes.c_int, P, P, P, P]
        L.orc_ltsolve.restype = None
        _lib = L
    return _lib


def _p(a):
    return a.ctypes.data_as(ctypes.c_void_p)


def nd_order(xadj: np.ndarray, adj: np.ndarray, leaf: int) -> np.ndarray:
    """Nested-dissection ordering of DESIGN.md §5; perm[k] = old index at new position k."""
    xadj = np.ascontiguousarray(xadj, dtype=np.int32)
    adj = np.ascontiguousarray(adj, dtype=np.int32)
    n = len(xadj) - 1
    perm = np.empty(n, dtype=np.int32)
    rc = lib().orc_nd_order(n, _p(xadj), _p(adj), int(leaf), _p(perm))
    if rc != 0:
        raise RuntimeError(f"orc_nd_order failed: {rc}")
    return perm


def symbolic(Ap: np.ndarray, Ai: np.ndarray):
    """(parent, colcount, Lp, Li) of the lower CSC pattern (Ap, Ai) incl. diagonal."""
    Ap = np.ascontiguousarray(Ap, dtype=np.int64)
    Ai = np.ascontiguousarray(Ai, dtype=np.int32)
    n = len(Ap) - 1
    parent = np.empty(n, dtype=np.int32)
    cc = np.empty(n, dtype=np.int32)
    Lp = np.empty(n + 1, dtype=np.int64)
    nnz = lib().orc_symbolic(n, _p(Ap), _p(Ai), _p(parent), _p(cc), _p(Lp), None)
    if nnz < 0:
        raise MemoryError("orc_symbolic")
    Li = np.empty(nnz, dtype=np.int32)
    lib().orc_symbolic(n, _p(Ap), _p(Ai), _p(parent), _p(cc), _p(Lp), _p(Li))
    return parent, cc, Lp, Li


def cholesky(Ap, Ai, Ax, Lp, Li):
    """Left-looking Cholesky.  Returns (Lx, fail) with fail = -1 or the first bad column."""
    n = len(Ap) - 1
    Lx = np.zeros(len(Li), dtype=np.float64)
    Ax = np.ascontiguousarray(Ax, dtype=np.float64)
    fail = lib().orc_cholesky(n, _p(Ap), _p(Ai), _p(Ax), _p(Lp), _p(Li), _p(Lx))
    return Lx, int(fail)


def lsolve(Lp, Li, Lx, b):
    x = np.array(b, dtype=np.float64, copy=True)
    lib().orc_lsolve(len(Lp) - 1, _p(Lp), _p(Li), _p(Lx), _p(x))
    return x


def ltsolve(Lp, Li, Lx, b):
    x = np.array(b, dtype=np.float64, copy=True)
    lib().orc_ltsolve(len(Lp) - 1, _p(Lp), _p(Li), _p(Lx), _p(x))
    return x
