"""ctypes wrapper of oracle/gbs_oracle.c (TEST INFRASTRUCTURE ONLY).

Builds the library on first use if it is missing (gcc -O2 -ffp-contract=off
-fopenmp).  See gbs_oracle.c for what it computes and which PAPER.md passages
it follows.
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from typing import Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "gbs_oracle.c")
_LIB = os.path.join(_HERE, "_build", "liboracle_gbs.so")

PDE_CODE = {"adv1d": 1, "acoustic2d": 2, "wave3d": 3}

_lib = None


def build(force: bool = False) -> str:
    """Compile the oracle shared library (plain C, no intrinsics)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        os.makedirs(os.path.dirname(_LIB), exist_ok=True)
        tmp = _LIB + f".tmp{os.getpid()}"
        cmd = ["gcc", "-O2", "-ffp-contract=off", "-fno-fast-math", "-fopenmp",
               "-std=c99", "-shared", "-fPIC", "-o", tmp, _SRC, "-lm"]
        subprocess.run(cmd, check=True)
        os.replace(tmp, _LIB)
    return _LIB


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB)
        i64p = ctypes.POINTER(ctypes.c_int64)
        dp = ctypes.POINTER(ctypes.c_double)
        i32p = ctypes.POINTER(ctypes.c_int32)
        L.oracle_advance.argtypes = [ctypes.c_int, ctypes.c_int, i64p, dp, ctypes.c_int, i32p,
                                     dp, ctypes.c_double, ctypes.c_int64, dp]
        L.oracle_advance.restype = ctypes.c_int
        L.oracle_rhs.argtypes = [ctypes.c_int, ctypes.c_int, i64p, dp, dp, dp]
        L.oracle_rhs.restype = ctypes.c_int
        L.oracle_fd_coeffs.argtypes = [ctypes.c_int, dp, dp, dp]
        L.oracle_fd_coeffs.restype = ctypes.c_int
        L.oracle_set_threads.argtypes = [ctypes.c_int]
        L.oracle_set_threads.restype = ctypes.c_int
        _lib = L
    return _lib


def set_threads(n: int) -> int:
    return lib().oracle_set_threads(int(n))


def _dims(state: np.ndarray, pde: str):
    """(nx, ny, nz) extents from an SoA state array [F][nz][ny][nx]."""
    sh = state.shape[1:]
    if pde == "adv1d":
        return (sh[0], 1, 1)
    if pde == "acoustic2d":
        return (sh[1], sh[0], 1)
    return (sh[2], sh[1], sh[0])


def _ptr(a, t):
    return a.ctypes.data_as(ctypes.POINTER(t))


def fd_coeffs(order: int):
    a = np.zeros(4)
    b = np.zeros(4)
    b0 = np.zeros(1)
    r = lib().oracle_fd_coeffs(order, _ptr(a, ctypes.c_double), _ptr(b0, ctypes.c_double),
                               _ptr(b, ctypes.c_double))
    if r < 0:
        raise ValueError(order)
    return a[:r].copy(), float(b0[0]), b[:r].copy()


def rhs(pde: str, order: int, y: np.ndarray, scale: Sequence[float] | None = None) -> np.ndarray:
    y = np.ascontiguousarray(y, dtype=np.float64)
    dims = np.array(_dims(y, pde), dtype=np.int64)
    sc = np.array(scale if scale is not None else dims, dtype=np.float64)
    f = np.empty_like(y)
    rc = lib().oracle_rhs(PDE_CODE[pde], order, _ptr(dims, ctypes.c_int64),
                          _ptr(sc, ctypes.c_double), _ptr(y, ctypes.c_double),
                          _ptr(f, ctypes.c_double))
    if rc:
        raise ValueError(f"oracle_rhs rc={rc}")
    return f


def advance(pde: str, order: int, y0: np.ndarray, n_k: Sequence[int], w_k: Sequence[float],
            H: float, M: int, scale: Sequence[float] | None = None,
            threads: int | None = None) -> np.ndarray:
    """Return Y after M macro steps from y0 (y0 is not modified)."""
    Y = np.array(y0, dtype=np.float64, order="C", copy=True)
    dims = np.array(_dims(Y, pde), dtype=np.int64)
    sc = np.array(scale if scale is not None else dims, dtype=np.float64)
    nk = np.array(n_k, dtype=np.int32)
    wk = np.array(w_k, dtype=np.float64)
    if threads is not None:
        set_threads(threads)
    rc = lib().oracle_advance(PDE_CODE[pde], order, _ptr(dims, ctypes.c_int64),
                              _ptr(sc, ctypes.c_double), len(nk), _ptr(nk, ctypes.c_int32),
                              _ptr(wk, ctypes.c_double), float(H), int(M),
                              _ptr(Y, ctypes.c_double))
    if rc:
        raise ValueError(f"oracle_advance rc={rc}")
    return Y
