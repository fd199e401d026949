"""Exact-rational brute-force GBS stepping on tiny grids (TEST INFRASTRUCTURE ONLY).

Second, independent implementation of PAPER.md Eq. (1) + the weighted
combination (lines 85-115, 221-225) in ``fractions.Fraction`` arithmetic on
numpy object arrays: no rounding anywhere, exact FD coefficients from the
Taylor conditions (oracle.fd), exact weights (oracle.weights), rational H.
Used to pin the fp64 C oracle (tests/test_oracle_exact.py): the two must
agree to rounding (about 1e-15 relative).
"""

from __future__ import annotations

from fractions import Fraction as Fr
from typing import Sequence

import numpy as np

from . import fd


def _to_obj(a: np.ndarray) -> np.ndarray:
    out = np.empty(a.shape, dtype=object)
    flat = out.reshape(-1)
    for i, v in enumerate(np.asarray(a, dtype=np.float64).reshape(-1)):
        flat[i] = Fr(float(v))   # exact binary value of the double
    return out


def _d1(u, axis, N, a):
    s = 0
    for j, aj in enumerate(a, start=1):
        s = s + aj * (np.roll(u, -j, axis=axis) - np.roll(u, j, axis=axis))
    return N * s


def _d2(u, axis, N, b0, b):
    s = b0 * u
    for j, bj in enumerate(b, start=1):
        s = s + bj * (np.roll(u, -j, axis=axis) + np.roll(u, j, axis=axis))
    return (N * N) * s


def rhs(pde: str, order: int, y, scale):
    a = fd.d1_coeffs(order)
    if pde == "adv1d":
        return np.stack([-_d1(y[0], 0, scale[0], a)])
    if pde == "acoustic2d":
        p, u, v = y[0], y[1], y[2]
        # arrays are [ny][nx]: x is axis 1, y is axis 0
        return np.stack([-(_d1(u, 1, scale[0], a) + _d1(v, 0, scale[1], a)),
                         -_d1(p, 1, scale[0], a),
                         -_d1(p, 0, scale[1], a)])
    if pde == "wave3d":
        b0, b = fd.d2_coeffs(order)
        u, v = y[0], y[1]
        lap = (_d2(u, 2, scale[0], b0, b) + _d2(u, 1, scale[1], b0, b)
               + _d2(u, 0, scale[2], b0, b))
        return np.stack([v, lap])
    raise ValueError(pde)


def advance(pde: str, order: int, y0: np.ndarray, counts: Sequence[int],
            weights: Sequence[Fr], H: Fr, M: int, scale=None):
    """Exact Y after M macro steps; returns an object array of Fractions."""
    Y = _to_obj(y0)
    if scale is None:
        sh = y0.shape[1:]
        scale = {"adv1d": lambda: (sh[0],), "acoustic2d": lambda: (sh[1], sh[0]),
                 "wave3d": lambda: (sh[2], sh[1], sh[0])}[pde]()
    scale = [Fr(s) for s in scale]
    H = Fr(H)
    for _ in range(M):
        acc = None
        for N, w in zip(counts, weights):
            h = H / N
            ym1 = Y
            y0_ = ym1 + h * rhs(pde, order, ym1, scale)                 # FE
            for n in range(1, N + 1):                                  # LF
                yp1 = ym1 + 2 * h * rhs(pde, order, y0_, scale)
                if n < N:
                    ym1, y0_ = y0_, yp1
            ystar = (ym1 + 2 * y0_ + yp1) / 4                           # averaging
            term = Fr(w) * ystar
            acc = term if acc is None else acc + term
        Y = acc
    return Y


def to_float(a) -> np.ndarray:
    return np.vectorize(float, otypes=[np.float64])(a)
