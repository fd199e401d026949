"""Centered periodic FD operators, exactly (TEST INFRASTRUCTURE ONLY).

The MOL right-hand sides of BASELINE.json's configs use centered
finite differences of order 4 (r = 2) and 8 (r = 4) in the pairing form
(SURVEY.md §8(c) item 3):

  D1 u_i = N sum_j a_j (u_{i+j} - u_{i-j}),   D2 u_i = N^2 (b0 u_i + sum_j b_j (u_{i+j} + u_{i-j})).

The coefficients are derived here from the Taylor conditions (exactness on
x^q), solved in exact rationals — not typed in — so that they pin the
literal tables in gbs_oracle.c:

  D1: 2 sum_j a_j j^q = [q == 1]      for odd q = 1, 3, ..., 2r-1
  D2: b0 + 2 sum_j b_j = 0;  2 sum_j b_j j^q = 2 [q == 2]  for even q = 2..2r

Fourier symbols on theta = 2 pi k / N (numpy DFT sign convention):
  D1 e^{i theta x} = i N k~(theta) e^{...},     k~(theta) = 2 sum_j a_j sin(j theta)
  D2 e^{i theta x} = -N^2 s2(theta) e^{...},    s2(theta) = -(b0 + 2 sum_j b_j cos(j theta)) >= 0
"""

from __future__ import annotations

from fractions import Fraction as Fr
from typing import List, Tuple

import numpy as np

from .weights import _solve


def radius(order: int) -> int:
    if order not in (2, 4, 6, 8):
        raise ValueError("order must be 2, 4, 6 or 8")
    return order // 2


def d1_coeffs(order: int) -> List[Fr]:
    r = radius(order)
    qs = [2 * i + 1 for i in range(r)]
    A = [[Fr(2 * j ** q) for j in range(1, r + 1)] for q in qs]
    b = [Fr(1) if q == 1 else Fr(0) for q in qs]
    return _solve(A, b)


def d2_coeffs(order: int) -> Tuple[Fr, List[Fr]]:
    r = radius(order)
    # unknowns (b0, b1..br); equations q = 0, 2, ..., 2r
    A = [[Fr(1)] + [Fr(2)] * r]
    rhs = [Fr(0)]
    for q in range(2, 2 * r + 1, 2):
        A.append([Fr(0)] + [Fr(2 * j ** q) for j in range(1, r + 1)])
        rhs.append(Fr(2) if q == 2 else Fr(0))
    sol = _solve(A, rhs)
    return sol[0], sol[1:]


def d1_symbol(order: int, theta) -> np.ndarray:
    a = [float(x) for x in d1_coeffs(order)]
    th = np.asarray(theta, dtype=np.float64)
    return 2.0 * sum(aj * np.sin((j + 1) * th) for j, aj in enumerate(a))


def d2_symbol_neg(order: int, theta) -> np.ndarray:
    b0, b = d2_coeffs(order)
    th = np.asarray(theta, dtype=np.float64)
    return -(float(b0) + 2.0 * sum(float(bj) * np.cos((j + 1) * th) for j, bj in enumerate(b)))
