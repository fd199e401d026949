"""Host-side scheme setup (layer L0): extrapolation weights, ISB and the H rule.

Not on the hot path: runs once per configuration and hands fp64 numbers to
``gbs_create`` / ``gbs_advance``.  Written independently of ``oracle/``
(different algorithms: Lagrange-basis inversion of the Vandermonde system here,
Gauss-Jordan there); tests/test_scheme.py checks the two agree exactly.

* Eq. (3): the order constraints are sum_i c_i x_i^j = b_j,
  j = 0..p/2-1, with x_i = h_i^2 = 1/n_i^2 (H = 1; the weights do not depend on
  H).  For p/2 dependent counts, V_dep^{-1} is the matrix of coefficients of the
  Lagrange basis polynomials L_i(x) = prod_{k != i} (x - x_k)/(x_i - x_k)
  (since sum_j l_ij x_k^j = L_i(x_k) = delta_ik).
* Eq. (6): c_dep = V_dep^{-1} (b - V_free c_free).
* Weights are rounded to fp64 once, correctly.
* ISB (§2.2): first y with |R(iy)| > 1 + 1e-10 on a 1e-4 grid,
  refined by bisection; R = sum_i c_i P_{n_i} evaluated by running Eq. (1) on
  y' = lambda y (App. A).
* H = h_factor * ISB / rho, rho the spectral radius of the FD operator
  (BASELINE.json configs; reading R7).
"""

from __future__ import annotations

import math
from fractions import Fraction
from typing import List, Sequence, Tuple

import numpy as np

# the paper's printed free weights
_PAPER = {
    "GBS_8_6": (8, (2, 4, 6, 10), (8, 12, 14, 16, 18, 20, 22),
                ("2165/767488", "13805/611712", "4553/72080", "14503/66520", "27058/7627",
                 "-86504/5761", "40916/3367")),
    # n_free printed as {4..22}; 11 weights are printed -> {4..24} (reading R4)
    "GBS_8_8": (8, (2, 26, 28, 30), (4, 6, 8, 10, 12, 14, 16, 18, 20, 22, 24),
                ("6833/476577792", "10847/91078656", "15235/34643968", "383/321152",
                 "543/198784", "9947/1741056", "6243/543104", "6875/296192", "1401/28496",
                 "17713/152688", "6375/19264")),
    "GBS_12_8": (12, (2, 8, 10, 16, 24, 26), (4, 6, 12, 14, 18, 20, 22, 28, 30),
                 ("235/21030240256", "4147/1612709888", "11521/39731200", "2375/3528704",
                  "6435/708736", "1291/15780", "11311/4672", "-180864/751", "222080/2079")),
}
# fully determined (square) systems: Table 1 and the configs' {2,4,6,8}
_SQUARE = {"FD8": (8, (2, 16, 18, 20)), "FD12": (12, (2, 8, 12, 14, 16, 20)),
           "FD16": (16, (2, 8, 10, 12, 14, 16, 18, 22)), "square8": (8, (2, 4, 6, 8))}


def _poly_mul_linear(p: List[Fraction], root: Fraction) -> List[Fraction]:
    """p(x) * (x - root), coefficient lists index = power."""
    out = [Fraction(0)] * (len(p) + 1)
    for i, c in enumerate(p):
        out[i + 1] += c
        out[i] -= c * root
    return out


def vandermonde_inverse(counts: Sequence[int]) -> List[List[Fraction]]:
    """l[i][j]: coefficient of x^j in the Lagrange basis L_i, x_k = 1/n_k^2."""
    xs = [Fraction(1, n * n) for n in counts]
    q = len(xs)
    inv = []
    for i in range(q):
        num = [Fraction(1)]
        den = Fraction(1)
        for k in range(q):
            if k != i:
                num = _poly_mul_linear(num, xs[k])
                den *= xs[i] - xs[k]
        inv.append([c / den for c in num])
    return inv


def weights_exact(n_dep: Sequence[int], n_free: Sequence[int] = (),
                  c_free: Sequence[Fraction] = ()) -> List[Fraction]:
    """c_dep from Eq. (6); order p = 2 * len(n_dep)."""
    allc = list(n_dep) + list(n_free)
    if any(n < 2 or n % 2 for n in allc) or len(set(allc)) != len(allc):
        raise ValueError("step counts must be even, >= 2 and distinct")
    q = len(n_dep)
    r = [Fraction(1 if j == 0 else 0) - sum((Fraction(c) * Fraction(1, n * n) ** j
                                             for n, c in zip(n_free, c_free)), Fraction(0))
         for j in range(q)]
    inv = vandermonde_inverse(n_dep)
    return [sum((inv[i][j] * r[j] for j in range(q)), Fraction(0)) for i in range(q)]


def weight_set(name: str, steps: Sequence[int] | None = None) -> Tuple[List[int], List[Fraction], int]:
    """(ascending step counts, exact weights, order) for a named weight set."""
    if name in _SQUARE:
        p, counts = _SQUARE[name]
        if steps is not None and sorted(steps) != list(counts):
            raise ValueError(f"{name} is defined on {counts}")
        return list(counts), weights_exact(counts), p
    if name in _PAPER:
        p, nd, nf, cf = _PAPER[name]
        cfree = [Fraction(x) for x in cf]
        cdep = weights_exact(nd, nf, cfree)
        w = dict(zip(nd, cdep))
        w.update(zip(nf, cfree))
        counts = sorted(w)
        if steps is not None and sorted(steps) != counts:
            raise ValueError(f"{name} is defined on {counts}")
        return counts, [w[n] for n in counts], p
    if name in ("fallback8", "nonzero8"):
        # configs 2-5: square order-8 weights on {2,4,6,8}, 0 elsewhere ("fallback8");
        # parity set: +1/50, -1/50, ... on the extra counts ("nonzero8").  DESIGN.md reading R3.
        counts = sorted(steps)
        nd = (2, 4, 6, 8)
        nf = [n for n in counts if n not in nd]
        cf = ([Fraction(0)] * len(nf) if name == "fallback8"
              else [Fraction(1 if i % 2 == 0 else -1, 50) for i in range(len(nf))])
        w = dict(zip(nd, weights_exact(nd, nf, cf)))
        w.update(zip(nf, cf))
        return counts, [w[n] for n in counts], 8
    if name == "opt8":
        # Appendix-B optimised free weights for these step counts (gbs_inputs/
        # optimized_schemes.json, written by tools/optimize_schemes.py); c_dep by Eq. (6)
        from gbs_inputs.schemes import optimized_for
        s = optimized_for(steps)
        nd, nf = tuple(s["n_dep"]), tuple(s["n_free"])
        cfree = [Fraction(x) for x in s["c_free"]]
        w = dict(zip(nd, weights_exact(nd, nf, cfree)))
        w.update(zip(nf, cfree))
        counts = sorted(w)
        return counts, [w[n] for n in counts], s["order"]
    raise KeyError(name)


def to_fp64(ws: Sequence[Fraction]) -> List[float]:
    return [w.numerator / w.denominator for w in ws]   # int/int true division: correctly rounded


def _gbs_component(n: int, z: np.ndarray) -> np.ndarray:
    """Eq. (1) on y' = lambda y, y0 = 1, z = H lambda: returns y*_n."""
    a = z / n
    prev = np.ones_like(z)
    cur = prev * (1.0 + a)
    nxt = cur
    for i in range(n):
        nxt = prev + 2.0 * a * cur
        if i < n - 1:
            prev, cur = cur, nxt
    return 0.25 * (prev + 2.0 * cur + nxt)


def stability_function(counts: Sequence[int], w: Sequence[float], z) -> np.ndarray:
    z = np.asarray(z, dtype=np.complex128)
    return sum(float(c) * _gbs_component(n, z) for n, c in zip(counts, w))


def imaginary_stability_boundary(counts: Sequence[int], w: Sequence[float],
                                 tol: float = 1e-10, dy: float = 1e-4, ymax: float = 200.0) -> float:
    y = 0.0
    block = 100_000
    while y < ymax:
        ys = y + dy * np.arange(1, block + 1)
        over = np.abs(stability_function(counts, w, 1j * ys)) > 1.0 + tol
        if over.any():
            k = int(np.argmax(over))
            lo, hi = (ys[k - 1] if k else y), ys[k]
            while hi - lo > 1e-12:
                mid = 0.5 * (lo + hi)
                if abs(stability_function(counts, w, np.array([1j * mid]))[0]) > 1.0 + tol:
                    hi = mid
                else:
                    lo = mid
            return float(lo)
        y = float(ys[-1])
    return ymax


def _d1_symbol_max(order: int) -> float:
    if order == 4:
        th = math.acos(1.0 - math.sqrt(6.0) / 2.0)      # root of 2c^2 - 4c - 1 = 0
        return 4.0 / 3.0 * math.sin(th) - 1.0 / 6.0 * math.sin(2 * th)
    a = {8: (4 / 5, -1 / 5, 4 / 105, -1 / 280), 2: (1 / 2,), 6: (3 / 4, -3 / 20, 1 / 60)}[order]
    f = lambda t: 2 * sum(aj * math.sin((j + 1) * t) for j, aj in enumerate(a))
    df = lambda t: 2 * sum(aj * (j + 1) * math.cos((j + 1) * t) for j, aj in enumerate(a))
    d2 = lambda t: -2 * sum(aj * (j + 1) ** 2 * math.sin((j + 1) * t) for j, aj in enumerate(a))
    ts = np.linspace(0, math.pi, 4097)
    t = float(ts[int(np.argmax([f(x) for x in ts]))])
    for _ in range(50):                                    # Newton on f'(t) = 0
        t -= df(t) / d2(t)
    return f(t)


def _d2_symbol_max(order: int) -> float:
    # -(b0 + 2 sum_j b_j cos(j theta)) is maximal at theta = pi for these stencils
    b0, b = {4: (-5 / 2, (4 / 3, -1 / 12)),
             8: (-205 / 72, (8 / 5, -1 / 5, 8 / 315, -1 / 560))}[order]
    return -(b0 + 2 * sum(bj * (-1) ** (j + 1) for j, bj in enumerate(b)))


def spectral_radius(pde: str, order: int, n: Sequence[int], length=(1.0, 1.0, 1.0)) -> float:
    s = [n[d] / length[d] for d in range(3)]
    if pde == "adv1d" and order == 0:
        return math.pi * s[0]               # spectral: pi / dx
    if pde == "adv1d":
        return s[0] * _d1_symbol_max(order)
    if pde == "acoustic2d":
        return math.hypot(s[0], s[1]) * _d1_symbol_max(order)
    if pde == "wave3d":
        return math.sqrt((s[0] ** 2 + s[1] ** 2 + s[2] ** 2) * _d2_symbol_max(order))
    raise ValueError(pde)


def macro_step(pde: str, order: int, n: Sequence[int], counts, w_fp64, h_factor: float = 0.5) -> float:
    """H = h_factor * ISB(R) / rho."""
    return h_factor * imaginary_stability_boundary(counts, w_fp64) / spectral_radius(pde, order, n)
