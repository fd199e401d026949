"""Exact-rational extrapolation weights (TEST INFRASTRUCTURE ONLY).

PAPER.md §3.2 Eq. (3) ("eq:vander", lines 186-225): with h_i = H/n_i the
p/2 order constraints are  sum_i c_i h_i^{2j} = delta_{j0},  j = 0..p/2-1
(odd powers vanish for even n, Eq. (2)).  The weights do not
depend on H (every row j scales by H^{2j}), so H = 1 here.

§3.7 Eqs. (5)-(6) (lines 403-425): for m > p/2 the weights split into
dependent and free parts, c_dep = V_dep^{-1} (b - V_free c_free).

All arithmetic is in ``fractions.Fraction``; conversion to fp64 happens once,
by correct rounding (``float(Fraction)``), PAPER.md:416-418 ("best computed
symbolically then converted").

Catalog (each entry cites where the paper prints it):
  FD8, FD12, FD16       Table 1 / §3.3.1-3.3.3
  GBS_8_6               §3.8.1
  GBS_8_8               §3.8.2, PAPER.md:492-501 (n_free read as {4..24},
                        DESIGN.md reading R4 / SURVEY.md S4)
  GBS_12_8              §3.8.3
  square8               square order-8 system on {2,4,6,8} (Eq. 3, m = p/2)
  fallback8(steps)      square8 on {2,4,6,8}, weight 0 on the other counts
                        (BASELINE.json configs 2-5 fallback; reading R3)
  nonzero8(steps)       n_dep = {2,4,6,8}, c_free = +1/50, -1/50, ... on the
                        other counts in ascending order, c_dep by Eq. (6)
                        (parity-only set; reading R3; parity unpinned by the
                        paper, pinned by Eq. (3) residual = 0)
"""

from __future__ import annotations

from fractions import Fraction as Fr
from typing import Dict, List, Sequence, Tuple


def _solve(A: List[List[Fr]], b: List[Fr]) -> List[Fr]:
    """Exact Gauss-Jordan elimination with row pivoting on nonzero pivots."""
    n = len(A)
    M = [list(row) + [bi] for row, bi in zip(A, b)]
    for col in range(n):
        piv = next((r for r in range(col, n) if M[r][col] != 0), None)
        if piv is None:
            raise ZeroDivisionError("singular Vandermonde system")
        M[col], M[piv] = M[piv], M[col]
        pv = M[col][col]
        M[col] = [x / pv for x in M[col]]
        for r in range(n):
            if r != col and M[r][col] != 0:
                fac = M[r][col]
                M[r] = [x - fac * y for x, y in zip(M[r], M[col])]
    return [M[r][n] for r in range(n)]


def vandermonde(counts: Sequence[int], p: int) -> List[List[Fr]]:
    """Eq. (3): p/2 x m matrix, row j holds h_i^{2j}, h_i = 1/n_i."""
    if p % 2:
        raise ValueError("order must be even")
    return [[Fr(1, n) ** (2 * j) for n in counts] for j in range(p // 2)]


def rhs_b(p: int) -> List[Fr]:
    return [Fr(1)] + [Fr(0)] * (p // 2 - 1)


def check_counts(counts: Sequence[int]) -> None:
    if len(set(counts)) != len(counts):
        raise ValueError("step counts must be distinct (PAPER.md:222-223)")
    for n in counts:
        if n < 2 or n % 2:
            raise ValueError("step counts must be even and >= 2 (PAPER.md:102-105)")


def full_weights(counts: Sequence[int], p: int) -> List[Fr]:
    """Square case m = p/2: solve V c = b."""
    check_counts(counts)
    if len(counts) != p // 2:
        raise ValueError("square system needs p/2 step counts")
    return _solve(vandermonde(counts, p), rhs_b(p))


def dependent_weights(n_dep: Sequence[int], n_free: Sequence[int],
                      c_free: Sequence[Fr], p: int) -> List[Fr]:
    """Eq. (6): c_dep = V_dep^{-1} (b - V_free c_free)."""
    check_counts(list(n_dep) + list(n_free))
    Vd = vandermonde(n_dep, p)
    Vf = vandermonde(n_free, p) if n_free else [[] for _ in range(p // 2)]
    b = rhs_b(p)
    rhs = [b[j] - sum((Vf[j][i] * c_free[i] for i in range(len(n_free))), Fr(0))
           for j in range(p // 2)]
    return _solve(Vd, rhs)


def residual(counts: Sequence[int], weights: Sequence[Fr], p: int) -> List[Fr]:
    """V c - b, exactly (Eq. 3)."""
    V = vandermonde(counts, p)
    b = rhs_b(p)
    return [sum((V[j][i] * weights[i] for i in range(len(counts))), Fr(0)) - b[j]
            for j in range(p // 2)]


def _F(s: str) -> Fr:
    return Fr(s)


# --- the paper's printed free weights, typed in from PAPER.md -------------
PAPER_SCHEMES: Dict[str, dict] = {
    "GBS_8_6": dict(order=8, n_dep=[2, 4, 6, 10], n_free=[8, 12, 14, 16, 18, 20, 22],
                    c_free=["2165/767488", "13805/611712", "4553/72080", "14503/66520",
                            "27058/7627", "-86504/5761", "40916/3367"],
                    cite="PAPER.md:455-461 (§3.8.1)"),
    "GBS_8_8": dict(order=8, n_dep=[2, 26, 28, 30],
                    n_free=[4, 6, 8, 10, 12, 14, 16, 18, 20, 22, 24],
                    c_free=["6833/476577792", "10847/91078656", "15235/34643968",
                            "383/321152", "543/198784", "9947/1741056", "6243/543104",
                            "6875/296192", "1401/28496", "17713/152688", "6375/19264"],
                    cite="PAPER.md:492-501 (§3.8.2); n_free read as {4..24} (reading R4)"),
    "GBS_12_8": dict(order=12, n_dep=[2, 8, 10, 16, 24, 26],
                     n_free=[4, 6, 12, 14, 18, 20, 22, 28, 30],
                     c_free=["235/21030240256", "4147/1612709888", "11521/39731200",
                             "2375/3528704", "6435/708736", "1291/15780", "11311/4672",
                             "-180864/751", "222080/2079"],
                     cite="PAPER.md:525-533 (§3.8.3)"),
}

FULL_SCHEMES: Dict[str, Tuple[int, List[int]]] = {
    "FD8": (8, [2, 16, 18, 20]),
    "FD12": (12, [2, 8, 12, 14, 16, 20]),
    "FD16": (16, [2, 8, 10, 12, 14, 16, 18, 22]),
    "square8": (8, [2, 4, 6, 8]),                      # Eq. (3), m = p/2
}


def scheme(name: str, steps: Sequence[int] | None = None) -> Tuple[List[int], List[Fr], int]:
    """Return (step counts ascending, exact weights aligned, order p)."""
    if name in FULL_SCHEMES:
        p, counts = FULL_SCHEMES[name]
        if steps is not None and sorted(steps) != sorted(counts):
            raise ValueError(f"{name} is defined on {counts}, not {list(steps)}")
        return list(counts), full_weights(counts, p), p
    if name in PAPER_SCHEMES:
        s = PAPER_SCHEMES[name]
        c_free = [_F(x) for x in s["c_free"]]
        c_dep = dependent_weights(s["n_dep"], s["n_free"], c_free, s["order"])
        pairs = sorted(list(zip(s["n_dep"], c_dep)) + list(zip(s["n_free"], c_free)))
        counts = [n for n, _ in pairs]
        if steps is not None and sorted(steps) != counts:
            raise ValueError(f"{name} is defined on {counts}, not {list(steps)}")
        return counts, [c for _, c in pairs], s["order"]
    if name in ("fallback8", "nonzero8"):
        if steps is None:
            raise ValueError(f"{name} needs the step counts")
        counts = sorted(steps)
        check_counts(counts)
        n_dep = [2, 4, 6, 8]
        if not set(n_dep) <= set(counts):
            raise ValueError(f"{name} needs {{2,4,6,8}} among the step counts")
        n_free = [n for n in counts if n not in n_dep]
        if name == "fallback8":
            c_free = [Fr(0)] * len(n_free)
        else:
            c_free = [Fr((-1) ** i, 50) for i in range(len(n_free))]
        c_dep = dependent_weights(n_dep, n_free, c_free, 8)
        wmap = dict(zip(n_dep, c_dep))
        wmap.update(zip(n_free, c_free))
        return counts, [wmap[n] for n in counts], 8
    if name == "opt8":
        # input data: the Appendix-B optimised free weights (gbs_inputs/optimized_schemes.json);
        # the dependent weights follow Eq. (6) here, by Gauss-Jordan
        from gbs_inputs.schemes import optimized_for
        if steps is None:
            raise ValueError("opt8 needs the step counts")
        s = optimized_for(steps)
        c_free = [_F(x) for x in s["c_free"]]
        c_dep = dependent_weights(s["n_dep"], s["n_free"], c_free, s["order"])
        pairs = sorted(list(zip(s["n_dep"], c_dep)) + list(zip(s["n_free"], c_free)))
        return [n for n, _ in pairs], [c for _, c in pairs], s["order"]
    raise KeyError(f"unknown weight set {name!r}")


def to_double(ws: Sequence[Fr]) -> List[float]:
    """Correctly rounded fp64 conversion."""
    return [float(w) for w in ws]
