"""GBS stability polynomials, imaginary stability boundary and the H rule
(TEST INFRASTRUCTURE ONLY).

* P_n(zeta): Eq. (1) applied to Dahlquist's y' = lambda y
  (App. A) with xi = zeta/n:  P_0 = 1, P_1 = 1 + xi,
  P_{k+1} = P_{k-1} + 2 xi P_k (k = 1..n), result (P_{n-1} + 2 P_n + P_{n+1})/4.
  Exact Fraction coefficients (``gbs_poly``) and a complex fp64 evaluation by
  the same recurrence (``gbs_eval``; the stable route).
* R(zeta) = sum_i c_i P_{n_i}(zeta)  (App. B).
* ISB: largest y with |R(iy)| <= 1 + tau on [0, y] (§2.2),
  by a dense scan (step 1e-4) then bisection to 1e-12; tau = 1e-10
  (SPEC.md:289).
* rho: spectral radius of the semi-discrete FD operator of each config
  (continuous-theta maximum of its Fourier symbol; reading R7).
* H rule: H = h_factor * ISB / rho (BASELINE.json configs, reading R7).
"""

from __future__ import annotations

from fractions import Fraction as Fr
from math import factorial
from typing import List, Sequence

import numpy as np

from . import fd


def _padd(p: List[Fr], q: List[Fr], s: Fr = Fr(1)) -> List[Fr]:
    n = max(len(p), len(q))
    out = [Fr(0)] * n
    for i, c in enumerate(p):
        out[i] += c
    for i, c in enumerate(q):
        out[i] += s * c
    while out and out[-1] == 0:
        out.pop()
    return out


def _pshift_scale(p: List[Fr], s: Fr) -> List[Fr]:
    """s * zeta * p(zeta)."""
    return [Fr(0)] + [s * c for c in p]


def gbs_poly(n: int) -> List[Fr]:
    """Exact coefficients of P_n(zeta), index k = coefficient of zeta^k."""
    if n < 2 or n % 2:
        raise ValueError("n must be even and >= 2")
    xi = Fr(1, n)                     # xi = zeta / n
    Pm, P = [Fr(1)], [Fr(1), xi]      # P_0, P_1
    levels = [Pm, P]
    for _ in range(1, n + 1):         # LF, k = 1..n
        Pn = _padd(levels[-2], _pshift_scale(levels[-1], 2 * xi))
        levels.append(Pn)
    PNm1, PN, PNp1 = levels[n - 1], levels[n], levels[n + 1]
    out = _padd(_padd(PNm1, PN, Fr(2)), PNp1)
    return [c / 4 for c in out]


def combined_poly(counts: Sequence[int], weights: Sequence[Fr]) -> List[Fr]:
    R: List[Fr] = []
    for n, c in zip(counts, weights):
        R = _padd(R, gbs_poly(n), Fr(c))
    return R


def order_of(counts: Sequence[int], weights: Sequence[Fr]) -> int:
    """Largest q with R(zeta) = e^zeta through zeta^q, exactly (Eq. (2) / SPEC verify_order)."""
    R = combined_poly(counts, weights)
    q = -1
    for k in range(len(R) + 2):
        ck = R[k] if k < len(R) else Fr(0)
        if ck != Fr(1, factorial(k)):
            return q
        q = k
    return q


def gbs_eval(n: int, zeta: np.ndarray) -> np.ndarray:
    """P_n(zeta) evaluated by running Eq. (1) on y' = lambda y in complex fp64."""
    z = np.asarray(zeta, dtype=np.complex128)
    xi = z / n
    ym1 = np.ones_like(z)
    y0 = ym1 + xi * ym1               # FE
    for k in range(1, n + 1):         # LF
        yp1 = ym1 + 2.0 * xi * y0
        if k < n:
            ym1, y0 = y0, yp1
    return 0.25 * ((ym1 + 2.0 * y0) + yp1)


def R_eval(counts: Sequence[int], weights: Sequence[float], zeta) -> np.ndarray:
    z = np.asarray(zeta, dtype=np.complex128)
    acc = np.zeros_like(z)
    for n, c in zip(counts, weights):
        acc = acc + float(c) * gbs_eval(n, z)
    return acc


def isb_fn(fun, tau: float = 1e-10, step: float = 1e-4, ymax: float = 200.0) -> float:
    """Largest y with |fun(i y')| <= 1 + tau for all y' in [0, y] (scan + bisection)."""
    chunk = 200_000
    y0 = 0.0
    while y0 < ymax:
        ys = y0 + step * np.arange(chunk)
        bad = np.abs(fun(1j * ys)) > 1.0 + tau
        if bad.any():
            i = int(np.argmax(bad))
            if i == 0 and y0 == 0.0:
                return 0.0
            lo = ys[i] - step
            hi = ys[i]
            while hi - lo > 1e-12:
                mid = 0.5 * (lo + hi)
                if abs(fun(np.array([1j * mid]))[0]) > 1.0 + tau:
                    hi = mid
                else:
                    lo = mid
            return float(lo)
        y0 = ys[-1] + step
    return ymax


def isb(counts: Sequence[int], weights: Sequence[float], tau: float = 1e-10,
        step: float = 1e-4, ymax: float = 200.0) -> float:
    """Imaginary stability boundary of R = sum c_i P_{n_i}."""
    w = [float(c) for c in weights]
    return isb_fn(lambda z: R_eval(counts, w, z), tau, step, ymax)


def critical_path(counts: Sequence[int], n_cores: int) -> int:
    """§3.6 folding rule: pair n with N_max - n on one core
    and share the first evaluation per core; return the max per-core count."""
    cs = sorted(counts, reverse=True)
    nmax = cs[0]
    loads = []
    used = set()
    for n in cs:
        if n in used:
            continue
        used.add(n)
        partner = nmax - n
        if partner in cs and partner not in used and partner != n:
            used.add(partner)
            loads.append((n + 1) + (partner + 1) - 1)
        else:
            loads.append(n + 1)
    # first-fit-decreasing onto n_cores if more groups than cores
    loads.sort(reverse=True)
    bins = [0] * n_cores
    cnt = [0] * n_cores
    for ld in loads:
        i = int(np.argmin(bins))
        bins[i] += ld - (1 if cnt[i] else 0)
        cnt[i] += 1
    return max(bins)


# --- spectral radius of the semi-discrete operators (reading R7) ----------
def _max_on_circle(fun, tol: float = 1e-15) -> float:
    th = np.linspace(0.0, np.pi, 200001)
    v = fun(th)
    i = int(np.argmax(v))
    lo, hi = th[max(i - 1, 0)], th[min(i + 1, len(th) - 1)]
    # golden-section refinement of the maximum
    g = (np.sqrt(5.0) - 1.0) / 2.0
    a, b = lo, hi
    c, d = b - g * (b - a), a + g * (b - a)
    while b - a > tol:
        if fun(np.array([c]))[0] > fun(np.array([d]))[0]:
            b = d
        else:
            a = c
        c, d = b - g * (b - a), a + g * (b - a)
    return float(max(v[i], fun(np.array([0.5 * (a + b)]))[0]))


def rho(pde: str, order: int, n: Sequence[int]) -> float:
    """max |lambda| over the continuous-theta symbol of the config's operator."""
    nx, ny, nz = n
    if pde == "adv1d" and order == 0:
        # spectral derivative: lambda = Delta t / Delta x = 0.99/pi ISB, "the factor of pi
        # arises from the spectral spatial derivatives": rho = pi / Delta x
        return float(np.pi * nx)
    if pde == "adv1d":
        kmax = _max_on_circle(lambda t: np.abs(fd.d1_symbol(order, t)))
        return nx * kmax
    if pde == "acoustic2d":
        kmax = _max_on_circle(lambda t: np.abs(fd.d1_symbol(order, t)))
        return float(np.sqrt(float(nx) ** 2 + float(ny) ** 2)) * kmax
    if pde == "wave3d":
        smax = _max_on_circle(lambda t: fd.d2_symbol_neg(order, t))
        return float(np.sqrt((float(nx) ** 2 + float(ny) ** 2 + float(nz) ** 2) * smax))
    raise ValueError(pde)


def macro_step_H(pde: str, order: int, n: Sequence[int], counts, weights,
                 h_factor: float = 0.5) -> float:
    """H = h_factor * ISB(R) / rho  (BASELINE.json configs; reading R7)."""
    return h_factor * isb(counts, weights) / rho(pde, order, n)
