"""Appendix-B ISB optimisation of the extrapolation weights (host side, layer L0).

Not on the hot path: runs offline and produces weight sets that ``gbs_create``
takes like any other.  Follows PAPER.md App. B
(lines 674-763) step by step:

* R(xi) = c_dep^T P_dep(xi) + c_free^T P_free(xi)  (App. B.3), with
  the order constraints eliminated exactly: c_dep = V_dep^{-1} (b - V_free c_free)
  (Eq. (6)), so R is affine in the free weights only.
* Convex subproblem (eq:cvx_subproblem): for a step h,
  r(h) = min over c_free of max over lambda in Lambda of |R(h lambda)| - 1, with
  Lambda = i [0, 1] (the imaginary-axis segment; wave-type problems, PAPER.md:
  129-149), sampled at N points.  The modulus constraints |z_j| <= t are second-
  order cones; they are solved exactly at the samples by a cutting-plane sequence
  of linear programs (scipy HiGHS): Re(z_j e^{-i phi}) <= t for a growing set of
  directions phi per sample, each new phi = arg z_j of the current iterate, until
  max_j |z_j| <= t (1 + 1e-10).  (The paper used CVX / OPTISB.)
* Outer problem (eq:reformulated_problem): bisection on h for
  the largest h with r(h) <= 0.
* The optimiser's free weights are taken exactly as binary fractions and the
  dependent weights recomputed exactly, so the order constraints hold exactly in
  the scheme handed to the GPU (the paper additionally searches
  small-integer rationals, which this does not).

The returned ISB is re-measured by the independent imaginary-axis scan of
``scheme.imaginary_stability_boundary`` (and, in the tests, by the oracle's).
"""

from __future__ import annotations

from fractions import Fraction
from typing import List, Sequence, Tuple

import numpy as np

from . import scheme as SC


# the plain subproblem counts h as feasible when max_j |R(i y_j)| <= 1 + PLAIN_TOL: the LP
# solver's own feasibility tolerance sits near 1e-9 for these ill-conditioned bases, and
# beyond the ISB |R| - 1 grows like (y - ISB)^1 so this moves h by < 1e-6
PLAIN_TOL = 1e-8
XMAX = 1000.0        # bound on |c_free| (the paper's schemes stay below 250)
TMIN = 0.01          # the margin problem's t >= -TMIN


def _component_values(n: int, z: np.ndarray) -> np.ndarray:
    """P_n(z) by running Eq. (1) on y' = lambda y (App. A)."""
    return SC._gbs_component(n, z)


def _affine_R(n_dep: Sequence[int], n_free: Sequence[int], ys: np.ndarray):
    """R(i y_j) = a_j + G_j @ c_free for the exact elimination of c_dep."""
    q, mf = len(n_dep), len(n_free)
    inv = SC.vandermonde_inverse(n_dep)                      # exact V_dep^{-1}
    # c_dep = inv @ (e_0 - V_free c_free): d0 = inv[:, 0], D = -inv @ V_free
    d0 = np.array([float(inv[i][0]) for i in range(q)])
    Vf = [[Fraction(1, n * n) ** j for n in n_free] for j in range(q)]
    D = np.array([[float(-sum((inv[i][j] * Vf[j][k] for j in range(q)), Fraction(0)))
                   for k in range(mf)] for i in range(q)])
    z = 1j * ys
    Pd = np.stack([_component_values(n, z) for n in n_dep], axis=1)       # [N, q]
    Pf = np.stack([_component_values(n, z) for n in n_free], axis=1)      # [N, mf]
    a = Pd @ d0
    G = Pf + Pd @ D
    return a, G


def minimax(n_dep: Sequence[int], n_free: Sequence[int], h: float, samples: int = 1500,
            max_rounds: int = 80, margin_power: int = 0) -> Tuple[float, np.ndarray]:
    """The convex subproblem at step h over the samples y_j of [0, h].

    margin_power = 0: r(h) + 1 = min_c max_j |R(i y_j)|; returns
    that value.  margin_power = k > 0: min t subject to |R(i y_j)| <= 1 + t (y_j/h)^k,
    a weighted form whose optimum t < 0 keeps |R| strictly below 1 away from the origin
    (where |R(iy)| = 1 - O(y^{p+2}) anyway), so the scheme survives fp64 rounding of
    its weights; returns 1 + t."""
    from scipy.optimize import linprog

    ys = np.linspace(0.0, h, samples)
    a, G = _affine_R(n_dep, n_free, ys)
    mf = len(n_free)
    wgt = np.ones(samples) if margin_power == 0 else np.maximum((ys / h) ** margin_power, 1e-300)
    off = 0.0 if margin_power == 0 else 1.0
    # rows: Re(e^{-i phi} (a_j + G_j x)) - w_j t <= off  (directions phi per sample, cutting planes)
    rows_j = np.repeat(np.arange(samples), 4)
    rows_p = np.tile(np.array([0.0, 0.5 * np.pi, np.pi, 1.5 * np.pi]), samples)
    # Well-conditioned variables: the P_n(iy) reach 1e5 on these segments while R stays
    # O(1), so the LP is posed in an orthonormal basis of the range of the map
    # x -> [Re G x; Im G x] (QR): z = z(x0) + Q y, y = Rr (x - x0), with x0 the least-
    # squares point and z(x0) = a + G x0 formed directly (accurate to ~1e-11).
    M = np.vstack([G.real, G.imag])
    Q, Rr = np.linalg.qr(M)
    ast = np.concatenate([a.real, a.imag])
    x0 = np.linalg.solve(Rr, -(Q.T @ ast))                    # least-squares shift
    ap = ast + M @ x0                                         # z(x0), O(1), formed directly
    Qre, Qim = Q[:samples], Q[samples:]
    Rinv = np.linalg.inv(Rr)
    apr, api = ap[:samples], ap[samples:]
    x = np.zeros(mf)
    t = np.inf
    for _ in range(max_rounds):
        cs, sn = np.cos(rows_p), np.sin(rows_p)
        A = np.hstack([cs[:, None] * Qre[rows_j] + sn[:, None] * Qim[rows_j], -wgt[rows_j][:, None]])
        b = off - (cs * apr[rows_j] + sn * api[rows_j])
        c = np.zeros(mf + 1)
        c[-1] = 1.0
        # |x_k| <= XMAX as rows in y (x = x0 + Rr^{-1} y), and t >= -TMIN: below the optimal
        # step the margin problem has a large optimal face; these keep the vertex the solver
        # returns at moderate weights instead of a huge cancelling combination
        Ab = np.vstack([np.hstack([Rinv, np.zeros((mf, 1))]), np.hstack([-Rinv, np.zeros((mf, 1))])])
        bb = np.concatenate([XMAX - x0, XMAX + x0])
        res = linprog(c, A_ub=np.vstack([A, Ab]), b_ub=np.concatenate([b, bb]),
                      bounds=[(None, None)] * mf + [(-TMIN if margin_power else None, None)], method="highs")
        if res.status != 0:
            raise RuntimeError(f"LP failed: {res.message}")
        yv, t = res.x[:mf], res.x[-1]
        x = x0 + np.linalg.solve(Rr, yv)
        zs = ap + Q @ yv
        zj = zs[:samples] + 1j * zs[samples:]
        lim = off + t * wgt
        viol = np.abs(zj) > lim + 1e-12 * np.maximum(1.0, np.abs(lim))
        if not viol.any():
            break
        new_j = np.nonzero(viol)[0]
        rows_j = np.concatenate([rows_j, new_j])
        rows_p = np.concatenate([rows_p, np.angle(zj[new_j])])
    if margin_power == 0:
        return float(np.max(np.abs(zj))), x
    return float(1.0 + t), x


def optimize_isb(n_dep: Sequence[int], n_free: Sequence[int], h_lo: float, h_hi: float,
                 tol: float = 1e-3, samples: int = 1500, margin_power: int = 0,
                 accept=None) -> Tuple[float, List[Fraction]]:
    """Bisection on h: the largest h whose subproblem value is
    <= 1 (+PLAIN_TOL; margin_power = 0) or < 1 (margin_power > 0) and, if given,
    accept(h, c_free) holds; returns h and that step's free weights as exact binary
    fractions."""
    def ok(h):
        m, x = minimax(n_dep, n_free, h, samples, margin_power=margin_power)
        good = m <= 1.0 + PLAIN_TOL if margin_power == 0 else m < 1.0
        cf = [Fraction(float(v)) for v in x]
        return (good and (accept is None or accept(h, cf))), cf

    good, cf = ok(h_lo)
    if not good:
        raise ValueError(f"h_lo = {h_lo} is not feasible")
    best = (h_lo, cf)
    lo, hi = h_lo, h_hi
    while hi - lo > tol:
        mid = 0.5 * (lo + hi)
        good, cf = ok(mid)
        if good:
            lo, best = mid, (mid, cf)
        else:
            hi = mid
    return best


def assemble(n_dep: Sequence[int], n_free: Sequence[int], cfree: Sequence[Fraction]):
    """(ascending counts, exact weights): c_dep from Eq. (6) in exact arithmetic."""
    cdep = SC.weights_exact(n_dep, n_free, cfree)
    w = dict(zip(n_dep, cdep))
    w.update(zip(n_free, cfree))
    counts = sorted(w)
    return counts, [w[n] for n in counts]


def optimized_scheme(n_dep: Sequence[int], n_free: Sequence[int], h_lo: float, h_hi: float,
                     tol: float = 1e-3, samples: int = 1500, margin_power: int = 10):
    """A usable optimised scheme: weighted-margin subproblem (so that |R(iy)| <= 1 +
    1e-10 survives the fp64 weights) and a bisection that accepts h only if the
    independent imaginary-axis scan of the fp64 scheme reaches h.  Returns
    (ascending counts, exact weights, scanned ISB)."""
    def accept(h, cf):
        counts, ws = assemble(n_dep, n_free, cf)
        return SC.imaginary_stability_boundary(counts, SC.to_fp64(ws), ymax=h * 1.01 + 1.0) >= h * (1 - 1e-9)

    h, cfree = optimize_isb(n_dep, n_free, h_lo, h_hi, tol, samples, margin_power, accept)
    counts, ws = assemble(n_dep, n_free, cfree)
    return counts, ws, SC.imaginary_stability_boundary(counts, SC.to_fp64(ws))
