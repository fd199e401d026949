"""Pins for oracle.stability: GBS polynomials, ISB and the paper's ISB_n table."""

import math
from fractions import Fraction as Fr

import numpy as np
import pytest

from oracle import stability as S
from oracle import weights as W


def test_p2_matches_hand_expansion(paper):
    g = paper["gbs_poly_n2"]
    assert S.gbs_poly(2) == [Fr(s) for s in g["coeffs"]]
    assert float(sum(S.gbs_poly(2))) == g["value_at_1"]
    assert S.gbs_eval(2, np.array([1.0 + 0j]))[0] == pytest.approx(g["value_at_1"], abs=0)


@pytest.mark.parametrize("n", [2, 4, 6, 8, 10, 16, 22, 30])
def test_poly_structure(n):
    P = S.gbs_poly(n)
    assert len(P) == n + 2                    # degree n + 1
    assert P[0] == 1 and P[1] == 1 and P[2] == Fr(1, 2)   # 2nd-order consistency
    assert P[3] != Fr(1, 6)                   # "accurate to at most second order"


@pytest.mark.parametrize("n", [2, 4, 8, 20, 30])
def test_recurrence_eval_matches_exact_coefficients(n):
    P = S.gbs_poly(n)
    zs = np.array([0.3 + 0.1j, 1j * 2.0, -0.7 + 0.4j, 1j * 0.5 * n])
    for z in zs:
        exact = sum(complex(float(c)) * z ** k for k, c in enumerate(P))
        got = S.gbs_eval(n, np.array([z]))[0]
        assert abs(got - exact) <= 1e-10 * max(1.0, abs(exact))


def test_rk4_isb(paper):
    rk4 = lambda z: 1 + z + z ** 2 / 2 + z ** 3 / 6 + z ** 4 / 24
    v = S.isb_fn(rk4)
    assert abs(v - 2 * math.sqrt(2)) < 1e-9          # closed form: |R(iy)|^2 = 1 - y^6/72 + y^8/576
    assert round(v, 4) == paper["rk4"]["isb"]
    assert round(v / 4, 4) == paper["rk4"]["isbn"]


def test_truncated_exponential_has_no_axis_coverage():
    # |R(iy)| ~ 1 + y^4/8: only the tau tolerance admits y <= (8 tau)^(1/4)
    v = S.isb_fn(lambda z: 1 + z + z ** 2 / 2)
    assert v < (8 * 1e-10) ** 0.25 + 1e-4


def test_partition_example(paper):
    g = paper["partition_example"]
    assert S.critical_path(g["counts"], g["cores"]) == g["evals_per_core"]


@pytest.mark.parametrize("name", ["FD8", "FD12", "FD16", "GBS_8_6", "GBS_8_8", "GBS_12_8"])
def test_isbn_matches_paper(paper, name):
    g = paper["isbn"][name]
    counts, w, _ = W.scheme(name)
    crit = S.critical_path(counts, g["cores"])
    v = S.isb(counts, W.to_double(w))
    assert round(v / crit, 4) == pytest.approx(g["value"], abs=1.01e-4), g["cite"]
    # |R(iy)| <= 1 + 1e-10 up to the paper-stated bound, trimmed for its 4-digit rounding
    ys = np.linspace(0.0, (g["value"] - 0.5e-4) * crit, 20001)
    assert np.max(np.abs(S.R_eval(counts, W.to_double(w), 1j * ys))) <= 1 + 1e-10
    # and just beyond the scanned ISB the method is unstable
    assert abs(S.R_eval(counts, W.to_double(w), np.array([1j * (v + 1e-3)]))[0]) > 1.0


@pytest.mark.parametrize("name", ["GBS_8_6", "GBS_8_8", "GBS_12_8"])
def test_rk4_step_ratios(paper, name):
    counts, w, _ = W.scheme(name)
    ratio = S.isb(counts, W.to_double(w)) / (2 * math.sqrt(2))
    assert ratio == pytest.approx(paper["rk4_step_ratio"][name], abs=0.02)


def test_combined_poly_equals_weighted_recurrence():
    counts, w, _ = W.scheme("GBS_8_6")
    R = S.combined_poly(counts, w)
    z = np.array([1j * 3.0])
    exact = sum(complex(float(c)) * z[0] ** k for k, c in enumerate(R))
    assert abs(S.R_eval(counts, W.to_double(w), z)[0] - exact) < 1e-9


def test_rho_closed_forms():
    # FD8 D2 symbol maximum is at theta = pi: s2(pi) = -(b0 + 2 sum_j b_j (-1)^j), exactly
    from oracle import fd
    b0, b = fd.d2_coeffs(8)
    s_pi = -(b0 + 2 * sum(bj * (-1) ** j for j, bj in enumerate(b, start=1)))
    assert s_pi == Fr(2048, 315)
    assert S.rho("wave3d", 8, (512, 512, 512)) == pytest.approx(math.sqrt(3 * 2048 / 315) * 512,
                                                                 rel=1e-12)
    # FD4 first-derivative symbol max: d/dtheta = 0 <=> 2c^2 - 4c - 1 = 0, c = cos(theta) = 1 - sqrt(6)/2
    th = math.acos(1 - math.sqrt(6) / 2)
    kmax = 2 * (2 / 3 * math.sin(th) - 1 / 12 * math.sin(2 * th))
    assert S.rho("adv1d", 4, (256, 1, 1)) == pytest.approx(256 * kmax, rel=1e-12)
