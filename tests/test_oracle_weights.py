"""Pins for oracle.weights: exact Eq. (3)/(6) weights against the paper's printed values."""

from fractions import Fraction as Fr

import pytest

from oracle import stability as S
from oracle import weights as W


@pytest.mark.parametrize("name", ["FD8", "FD12"])
def test_fully_determined_weights_match_paper(paper, name):
    g = paper["fd_weights"][name]
    counts, w, p = W.scheme(name)
    assert counts == g["counts"] and p == g["order"]
    assert w == [Fr(s) for s in g["weights"]], g["cite"]


def test_square_p4_hand_solution(paper):
    g = paper["square_p4"]
    assert W.full_weights(g["counts"], 4) == [Fr(s) for s in g["weights"]]


@pytest.mark.parametrize("name", ["FD8", "FD12", "FD16", "GBS_8_6", "GBS_8_8", "GBS_12_8",
                                  "square8"])
def test_order_constraints_exact(name):
    counts, w, p = W.scheme(name)
    assert all(r == 0 for r in W.residual(counts, w, p))
    assert sum(w) == 1


@pytest.mark.parametrize("steps", [(2, 4, 6, 8, 10, 12), (2, 4, 6, 8, 10, 12, 14, 16)])
@pytest.mark.parametrize("name", ["fallback8", "nonzero8"])
def test_config_weight_sets(name, steps):
    counts, w, p = W.scheme(name, steps)
    assert counts == list(steps) and p == 8
    assert all(r == 0 for r in W.residual(counts, w, 8))
    if name == "fallback8":
        assert w[4:] == [0] * (len(steps) - 4)
        assert w[:4] == W.full_weights([2, 4, 6, 8], 8)
    else:
        assert all(x != 0 for x in w)
        assert w[4:] == [Fr((-1) ** i, 50) for i in range(len(steps) - 4)]


@pytest.mark.parametrize("name", ["FD8", "FD12", "FD16", "GBS_8_6", "GBS_8_8", "GBS_12_8"])
def test_order_matches_paper(paper, name):
    counts, w, _ = W.scheme(name)
    assert S.order_of(counts, w) == paper["orders"][name]


def test_perturbed_weight_breaks_order():
    counts, w, _ = W.scheme("FD8")
    w2 = list(w)
    w2[1] += Fr(1, 1000)
    assert S.order_of(counts, w2) < 8


def test_gbs88_free_list_reading():
    """Reading R4: with n_free = {4..22} (10 counts) the 11 printed c_free cannot align."""
    s = W.PAPER_SCHEMES["GBS_8_8"]
    assert len(s["c_free"]) == 11 and len(s["n_free"]) == 11
    assert s["n_free"][-1] == 24


def test_invalid_counts_rejected():
    with pytest.raises(ValueError):
        W.full_weights([2, 3], 4)
    with pytest.raises(ValueError):
        W.full_weights([2, 2], 4)


def test_to_double_is_correctly_rounded():
    x = Fr(1, 3)
    d = W.to_double([x])[0]
    # the neighbours of d are farther from 1/3 than d is
    import math
    lo, hi = math.nextafter(d, 0.0), math.nextafter(d, 1.0)
    assert abs(Fr(d) - x) <= abs(Fr(lo) - x) and abs(Fr(d) - x) <= abs(Fr(hi) - x)
