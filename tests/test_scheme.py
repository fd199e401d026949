"""Host-side scheme setup of the product (paper_1907_11771_b200.scheme) against the oracle:
identical exact weights, identical fp64 weights, H within the ISB bisection tolerance."""

import pytest

from gbs_inputs import CONFIGS
from oracle import stability as OS
from oracle import weights as OW
from paper_1907_11771_b200 import scheme as PS


@pytest.mark.parametrize("name", ["FD8", "FD12", "FD16", "GBS_8_6", "GBS_8_8", "GBS_12_8",
                                  "square8"])
def test_catalog_weights_identical(name):
    c1, w1, p1 = PS.weight_set(name)
    c2, w2, p2 = OW.scheme(name)
    assert (c1, w1, p1) == (c2, w2, p2)
    assert PS.to_fp64(w1) == OW.to_double(w2)


@pytest.mark.parametrize("steps", [(2, 4, 6, 8, 10, 12), (2, 4, 6, 8, 10, 12, 14, 16)])
@pytest.mark.parametrize("name", ["fallback8", "nonzero8"])
def test_config_weights_identical(name, steps):
    assert PS.weight_set(name, steps) == OW.scheme(name, steps)


@pytest.mark.parametrize("cfg", sorted(CONFIGS))
def test_H_rule_agrees(cfg):
    w = CONFIGS[cfg]
    counts, ws, _ = PS.weight_set(w.weights, w.steps)
    wd = PS.to_fp64(ws)
    Hp = PS.macro_step(w.pde, w.order, w.n, counts, wd, w.h_factor)
    Ho = OS.macro_step_H(w.pde, w.order, w.n, counts, wd, w.h_factor)
    assert Hp == pytest.approx(Ho, rel=1e-11)


def test_survey_H_values():
    """SURVEY.md §8(c) S7 lists H = 5.4839e-3 / 9.6943e-4 / 1.9217e-4 / 8.5195e-4 / 4.2597e-4."""
    want = {"c1": 5.4839e-3, "c2": 9.6943e-4, "c3": 1.9217e-4, "c4": 8.5195e-4, "c5": 4.2597e-4}
    for cfg, h in want.items():
        w = CONFIGS[cfg]
        counts, ws, _ = PS.weight_set(w.weights, w.steps)
        H = PS.macro_step(w.pde, w.order, w.n, counts, PS.to_fp64(ws), w.h_factor)
        assert H == pytest.approx(h, rel=1e-4)


def test_spectral_radius_agrees():
    for pde, order, n in [("adv1d", 4, (256, 1, 1)), ("acoustic2d", 8, (4096, 4096, 1)),
                          ("acoustic2d", 4, (100, 60, 1)), ("wave3d", 8, (512, 256, 128))]:
        assert PS.spectral_radius(pde, order, n) == pytest.approx(OS.rho(pde, order, n), rel=1e-12)
