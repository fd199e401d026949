"""Pins for the C oracle's GBS stepping (gbs_oracle.c) against things other than itself:
exact-rational brute force, the per-mode closed form, the scalar stability polynomial,
invariants, the observed order of accuracy and the instability threshold."""

from fractions import Fraction as Fr

import numpy as np
import pytest

from gbs_inputs import get_config, make_ic, reduced
from oracle import c_oracle as C
from oracle import exact as E
from oracle import fourier as FO
from oracle import stability as S
from oracle import weights as W


def rel_l2(a, b):
    return float(np.linalg.norm((a - b).ravel()) / np.linalg.norm(b.ravel()))


def _dyadic_ic(shape, seed):
    rng = np.random.default_rng(seed)
    return rng.integers(-1024, 1025, size=shape).astype(np.float64) / 1024.0


# ---------------------------------------------------------------- exact brute force
@pytest.mark.parametrize("pde,order,shape,steps,M", [
    ("adv1d", 4, (1, 16), (2, 4, 6, 8), 3),
    ("adv1d", 8, (1, 12), (2, 4, 6, 8), 1),
    ("acoustic2d", 4, (3, 6, 7), (2, 4, 6, 8, 10, 12), 1),
    ("wave3d", 8, (2, 5, 6, 5), (2, 4, 6, 8), 1),
])
def test_matches_exact_rational_stepping(pde, order, shape, steps, M):
    y0 = _dyadic_ic(shape, 7)
    name = "square8" if steps == (2, 4, 6, 8) else "nonzero8"
    counts, w, _ = W.scheme(name, steps)
    H = Fr(1, 64) if pde == "adv1d" else Fr(1, 256)
    ex = E.to_float(E.advance(pde, order, y0, counts, w, H, M))
    got = C.advance(pde, order, y0, counts, W.to_double(w), float(H), M)
    assert rel_l2(got, ex) < 1e-13


# ---------------------------------------------------------------- Fourier closed form
@pytest.mark.parametrize("cfg,n,M,wset", [
    ("c1", (256, 1, 1), 200, "square8"),
    ("c2", (64, 48, 1), 20, "fallback8"),
    ("c2", (64, 48, 1), 20, "nonzero8"),
    ("c3", (40, 64, 1), 10, "nonzero8"),
    ("c4", (24, 20, 16), 6, "fallback8"),
    ("c5", (20, 16, 24), 3, "nonzero8"),
])
def test_matches_fourier_closed_form(cfg, n, M, wset):
    w_ = reduced(cfg, n, macro_steps=M, weights=wset)
    y0 = make_ic(w_)
    counts, w, _ = W.scheme(w_.weights, w_.steps)
    wd = W.to_double(w)
    H = S.macro_step_H(w_.pde, w_.order, w_.n, counts, wd, w_.h_factor)
    got = C.advance(w_.pde, w_.order, y0, counts, wd, H, M)
    ref = FO.gbs_closed_form(w_.pde, w_.order, y0, counts, wd, H, M)
    assert rel_l2(got, ref) < 1e-12


# ---------------------------------------------------------------- scalar stability function
@pytest.mark.parametrize("N", [2, 4, 8, 12])
def test_single_mode_is_stability_polynomial(N):
    """ADV1D on one Fourier mode is Dahlquist's y' = lambda y with lambda = -i nx k~(theta);
    stepping it must reproduce P_N(H lambda) computed from the exact coefficients."""
    nx, k, order = 32, 3, 4
    x = np.arange(nx) / nx
    lam = -1j * nx * float(np.asarray(__import__("oracle.fd", fromlist=["fd"]).d1_symbol(order, 2 * np.pi * k / nx)))
    H = 0.05
    P = S.gbs_poly(N)
    Rz = sum(complex(float(c)) * (H * lam) ** j for j, c in enumerate(P))
    y0c = np.cos(2 * np.pi * k * x)[None, :]
    y0s = np.sin(2 * np.pi * k * x)[None, :]
    outc = C.advance("adv1d", order, y0c, [N], [1.0], H, 1)
    outs = C.advance("adv1d", order, y0s, [N], [1.0], H, 1)
    z = outc[0] + 1j * outs[0]                   # = R * e^{i theta x}
    assert np.max(np.abs(z - Rz * np.exp(2j * np.pi * k * x))) < 1e-13


# ---------------------------------------------------------------- invariants
def test_constant_state_is_steady():
    for pde, shape in (("adv1d", (1, 20)), ("acoustic2d", (3, 9, 11)), ("wave3d", (2, 9, 9, 10))):
        y0 = np.full(shape, 0.75)
        if pde == "wave3d":
            y0[1] = 0.0                          # u const, v = 0 is steady (u_t = v = 0)
        counts, w, _ = W.scheme("fallback8", (2, 4, 6, 8, 10, 12))
        got = C.advance(pde, 8 if pde == "wave3d" else 4, y0, counts, W.to_double(w), 1e-3, 3)
        assert np.max(np.abs(got - y0)) <= 4e-15


def test_mean_is_conserved():
    w_ = reduced("c2", (48, 40, 1), macro_steps=10)
    y0 = make_ic(w_)
    counts, w, _ = W.scheme("nonzero8", w_.steps)
    wd = W.to_double(w)
    H = S.macro_step_H(w_.pde, w_.order, w_.n, counts, wd)
    got = C.advance(w_.pde, w_.order, y0, counts, wd, H, 10)
    assert abs(got[0].mean() - y0[0].mean()) < 1e-13


def test_zero_rhs_keeps_state_and_unit_weight_sum():
    y0 = np.zeros((2, 6, 6, 6))
    counts, w, _ = W.scheme("square8")
    got = C.advance("wave3d", 8, y0, counts, W.to_double(w), 0.1, 2)
    assert np.array_equal(got, y0)


# ---------------------------------------------------------------- order of accuracy (reading R9)
def test_observed_order_eight():
    w_ = get_config("c1")
    y0 = make_ic(w_)
    counts, w, _ = W.scheme("square8")
    wd = W.to_double(w)
    T = 200 * S.macro_step_H(w_.pde, w_.order, w_.n, counts, wd)
    ref = FO.exact_semidiscrete("adv1d", 4, y0, T)
    errs = []
    for M in (100, 200):
        got = C.advance("adv1d", 4, y0, counts, wd, T / M, M)
        errs.append(np.max(np.abs(got - ref)))
    ratio = errs[0] / errs[1]
    assert 2 ** 7.6 < ratio < 2 ** 8.4, (errs, ratio)


# ---------------------------------------------------------------- stability threshold
@pytest.mark.parametrize("fac,grows", [(1.05, True), (0.99, False)])
def test_instability_threshold(fac, grows):
    """Unit-amplitude extreme mode of the 3-D wave: above the ISB it grows as |R|^M."""
    n = 16
    counts, w, _ = W.scheme("square8")
    wd = W.to_double(w)
    x = np.arange(n) / n
    z, yy, xx = np.meshgrid(x, x, x, indexing="ij")
    u = np.cos(np.pi * n * xx) * np.cos(np.pi * n * yy) * np.cos(np.pi * n * z)  # theta = pi
    y0 = np.stack([u, np.zeros_like(u)])
    rho = S.rho("wave3d", 8, (n, n, n))
    H = fac * S.isb(counts, wd) / rho
    M = 60
    got = C.advance("wave3d", 8, y0, counts, wd, H, M)
    ref = FO.gbs_closed_form("wave3d", 8, y0, counts, wd, H, M)
    assert rel_l2(got, ref) < 1e-10
    amp = np.max(np.abs(got[0]))
    if grows:
        R = abs(S.R_eval(counts, wd, np.array([1j * H * rho]))[0])
        assert R > 1.01 and amp > 0.5 * R ** M
    else:
        assert amp <= 1.0 + 1e-9


# ---------------------------------------------------------------- sampled-output method
def test_box_sample_reproduces_full_grid_value_bitwise():
    """The sampled-parity method: the oracle run on a periodically extracted box of
    half-width >= r * (max n_k + 1) * M, with the full grid's spacing, gives the
    full-grid value at the box centre bit for bit (same arithmetic, same inputs)."""
    w_ = reduced("c4", (40, 36, 38), macro_steps=1)
    y0 = make_ic(w_)
    counts, w, _ = W.scheme("nonzero8", w_.steps)
    wd = W.to_double(w)
    H = S.macro_step_H(w_.pde, w_.order, w_.n, counts, wd)
    full = C.advance(w_.pde, w_.order, y0, counts, wd, H, 1)
    R = 4 * (max(counts) + 1)
    for (cz, cy, cx) in [(0, 0, 0), (17, 35, 3), (37, 10, 20)]:
        iz = np.arange(cz - R, cz + R + 1) % 38
        iy = np.arange(cy - R, cy + R + 1) % 36
        ix = np.arange(cx - R, cx + R + 1) % 40
        box = y0[:, iz][:, :, iy][:, :, :, ix]
        out = C.advance(w_.pde, w_.order, box, counts, wd, H, 1, scale=(40, 36, 38))
        assert np.array_equal(out[:, R, R, R], full[:, cz, cy, cx])


def test_thread_count_does_not_change_bits():
    w_ = reduced("c4", (20, 18, 16), macro_steps=1)
    y0 = make_ic(w_)
    counts, w, _ = W.scheme("nonzero8", w_.steps)
    wd = W.to_double(w)
    a = C.advance(w_.pde, w_.order, y0, counts, wd, 1e-3, 1, threads=1)
    b = C.advance(w_.pde, w_.order, y0, counts, wd, 1e-3, 1, threads=4)
    C.set_threads(__import__("os").cpu_count() or 1)
    assert np.array_equal(a, b)
