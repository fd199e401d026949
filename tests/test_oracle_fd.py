"""Pins for the C oracle's FD right-hand sides (gbs_oracle.c)."""

import math

import numpy as np
import pytest

from oracle import c_oracle as C
from oracle import fd


@pytest.mark.parametrize("order", [4, 8])
def test_c_tables_equal_taylor_solution(order):
    a, b0, b = C.fd_coeffs(order)
    assert list(a) == [float(x) for x in fd.d1_coeffs(order)]
    eb0, eb = fd.d2_coeffs(order)
    assert b0 == float(eb0) and list(b) == [float(x) for x in eb]


def test_taylor_solution_textbook_fd4():
    # the two classic 4th-order stencils, derivable by hand
    from fractions import Fraction as Fr
    assert fd.d1_coeffs(4) == [Fr(2, 3), Fr(-1, 12)]
    assert fd.d2_coeffs(4) == (Fr(-5, 2), [Fr(4, 3), Fr(-1, 12)])


def _err_1d(order, n):
    x = np.arange(n) / n
    u = np.sin(2 * np.pi * x)[None, :]
    f = C.rhs("adv1d", order, u)                 # f = -u_x
    return np.max(np.abs(f[0] + 2 * np.pi * np.cos(2 * np.pi * x)))


@pytest.mark.parametrize("order", [4, 8])
def test_adv1d_convergence_order(order):
    e1, e2 = _err_1d(order, 32), _err_1d(order, 64)
    assert math.log2(e1 / e2) == pytest.approx(order, abs=0.1)


def test_acoustic2d_rhs_closed_form():
    n = 64
    x = np.arange(n) / n
    X, Y = np.meshgrid(x, x, indexing="xy")       # arrays [ny][nx]
    p = np.sin(2 * np.pi * X) * np.cos(4 * np.pi * Y)
    u = np.cos(2 * np.pi * X)
    v = np.sin(2 * np.pi * Y)
    y = np.stack([p, u, v])
    for order in (4, 8):
        f = C.rhs("acoustic2d", order, y)
        ex_p = -(-2 * np.pi * np.sin(2 * np.pi * X) + 2 * np.pi * np.cos(2 * np.pi * Y))
        ex_u = -(2 * np.pi * np.cos(2 * np.pi * X) * np.cos(4 * np.pi * Y))
        ex_v = -(-4 * np.pi * np.sin(2 * np.pi * X) * np.sin(4 * np.pi * Y))
        tol = {4: 2e-2, 8: 5e-5}[order]
        for got, ex in zip(f, (ex_p, ex_u, ex_v)):
            assert np.max(np.abs(got - ex)) < tol


def test_wave3d_rhs_closed_form():
    nx, ny, nz = 24, 20, 16
    z, yy, x = np.meshgrid(np.arange(nz) / nz, np.arange(ny) / ny, np.arange(nx) / nx,
                           indexing="ij")
    u = np.sin(2 * np.pi * x) * np.cos(2 * np.pi * yy) * np.sin(2 * np.pi * z)
    v = np.cos(2 * np.pi * (x + z))
    f = C.rhs("wave3d", 8, np.stack([u, v]))
    assert np.array_equal(f[0], v)                       # u_t = v, exactly
    lap = -3 * (2 * np.pi) ** 2 * u
    assert np.max(np.abs(f[1] - lap)) < 1e-4 * np.max(np.abs(lap))


def test_wave3d_rhs_symbol_matches_fourier():
    """Single Fourier mode: D2 e^{i theta x} = -N^2 s2(theta) e^{i theta x}."""
    nx, ny, nz = 16, 12, 10
    k = 5
    x = np.arange(nx) / nx
    u = np.broadcast_to(np.cos(2 * np.pi * k * x), (nz, ny, nx))
    f = C.rhs("wave3d", 8, np.stack([u, np.zeros_like(u)]))
    s2 = fd.d2_symbol_neg(8, 2 * np.pi * k / nx)
    assert np.allclose(f[1], -(nx ** 2) * s2 * u, rtol=0, atol=1e-9 * nx ** 2)
