"""Closed-form solution of the linear periodic configs, mode by mode
(TEST INFRASTRUCTURE ONLY).

Every BASELINE.json config is linear, constant-coefficient and periodic, so
the DFT diagonalises the semi-discrete operator into small per-mode blocks.
For a one-step method with stability function R (App. A, PAPER.md:631-633;
R = sum c_i P_{n_i}, App. B) one macro step maps each block to
R(H A_k); M macro steps to R(H A_k)^M.  The exact semi-discrete solution is
exp(T A_k) (used for the order-8 convergence pin, reading R9).

Blocks (symbols from oracle.fd, theta_d = 2 pi k_d / N_d):
  adv1d       A = -i N k~(theta)                              (scalar)
  acoustic2d  A = -i S, S = [[0, ax, ay], [ax, 0, 0], [ay, 0, 0]],
              a_d = N_d k~(theta_d); S = Q diag(0, +r, -r) Q^T, r = |a|
  wave3d      A = [[0, 1], [-sigma, 0]], sigma = sum_d N_d^2 s2(theta_d);
              eigenvalues +-i sqrt(sigma); the sigma = 0 mode is the Jordan
              block phi(A) = phi(0) I + phi'(0) A.

``phi`` maps an array of eigenvalues lambda to the multiplier phi(lambda);
``dphi0`` is phi'(0), needed only for the 3-D zero mode.
"""

from __future__ import annotations

from typing import Callable, Sequence

import numpy as np

from . import fd
from .stability import R_eval


def _thetas(n: int) -> np.ndarray:
    return 2.0 * np.pi * np.fft.fftfreq(n) * 1.0  # fftfreq gives k/n in [-1/2, 1/2)


def modal_apply(pde: str, order: int, y0: np.ndarray, phi: Callable, dphi0: float,
                scale: Sequence[float] | None = None) -> np.ndarray:
    y0 = np.asarray(y0, dtype=np.float64)
    if pde == "adv1d":
        nx = y0.shape[1]
        N = scale[0] if scale else nx
        lam = -1j * N * fd.d1_symbol(order, _thetas(nx))
        return np.real(np.fft.ifft(phi(lam) * np.fft.fft(y0[0])))[None, :]
    if pde == "acoustic2d":
        _, ny, nx = y0.shape
        Nx, Ny = (scale[0], scale[1]) if scale else (nx, ny)
        ax = (Nx * fd.d1_symbol(order, _thetas(nx)))[None, :] * np.ones((ny, 1))
        ay = (Ny * fd.d1_symbol(order, _thetas(ny)))[:, None] * np.ones((1, nx))
        P, U, V = (np.fft.fft2(y0[i]) for i in range(3))
        r = np.sqrt(ax * ax + ay * ay)
        safe = np.where(r > 0, r, 1.0)
        ex, ey = ax / safe, ay / safe
        s2 = np.sqrt(0.5)
        # eigenvectors of S: v+ = [1, ex, ey]/sqrt2 (mu=+r), v- = [1,-ex,-ey]/sqrt2, v0 = [0, ey, -ex]
        cp = s2 * (P + ex * U + ey * V)
        cm = s2 * (P - ex * U - ey * V)
        c0 = ey * U - ex * V
        fp, fm, f0 = phi(-1j * r), phi(1j * r), phi(np.zeros_like(r) + 0j)
        Pn = s2 * (fp * cp + fm * cm)
        Un = s2 * ex * (fp * cp - fm * cm) + ey * f0 * c0
        Vn = s2 * ey * (fp * cp - fm * cm) - ex * f0 * c0
        zero = r == 0
        f00 = phi(np.array([0j]))[0]
        Pn = np.where(zero, f00 * P, Pn)
        Un = np.where(zero, f00 * U, Un)
        Vn = np.where(zero, f00 * V, Vn)
        return np.stack([np.real(np.fft.ifft2(X)) for X in (Pn, Un, Vn)])
    if pde == "wave3d":
        _, nz, ny, nx = y0.shape
        Nx, Ny, Nz = scale if scale else (nx, ny, nz)
        sig = ((Nx ** 2) * fd.d2_symbol_neg(order, _thetas(nx))[None, None, :]
               + (Ny ** 2) * fd.d2_symbol_neg(order, _thetas(ny))[None, :, None]
               + (Nz ** 2) * fd.d2_symbol_neg(order, _thetas(nz))[:, None, None])
        sig = np.maximum(sig, 0.0)
        w = np.sqrt(sig)
        U, V = np.fft.fftn(y0[0]), np.fft.fftn(y0[1])
        safe = np.where(w > 0, w, 1.0)
        cp = 0.5 * (U - 1j * V / safe)
        cm = 0.5 * (U + 1j * V / safe)
        fp, fm = phi(1j * w), phi(-1j * w)
        Un = fp * cp + fm * cm
        Vn = 1j * w * (fp * cp - fm * cm)
        zero = w == 0
        f00 = phi(np.array([0j]))[0]
        Un = np.where(zero, f00 * U + dphi0 * V, Un)
        Vn = np.where(zero, f00 * V, Vn)
        return np.stack([np.real(np.fft.ifftn(Un)), np.real(np.fft.ifftn(Vn))])
    raise ValueError(pde)


def gbs_closed_form(pde: str, order: int, y0: np.ndarray, counts, weights, H: float, M: int,
                    scale=None) -> np.ndarray:
    """Y after M macro steps: each mode multiplied by R(H lambda)^M."""
    w = [float(c) for c in weights]

    def phi(lam):
        return R_eval(counts, w, H * np.asarray(lam)) ** M

    dphi0 = M * H * float(sum(w))     # d/dlam R(H lam)^M at 0, R'(0) = sum_i c_i P_i'(0) = sum c_i
    return modal_apply(pde, order, y0, phi, dphi0, scale)


def exact_semidiscrete(pde: str, order: int, y0: np.ndarray, T: float, scale=None) -> np.ndarray:
    """exp(T A) y0: the exact solution of the semi-discrete ODE system (reading R9)."""
    return modal_apply(pde, order, y0, lambda lam: np.exp(T * np.asarray(lam)), T, scale)
