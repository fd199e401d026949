"""Seeded initial conditions (BASELINE.json configs).

All generators return a C-contiguous float64 numpy array shaped like the SoA
state ``[F][nz][ny][nx]`` (unused axes dropped), on the unit periodic box
with grid points x_i = i / n (S6).  They are pure input plumbing: the same
bytes are handed to the oracle and to the CUDA path (S12).

Recipes (draw order is part of the recipe; ``numpy.random.default_rng(seed)``):

* ``gauss1d``: c ~ U(0.3, 0.7), then s ~ U(0.03, 0.08);
  u = exp(-(d/s)^2), d = minimum-image distance ((x - c + 1/2) mod 1) - 1/2.
* ``gauss2d_sum8``: for each of 8 pulses: (cx, cy) ~ U[0,1)^2, then
  s ~ U(0.03, 0.08); p = sum_i exp(-(dx/s)^2) * exp(-(dy/s)^2); u = v = 0.
* ``gauss3d``: (cx, cy, cz) ~ U(0.3, 0.7)^3, then s ~ U(0.03, 0.08);
  u = exp(-(dx/s)^2) * exp(-(dy/s)^2) * exp(-(dz/s)^2); v = 0.
* ``bandlimited2d`` / ``bandlimited3d``: integer wavevectors k with
  1 <= |k| <= 64 and |k_d| < n_d / 2 on every axis, restricted to the half
  space (kx > 0) or (kx = 0, ky > 0) or (kx = ky = 0, kz > 0), enumerated in
  ascending lexicographic (kz, ky, kx) order; one phase phi_k ~ U[0, 2*pi)
  per mode in that order; field = sum_k |k|^-2 cos(2*pi k.x + phi_k)
  (a real, i.e. Hermitian-symmetric, band-limited field), divided by its exact RMS
  sqrt(sum_k |k|^-4 / 2) (Parseval), i.e. unit RMS.
  Placed in p (2-D acoustics, u = v = 0) or in u (3-D wave, v = 0).
"""

from __future__ import annotations

import numpy as np

from .configs import Workload

KMAX = 64


def _min_image(x: np.ndarray, c: float) -> np.ndarray:
    return np.mod(x - c + 0.5, 1.0) - 0.5


def _axis(n: int) -> np.ndarray:
    return np.arange(n, dtype=np.float64) / n


def gauss1d(nx: int, seed: int) -> np.ndarray:
    rng = np.random.default_rng(seed)
    c = rng.uniform(0.3, 0.7)
    s = rng.uniform(0.03, 0.08)
    d = _min_image(_axis(nx), c)
    return np.exp(-(d / s) ** 2)[None, :].copy()


def gauss2d_sum8(nx: int, ny: int, seed: int) -> np.ndarray:
    rng = np.random.default_rng(seed)
    out = np.zeros((3, ny, nx), dtype=np.float64)
    x, y = _axis(nx), _axis(ny)
    for _ in range(8):
        cx, cy = rng.uniform(0.0, 1.0, size=2)
        s = rng.uniform(0.03, 0.08)
        gx = np.exp(-(_min_image(x, cx) / s) ** 2)
        gy = np.exp(-(_min_image(y, cy) / s) ** 2)
        out[0] += gy[:, None] * gx[None, :]
    return out


def gauss3d(nx: int, ny: int, nz: int, seed: int, srange=None) -> np.ndarray:
    rng = np.random.default_rng(seed)
    cx, cy, cz = rng.uniform(0.3, 0.7, size=3)
    s = rng.uniform(0.03, 0.08)
    gx = np.exp(-(_min_image(_axis(nx), cx) / s) ** 2)
    gy = np.exp(-(_min_image(_axis(ny), cy) / s) ** 2)
    gz = np.exp(-(_min_image(_axis(nz), cz) / s) ** 2)
    lo, hi = (0, nz) if srange is None else srange
    out = np.zeros((2, hi - lo, ny, nx), dtype=np.float64)
    gyx = gy[:, None] * gx[None, :]
    for z in range(lo, hi):
        out[0, z - lo] = gz[z] * gyx
    return out


def _half_space_modes(dims: tuple, kmax: int = KMAX):
    """Integer wavevectors (per axis, fastest = x last) of the band-limited recipe."""
    nd = len(dims)  # dims = (nx,) / (nx, ny) / (nx, ny, nz)
    lim = [min(kmax, (n - 1) // 2) for n in dims]   # |k_d| < n_d/2
    rng_z = range(-lim[2], lim[2] + 1) if nd == 3 else [0]
    rng_y = range(-lim[1], lim[1] + 1) if nd >= 2 else [0]
    modes = []
    for kz in rng_z:
        for ky in rng_y:
            for kx in range(0, lim[0] + 1):
                k2 = kx * kx + ky * ky + kz * kz
                if k2 < 1 or k2 > kmax * kmax:
                    continue
                if kx > 0 or (kx == 0 and ky > 0) or (kx == 0 and ky == 0 and kz > 0):
                    modes.append((kx, ky, kz))
    return np.array(modes, dtype=np.int64).reshape(-1, 3), lim


def bandlimited(dims: tuple, seed: int, srange=None) -> np.ndarray:
    """Real band-limited field on the grid `dims` = (nx[, ny[, nz]]), unit RMS.

    Evaluated as Re(sum_k A_k e^{i phi_k} e^{2 pi i k.x}) by staged inverse
    transforms (z, y by small dense matrices; x by a real inverse FFT) and scaled by
    the exact RMS sqrt(sum_k A_k^2 / 2) (Parseval: the half-space modes are distinct,
    none is a Nyquist mode).  `srange` = (lo, hi) returns only planes [lo, hi) of the
    slowest axis (z in 3-D, y in 2-D), identical to the same planes of the full field.
    """
    rng = np.random.default_rng(seed)
    modes, lim = _half_space_modes(dims)
    phase = rng.uniform(0.0, 2.0 * np.pi, size=len(modes))
    amp = 1.0 / (modes ** 2).sum(axis=1).astype(np.float64)   # |k|^-2
    coef = amp * np.exp(1j * phase)
    rms = np.sqrt(0.5 * np.sum(amp * amp))
    nd = len(dims)
    nx = dims[0]
    ny = dims[1] if nd >= 2 else 1
    nz = dims[2] if nd == 3 else 1
    slow = nz if nd == 3 else ny
    lo, hi = (0, slow) if srange is None else (int(srange[0]), int(srange[1]))
    Kx, Ky, Kz = lim[0], (lim[1] if nd >= 2 else 0), (lim[2] if nd == 3 else 0)
    T = np.zeros((2 * Kz + 1, 2 * Ky + 1, Kx + 1), dtype=np.complex128)
    T[modes[:, 2] + Kz, modes[:, 1] + Ky, modes[:, 0]] = coef
    # irfft convention: f(x) = nx * irfft(G')[x], G'_0 = G_0, G'_k = G_k / 2
    T[:, :, 1:] *= 0.5
    zs = np.arange(lo, hi) if nd == 3 else np.arange(1)
    ys = np.arange(ny) if nd == 3 else np.arange(lo, hi)
    Ez = np.exp(2j * np.pi * np.outer(zs, np.arange(-Kz, Kz + 1)) / nz)
    Ey = np.exp(2j * np.pi * np.outer(ys, np.arange(-Ky, Ky + 1)) / ny)
    # one plane at a time, so a plane's bytes do not depend on the requested range
    T2 = T.reshape(T.shape[0], -1)
    Tz = np.stack([(Ez[i:i + 1] @ T2).reshape(T.shape[1:]) for i in range(len(zs))])   # (nzr, 2Ky+1, Kx+1)
    out = np.empty((len(zs), len(ys), nx), dtype=np.float64)
    chunk = max(1, (1 << 26) // max(1, len(ys) * (nx // 2 + 1)))
    for z0 in range(0, len(zs), chunk):
        z1 = min(len(zs), z0 + chunk)
        G = np.matmul(Ey[None, :, :], Tz[z0:z1])          # (zc, nyr, Kx+1)
        Gp = np.zeros((z1 - z0, len(ys), nx // 2 + 1), dtype=np.complex128)
        Gp[:, :, : Kx + 1] = G
        out[z0:z1] = nx * np.fft.irfft(Gp, n=nx, axis=2)
    out /= rms
    if nd == 1:
        return out[0, 0]
    if nd == 2:
        return out[0]
    return out


def make_ic(w: Workload, srange=None) -> np.ndarray:
    """Initial state for workload `w`, shaped ``w.state_shape``, float64.

    `srange` = (lo, hi): only planes [lo, hi) of the slowest axis (z in 3-D, y in 2-D),
    bit-identical to the same planes of the full state (for multi-GPU slabs)."""
    nx, ny, nz = w.n
    if srange is not None and w.ndim == 1:
        raise ValueError("1-D states are not slabbed")
    if w.ic == "gauss1d":
        y = gauss1d(nx, w.seed)
    elif w.ic == "cos1d":
        # PAPER.md §4.1 (line 560): u(x, 0) = (1 - cos 2 pi x) / 2 on [0, 1) (no random draw)
        y = (0.5 * (1.0 - np.cos(2.0 * np.pi * np.arange(nx) / nx)))[None, :]
    elif w.ic == "gauss2d_sum8":
        y = gauss2d_sum8(nx, ny, w.seed)
        if srange is not None:
            y = y[:, srange[0]:srange[1]]
    elif w.ic == "gauss3d":
        y = gauss3d(nx, ny, nz, w.seed, srange)
    elif w.ic == "bandlimited2d":
        p = bandlimited((nx, ny), w.seed, srange)
        y = np.zeros((3,) + p.shape, dtype=np.float64)
        y[0] = p
    elif w.ic == "bandlimited3d":
        u = bandlimited((nx, ny, nz), w.seed, srange)
        y = np.zeros((2,) + u.shape, dtype=np.float64)
        y[0] = u
    else:
        raise ValueError(f"unknown IC recipe {w.ic!r}")
    if srange is None:
        assert y.shape == w.state_shape, (y.shape, w.state_shape)
    return np.ascontiguousarray(y, dtype=np.float64)
