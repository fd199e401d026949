"""The seeded input generators (gbs_inputs): shapes, determinism, recipe properties."""

import numpy as np
import pytest

from gbs_inputs import CONFIGS, get_config, make_ic, reduced


def test_config_table_matches_baseline():
    c = CONFIGS
    assert c["c1"].n == (256, 1, 1) and c["c1"].macro_steps == 200 and c["c1"].order == 4
    assert c["c2"].n == (1024, 1024, 1) and c["c2"].macro_steps == 50
    assert c["c3"].n == (4096, 4096, 1) and c["c3"].order == 8 and c["c3"].macro_steps == 20
    assert c["c4"].n == (512, 512, 512) and c["c4"].macro_steps == 10
    assert c["c5"].n == (1024,) * 3 and c["c5"].steps == (2, 4, 6, 8, 10, 12, 14, 16)
    assert [w.substeps for w in c.values()] == [24, 48, 48, 48, 80]


@pytest.mark.parametrize("name,n", [("c1", (256, 1, 1)), ("c2", (96, 80, 1)),
                                    ("c3", (128, 96, 1)), ("c4", (24, 20, 16)),
                                    ("c5", (32, 24, 20))])
def test_ic_shape_and_determinism(name, n):
    w = reduced(name, n)
    a, b = make_ic(w), make_ic(w)
    assert a.shape == w.state_shape and a.dtype == np.float64 and a.flags.c_contiguous
    assert np.array_equal(a, b)
    assert np.all(np.isfinite(a))


def test_bandlimited_recipe():
    w = reduced("c3", (256, 192, 1))
    p = make_ic(w)[0]
    assert np.sqrt(np.mean(p * p)) == pytest.approx(1.0, rel=1e-12)
    P = np.fft.fft2(p)
    ky = np.fft.fftfreq(192) * 192
    kx = np.fft.fftfreq(256) * 256
    K2 = ky[:, None] ** 2 + kx[None, :] ** 2
    assert np.max(np.abs(P[K2 > 64 ** 2])) < 1e-9 * np.max(np.abs(P))
    assert abs(P[0, 0]) < 1e-9 * np.max(np.abs(P))        # no mean
    # amplitude ~ |k|^-2: |P(k)| * |k|^2 is constant over the band
    band = (K2 >= 1) & (K2 <= 64 ** 2)
    r = np.abs(P[band]) * K2[band]
    assert np.max(r) / np.min(r) < 1 + 1e-8


def test_gauss1d_recipe():
    w = get_config("c1")
    u = make_ic(w)[0]
    rng = np.random.default_rng(w.seed)
    c, s = rng.uniform(0.3, 0.7), rng.uniform(0.03, 0.08)
    i = int(np.argmax(u))
    assert abs(i / 256 - c) <= 1 / 256 and u.max() <= 1.0
    assert 0.3 <= c <= 0.7 and 0.03 <= s <= 0.08


@pytest.mark.parametrize("name,n", [("c2", (48, 40, 1)), ("c3", (96, 80, 1)), ("c4", (40, 36, 32)),
                                    ("c5", (64, 48, 40))])
def test_slab_ic_equals_planes_of_full_ic(name, n):
    """Multi-GPU ranks generate only their slab; the bytes must equal the full IC's planes."""
    w = reduced(name, n)
    full = make_ic(w)
    slow = n[2] if w.ndim == 3 else n[1]
    parts = [make_ic(w, (a, min(a + 13, slow))) for a in range(0, slow, 13)]
    assert np.array_equal(np.concatenate(parts, axis=1), full)
