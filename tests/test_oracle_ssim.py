"""Pins of the SSIM oracle (oracle/ssim.py; reading A18 = SPEC S:L605 parameters) against
closed forms that do not re-type its formula.

Periodic images with period 8 in both directions put every sample of one period in every
8x8 window, so all windows share the same mean, variance and covariance; for y = a*x + b the
SSIM then has the closed form  l * s  with
   l = (2 mu (a mu + b) + C1) / (mu^2 + (a mu + b)^2 + C1),
   s = (2 a var + C2) / (var + a^2 var + C2),
where mu, var are the mean and (1/64) variance of one period, computed here by plain sums.
"""
import itertools

import numpy as np
import pytest

from oracle import ssim as S

C1, C2 = (0.01 * 255) ** 2, (0.03 * 255) ** 2


def periodic(h, w, seed):
    rng = np.random.default_rng(seed)
    period = rng.integers(0, 256, size=(8, 8)).astype(np.float64)
    return np.tile(period, (h // 8 + 1, w // 8 + 1))[:h, :w], period


def test_identical_images_score_one():
    x = np.random.default_rng(0).integers(0, 256, size=(24, 40))
    assert np.allclose(S.ssim_map(x, x), 1.0, rtol=0, atol=1e-15)
    assert S.ssim(x, x)[0] == pytest.approx(1.0, abs=1e-15)


@pytest.mark.parametrize("a,b", [(1.0, 0.0), (1.0, 17.0), (0.5, 40.0), (-1.0, 255.0), (2.0, -30.0)])
def test_affine_change_of_periodic_image_closed_form(a, b):
    x, period = periodic(27, 35, seed=3)
    y = a * x + b
    n = 64
    mu = sum(period.ravel()) / n
    var = sum((v - mu) ** 2 for v in period.ravel()) / n
    l = (2 * mu * (a * mu + b) + C1) / (mu ** 2 + (a * mu + b) ** 2 + C1)
    s = (2 * a * var + C2) / (var + a * a * var + C2)
    m = S.ssim_map(x, y)
    assert m.shape == (20, 28)
    assert np.allclose(m, l * s, rtol=1e-12, atol=0)


def test_constant_images_closed_form():
    for a, b in itertools.product([0.0, 30.0, 128.0], [0.0, 64.0, 255.0]):
        x = np.full((8, 8), a)
        y = np.full((8, 8), b)
        assert S.ssim_map(x, y)[0, 0] == pytest.approx((2 * a * b + C1) / (a * a + b * b + C1), rel=1e-14)


def test_symmetry_and_window_count():
    rng = np.random.default_rng(5)
    x = rng.integers(0, 256, size=(16, 24)).astype(float)
    y = x + rng.normal(0, 10, size=x.shape)
    assert np.allclose(S.ssim_map(x, y), S.ssim_map(y, x), rtol=1e-14)
    assert S.ssim_map(x, y).shape == (9, 17)
    assert np.all(S.ssim_map(x, y) <= 1.0)


def test_single_window_brute_force_loops():
    """One 8x8 window, statistics accumulated sample by sample in plain Python."""
    rng = np.random.default_rng(6)
    x = rng.integers(0, 256, size=(8, 8)).tolist()
    y = [[v + int(rng.integers(-20, 21)) for v in row] for row in x]
    sx = sy = sxx = syy = sxy = 0.0
    for i in range(8):
        for j in range(8):
            sx += x[i][j]
            sy += y[i][j]
    mx, my = sx / 64, sy / 64
    for i in range(8):
        for j in range(8):
            sxx += (x[i][j] - mx) ** 2
            syy += (y[i][j] - my) ** 2
            sxy += (x[i][j] - mx) * (y[i][j] - my)
    want = ((2 * mx * my + C1) * (2 * sxy / 64 + C2)) / ((mx * mx + my * my + C1) * (sxx / 64 + syy / 64 + C2))
    assert S.ssim_map(np.array(x), np.array(y))[0, 0] == pytest.approx(want, rel=1e-13)


def test_clip_policies():
    x = np.full((1, 8, 8), 250.0)
    r = np.full((1, 8, 8), 300.0)
    assert S.ssim(x, r, clip=1)[0] == pytest.approx((2 * 250 * 255 + C1) / (250 ** 2 + 255 ** 2 + C1))
    r2 = np.full((1, 8, 8), 100.4)
    assert S.ssim(x, r2, clip=2)[0] == pytest.approx((2 * 250 * 100 + C1) / (250 ** 2 + 100 ** 2 + C1))
