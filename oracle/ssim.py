"""Structural similarity (SSIM) of a reconstruction — ORACLE SIDE (test infrastructure).

PAPER.md §6.1 scores reconstructions by MSE, PSNR and SSIM (citing Wang et
al. 2004); the paper does not print the SSIM parameters.  Reading A18, after
SPEC.md S:L605: an 8x8 moving window (every position fully inside the image, stride 1) with
uniform weights, K1 = 0.01, K2 = 0.03, dynamic range L = peak = 255, local statistics with
the 1/N normalisation of uniform weights summing to one:

    mu_x = E[x], sigma_x^2 = E[(x - mu_x)^2], sigma_xy = E[(x - mu_x)(y - mu_y)]
    SSIM_w = (2 mu_x mu_y + C1)(2 sigma_xy + C2) / ((mu_x^2 + mu_y^2 + C1)(sigma_x^2 + sigma_y^2 + C2))
    C1 = (K1 L)^2, C2 = (K2 L)^2,  SSIM(image) = mean over windows.

Plain fp64 numpy, window by window as written (numpy's sliding-window view gathers the 64
samples of every window; no running sums, no separable filtering).  Only tests/, smoke() and
bench.py's CPU legs may use it.  Pins: tests/test_oracle_ssim.py.
"""
from __future__ import annotations

import numpy as np

K1, K2, WIN = 0.01, 0.03, 8


def ssim_map(x: np.ndarray, y: np.ndarray, peak: float = 255.0) -> np.ndarray:
    """SSIM of every 8x8 window of two [H, W] images: array [H-7, W-7] (fp64)."""
    x = np.asarray(x, dtype=np.float64)
    y = np.asarray(y, dtype=np.float64)
    if x.shape != y.shape or x.ndim != 2 or min(x.shape) < WIN:
        raise ValueError("two [H, W] images with H, W >= 8")
    c1, c2 = (K1 * peak) ** 2, (K2 * peak) ** 2
    wx = np.lib.stride_tricks.sliding_window_view(x, (WIN, WIN))   # [H-7, W-7, 8, 8]
    wy = np.lib.stride_tricks.sliding_window_view(y, (WIN, WIN))
    mx = wx.mean(axis=(2, 3))
    my = wy.mean(axis=(2, 3))
    dx = wx - mx[:, :, None, None]
    dy = wy - my[:, :, None, None]
    vx = (dx * dx).mean(axis=(2, 3))
    vy = (dy * dy).mean(axis=(2, 3))
    cxy = (dx * dy).mean(axis=(2, 3))
    return ((2 * mx * my + c1) * (2 * cxy + c2)) / ((mx * mx + my * my + c1) * (vx + vy + c2))


def ssim(orig: np.ndarray, recon: np.ndarray, peak: float = 255.0, clip: int = 0) -> np.ndarray:
    """Mean SSIM per image of stacks [n, H, W] (or one [H, W] image).  clip: the policy of
    reading A6 applied to the reconstruction first (0 none, 1 clip to [0, peak], 2 clip and
    round half to even)."""
    o = np.asarray(orig, dtype=np.float64)
    r = np.asarray(recon, dtype=np.float64)
    if o.ndim == 2:
        o, r = o[None], r[None]
    if clip:
        r = np.clip(r, 0.0, peak)
        if clip == 2:
            r = np.rint(r)
    return np.array([ssim_map(o[i], r[i], peak).mean() for i in range(o.shape[0])])
