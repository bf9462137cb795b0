"""16- and 32-point transforms of §6.2 (JAM scaling of T1) — ORACLE SIDE (test infrastructure).

PAPER.md P:L2593-2836: the Jridi-Alfalou-Meher algorithm builds an N-point transform from two
copies of the N/2-point one (Eq. 7); the paper prints the results T(16) and
T(32) (transcribed to oracle/data/*.txt by tools/extract_jam.py), their
diagonal D(N) = T T^T and the costs of Table 8.

Reading A19: the printed block dimensions of M_per / M_add are garbled; the
printed T(16), T(32) are reproduced by the butterfly u_i = x_i + x_{N-1-i},
v_i = x_i - x_{N-1-i} (i < N/2) followed by T(N/2) on u (rows 0, 2, 4, ...) and on v (rows
1, 3, 5, ...) — the recursion below.  Reading A20: zonal retention on N x N blocks keeps the
first r coefficients of the JPEG-style zig-zag walk of the N x N grid (the 8 x 8 rule of
reading A5, one size up).

Everything here is plain numpy by definition: Y = T X T^T (int64), S = diag(1/sqrt(d_k)),
B = S Y S, x_hat = C_hat^T B' C_hat, SSE in fp64.
"""
from __future__ import annotations

import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))


def _load(name: str) -> np.ndarray:
    rows = []
    with open(os.path.join(_HERE, "data", name)) as f:
        for line in f:
            line = line.split("#", 1)[0].strip()
            if line:
                rows.append([int(v) for v in line.split()])
    return np.array(rows, dtype=np.int64)


T16 = _load("t16.txt")
T32 = _load("t32.txt")


def jam(t_half: np.ndarray) -> np.ndarray:
    """T(N) from T(N/2) (Eq. 7 under reading A19): row 2k = row k of T(N/2) on u, row 2k+1 =
    row k of T(N/2) on v, with u = x_top + reverse(x_bottom), v = x_top - reverse(x_bottom)."""
    h = t_half.shape[0]
    n = 2 * h
    t = np.zeros((n, n), dtype=np.int64)
    for k in range(h):
        for i in range(h):
            t[2 * k, i] = t_half[k, i]
            t[2 * k, n - 1 - i] = t_half[k, i]
            t[2 * k + 1, i] = t_half[k, i]
            t[2 * k + 1, n - 1 - i] = -t_half[k, i]
    return t


def jam_cost(n: int, base=(24, 6)) -> tuple[int, int]:
    """(additions, shifts) of the N-point JAM transform built from T1: twice
    the N/2 cost plus N additions for the butterfly."""
    if n == 8:
        return base
    a, s = jam_cost(n // 2, base)
    return 2 * a + n, 2 * s


def zigzag_order_n(n: int) -> np.ndarray:
    """order[z] = k*n + l of the z-th coefficient of the n x n zig-zag walk (reading A20)."""
    order = []
    for d in range(2 * n - 1):
        cells = [(k, d - k) for k in range(n) if 0 <= d - k < n]
        if d % 2 == 0:
            cells = cells[::-1]   # even anti-diagonals run bottom-left -> top-right
        order.extend(k * n + l for k, l in cells)
    return np.array(order, dtype=np.int64)


def blocks_n(img: np.ndarray, n: int) -> np.ndarray:
    """[N_img, H, W] -> [N_img, H/n, W/n, n, n] blocks (H, W multiples of n)."""
    x = np.asarray(img)
    if x.ndim == 2:
        x = x[None]
    m, h, w = x.shape
    return x.reshape(m, h // n, n, w // n, n).transpose(0, 1, 3, 2, 4)


def unblocks_n(b: np.ndarray) -> np.ndarray:
    m, bh, bw, n, _ = b.shape
    return b.transpose(0, 1, 3, 2, 4).reshape(m, bh * n, bw * n)


def forward_n(t: np.ndarray, img: np.ndarray) -> np.ndarray:
    """Y = T X T^T of every n x n block, exact int64 (two plain matrix products)."""
    n = t.shape[0]
    x = blocks_n(img, n).astype(np.int64)
    return np.einsum("ki,abcij,lj->abckl", t, x, t)


def recon_n(t: np.ndarray, img: np.ndarray, r: int) -> np.ndarray:
    """x_hat = C_hat^T B' C_hat with C_hat = S T, B = S Y S, B' = first r zig-zag coefficients."""
    n = t.shape[0]
    d = np.diag(t @ t.T).astype(np.float64)
    s = 1.0 / np.sqrt(d)
    chat = s[:, None] * t
    y = forward_n(t, img).astype(np.float64)
    b = y * s[:, None] * s[None, :]
    keep = np.zeros(n * n, dtype=bool)
    keep[zigzag_order_n(n)[:r]] = True
    b = b * keep.reshape(n, n)
    xh = np.einsum("ki,abckl,lj->abcij", chat, b, chat)
    return unblocks_n(xh)


def codec_sse_n(t: np.ndarray, img: np.ndarray, r: int) -> np.ndarray:
    """Per-image SSE of the n x n codec at r (no clip, reading A6)."""
    x = np.asarray(img, dtype=np.float64)
    if x.ndim == 2:
        x = x[None]
    return ((x - recon_n(t, x, r)) ** 2).sum(axis=(1, 2))
