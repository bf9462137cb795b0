"""Matrices of arXiv 1808.02950 as printed in PAPER.md — ORACLE SIDE (test infrastructure).

Every integer table below is typed from the LaTeX source of the paper; `P:L<n>` is a
line of /root/reference/PAPER.md.  This module is independent of the CUDA path
(paper_1808_02950_b200/catalog.py types the same matrices a second time); neither
imports the other, and tests check that the two transcriptions agree.

Readings:
  A1  the printed exact DCT C (§2) has rows of norm 2; the orthonormal DCT
      is printed C / 2.
  A11 T_LO has +-1/2 entries (Table 2); it is stored here as 2*T_LO.  The
      row-norm scaling S = diag(1/||t_k||) absorbs the factor 2.
"""
from __future__ import annotations

import math

import numpy as np

# --- exact DCT, §2:  gamma_k = cos(2*pi*(k+1)/32), k = 0..6 -------------------
_GAMMA = [math.cos(2.0 * math.pi * (k + 1) / 32.0) for k in range(7)]


def _printed_c() -> np.ndarray:
    """The matrix C exactly as printed at P:L260-271 (entries gamma_k, rows of norm 2)."""
    g = _GAMMA
    rows = [
        [g[3], g[3], g[3], g[3], g[3], g[3], g[3], g[3]],
        [g[0], g[2], g[4], g[6], -g[6], -g[4], -g[2], -g[0]],
        [g[1], g[5], -g[5], -g[1], -g[1], -g[5], g[5], g[1]],
        [g[2], -g[6], -g[0], -g[4], g[4], g[0], g[6], -g[2]],
        [g[3], -g[3], -g[3], g[3], g[3], -g[3], -g[3], g[3]],
        [g[4], -g[0], g[6], g[2], -g[2], -g[6], g[0], -g[4]],
        [g[5], -g[1], g[1], -g[5], -g[5], g[1], -g[1], g[5]],
        [g[6], -g[4], g[2], -g[0], g[0], -g[2], g[4], -g[6]],
    ]
    return np.array(rows, dtype=np.float64)


PRINTED_C = _printed_c()
#: orthonormal exact DCT (reading A1: printed C / 2)
C = PRINTED_C / 2.0

# --- T1, T2: §4.1 P:L1116-1145 --------------------------------------------------------------
T1 = np.array([
    [1, 1, 1, 1, 1, 1, 1, 1],
    [2, 2, 1, 0, 0, -1, -2, -2],
    [2, 1, -1, -2, -2, -1, 1, 2],
    [1, 0, -2, -2, 2, 2, 0, -1],
    [1, -1, -1, 1, 1, -1, -1, 1],
    [2, -2, 0, 1, -1, 0, 2, -2],
    [1, -2, 2, -1, -1, 2, -2, 1],
    [0, -1, 2, -2, 2, -2, 1, 0],
], dtype=np.int64)

T2 = np.array([
    [1, 1, 1, 1, 1, 1, 1, 1],
    [2, 1, 2, 0, 0, -2, -1, -2],
    [2, 1, -1, -2, -2, -1, 1, 2],
    [2, 0, -2, -1, 1, 2, 0, -2],
    [1, -1, -1, 1, 1, -1, -1, 1],
    [1, -2, 0, 2, -2, 0, 2, -1],
    [1, -2, 2, -1, -1, 2, -2, 1],
    [0, -2, 1, -2, 2, -1, 2, 0],
], dtype=np.int64)

# --- Table 2 -------------------------------------------------------------------
T_RDCT = np.array([
    [1, 1, 1, 1, 1, 1, 1, 1],
    [1, 1, 1, 0, 0, -1, -1, -1],
    [1, 0, 0, -1, -1, 0, 0, 1],
    [1, 0, -1, -1, 1, 1, 0, -1],
    [1, -1, -1, 1, 1, -1, -1, 1],
    [1, -1, 0, 1, -1, 0, 1, -1],
    [0, -1, 1, 0, 0, 1, -1, 0],
    [0, -1, 1, -1, 1, -1, 1, 0],
], dtype=np.int64)

T_BAS2008B = np.array([
    [1, 1, 1, 1, 1, 1, 1, 1],
    [1, 1, 1, 0, 0, -1, -1, -1],
    [1, 1, -1, -1, -1, -1, 1, 1],
    [1, 0, -1, 0, 0, 1, 0, -1],
    [1, -1, -1, 1, 1, -1, -1, 1],
    [1, -1, 1, 0, 0, -1, 1, -1],
    [1, -1, 1, -1, -1, 1, -1, 1],
    [1, -1, 1, -1, 1, -1, 1, -1],
], dtype=np.int64)

# P:L469-477, stored as 2*T_LO (reading A11)
T_LO_X2 = np.array([
    [2, 2, 2, 2, 2, 2, 2, 2],
    [2, 2, 2, 0, 0, -2, -2, -2],
    [2, 1, -1, -2, -2, -1, 1, 2],
    [2, 0, -2, -2, 2, 2, 0, -2],
    [2, -2, -2, 2, 2, -2, -2, 2],
    [2, -2, 0, 2, -2, 0, 2, -2],
    [1, -2, 2, -1, -1, 2, -2, 1],
    [0, -2, 2, -2, 2, -2, 2, 0],
], dtype=np.int64)

T6 = np.array([
    [1, 1, 1, 1, 1, 1, 1, 1],
    [2, 1, 1, 0, 0, -1, -1, -2],
    [2, 1, -1, -2, -2, -1, 1, 2],
    [1, 0, -2, -1, 1, 2, 0, -1],
    [1, -1, -1, 1, 1, -1, -1, 1],
    [1, -2, 0, 1, -1, 0, 2, -1],
    [1, -2, 2, -1, -1, 2, -2, 1],
    [0, -1, 1, -2, 2, -1, 1, 0],
], dtype=np.int64)

T4 = np.array([
    [1, 1, 1, 1, 1, 1, 1, 1],
    [1, 1, 1, 0, 0, -1, -1, -1],
    [1, 1, -1, -1, -1, -1, 1, 1],
    [1, 0, -1, -1, 1, 1, 0, -1],
    [1, -1, -1, 1, 1, -1, -1, 1],
    [1, -1, 0, 1, -1, 0, 1, -1],
    [1, -1, 1, -1, -1, 1, -1, 1],
    [0, -1, 1, -1, 1, -1, 1, 0],
], dtype=np.int64)

# SDCT: T = sgn(C), P:L387-402 (entry-wise signum of the exact DCT)
T_SDCT = np.sign(PRINTED_C).astype(np.int64)

#: the integer matrices of the paper that can be run (name -> T); LO stored x2 (A11)
INT_MATRICES = {
    "T1": T1,
    "T2": T2,
    "LO": T_LO_X2,
    "SDCT": T_SDCT,
    "RDCT": T_RDCT,
    "BAS-2008b": T_BAS2008B,
    "T4": T4,
    "T6": T6,
}


def row_norm_scaling(t: np.ndarray) -> np.ndarray:
    """S = diag(1/||t_k||) — Eq. (2) P:L363-367 for row-orthogonal T (polar decomposition
    of a matrix with orthogonal rows is diagonal); reading A2 uses the same
    row-norm S for the non-orthogonal SDCT and BAS-2008b."""
    n = (t.astype(np.int64) ** 2).sum(axis=1)
    return np.diag(1.0 / np.sqrt(n.astype(np.float64)))


def polar_scaling(t: np.ndarray) -> np.ndarray:
    """S = sqrt((T T^T)^{-1}) by symmetric eigendecomposition — Eq. (2) P:L363-367 literally."""
    m = t.astype(np.float64) @ t.astype(np.float64).T
    w, v = np.linalg.eigh(m)
    return v @ np.diag(1.0 / np.sqrt(w)) @ v.T


def c_hat(t: np.ndarray) -> np.ndarray:
    """C_hat = S T, Eq. (1), with S = diag(1/||t_k||) (reading A2)."""
    return row_norm_scaling(t) @ t.astype(np.float64)
