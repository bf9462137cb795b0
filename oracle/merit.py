"""Matrix-level figures of merit of §4.2 (Tables 4-5) — ORACLE SIDE (test infrastructure).

These are not on the GPU path.  They exist to pin the oracle's transcription of the
matrices (oracle/matrices.py) to numbers the paper prints: if an entry of T1 were
mistyped, Table 4 / Table 5 would not reproduce to the printed decimals.

All arithmetic is fp64 numpy, written as the paper states each measure.
"""
from __future__ import annotations

import math

import numpy as np

from . import matrices as M

RHO = 0.95  # interpixel correlation


def markov_covariance(rho: float = RHO) -> np.ndarray:
    """R_x with entries rho^|i-j|, i,j = 1..8 — P:L1298-1304."""
    i = np.arange(8)
    return rho ** np.abs(i[:, None] - i[None, :])


def total_error_energy(chat: np.ndarray) -> float:
    """epsilon(C_hat) = pi * ||C - C_hat||_F^2 — §4.2.1 P:L1318-1326."""
    return math.pi * float(np.sum((M.C - chat) ** 2))


def mse_matrix(chat: np.ndarray, rho: float = RHO) -> float:
    """MSE(C_hat) = 1/8 tr((C - C_hat) R_x (C - C_hat)^T) — §4.2.2 P:L1344-1356."""
    d = M.C - chat
    return float(np.trace(d @ markov_covariance(rho) @ d.T)) / 8.0


def unified_coding_gain(chat: np.ndarray, rho: float = RHO) -> float:
    """C*_g = 10 log10 prod_i 1/(A_i B_i)^(1/8), A_i = su[(c_i c_i^T) o R_x], B_i = ||g_i||^2
    with g_i^T the i-th ROW of C_hat^{-1} (reading A3) — §4.2.3 P:L1419-1468."""
    rx = markov_covariance(rho)
    g = np.linalg.inv(chat)
    prod = 1.0
    for i in range(8):
        ci = chat[i, :]
        a = float(np.sum(np.outer(ci, ci) * rx))
        b = float(np.sum(g[i, :] ** 2))
        prod *= 1.0 / (a * b) ** (1.0 / 8.0)
    return 10.0 * math.log10(prod)


def transform_efficiency(chat: np.ndarray, rho: float = RHO) -> float:
    """eta = sum_i |r_ii| / sum_ij |r_ij| * 100, R_y = C_hat R_x C_hat^T — §4.2.4 P:L1478-1494."""
    ry = chat @ markov_covariance(rho) @ chat.T
    return float(np.sum(np.abs(np.diag(ry))) / np.sum(np.abs(ry)) * 100.0)


def angle(a: np.ndarray, q: np.ndarray) -> float:
    """angle(u, v) = arccos(<u, v> / (||u|| ||v||)) — §3.3, Table 5 uses q = e_1
    and the normalised vector a' = a/||a||."""
    a = np.asarray(a, dtype=np.float64)
    q = np.asarray(q, dtype=np.float64)
    cosv = float(a @ q) / (float(np.linalg.norm(a)) * float(np.linalg.norm(q)))
    return math.acos(max(-1.0, min(1.0, cosv)))


def row_angles(m: np.ndarray) -> np.ndarray:
    q = np.zeros(8)
    q[0] = 1.0
    return np.array([angle(m[k, :], q) for k in range(8)])


def circular_mean(theta: np.ndarray) -> float:
    """Circular mean, cases as printed at P:L1526-1549 (radians)."""
    cc = float(np.sum(np.cos(theta)))
    ss = float(np.sum(np.sin(theta)))
    if cc > 0 and ss >= 0:
        return math.atan(ss / cc)
    if cc == 0 and ss > 0:
        return math.pi / 2
    if cc < 0:
        return math.atan(ss / cc) + math.pi
    if cc >= 0 and ss < 0:
        return math.atan(ss / cc) + 2 * math.pi
    raise ValueError("circular mean undefined (C = S = 0)")


def circular_variance(theta: np.ndarray) -> float:
    """V = 1 - sqrt(C^2 + S^2)/8 — P:L1563-1566."""
    cc = float(np.sum(np.cos(theta)))
    ss = float(np.sum(np.sin(theta)))
    return 1.0 - math.sqrt(cc * cc + ss * ss) / 8.0


def circular_mean_difference_mod(theta_c: np.ndarray, theta_t: np.ndarray) -> float:
    """D_mod = 1/8 sum_i (pi - |pi - |theta_ci - theta_ti||) — P:L1632-1639 (radians)."""
    return float(np.sum(math.pi - np.abs(math.pi - np.abs(theta_c - theta_t)))) / 8.0


def table5_row(t: np.ndarray) -> tuple[float, float, float]:
    """(theta_bar in degrees, V, D_mod) of the row angles of T vs the exact DCT rows."""
    th_t = row_angles(t.astype(np.float64))
    th_c = row_angles(M.C)
    return (math.degrees(circular_mean(th_t)), circular_variance(th_t),
            circular_mean_difference_mod(th_c, th_t))


# --- §5.1 fast algorithm T1 = D A4 A3 A2 A1, P:L1886-1951 ---------------------------------
A1 = np.array([
    [1, 0, 0, 0, 0, 0, 0, 1],
    [0, 1, 0, 0, 0, 0, 1, 0],
    [0, 0, 1, 0, 0, 1, 0, 0],
    [0, 0, 0, 1, 1, 0, 0, 0],
    [0, 0, 0, 1, -1, 0, 0, 0],
    [0, 0, 1, 0, 0, -1, 0, 0],
    [0, 1, 0, 0, 0, 0, -1, 0],
    [1, 0, 0, 0, 0, 0, 0, -1],
], dtype=np.float64)
A2 = np.array([
    [1, 0, 0, 1, 0, 0, 0, 0],
    [0, 1, 1, 0, 0, 0, 0, 0],
    [0, 1, -1, 0, 0, 0, 0, 0],
    [1, 0, 0, -1, 0, 0, 0, 0],
    [0, 0, 0, 0, 1, 0, 0, 0],
    [0, 0, 0, 0, 0, 1, 0, 0],
    [0, 0, 0, 0, 0, 0, 1, 0],
    [0, 0, 0, 0, 0, 0, 0, 1],
], dtype=np.float64)
A3 = np.array([
    [1, 1, 0, 0, 0, 0, 0, 0],
    [1, -1, 0, 0, 0, 0, 0, 0],
    [0, 0, 1, 0, 0, 0, 0, 0],
    [0, 0, 0, 1, 0, 0, 0, 0],
    [0, 0, 0, 0, 1, 0, 0, 0],
    [0, 0, 0, 0, 0, 1, 0, 0],
    [0, 0, 0, 0, 0, 0, 1, 0],
    [0, 0, 0, 0, 0, 0, 0, 1],
], dtype=np.float64)
A4 = np.array([
    [1, 0, 0, 0, 0, 0, 0, 0],
    [0, 0, 0, 0, 0, 0.5, 1, 1],
    [0, 0, 1, 2, 0, 0, 0, 0],
    [0, 0, 0, 0, -1, -1, 0, 0.5],
    [0, 1, 0, 0, 0, 0, 0, 0],
    [0, 0, 0, 0, 0.5, 0, -1, 1],
    [0, 0, -2, 1, 0, 0, 0, 0],
    [0, 0, 0, 0, -1, 1, -0.5, 0],
], dtype=np.float64)
D = np.diag([1.0, 2.0, 1.0, 2.0, 1.0, 2.0, 1.0, 2.0])


def fast_factor_product() -> np.ndarray:
    """D A4 A3 A2 A1 as printed — equals T1 exactly if both transcriptions hold."""
    return D @ A4 @ A3 @ A2 @ A1


class CountedInt:
    """Integer with add/shift accounting, to count the arithmetic of a network (Table 6)."""

    adds = 0
    shifts = 0

    def __init__(self, v: int):
        self.v = int(v)

    def __add__(self, o):
        CountedInt.adds += 1
        return CountedInt(self.v + o.v)

    def __sub__(self, o):
        CountedInt.adds += 1
        return CountedInt(self.v - o.v)

    def shl1(self):
        CountedInt.shifts += 1
        return CountedInt(self.v * 2)


def t1_fast_network(x):
    """T1 x through the factorization D A4 A3 A2 A1 as an add/shift network.

    A1 (8 additions), A2 (4), A3 (2), then the rows of D*A4 (the +-1/2 of A4 cancel the x2
    of D): 10 additions and 6 doublings.  Works on CountedInt or plain ints.
    """
    def add(a, b):
        return a + b

    def sub(a, b):
        return a - b

    def dbl(a):
        return a.shl1() if isinstance(a, CountedInt) else a * 2

    # A1
    a = [add(x[0], x[7]), add(x[1], x[6]), add(x[2], x[5]), add(x[3], x[4]),
         sub(x[3], x[4]), sub(x[2], x[5]), sub(x[1], x[6]), sub(x[0], x[7])]
    # A2
    b = [add(a[0], a[3]), add(a[1], a[2]), sub(a[1], a[2]), sub(a[0], a[3]), a[4], a[5], a[6], a[7]]
    # A3
    c = [add(b[0], b[1]), sub(b[0], b[1]), b[2], b[3], b[4], b[5], b[6], b[7]]
    # D * A4 (integer rows)
    y = [None] * 8
    y[0] = c[0]
    y[1] = add(c[5], dbl(add(c[6], c[7])))        # 2*(1/2 c5 + c6 + c7)
    y[2] = add(c[2], dbl(c[3]))                   # c2 + 2 c3
    y[3] = sub(c[7], dbl(add(c[4], c[5])))        # 2*(-c4 - c5 + 1/2 c7)
    y[4] = c[1]
    y[5] = add(c[4], dbl(sub(c[7], c[6])))        # 2*(1/2 c4 - c6 + c7)
    y[6] = sub(c[3], dbl(c[2]))                   # -2 c2 + c3
    y[7] = sub(dbl(sub(c[5], c[4])), c[6])        # 2*(-c4 + c5 - 1/2 c6)
    return y


def t1_fast_cost() -> tuple[int, int]:
    """(additions, shifts) of one 8-point T1 evaluation through t1_fast_network."""
    CountedInt.adds = 0
    CountedInt.shifts = 0
    t1_fast_network([CountedInt(i) for i in range(8)])
    return CountedInt.adds, CountedInt.shifts


def direct_cost(t: np.ndarray) -> tuple[int, int]:
    """(additions, shifts) of the direct product T x: (nnz_k - 1) additions per row and one
    shift per +-2 entry (P:L1868-1872 quotes 48 and 24 for T1)."""
    adds = int(sum(np.count_nonzero(t[k]) - 1 for k in range(8)))
    shifts = int(np.count_nonzero(np.abs(t) == 2))
    return adds, shifts
