"""The greedy angle search of §3 (Eq. 5-6, Fig. 2 "abmApprox") — ORACLE SIDE (test infrastructure).

For a permutation sequence p of the rows, row p(k) of the approximation is the vector d of the
search space D = P^8 with the smallest angle to row p(k) of the exact DCT C,
among the vectors orthogonal to every row already placed (Eq. 6).  §4.1
 fixes rows 1 and 5 to [1 1 1 1 1 1 1 1] and [1 -1 -1 1 1 -1 -1 1] and searches
the other six rows in all 6! = 720 orders.

Readings:
  A21  angle(c, d) = arccos(<c,d> / (|c| |d|)) is decreasing in the cosine, so the minimum
       angle is the maximum of  s(d) = <c,d> / (|d| |c|), evaluated in fp64 in this order:
       <c,d> = ((c0 d0 + c1 d1) + ...) sequentially, |d| = sqrt(sum d_i^2) (exact integer
       sum), |c| = sqrt(sequential sum c_i^2), s = <c,d> / (|d| * |c|).  The CUDA path computes
       the same sequence, so both take every argmax decision on identical fp64 values.
  A22  D is enumerated lexicographically, first coordinate most significant, digits in the
       ascending order of P (P1 = (-1, 0, 1), P2 = (-2, -1, 0, 1, 2)); the listings of
       Tables 3-4 are self-inconsistent.  Fig. 2 keeps the first strictly better candidate
       ("theta < theta_min"): ties go to the earliest vector.  The zero vector is excluded.
  A23  orthogonality is every dot product with a placed row equal to 0 (Eq. 6), not the
       "sum(aux) = 0" shortcut of Fig. 2.
  A24  an order that runs out of orthogonal candidates is reported infeasible (Fig. 2 would
       silently place D(1,:)); with rows 1 and 5 fixed, 480 of the 720 D2 orders are.
Exact ties exist (e.g. two D1 vectors at exactly cos(pi/8) to c_2), so outcomes depend on
A22; ties met during a search are reported by `greedy_solve(..., ties=list)`.
"""
from __future__ import annotations

import itertools
import math

import numpy as np

from . import matrices as M

P1 = (-1, 0, 1)
P2 = (-2, -1, 0, 1, 2)
FIXED_ROWS = {0: (1, 1, 1, 1, 1, 1, 1, 1), 4: (1, -1, -1, 1, 1, -1, -1, 1)}  # §4.1


def search_space(entries) -> np.ndarray:
    """All |P|^8 vectors in the order of reading A22 (int64 [|P|^8, 8])."""
    return np.array(list(itertools.product(sorted(entries), repeat=8)), dtype=np.int64)


def scores(D: np.ndarray, c: np.ndarray) -> np.ndarray:
    """s(d) of reading A21 for every d in D (fp64; NaN for the zero vector)."""
    dot = np.zeros(len(D))
    for j in range(8):
        dot = dot + float(c[j]) * D[:, j].astype(np.float64)
    nd = np.sqrt((D * D).sum(axis=1).astype(np.float64))
    nc = 0.0
    for j in range(8):
        nc = nc + float(c[j]) * float(c[j])
    nc = math.sqrt(nc)
    with np.errstate(invalid="ignore", divide="ignore"):
        return dot / (nd * nc)


class Search:
    """Greedy solver over one search space (masks of orthogonal vectors are memoised)."""

    def __init__(self, entries, c: np.ndarray = M.C):
        self.D = search_space(entries)
        self.c = np.asarray(c, dtype=np.float64)
        self.s = [scores(self.D, self.c[k]) for k in range(8)]
        self.nonzero = np.any(self.D != 0, axis=1)
        self._orth = {}

    def orth_mask(self, v) -> np.ndarray:
        key = tuple(int(x) for x in v)
        if key not in self._orth:
            self._orth[key] = (self.D @ np.array(key, dtype=np.int64)) == 0
        return self._orth[key]

    def solve(self, order, fixed=None, ties=None) -> np.ndarray | None:
        """Rows placed in `order` (0-based row indices) after the `fixed` rows; None when no
        orthogonal candidate remains."""
        T = np.zeros((8, 8), dtype=np.int64)
        placed = []
        for k, v in (fixed or {}).items():
            T[k] = v
            placed.append(k)
        for k in order:
            ok = self.nonzero.copy()
            for p in placed:
                ok &= self.orth_mask(T[p])
            if not ok.any():
                return None
            s = np.where(ok, self.s[k], -np.inf)
            i = int(np.argmax(s))  # first maximum: the earliest vector wins a tie
            if ties is not None and np.count_nonzero(s == s[i]) > 1:
                ties.append((tuple(order), k, np.flatnonzero(s == s[i]).tolist()))
            T[k] = self.D[i]
            placed.append(k)
        return T

    def derive_all(self, fixed=FIXED_ROWS):
        """Every order of the free rows (720 with rows 1 and 5 fixed): list of (order, T)."""
        free = [k for k in range(8) if k not in fixed]
        return [(order, self.solve(order, fixed)) for order in itertools.permutations(free)]
