"""Pins of the oracle's matrix transcription against numbers PAPER.md prints.

If any entry of a transcribed matrix were wrong, one of Table 4,
Table 5, the printed S1 or the factorization
T1 = D A4 A3 A2 A1 (a second, independent transcription of T1) would fail.
"""
import math

import numpy as np
import pytest

from oracle import matrices as M
from oracle import merit as R

NAMES = {"DCT": None, "T1": M.T1, "T2": M.T2, "LO": M.T_LO_X2, "SDCT": M.T_SDCT, "RDCT": M.T_RDCT,
         "BAS-2008b": M.T_BAS2008B, "T4": M.T4, "T6": M.T6}


def _chat(name):
    return M.C if name == "DCT" else M.c_hat(NAMES[name])


def test_exact_dct_printed_norm_and_orthonormal():
    # reading A1: printed C has rows of norm 2; C/2 is orthonormal
    assert np.allclose(np.linalg.norm(M.PRINTED_C, axis=1), 2.0, atol=1e-14)
    assert np.allclose(M.C @ M.C.T, np.eye(8), atol=1e-12)
    # equals the textbook orthonormal DCT-II alpha_k cos((2i+1) k pi / 16)
    k = np.arange(8)[:, None]
    i = np.arange(8)[None, :]
    alpha = np.where(k == 0, 1 / math.sqrt(8), 0.5)
    assert np.allclose(M.C, alpha * np.cos((2 * i + 1) * k * math.pi / 16), atol=1e-14)


def test_t1_orthogonality_and_s1(golden):
    rows = dict((r[0], r[1:]) for r in golden("t1_facts.txt"))
    n = [int(v) for v in rows["s1_squared_inverse"]]
    tt = M.T1 @ M.T1.T
    assert np.array_equal(tt, np.diag(n))  # T1 T1^T diagonal
    s_polar = M.polar_scaling(M.T1)
    assert np.allclose(s_polar, np.diag(1 / np.sqrt(n)), atol=1e-12)  # Eq. (2) = printed S1
    assert np.allclose(M.c_hat(M.T1) @ M.c_hat(M.T1).T, np.eye(8), atol=1e-12)
    assert np.array_equal(M.T1[0], [int(v) for v in rows["row0"]])
    assert np.array_equal(M.T1[4], [int(v) for v in rows["row4"]])
    assert np.array_equal(M.T2 @ M.T2.T, np.diag(n))  # S1 = S2


def test_t1_factorization_is_exact():
    # two independent transcriptions of T1 agree exactly
    assert np.array_equal(R.fast_factor_product(), M.T1.astype(float))
    assert np.array_equal(R.A1 @ R.A1, 2 * np.eye(8))


def test_arithmetic_costs(golden):
    rows = dict((r[0], r[1:]) for r in golden("t1_facts.txt"))
    assert R.t1_fast_cost() == tuple(int(v) for v in rows["fast_cost"])      # Table 6
    assert R.direct_cost(M.T1) == tuple(int(v) for v in rows["direct_cost"])


def test_fast_network_matches_matrix():
    rng = np.random.default_rng(11)
    for _ in range(2000):
        x = rng.integers(-255, 256, size=8)
        assert list(R.t1_fast_network([int(v) for v in x])) == list(M.T1 @ x)


@pytest.mark.parametrize("row", range(9))
def test_table4(golden, row):
    name, eps, mse, cg, eta = golden("table4.txt")[row]
    ch = _chat(name)
    assert abs(R.total_error_energy(ch) - float(eps)) <= 6e-5
    assert abs(R.mse_matrix(ch) - float(mse)) <= 6e-5
    assert abs(R.unified_coding_gain(ch) - float(cg)) <= 6e-5
    assert abs(R.transform_efficiency(ch) - float(eta)) <= 6e-5


@pytest.mark.parametrize("row", range(9))
def test_table5(golden, row):
    name, theta, v, dmod = golden("table5.txt")[row]
    t = M.C if name == "DCT" else NAMES[name]
    th, var, dm = R.table5_row(t)
    # printed to 2 decimals (degrees; DCT and SDCT are truncated, not rounded) and 4 decimals
    assert abs(th - float(theta)) <= 0.01
    assert abs(var - float(v)) <= 6e-5
    assert abs(dm - float(dmod)) <= 6e-5


def test_row_norm_scaling_needed_for_bas2008b():
    # reading A2: for the non-orthogonal BAS-2008b only S = diag(1/||t_k||) reproduces Table 4;
    # Eq. (2) taken literally (polar S) does not.
    t = M.T_BAS2008B
    assert not np.allclose(t @ t.T, np.diag(np.diag(t @ t.T)))
    polar = M.polar_scaling(t) @ t
    assert abs(R.total_error_energy(polar) - 4.1875) > 1e-2
    assert abs(R.total_error_energy(M.c_hat(t)) - 4.1875) <= 6e-5


def test_even_odd_symmetry_of_all_matrices():
    # T J = diag((-1)^k) T: every printed matrix (and C) is even/odd symmetric, so the
    # partial-butterfly structure of the transform applies to each of them
    J = np.eye(8)[::-1]
    sg = np.diag([(-1) ** k for k in range(8)])
    for t in list(M.INT_MATRICES.values()) + [M.C]:
        assert np.allclose(t @ J, sg @ t)
