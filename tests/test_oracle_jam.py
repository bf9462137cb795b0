"""Pins of the 16/32-point oracle (oracle/jam.py) to what §6.2 prints.

  transcription  the JAM recursion (reading A19) applied to T1 reproduces the printed T(16),
                 and applied to T(16) the printed T(32), entry for entry;
  scaling        T T^T is diagonal and equals D(16) = 4 (I2 x diag(4,9,10,9) x I2),
                 D(32) = 2 D(16) x I2, built here with np.kron;
  costs          Table 8: 24/6, 64/12, 160/24 additions/shifts;
  zig-zag        the n x n walk at n = 8 equals the C oracle's 8 x 8 order; prefixes nest;
  codec          the n = 8 forward equals the C oracle's forward for T1; unit impulses give
                 outer products; r = n^2 reconstructs exactly; constant image -> DC only.
"""
import numpy as np
import pytest

import oracle
from oracle import jam as J
from oracle import matrices as M


def test_jam_recursion_reproduces_printed_matrices():
    assert np.array_equal(J.jam(np.array(M.T1)), J.T16)
    assert np.array_equal(J.jam(J.T16), J.T32)


def test_printed_diagonals():
    d16 = 4 * np.kron(np.kron(np.eye(2), np.diag([4, 9, 10, 9])), np.eye(2))
    d32 = 2 * np.kron(d16, np.eye(2))
    assert np.array_equal(J.T16 @ J.T16.T, d16.astype(np.int64))
    assert np.array_equal(J.T32 @ J.T32.T, d32.astype(np.int64))


def test_table8_costs():
    assert [J.jam_cost(n) for n in (8, 16, 32)] == [(24, 6), (64, 12), (160, 24)]


@pytest.mark.parametrize("n", [8, 16, 32])
def test_zigzag_walk(n):
    o = J.zigzag_order_n(n)
    assert sorted(o.tolist()) == list(range(n * n))
    if n == 8:
        assert np.array_equal(o, oracle.zigzag_order())
    assert o[:3].tolist() == [0, 1, n]
    k, l = o // n, o % n
    assert np.all(np.abs(np.diff(k)) + np.abs(np.diff(l)) <= 2)  # each step moves to a neighbour
    assert np.all(np.diff(k + l) >= 0)                            # anti-diagonals in order


def test_forward_n8_equals_c_oracle():
    img = np.random.default_rng(1).integers(0, 256, size=(2, 16, 24)).astype(np.uint8)
    assert np.array_equal(J.forward_n(np.array(M.T1), img), oracle.forward_int(M.T1, img))


@pytest.mark.parametrize("t", [J.T16, J.T32], ids=["T16", "T32"])
def test_forward_impulses_and_constant(t):
    n = t.shape[0]
    for i, j in [(0, 0), (1, n - 1), (n // 2, 3), (n - 1, n - 1)]:
        x = np.zeros((1, n, n), dtype=np.int64)
        x[0, i, j] = 1
        assert np.array_equal(J.forward_n(t, x)[0, 0, 0], np.outer(t[:, i], t[:, j]))
    c = np.full((1, n, n), 77, dtype=np.int64)
    y = J.forward_n(t, c)[0, 0, 0]
    assert y[0, 0] == 77 * n * n and np.count_nonzero(y) == 1


@pytest.mark.parametrize("t", [J.T16, J.T32], ids=["T16", "T32"])
def test_roundtrip_and_monotone_error(t):
    n = t.shape[0]
    img = np.random.default_rng(2).integers(0, 256, size=(1, 2 * n, 2 * n))
    assert np.allclose(J.recon_n(t, img, n * n), img, atol=1e-9)
    sse = [J.codec_sse_n(t, img, r)[0] for r in (1, 3, 10, n * n // 2, n * n - 1)]
    assert all(a >= b - 1e-6 for a, b in zip(sse, sse[1:]))  # nested retention, orthogonal C_hat
    # r = 1 keeps the block means: SSE = sum of squared deviations from each block mean
    b = J.blocks_n(img, n).astype(float)
    dev = ((b - b.mean(axis=(3, 4), keepdims=True)) ** 2).sum()
    assert J.codec_sse_n(t, img, 1)[0] == pytest.approx(dev, rel=1e-12)
