"""CPU checks of arithmetic claims the kernels rely on (no GPU, no library call).

The C3 quantiser (blockmajor.cu, ADCT_Q_FAST) takes |q| = floor((|Y| + c/2) / c) at the 40
positions where c = step * sqrt(n_k n_l) is an integer (T1: sqrt(n_k n_l) in {8, 12, 18, 20},
P:L1195-1203 with reading A10) from ONE fp32 FMA rounding toward -inf: A * u + 1.5 * 2^23 with
u = fp32(1/c) rounded up.  That equals floor(A / c) iff floor(A * u) = floor(A / c), u taken as the
exact binary fraction it is -- checked here for every integer A the kernel can see (|Y| <= 18360
for u8 and T1, so A < 18360 + c/2 + 1) at every step the TMA path accepts that matters for the
bound (the largest c gives the tightest margin 1/c, the largest A the largest error A 2^-23 / c).
"""
import numpy as np
import pytest

SQRT_NN = (8, 12, 18, 20)  # sqrt(n_k n_l) at the rational positions of T1 (n = 8, 18, 20)


def _round_up_recip(c: int):
    """fp32 1/c rounded up, as (mantissa, exponent) with value mant * 2^exp exactly."""
    u = np.float32(1.0 / c)
    if float(u) * c < 1.0:  # exact in fp64: 24-bit mantissa times c < 2^17
        u = np.nextafter(u, np.float32(1.0))
    m, e = np.frexp(np.float64(u))  # u = m * 2^e, m in [0.5, 1)
    mant = int(m * (1 << 24))
    assert mant * 2.0 ** (e - 24) == float(u)
    return mant, e - 24


@pytest.mark.parametrize("step", [1, 2, 3, 7, 16, 17, 100, 255, 1000, 4095, 4096])
def test_c3_directed_rounding_floor_is_exact(step):
    a_max = 18360 + (step * 20) // 2 + 1
    A = np.arange(0, a_max + 1, dtype=np.int64)
    for s in SQRT_NN:
        c = step * s
        assert c % 2 == 0  # c/2 is an integer: A is an exact fp32 integer
        mant, sh = _round_up_recip(c)
        assert sh < 0
        # floor(A * mant * 2^sh) with exact integer arithmetic (A * mant < 2^41)
        got = (A * mant) >> (-sh)
        assert np.array_equal(got, A // c), (step, c)


def test_c3_negative_two_complement():
    """3 * 2^23 - (1.5 * 2^23 + |q|) is exact and its low 16 bits are -|q| in two's complement."""
    M = np.float32(12582912.0)
    q = np.arange(0, 1 << 15, dtype=np.int64)
    up = (M + q.astype(np.float32)).astype(np.float32)
    assert np.array_equal(up.astype(np.int64), 12582912 + q)
    neg = (np.float32(25165824.0) - up).astype(np.float32)
    low = neg.view(np.uint32) & 0xFFFF
    assert np.array_equal(low.astype(np.int64), (-q) & 0xFFFF)
    pos = up.view(np.uint32) & 0xFFFF
    assert np.array_equal(pos.astype(np.int64), q)
