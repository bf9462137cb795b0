"""Pins of the C oracle (oracle/adct_oracle.c) against closed forms, special cases,
invariants and brute force — none of which re-types the oracle's own formula.

  forward    unit-impulse response = outer product of T's columns (basis, exhaustive);
             constant block -> DC only; worst case |Y| = 18360 for u8 (extremal blocks);
             the §5.1 add/shift network row/column; textbook DCT-II sum
  zig-zag    SPEC S:L559-567 examples, the JPEG prefix, walk adjacency, symmetric sets
  inverse    r = 64 round trip; single-coefficient closed form; Parseval for orthogonal C_hat
  error      constant image; cross-matrix r = 1 identity; MSE monotone in r; tiling commutes
  quantiser  exhaustive over Y in [-36720, 36720] against decimal arithmetic
"""
import decimal
import fractions
import itertools
import math

import numpy as np
import pytest

import oracle
from oracle import matrices as M
from oracle import merit as R
import synth

ORTHO = {"T1": M.T1, "T2": M.T2, "LO": M.T_LO_X2, "RDCT": M.T_RDCT, "T4": M.T4, "T6": M.T6}
ALL_INT = dict(M.INT_MATRICES)


def blocks_to_image(a):
    n, bh, bw = a.shape[:3]
    return a.transpose(0, 1, 3, 2, 4).reshape(n, bh * 8, bw * 8)


# --- zig-zag ------------------------------------------------------------------------------

def test_zigzag_pins():
    o = oracle.zigzag_order()
    assert sorted(o.tolist()) == list(range(64))
    assert o[:10].tolist() == [0, 1, 8, 16, 9, 2, 3, 10, 17, 24]  # JPEG order (reading A5)
    assert set(o[:1].tolist()) == {0} and set(o[:3].tolist()) == {0, 1, 8}
    assert o[63] == 63
    for a, b in zip(o[:-1], o[1:]):  # the scan moves to a neighbouring coefficient each step
        assert max(abs(a // 8 - b // 8), abs(a % 8 - b % 8)) == 1


def test_zigzag_symmetric_prefixes():
    o = oracle.zigzag_order()
    sym = [r for r in range(1, 65) if {(z % 8) * 8 + z // 8 for z in o[:r]} == set(o[:r].tolist())]
    assert sym == [1, 3, 6, 10, 15, 21, 28, 36, 43, 49, 54, 58, 61, 63, 64]


def test_retain_counts_and_nesting():
    rng = np.random.default_rng(0)
    y = rng.integers(1, 100, size=(3, 1, 1, 8, 8)).astype(np.int64)
    prev = None
    for r in range(1, 65):
        kept = oracle.retain(y, r)
        nz = (kept != 0)
        assert nz.reshape(3, 64).sum(axis=1).tolist() == [r] * 3
        if prev is not None:
            assert np.all(nz >= prev)
        prev = nz
    with pytest.raises(ValueError):
        oracle.retain(y, 0)
    with pytest.raises(ValueError):
        oracle.retain(y, 65)


# --- forward ------------------------------------------------------------------------------

@pytest.mark.parametrize("name", list(ALL_INT))
def test_forward_impulse_basis(name):
    t = ALL_INT[name]
    imgs = np.zeros((64, 8, 8), dtype=np.int16)
    for idx in range(64):
        imgs[idx, idx // 8, idx % 8] = 1
    y = oracle.forward_int(t, imgs)[:, 0, 0]
    for idx in range(64):
        i, j = divmod(idx, 8)
        assert np.array_equal(y[idx], np.outer(t[:, i], t[:, j]))


def test_forward_constant_block_dc_only():
    for v in (0, 1, 77, 255):
        img = np.full((1, 16, 16), v, dtype=np.uint8)
        for name, t in ALL_INT.items():
            y = oracle.forward_int(t, img)
            dc = int(t[0].sum()) ** 2 * v
            assert np.all(y[..., 0, 0] == dc)
            y2 = y.copy()
            y2[..., 0, 0] = 0
            assert not y2.any(), name


def test_forward_extremal_u8_bound():
    # max |Y_kl| over u8 blocks: X_ij = 255 where T_ki T_lj > 0 (or < 0), 0 elsewhere
    t = M.T1
    best = 0
    for k, l in itertools.product(range(8), range(8)):
        w = np.outer(t[k], t[l])
        for sgn in (1, -1):
            x = np.where(sgn * w > 0, 255, 0).astype(np.uint8)[None]
            y = oracle.forward_int(t, x)[0, 0, 0, k, l]
            assert abs(y) == 255 * int(np.sum(np.abs(w[sgn * w > 0])))
            best = max(best, abs(int(y)))
    assert best == 18360  # fits int16


def test_forward_matches_fast_network():
    rng = np.random.default_rng(3)
    img = rng.integers(-255, 256, size=(1, 32, 40)).astype(np.int16)
    y = oracle.forward_int(M.T1, img)
    x = img[0]
    for by in range(4):
        for bx in range(5):
            blk = x[by * 8:by * 8 + 8, bx * 8:bx * 8 + 8].astype(int).tolist()
            cols = [R.t1_fast_network([blk[i][j] for i in range(8)]) for j in range(8)]   # T X
            p = [[cols[j][k] for j in range(8)] for k in range(8)]
            yy = [R.t1_fast_network(p[k]) for k in range(8)]                            # (T X) T^T
            assert np.array_equal(y[0, by, bx], np.array(yy))


def test_forward_real_matches_textbook_dct():
    rng = np.random.default_rng(5)
    img = rng.integers(0, 256, size=(2, 16, 24)).astype(np.uint8)
    b = oracle.forward_real(M.C, img)
    for n in range(2):
        for by in range(2):
            for bx in range(3):
                x = img[n, by * 8:by * 8 + 8, bx * 8:bx * 8 + 8].astype(float)
                for k in range(8):
                    for l in range(8):
                        ak = 1 / math.sqrt(8) if k == 0 else 0.5
                        al = 1 / math.sqrt(8) if l == 0 else 0.5
                        s = 0.0
                        for i in range(8):
                            for j in range(8):
                                s += x[i, j] * math.cos((2 * i + 1) * k * math.pi / 16) * \
                                    math.cos((2 * j + 1) * l * math.pi / 16)
                        assert abs(b[n, by, bx, k, l] - ak * al * s) < 1e-9


# --- inverse / error --------------------------------------------------------------------

@pytest.mark.parametrize("name", list(ALL_INT))
def test_roundtrip_r64(name):
    t = ALL_INT[name]
    img = synth.ar1_field(2, 32, 48, 0.95, seed=9).numpy()
    n, s = oracle.row_scaling(t)
    g, kind = oracle.synthesis_matrix(oracle.chat_from_int(t))
    assert kind == (1 if name in ORTHO else 0)
    assert np.allclose(g @ oracle.chat_from_int(t), np.eye(8), atol=1e-12)
    b = oracle.scale(oracle.forward_int(t, img), s)
    a = blocks_to_image(oracle.inverse(g, b))
    assert np.max(np.abs(a - img)) < 1e-9
    assert np.all(oracle.codec_sse(img, [64], t=t) < 1e-16 * img[0].size)


def test_single_coefficient_inverse_closed_form():
    ch = oracle.chat_from_int(M.T1)
    g, _ = oracle.synthesis_matrix(ch)
    for k, l in [(0, 0), (1, 0), (0, 1), (3, 5), (7, 7)]:
        bp = np.zeros((1, 1, 1, 8, 8))
        bp[0, 0, 0, k, l] = 2.5
        a = oracle.inverse(g, bp)[0, 0, 0]
        assert np.allclose(a, 2.5 * np.outer(ch[k], ch[l]), atol=1e-14)
    bp = np.zeros((1, 1, 1, 8, 8))
    bp[0, 0, 0, 0, 0] = 80.0
    assert np.allclose(oracle.inverse(g, bp), 10.0)  # single DC b -> constant b/8


@pytest.mark.parametrize("name", list(ORTHO))
def test_parseval_sse_equals_dropped_energy(name):
    t = ORTHO[name]
    img = synth.ar1_field(1, 64, 64, 0.95, seed=4).numpy()
    n, s = oracle.row_scaling(t)
    b = oracle.scale(oracle.forward_int(t, img), s)
    order = oracle.zigzag_order()
    rs = [1, 2, 3, 10, 17, 32, 40, 63]
    sse = oracle.codec_sse(img, rs, t=t)[0]
    bb = b.reshape(-1, 64)
    for r, e in zip(rs, sse):
        dropped = float(np.sum(bb[:, order[r:]] ** 2))
        assert abs(e - dropped) <= 1e-9 * dropped


def test_codec_is_composition_of_steps():
    img = synth.ar1_field(2, 24, 32, 0.9, seed=2).numpy()
    for t in (M.T1, M.T_SDCT):
        n, s = oracle.row_scaling(t)
        g, _ = oracle.synthesis_matrix(oracle.chat_from_int(t))
        b = oracle.scale(oracle.forward_int(t, img), s)
        for r in (1, 5, 10, 33):
            a = oracle.inverse(g, oracle.retain(b, r))
            for clip in (oracle.CLIP_NONE, oracle.CLIP, oracle.CLIP_ROUND):
                e1 = oracle.sse(img, a, clip)
                e2 = oracle.codec_sse(img, [r], t=t, clip=clip)[:, 0]
                assert np.allclose(e1, e2, rtol=1e-12)
    b = oracle.forward_real(M.C, img)
    a = oracle.inverse(M.C.T, oracle.retain(b, 7))
    assert np.allclose(oracle.sse(img, a), oracle.codec_sse(img, [7], c=M.C)[:, 0], rtol=1e-12)


def test_constant_image_zero_error():
    img = np.full((1, 16, 16), 93, dtype=np.uint8)
    for t in ALL_INT.values():
        assert np.all(oracle.codec_sse(img, [1, 2, 10, 64], t=t) < 1e-18)


def test_r1_identical_for_every_matrix():
    # every printed matrix (and C) has DC row ∝ 1 and AC rows summing to 0, so r=1
    # reconstructs block means whatever the matrix (true inverse for SDCT/BAS-2008b)
    img = synth.ar1_field(2, 64, 64, 0.95, seed=6).numpy()
    ref = oracle.codec_sse(img, [1], c=M.C)
    x = img.astype(float).reshape(2, 8, 8, 8, 8)
    means = x.mean(axis=(2, 4), keepdims=True)
    assert np.allclose(ref[:, 0], ((x - means) ** 2).sum(axis=(1, 2, 3, 4)), rtol=1e-12)
    for t in ALL_INT.values():
        assert np.allclose(oracle.codec_sse(img, [1], t=t), ref, rtol=1e-11)


def test_mse_monotone_for_orthogonal_only():
    img = synth.ar1_field(1, 64, 64, 0.95, seed=8).numpy()
    rs = list(range(1, 65))
    for t in ORTHO.values():
        e = oracle.codec_sse(img, rs, t=t)[0]
        assert np.all(np.diff(e) <= 1e-9 * e[0])


def test_tiling_commutes():
    img = synth.ar1_field(1, 32, 64, 0.95, seed=1).numpy()
    whole = oracle.codec_sse(img, [3, 10], t=M.T1)
    left = oracle.codec_sse(np.ascontiguousarray(img[:, :, :32]), [3, 10], t=M.T1)
    right = oracle.codec_sse(np.ascontiguousarray(img[:, :, 32:]), [3, 10], t=M.T1)
    assert np.allclose(whole, left + right, rtol=1e-12)


def test_clip_policies():
    # a single huge DC coefficient drives the reconstruction outside [0, 255]
    img = np.full((1, 8, 8), 250, dtype=np.uint8)
    img[0, 0, 0] = 0
    e_none = oracle.codec_sse(img, [1], t=M.T1, clip=oracle.CLIP_NONE)[0, 0]
    mean = img.mean()
    assert abs(e_none - float(((img - mean) ** 2).sum())) < 1e-9
    bp = np.zeros((1, 1, 1, 8, 8))
    bp[..., 0, 0] = 8 * 300.4  # constant block 300.4
    recon = np.full((1, 1, 1, 8, 8), 300.4)
    assert abs(oracle.sse(img, recon, oracle.CLIP)[0] - float(((img - 255.0) ** 2).sum())) < 1e-9
    recon[...] = 2.5
    assert abs(oracle.sse(img, recon, oracle.CLIP_ROUND)[0] - float(((img - 2.0) ** 2).sum())) < 1e-9


def test_psnr_closed_forms():
    npix = 512 * 512
    assert oracle.psnr(0.0, npix) == math.inf
    assert abs(oracle.psnr(255.0 ** 2 * npix, npix)) < 1e-12           # MSE = peak^2 -> 0 dB
    assert abs(oracle.psnr(npix, npix) - 20 * math.log10(255)) < 1e-12  # MSE = 1 -> 48.13 dB


# (position, n_k * n_l) for T1, n = diag(T1 T1^T) = (8, 18, 20, 18, 8, 18, 20, 18): one position per
# distinct product; 64, 144, 324, 400 have a rational sqrt (ties possible), 160 and 360 do not
QUANT_POSITIONS = [((0, 0), 64), ((0, 1), 144), ((0, 2), 160), ((1, 1), 324), ((1, 2), 360), ((2, 2), 400)]
Y_MAX = 36720  # 2 * 18360: covers the int16 sources' range of Y for T1 with margin


def _quantize_at(ys, pos):
    """Oracle quantiser on blocks that hold Y only at `pos` (T1's row norms n)."""
    n, _ = oracle.row_scaling(M.T1)
    yb = np.zeros((ys.size, 1, 1, 8, 8), dtype=np.int64)
    yb[:, 0, 0, pos[0], pos[1]] = ys
    q = oracle.quantize(yb, n, 16)
    rest = q.copy()
    rest[:, 0, 0, pos[0], pos[1]] = 0
    assert not rest.any()  # zero coefficients quantise to zero
    return q[:, 0, 0, pos[0], pos[1]].astype(np.int64)


def test_quantiser_exhaustive():
    """Reading A10: q = round half away from zero of the real Y / (16 sqrt(n_k n_l)).  For EVERY
    Y in [-36720, 36720] and each of the six products n_k n_l of T1 (S_1) the oracle
    equals exact arithmetic done another way: rational products with Fraction (exact, ties
    included), irrational ones with 50-digit decimals (no ties exist there).  The exact tie counts
    of SURVEY.md §8(c) A10 follow from the mathematics (|Y| = (2m+1) * 8 sqrt(n_k n_l)) and are
    asserted, as is the number of ties on which round-half-even (rint) would disagree."""
    ys = np.arange(-Y_MAX, Y_MAX + 1, dtype=np.int64)
    decimal.getcontext().prec = 50
    half = fractions.Fraction(1, 2)
    expect_ties = {64: (574, 288), 144: (382, 192), 324: (256, 128), 400: (230, 116)}
    for pos, prod in QUANT_POSITIONS:
        q = _quantize_at(ys, pos).tolist()
        root = math.isqrt(prod)
        ties = rint_disagree = 0
        if root * root == prod:
            step = 16 * root
            for yv, qv in zip(ys.tolist(), q):
                f = fractions.Fraction(abs(yv), step)
                fl = f.numerator // f.denominator
                frac = f - fl
                ref = fl + 1 if frac >= half else fl
                if frac == half:
                    ties += 1
                    if fl % 2 == 0:  # half-even would keep fl, half-away takes fl + 1
                        rint_disagree += 1
                assert qv == (-ref if yv < 0 else ref), (prod, yv)
            assert (ties, rint_disagree) == expect_ties[prod], prod
        else:
            step = decimal.Decimal(16) * decimal.Decimal(prod).sqrt()
            for yv, qv in zip(ys.tolist(), q):
                d = decimal.Decimal(abs(yv)) / step
                fl = int(d)
                assert abs((d - fl) - decimal.Decimal("0.5")) > decimal.Decimal("1e-30")  # never a tie
                ref = fl + 1 if d - fl > decimal.Decimal("0.5") else fl
                assert qv == (-ref if yv < 0 else ref), (prod, yv)
    # the smallest tie: Y = +-64 at (0, 0) is exactly +-0.5 and rounds away from zero
    assert _quantize_at(np.array([64, -64, 63, -63, 192, -192]), (0, 0)).tolist() == [1, -1, 0, 0, 2, -2]


def test_paper_psnr_ordering_on_ar1_image():
    # C_hat_1 outperforms C_hat_LO and C_hat_6 in PSNR; the DCT is best
    img = synth.ar1_field(1, 256, 256, 0.95, seed=1).numpy()
    rs = [3, 6, 10, 15, 21, 28]
    e1 = oracle.codec_sse(img, rs, t=M.T1)[0]
    for other in (M.T_LO_X2, M.T6):
        assert np.all(e1 <= oracle.codec_sse(img, rs, t=other)[0])
    assert np.all(oracle.codec_sse(img, rs, c=M.C)[0] <= e1)
