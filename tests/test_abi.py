"""C-ABI checks that need no GPU: the library loads, exports every symbol include/adct.h
declares, validates arguments before any launch, and its host-side descriptors and tables
agree with the independently written oracle."""
import math
import os
import re

import numpy as np
import pytest
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

adct = pytest.importorskip("paper_1808_02950_b200.adct", reason="libadct.so not built")
from paper_1808_02950_b200 import catalog  # noqa: E402

import oracle  # noqa: E402
from oracle import matrices as M  # noqa: E402


def header_functions():
    src = open(os.path.join(ROOT, "include", "adct.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(?:adct_status|size_t|void|int64_t|const char\*)\s+(\w+)\s*\(", src)))


def test_exports_every_declared_symbol():
    names = header_functions()
    assert len(names) >= 15
    for n in names:
        assert hasattr(adct.lib, n), n
    assert set(names) == set(adct.SYMBOLS)


def test_catalog_matches_oracle_transcription():
    pairs = {"T1": M.T1, "T2": M.T2, "LO": M.T_LO_X2, "SDCT": M.T_SDCT, "RDCT": M.T_RDCT,
             "BAS-2008b": M.T_BAS2008B, "T4": M.T4, "T6": M.T6}
    for name, t in pairs.items():
        assert np.array_equal(np.array(catalog.INTEGER[name]).reshape(8, 8), t), name
    assert np.allclose(np.array(catalog.exact_dct()).reshape(8, 8), M.C, atol=1e-15)


def test_zigzag_matches_oracle():
    assert adct.zigzag_order() == oracle.zigzag_order().tolist()


@pytest.mark.parametrize("name", list(catalog.INTEGER))
def test_descriptor_integer(name):
    t = np.array(catalog.INTEGER[name]).reshape(8, 8)
    m = adct.Matrix.from_int(catalog.INTEGER[name], name)
    info = m.info()
    n, s = oracle.row_scaling(t)
    assert np.allclose(info.s, s, rtol=1e-15)
    g_ref, kind = oracle.synthesis_matrix(oracle.chat_from_int(t))
    assert info.row_orthogonal == (kind == 1)
    assert np.allclose(np.array(info.g).reshape(8, 8), g_ref, atol=1e-12)
    assert info.is_integer
    assert info.specialized == (name == "T1")
    # worst case |Y| over u8 blocks, by brute force over the sign-pattern extremal blocks
    best = 0
    for k in range(8):
        for l in range(8):
            w = np.outer(t[k], t[l])
            best = max(best, 255 * max(w[w > 0].sum(), -w[w < 0].sum()))
    assert info.max_abs_y_u8 == best
    if name == "T1":
        assert best == 18360
    m.close()


def test_descriptor_real_dct():
    m = adct.Matrix.from_real(catalog.exact_dct(), "DCT")
    info = m.info()
    assert info.row_orthogonal and not info.is_integer and not info.specialized
    assert np.allclose(np.array(info.g).reshape(8, 8), M.C.T, atol=1e-15)


def test_descriptor_errors():
    bad = list(catalog.T1)
    bad[1] = 3  # breaks the even/odd symmetry T J = diag((-1)^k) T
    with pytest.raises(adct.AdctError) as e:
        adct.Matrix.from_int(bad)
    assert e.value.status == 2
    zero_row = list(catalog.T1)
    zero_row[8:16] = [0] * 8
    with pytest.raises(adct.AdctError) as e:
        adct.Matrix.from_int(zero_row)
    assert e.value.status == 3
    big = [v * 300 for v in catalog.T1]  # |Y| for int16 input would exceed 2^24
    with pytest.raises(adct.AdctError) as e:
        adct.Matrix.from_int(big)
    assert e.value.status == 4
    with pytest.raises(adct.AdctError):
        adct.Matrix.from_real([float("nan")] * 64)


def _fake(n=1, h=16, w=16):
    return adct.Geom(n, h, w, h * w, w)


def test_argument_validation_before_launch():
    """Shape/argument errors are returned synchronously, without touching a device."""
    m = adct.Matrix.from_int(catalog.T1)
    L = adct.lib
    fake = 1 << 20  # aligned non-null pointer, never dereferenced
    assert L.zonal_retain(fake, adct.I32, 4, 0, None) == 1
    assert L.zonal_retain(fake, adct.I32, 4, 65, None) == 1
    assert L.zonal_retain(fake + 4, adct.I32, 4, 3, None) == 5
    assert L.approx_dct8x8_fwd(m.handle, fake, adct.U8, adct.Geom(1, 12, 16, 192, 16), fake, adct.I32, None) == 1
    assert L.approx_dct8x8_fwd(m.handle, fake, adct.U8, adct.Geom(1, 16, 16, 256, 12), fake, adct.I32, None) == 5
    assert L.approx_dct8x8_fwd(m.handle, None, adct.U8, _fake(), fake, adct.I32, None) == 1
    assert L.approx_dct8x8_fwd(m.handle, fake, adct.F32, _fake(), fake, adct.I32, None) == 1
    # int16 coefficients cannot hold |Y| for int16 samples (bound 4.7e6)
    assert L.approx_dct8x8_fwd(m.handle, fake, adct.I16, _fake(), fake, adct.I16, None) == 4
    dct = adct.Matrix.from_real(catalog.exact_dct())
    assert L.approx_dct8x8_fwd(dct.handle, fake, adct.U8, _fake(), fake, adct.I32, None) == 4
    assert L.approx_dct8x8_inv(m.handle, fake, adct.I32, _fake(), fake, adct.U8, adct.CLIP_NONE, None) == 1
    rl = (adct.ctypes.c_int32 * 2)(10, 0)
    assert L.approx_dct8x8_fused_sse(m.handle, fake, adct.U8, _fake(), adct.ctypes.cast(rl, adct.ctypes.c_void_p),
                                     2, 0, fake, None, fake, 1 << 30, None) == 1
    rl = (adct.ctypes.c_int32 * 1)(10)
    assert L.approx_dct8x8_fused_sse(m.handle, fake, adct.U8, _fake(), adct.ctypes.cast(rl, adct.ctypes.c_void_p),
                                     1, 0, fake, fake, fake, 8, None) == 7
    assert L.psnr_reduce(fake, adct.U8, fake, adct.F32, _fake(), 0.0, 0, fake, fake, fake, 1 << 30, None) == 1


def test_host_workspace_lone_image_stride():
    """A lone image's image_stride is ignored by the host path: its workspace is sized
    from H * row_stride, so image_stride = 0 and = H * row_stride give the same size."""
    g0 = adct.Geom(1, 2160, 3840, 0, 3840)
    g1 = adct.Geom(1, 2160, 3840, 2160 * 3840, 3840)
    assert adct.host_workspace_bytes(g0, 1, 16) == adct.host_workspace_bytes(g1, 1, 16)
    assert adct.host_workspace_bytes(g0, 1, 1) >= 2 * 2160 * 3840


def test_workspace_sizes_monotone():
    g1 = adct.Geom(1, 512, 512, 512 * 512, 512)
    g2 = adct.Geom(45, 512, 512, 512 * 512, 512)
    assert adct.workspace_bytes(g2, 64) >= 45 * adct.workspace_bytes(g1, 64) - 45 * 256
    assert adct.host_workspace_bytes(g2, 1, 8) > 2 * 8 * 512 * 512


def test_status_strings():
    for s in range(8):
        assert adct.lib.adct_status_str(s)
    assert math.isfinite(adct.launch_count())


def test_catalog_greedy_constants_match_oracle():
    from oracle import greedy as OG
    from paper_1808_02950_b200 import catalog
    assert tuple(catalog.P1) == OG.P1 and tuple(catalog.P2) == OG.P2
    assert catalog.GREEDY_FIXED_ROWS == OG.FIXED_ROWS


def test_argument_validation_next_rows():
    """The next-row entry points reject bad arguments before any launch."""
    L = adct.lib
    fake = 1 << 20
    c = (adct.ctypes.c_double * 64)(*catalog.exact_dct())
    cp = adct.ctypes.cast(c, adct.ctypes.c_void_p)
    ent = (adct.ctypes.c_int32 * 3)(-1, 0, 1)
    ep = adct.ctypes.cast(ent, adct.ctypes.c_void_p)
    dup = (adct.ctypes.c_int32 * 3)(-1, 0, 0)
    # greedy: no entries, duplicate entries, workspace too small
    assert L.adct_greedy_search(cp, ep, 0, None, 0, fake, 1, fake, fake, None, fake, 1 << 30, None) == 1
    assert L.adct_greedy_search(cp, adct.ctypes.cast(dup, adct.ctypes.c_void_p), 3, None, 0, fake, 1, fake, fake,
                                None, fake, 1 << 30, None) == 1
    assert L.adct_greedy_search(cp, ep, 3, None, 0, fake, 1, fake, fake, fake, fake, 16, None) == 7
    assert L.adct_greedy_workspace_bytes(3) >= 9 * 8 * 6561
    # JAM: block size, r range, geometry, alignment
    g16 = adct.Geom(1, 32, 32, 1024, 32)
    assert L.approx_dct_jam_roundtrip(8, fake, adct.U8, g16, 1, fake, adct.F32, 0, None) == 1
    assert L.approx_dct_jam_roundtrip(16, fake, adct.U8, g16, 257, fake, adct.F32, 0, None) == 1
    assert L.approx_dct_jam_roundtrip(32, fake, adct.U8, adct.Geom(1, 16, 32, 512, 32), 1, fake, adct.F32, 0,
                                      None) == 1
    assert L.approx_dct_jam_roundtrip(16, fake + 8, adct.U8, g16, 1, fake, adct.F32, 0, None) == 5
    assert L.approx_dct_jam_roundtrip(16, fake, adct.U8, g16, 10, fake, adct.I16, 0, None) == 1  # needs ROUND
    # round trip and SSIM
    assert L.approx_dct8x8_roundtrip(adct.Matrix.from_int(catalog.T1).handle, fake, adct.I16, _fake(), 0, fake,
                                     adct.I16, 2, None) == 1
    assert L.ssim_reduce(fake, adct.U8, fake, adct.F32, _fake(), -1.0, 0, fake, fake, 1 << 30, None) == 1
    assert L.ssim_reduce(fake, adct.U8, fake, adct.F32, _fake(), 255.0, 0, fake, fake, 8, None) == 7
    # merit: negative counts
    assert L.adct_merit_batch(cp, fake, fake, -1, fake, 4, fake, None) == 1


def test_binding_validates_caller_outputs():
    """Output tensors a caller passes are written through their data pointer, so the binding
    checks dtype, contiguity, size and shape before any call reaches the library (CPU tensors:
    the checks run before any launch)."""
    m = adct.Matrix.from_int(catalog.T1)
    src = torch.zeros((2, 16, 16), dtype=torch.uint8)
    with pytest.raises(ValueError):
        adct.approx_dct8x8_fused_sse(m, src, [10], sse=torch.empty((2, 1), dtype=torch.float32))
    with pytest.raises(ValueError):
        adct.approx_dct8x8_fused_sse(m, src, [3, 10], sse=torch.empty((2, 1), dtype=torch.float64))
    with pytest.raises(ValueError):
        adct.approx_dct8x8_fused_sse(m, src, [10], sse=torch.empty((2, 2), dtype=torch.float64)[:, :1])
    with pytest.raises(ValueError):
        adct.approx_dct8x8_fwd_quant(m, src, q=torch.empty((2, 2, 2, 8, 8), dtype=torch.int32))
    with pytest.raises(ValueError):
        adct.approx_dct8x8_fwd(m, src, coef=torch.empty((1, 2, 2, 8, 8), dtype=torch.int32))
    with pytest.raises(ValueError):
        adct.approx_dct8x8_roundtrip(m, src, 10, recon=torch.empty((1, 16, 16), dtype=torch.int16))
    with pytest.raises(ValueError):
        adct.approx_dct_jam_roundtrip(16, src, 10, recon=torch.empty((2, 16, 8), dtype=torch.float32))
