"""GPU parity of the streaming hot kernel (fused_u8_wtile_kernel, per-warp TMA tile ring)
against the CPU oracle, on the geometries that stress its tiling: 256-byte row slices that
are exact / ragged / narrower than one slice, 16-row tiles cut by the image bottom, padded
row and image strides (tensor-map strides), stacks with more chunks than CTAs, chunks in
which some warps have no tile, every compiled r and both compile-time (T1) and runtime
matrices.  Tolerance: BASELINE.json north_star (1e-5 relative on SSE, 0 where the oracle's
SSE is 0).  The streaming kernel and the generic fused kernels (ADCT_DISABLE_STREAM=1) are run
in subprocesses and must both match the oracle.
"""
import os
import subprocess
import sys
import textwrap

import numpy as np
import pytest
import torch

import oracle
from oracle import matrices as M
import synth

pytestmark = pytest.mark.gpu

adct = pytest.importorskip("paper_1808_02950_b200.adct")
from paper_1808_02950_b200 import catalog  # noqa: E402

DEV = torch.device("cuda:0") if torch.cuda.is_available() else None
RTOL = 1e-5
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
STREAM_R = [1, 3, 6, 10, 14, 15, 21, 28, 36]


def _check(got, ref):
    """1e-5 relative; where the oracle's fp64 SSE is at rounding level (r = 64: the exact
    value is 0, reading A17) the GPU's must be exactly 0."""
    got = np.asarray(got, dtype=np.float64)
    zero = ref <= 1e-16 * 64 * 1e6
    assert np.all(got[zero] == 0.0)
    rel = np.abs(got[~zero] - ref[~zero]) / ref[~zero]
    assert rel.size == 0 or rel.max() <= RTOL, rel.max()


@pytest.fixture(scope="module")
def mats():
    return {n: adct.Matrix.from_int(catalog.INTEGER[n], n) for n in catalog.INTEGER}


# (n_images, H, W): exact slices, ragged slice, sub-slice width, bottom-cut tiles, tall/narrow
GEOMS = [(2, 16, 256), (3, 24, 272), (2, 8, 16), (1, 136, 1040), (4, 40, 512), (1, 2160, 3840), (2, 1080, 1920)]


@pytest.mark.parametrize("geom", GEOMS)
def test_stream_geometries_t1_r10(mats, geom):
    n, h, w = geom
    img = synth.ar1_field(n, h, w, 0.95, seed=h * 7 + w)
    sse = adct.approx_dct8x8_fused_sse(mats["T1"], img.to(DEV), [10]).cpu().numpy()
    _check(sse, oracle.codec_sse(img.numpy(), [10], t=M.T1))


@pytest.mark.parametrize("r", STREAM_R + [64])
@pytest.mark.parametrize("name", ["T1", "T2", "LO", "T6", "SDCT", "BAS-2008b"])
def test_stream_every_r_and_matrix(mats, name, r):
    img = synth.ar1_field(3, 48, 272, 0.9, seed=r)
    sse = adct.approx_dct8x8_fused_sse(mats[name], img.to(DEV), [r]).cpu().numpy()
    _check(sse, oracle.codec_sse(img.numpy(), [r], t=np.array(catalog.INTEGER[name]).reshape(8, 8)))


@pytest.mark.parametrize("r", [1, 3, 6, 14, 15, 36])
@pytest.mark.parametrize("geom", [(3, 72, 384), (2, 136, 1920), (2, 40, 2048)])
def test_tensor_core_kernel_other_r(mats, geom, r):
    """Whole 128-byte chunks: the tensor-core kernel's other compiled retentions for T1 (kept form
    r <= 15, dropped-coefficient form r = 36) on its three tile shapes (2-chunk, donor, 16-chunk)."""
    n, h, w = geom
    img = synth.ar1_field(n, h, w, 0.93, seed=31 * r + w)
    sse = adct.approx_dct8x8_fused_sse(mats["T1"], img.to(DEV), [r]).cpu().numpy()
    _check(sse, oracle.codec_sse(img.numpy(), [r], t=M.T1))


@pytest.mark.parametrize("kind", ["ar1", "uniform", "extreme"])
@pytest.mark.parametrize("geom", [(3, 72, 384), (2, 136, 1920), (2, 40, 2048), (1, 2160, 3840)])
def test_tensor_core_kernel_clip_policy(mats, geom, kind):
    """ADCT_CLIP (reconstruction clipped to [0, 255], no rounding, before the error;
    reading A6) on the tensor-core kernel, T1 at r = 10: AR(1) frames, uniform noise, and extremal
    0 / 255 images whose reconstructions overshoot in most blocks."""
    n, h, w = geom
    if kind == "ar1":
        img = synth.ar1_field(n, h, w, 0.95, seed=h + w)
    elif kind == "uniform":
        img = synth.uniform_blocks_u8(n, h, w, seed=h + w)
    else:
        img = (torch.randint(0, 2, (n, h, w), generator=torch.Generator().manual_seed(h + w)) * 255).to(torch.uint8)
    sse = adct.approx_dct8x8_fused_sse(mats["T1"], img.to(DEV), [10], clip=adct.CLIP).cpu().numpy()
    ref = oracle.codec_sse(img.numpy(), [10], t=M.T1, clip=adct.CLIP)
    _check(sse, ref)
    if kind == "extreme":  # the case really exercises the clip: the policies differ by > 10x the 1e-5 tolerance
        plain = oracle.codec_sse(img.numpy(), [10], t=M.T1)
        assert np.all(np.abs(plain - ref) > 1e-4 * ref)


def test_stream_padded_strides(mats):
    """row_stride > W and image_stride > H*row_stride (16-byte multiples): tensor-map strides."""
    img = synth.uniform_blocks_u8(3, 40, 272, seed=5)
    big = torch.zeros((3, 48, 304), dtype=torch.uint8)
    big[:, 4:44, 16:288] = img
    view = big.to(DEV)[:, 4:44, 16:288]  # row stride 304, image stride 48*304
    assert view.stride() == (48 * 304, 304, 1)
    sse = adct.approx_dct8x8_fused_sse(mats["T1"], view, [10]).cpu().numpy()
    _check(sse, oracle.codec_sse(img.numpy(), [10], t=M.T1))


def test_stream_many_chunks_and_idle_warps(mats):
    """300 one-tile images: more chunks than CTAs, and 15 of 16 warps idle in every chunk."""
    img = synth.uniform_blocks_u8(300, 16, 256, seed=6)
    sse = adct.approx_dct8x8_fused_sse(mats["T1"], img.to(DEV), [10]).cpu().numpy()
    _check(sse, oracle.codec_sse(img.numpy(), [10], t=M.T1))


def test_stream_extreme_and_constant_blocks(mats):
    ext = (torch.randint(0, 2, (2, 32, 256), generator=torch.Generator().manual_seed(3)) * 255).to(torch.uint8)
    const = torch.full((1, 32, 256), 77, dtype=torch.uint8)
    for img in (ext, const):
        for r in (1, 10, 36):
            sse = adct.approx_dct8x8_fused_sse(mats["T1"], img.to(DEV), [r]).cpu().numpy()
            _check(sse, oracle.codec_sse(img.numpy(), [r], t=M.T1))
    sse = adct.approx_dct8x8_fused_sse(mats["T1"], const.to(DEV), [1]).cpu().numpy()
    assert np.all(sse == 0.0)  # a constant image is reconstructed exactly at every r


def test_stream_config4_full_size_sampled(mats):
    """BASELINE config 4 at full size in the bench's launch configuration: the 512-frame
    3840x2160 luma stack and both 1920x1080 chroma stacks of bench.py (same generator and
    seed), one call per plane; the oracle on frames 0, 255 and 511 of every plane."""
    planes = synth.yuv420_stack(512, 2160, 3840, seed=4, device=DEV, batch=8)
    for plane in planes:
        sse = adct.approx_dct8x8_fused_sse(mats["T1"], plane, [10]).cpu().numpy()
        for f in (0, 255, 511):
            _check(sse[f:f + 1], oracle.codec_sse(plane[f:f + 1].cpu().numpy(), [10], t=M.T1))
        # shard invariance: the same frames in a different stack give identical sums
        part = adct.approx_dct8x8_fused_sse(mats["T1"], plane[250:260], [10]).cpu().numpy()
        assert np.array_equal(part, sse[250:260])
    del planes
    torch.cuda.empty_cache()


_VARIANT_SCRIPT = textwrap.dedent("""
    import sys, numpy as np, torch
    sys.path.insert(0, {root!r})
    import synth
    from paper_1808_02950_b200 import adct, catalog
    m = adct.Matrix.from_int(catalog.T1, "T1")
    out = []
    for (n, h, w) in [(2, 24, 272), (1, 2160, 3840), (3, 1080, 1920), (2, 40, 1280), (1, 136, 384)]:
        img = synth.ar1_field(n, h, w, 0.95, seed=h + w)
        out.append(adct.approx_dct8x8_fused_sse(m, img.cuda(), [10]).cpu().numpy().ravel())
    np.save(sys.argv[1], np.concatenate(out))
""")


@pytest.mark.parametrize("env", [{}, {"ADCT_DISABLE_STREAM": "1"}, {"ADCT_HOT": "simt"}, {"ADCT_TC_CW": "1"},
                                 {"ADCT_TC_CW": "16"}, {"ADCT_TC_CW": "15"}])
def test_kernel_variants_agree_with_oracle(tmp_path, env):
    """Every kernel variant on the same geometries: the tensor-core kernel with its automatic tile
    shape and with forced 1- and 16-chunk-wide tiles; the SIMT streaming kernel; the generic fused
    kernels."""
    script = tmp_path / "v.py"
    script.write_text(_VARIANT_SCRIPT.format(root=ROOT))
    out = tmp_path / "o.npy"
    e = dict(os.environ)
    e.update(env)
    subprocess.run([sys.executable, str(script), str(out)], check=True, env=e, timeout=600)
    got = np.load(out)
    ref = []
    for (n, h, w) in [(2, 24, 272), (1, 2160, 3840), (3, 1080, 1920), (2, 40, 1280), (1, 136, 384)]:
        img = synth.ar1_field(n, h, w, 0.95, seed=h + w)
        ref.append(oracle.codec_sse(img.numpy(), [10], t=M.T1).ravel())
    _check(got, np.concatenate(ref))


# --- donor tiling of 15-chunk rows (1920-byte planes: config 4's chroma, tc.cu CW = 15) ----------
# bands = H / 8 across the cases the plan distinguishes: fewer than 16 (no main tile, only the
# leftover), exactly 16 (no leftover), 17 / 31 / 33 (a leftover of 15 / 1 / 15 chunk-bands), 135
DONOR_GEOMS = [(3, 8, 1920), (2, 120, 1920), (2, 128, 1920), (2, 136, 1920), (2, 248, 1920), (1, 264, 1920),
               (3, 1080, 1920)]


@pytest.mark.parametrize("geom", DONOR_GEOMS)
def test_donor_tiles(mats, geom):
    """Main tiles (one band + one donor chunk-band), the leftover tile (the last band's tail, its
    16th KB a fully out-of-bounds box) and the per-image sums over them equal the oracle for T1
    at r = 3, 10, 14 and a runtime matrix at r = 10."""
    n, h, w = geom
    img = synth.ar1_field(n, h, w, 0.95, seed=h + 3 * n)
    for name, r in (("T1", 3), ("T1", 10), ("T1", 14), ("T2", 10)):
        sse = adct.approx_dct8x8_fused_sse(mats[name], img.to(DEV), [r]).cpu().numpy()
        _check(sse, oracle.codec_sse(img.numpy(), [r], t=np.array(catalog.INTEGER[name]).reshape(8, 8)))


def test_donor_tiles_padded_strides(mats):
    """Donor boxes through padded row / image strides: the 15-chunk map's out-of-bounds chunk is
    the 16th 128-byte chunk of the WIDTH, never the row padding."""
    img = synth.ar1_field(2, 136, 1920, 0.9, seed=9)
    big = torch.full((2, 144, 2048), 255, dtype=torch.uint8)
    big[:, :136, :1920] = img
    view = big.to(DEV)[:, :136, :1920]
    assert view.stride() == (144 * 2048, 2048, 1)
    sse = adct.approx_dct8x8_fused_sse(mats["T1"], view, [10]).cpu().numpy()
    _check(sse, oracle.codec_sse(img.numpy(), [10], t=M.T1))


# --- several planes in one launch (approx_dct8x8_fused_sse_planes; the Y, U, V planes of C4) ------

@pytest.mark.parametrize("shapes", [
    [(3, 2160, 3840), (3, 1080, 1920), (3, 1080, 1920)],   # C4 frames: Y + U + V, one launch
    [(2, 136, 384), (5, 72, 256)],                          # planes with different image counts
    [(1, 64, 128), (0, 64, 128), (2, 40, 1280)],            # an empty plane, ragged bands
    [(2, 64, 200), (2, 64, 256)],                           # width % 128 != 0: per-plane fallback
])
def test_planes_equal_per_plane_calls(mats, shapes):
    """The planes call equals the per-plane approx_dct8x8_fused_sse bit for bit (SSE and PSNR) and
    the oracle; per-image sums do not depend on which planes share the launch."""
    planes = [synth.ar1_field(n, h, w, 0.95, seed=100 + i) if n else torch.empty((0, h, w), dtype=torch.uint8)
              for i, (n, h, w) in enumerate(shapes)]
    dp = [p.to(DEV) for p in planes]
    sse, psnr = adct.approx_dct8x8_fused_sse_planes(mats["T1"], dp, 10)
    for p, d, s, q in zip(planes, dp, sse, psnr):
        if p.shape[0] == 0:
            assert s.numel() == 0
            continue
        s1, q1 = adct.approx_dct8x8_fused_sse(mats["T1"], d, [10], return_psnr=True)
        assert torch.equal(s, s1[:, 0]) and torch.equal(q, q1[:, 0])
        if p.shape[1] * p.shape[2] <= 1080 * 1920:
            ref = oracle.codec_sse(p.numpy(), [10], t=M.T1)[:, 0]
            assert np.all(np.abs(s.cpu().numpy() - ref) <= 1e-5 * ref)


@pytest.mark.parametrize("counts,h,w", [((3, 3), 1080, 1920), ((2, 5), 136, 384), ((1, 1), 64, 1920),
                                        ((4, 2), 40, 1280)])
def test_planes_back_to_back_one_launch(mats, counts, h, w):
    """Two planes of one geometry stored back to back (plane 2 starts where plane 1's last image
    ends: bench.py's U and V) run as ONE launch over both image ranges; SSE and PSNR equal the
    per-plane calls bit for bit (chunks follow the geometry), and one launch fewer is counted."""
    na, nb = counts
    both = synth.ar1_field(na + nb, h, w, 0.9, seed=na * 10 + nb).to(DEV)
    a, b = both[:na], both[na:]
    y = synth.ar1_field(2, 2 * h, 2 * w, 0.95, seed=1).to(DEV)
    for planes in ([a, b], [y, a, b]):
        n0 = adct.launch_count()
        sse, psnr = adct.approx_dct8x8_fused_sse_planes(mats["T1"], planes, 10)
        torch.cuda.synchronize()
        merged = adct.launch_count() - n0
        n0 = adct.launch_count()
        for p, s, q in zip(planes, sse, psnr):
            s1, q1 = adct.approx_dct8x8_fused_sse(mats["T1"], p, [10], return_psnr=True)
            assert torch.equal(s, s1[:, 0]) and torch.equal(q, q1[:, 0])
        torch.cuda.synchronize()
        assert merged == adct.launch_count() - n0 - 1  # one hot-kernel launch fewer (the finalizes stay per plane)
    ref = oracle.codec_sse(both.cpu().numpy(), [10], t=M.T1)[:, 0]
    sse, _ = adct.approx_dct8x8_fused_sse_planes(mats["T1"], [a, b], 10)
    _check(torch.cat(sse).cpu().numpy(), ref)


def test_planes_not_back_to_back(mats):
    """Same geometry with a gap between the planes, or a different row stride: separate launches,
    same results as the per-plane calls."""
    buf = synth.ar1_field(5, 136, 384, 0.9, seed=3).to(DEV)
    a, b = buf[:2], buf[3:]  # one image gap
    sse, psnr = adct.approx_dct8x8_fused_sse_planes(mats["T1"], [a, b], 10)
    for p, s in zip((a, b), sse):
        assert torch.equal(s, adct.approx_dct8x8_fused_sse(mats["T1"], p, [10])[:, 0])


def test_planes_argument_errors(mats):
    y = torch.zeros((1, 64, 128), dtype=torch.uint8, device=DEV)
    with pytest.raises(ValueError):
        adct.approx_dct8x8_fused_sse_planes(mats["T1"], [y] * 4, 10)
    with pytest.raises(adct.AdctError):
        adct.approx_dct8x8_fused_sse_planes(mats["T1"], [y], 0)
    with pytest.raises(ValueError):
        adct.approx_dct8x8_fused_sse_planes(mats["T1"], [y, y.to(torch.int16)], 10)
