"""GPU parity: the CUDA path (through the C-ABI) against the CPU oracle on the same seeded
inputs.  Integer transform / retention / quantiser: bit-exact.  Floating point (after S,
inverse, error): <= 1e-5 relative (per-block max-norm for arrays; per value for SSE) and
<= 1e-3 dB PSNR (BASELINE.json north_star); SSE exactly 0 where the oracle's is 0 (r = 64).
"""
import ctypes
import fractions
import math

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
INT_NAMES = list(catalog.INTEGER)
ORTHO = ["T1", "T2", "LO", "RDCT", "T4", "T6"]


def tmat(name):
    return np.array(catalog.INTEGER[name]).reshape(8, 8)


@pytest.fixture(scope="module")
def mats():
    d = {n: adct.Matrix.from_int(catalog.INTEGER[n], n) for n in INT_NAMES}
    d["DCT"] = adct.Matrix.from_real(catalog.exact_dct(), "DCT")
    return d


def blocks_to_image(a):
    n, bh, bw = a.shape[:3]
    return a.transpose(0, 1, 3, 2, 4).reshape(n, bh * 8, bw * 8)


def rel_block_err(got, ref):
    """per-block max-norm relative error, ||g - o||_inf / max(||o||_inf, 1) (reading A17)"""
    g = got.reshape(-1, 64).astype(np.float64)
    o = ref.reshape(-1, 64).astype(np.float64)
    return float(np.max(np.abs(g - o).max(axis=1) / np.maximum(np.abs(o).max(axis=1), 1.0)))


def images(kind, n, h, w, seed):
    if kind == "ar1":
        return synth.ar1_field(n, h, w, 0.95, seed=seed)
    if kind == "uniform":
        return synth.uniform_blocks_u8(n, h, w, seed=seed)
    if kind == "laplace":
        b = synth.laplace_blocks(n * (h // 8) * (w // 8), seed=seed)
        return torch.from_numpy(blocks_to_image(b.numpy().reshape(n, h // 8, w // 8, 8, 8)).copy())
    if kind == "extreme":
        g = torch.Generator().manual_seed(seed)
        return (torch.randint(0, 2, (n, h, w), generator=g) * 255).to(torch.uint8)
    raise ValueError(kind)


SHAPES = [(1, 8, 8), (3, 40, 56), (2, 64, 1032), (1, 136, 520)]  # one block .. several tiles + ragged tails


# --- forward -------------------------------------------------------------------------------

@pytest.mark.parametrize("name", INT_NAMES)
@pytest.mark.parametrize("kind", ["ar1", "uniform", "extreme", "laplace"])
def test_forward_int32_bit_exact(mats, name, kind):
    for (n, h, w) in SHAPES[:3]:
        img = images(kind, n, h, w, seed=n * 1000 + w)
        y = adct.approx_dct8x8_fwd(mats[name], img.to(DEV), torch.int32).cpu().numpy()
        assert np.array_equal(y, oracle.forward_int(tmat(name), img.numpy()))


def test_forward_int16_output_and_strided_view(mats):
    img = images("uniform", 2, 48, 80, seed=3)
    big = torch.zeros((2, 64, 128), dtype=torch.uint8)
    big[:, 8:56, 16:96] = img
    view = big.to(DEV)[:, 8:56, 16:96]  # row stride 128, image stride 8192
    y16 = adct.approx_dct8x8_fwd(mats["T1"], view, torch.int16).cpu().numpy()
    assert np.array_equal(y16.astype(np.int64), oracle.forward_int(M.T1, img.numpy()))


@pytest.mark.parametrize("name", INT_NAMES)
def test_forward_f32_scaled(mats, name):
    img = images("ar1", 2, 40, 56, seed=5)
    b = adct.approx_dct8x8_fwd(mats[name], img.to(DEV), torch.float32).cpu().numpy()
    n, s = oracle.row_scaling(tmat(name))
    ref = oracle.scale(oracle.forward_int(tmat(name), img.numpy()), s)
    assert rel_block_err(b, ref) <= RTOL


@pytest.mark.parametrize("kind", ["ar1", "laplace"])
def test_forward_exact_dct(mats, kind):
    img = images(kind, 2, 40, 56, seed=6)
    b = adct.approx_dct8x8_fwd(mats["DCT"], img.to(DEV), torch.float32).cpu().numpy()
    ref = oracle.forward_real(M.C, img.numpy())
    assert rel_block_err(b, ref) <= RTOL


# --- retention -----------------------------------------------------------------------------

@pytest.mark.parametrize("dtype", [torch.int32, torch.int16, torch.float32])
def test_retain_bit_exact(mats, dtype):
    img = images("uniform", 2, 24, 40, seed=8)
    y = oracle.forward_int(M.T1, img.numpy())
    for r in [1, 2, 3, 10, 33, 63, 64]:
        c = torch.from_numpy(y.astype({torch.int32: np.int32, torch.int16: np.int16,
                                       torch.float32: np.float32}[dtype])).to(DEV)
        adct.zonal_retain(c, r)
        assert np.array_equal(c.cpu().numpy().astype(np.int64), oracle.retain(y, r))
    with pytest.raises(adct.AdctError):
        adct.zonal_retain(torch.zeros(64, dtype=dtype, device=DEV), 0)


# --- inverse -------------------------------------------------------------------------------

@pytest.mark.parametrize("name", INT_NAMES + ["DCT"])
@pytest.mark.parametrize("r", [1, 6, 10, 40, 64])
def test_inverse_f32(mats, name, r):
    img = images("ar1", 2, 40, 56, seed=9)
    if name == "DCT":
        chat = M.C
        bref = oracle.forward_real(M.C, img.numpy())
        coef = torch.from_numpy(oracle.retain(bref, r).astype(np.float32)).to(DEV)
    else:
        chat = oracle.chat_from_int(tmat(name))
        n, s = oracle.row_scaling(tmat(name))
        yr = oracle.retain(oracle.forward_int(tmat(name), img.numpy()), r)
        bref = oracle.scale(yr, s)
        coef = torch.from_numpy(yr.astype(np.int32)).to(DEV)
    g, _ = oracle.synthesis_matrix(chat)
    ref = blocks_to_image(oracle.inverse(g, oracle.retain(bref, r)))
    rec = adct.approx_dct8x8_inv(mats[name], coef, 40, 56).cpu().numpy()
    assert rel_block_err(rec, ref) <= RTOL
    if name != "DCT":  # B' (f32 scaled coefficients) input gives the same reconstruction
        rec2 = adct.approx_dct8x8_inv(mats[name], torch.from_numpy(oracle.retain(bref, r).astype(np.float32))
                                      .to(DEV), 40, 56).cpu().numpy()
        assert rel_block_err(rec2, ref) <= RTOL


@pytest.mark.parametrize("name", ["T1", "DCT"])
def test_config5_roundtrip_int16_bit_exact(mats, name):
    """C5 pin: rint(inverse(forward(X))) == X for int16 Laplace blocks."""
    n_blocks = 1 << 16
    x = synth.laplace_blocks(n_blocks, seed=5).reshape(n_blocks, 8, 8)  # images of one block
    xd = x.to(DEV)
    ct = torch.int32 if name == "T1" else torch.float32
    coef = adct.approx_dct8x8_fwd(mats[name], xd, ct)
    rec = adct.approx_dct8x8_inv(mats[name], coef, 8, 8, torch.int16, adct.CLIP_ROUND)
    assert torch.equal(rec.cpu(), x)


def test_inverse_u8_round_clip(mats):
    img = images("ar1", 1, 32, 32, seed=2)
    y = adct.approx_dct8x8_fwd(mats["T1"], img.to(DEV), torch.int32)
    adct.zonal_retain(y, 6)
    rec = adct.approx_dct8x8_inv(mats["T1"], y, 32, 32, torch.uint8, adct.CLIP_ROUND).cpu().numpy()
    n, s = oracle.row_scaling(M.T1)
    g, _ = oracle.synthesis_matrix(oracle.chat_from_int(M.T1))
    ref = blocks_to_image(oracle.inverse(g, oracle.scale(oracle.retain(oracle.forward_int(M.T1, img.numpy()), 6), s)))
    ref_u8 = np.clip(np.rint(ref), 0, 255)
    # rounding may differ only where the exact value is within fp32 error of .5
    diff = np.abs(rec.astype(np.int64) - ref_u8)
    assert diff.max() <= 1
    assert np.all(np.abs(np.abs(ref - np.floor(ref)) - 0.5)[diff > 0] < 1e-3)


# --- psnr_reduce -----------------------------------------------------------------------------

@pytest.mark.parametrize("clip", [adct.CLIP_NONE, adct.CLIP, adct.CLIP_ROUND])
def test_psnr_reduce(mats, clip):
    img = images("ar1", 3, 40, 56, seed=12)
    y = adct.approx_dct8x8_fwd(mats["T1"], img.to(DEV), torch.int32)
    adct.zonal_retain(y, 3)
    rec = adct.approx_dct8x8_inv(mats["T1"], y, 40, 56)
    sse, psnr = adct.psnr_reduce(img.to(DEV), rec, clip=clip)
    rec_blocks = rec.cpu().numpy().astype(np.float64).reshape(3, 5, 8, 7, 8).transpose(0, 1, 3, 2, 4)
    ref = oracle.sse(img.numpy(), rec_blocks, clip)
    assert np.allclose(sse.cpu().numpy(), ref, rtol=RTOL, atol=0)
    for i in range(3):
        assert abs(psnr[i].item() - oracle.psnr(ref[i], 40 * 56)) <= 1e-3
    s0, p0 = adct.psnr_reduce(img.to(DEV), img.to(DEV).float())
    assert torch.all(s0 == 0) and torch.all(torch.isinf(p0))


# --- fused paths -------------------------------------------------------------------------------

def _check_sse(got, ref):
    got = np.asarray(got, dtype=np.float64)
    zero = ref <= 1e-16 * 64 * 1e6
    assert np.all(got[zero] == 0.0)
    assert np.allclose(got[~zero], ref[~zero], rtol=RTOL, atol=0)


@pytest.mark.parametrize("name", INT_NAMES + ["DCT"])
def test_fused_sweep_all_r(mats, name):
    img = images("ar1", 2, 64, 72, seed=21)
    rs = list(range(1, 65))
    sse = adct.approx_dct8x8_fused_sse(mats[name], img.to(DEV), rs).cpu().numpy()
    kw = {"c": M.C} if name == "DCT" else {"t": tmat(name)}
    _check_sse(sse, oracle.codec_sse(img.numpy(), rs, **kw))


@pytest.mark.parametrize("r", [1, 3, 6, 10, 14, 15, 21, 28, 36, 64])
@pytest.mark.parametrize("name", ["T1", "T6", "LO", "SDCT"])
def test_fused_single_r(mats, name, r):
    img = images("ar1", 3, 72, 200, seed=r)  # ragged chunks
    sse = adct.approx_dct8x8_fused_sse(mats[name], img.to(DEV), [r]).cpu().numpy()
    _check_sse(sse, oracle.codec_sse(img.numpy(), [r], t=tmat(name)))


@pytest.mark.parametrize("clip", [adct.CLIP, adct.CLIP_ROUND])
def test_fused_clip(mats, clip):
    img = images("uniform", 2, 32, 48, seed=4)  # saturates often
    for rs in ([10], [2, 10, 30]):
        sse = adct.approx_dct8x8_fused_sse(mats["T1"], img.to(DEV), rs, clip=clip).cpu().numpy()
        ref = oracle.codec_sse(img.numpy(), rs, t=M.T1, clip=clip)
        if clip == adct.CLIP_ROUND:
            _check_sse_round(sse, ref, img.numpy(), rs)
        else:
            _check_sse(sse, ref)


def _check_sse_round(sse, ref, img, rs):
    """Tie-aware SSE rule for CLIP_ROUND (reading A6 + A17): fp32 may round a reconstructed
    pixel to the other neighbour only where the exact value is within 1e-3 of a .5 tie.  Each such
    pixel may move the image's SSE by at most |(x - lo)^2 - (x - hi)^2|; everything else is held
    to the north-star 1e-5."""
    for j, r in enumerate(rs):
        rec = _oracle_recon("T1", img, r)  # exact (fp64) reconstruction image
        lo = np.clip(np.floor(rec), 0, 255)
        hi = np.clip(np.floor(rec) + 1, 0, 255)
        near = np.abs(rec - np.floor(rec) - 0.5) < 1e-3
        x = img.astype(np.float64)
        slack = (np.abs((x - lo) ** 2 - (x - hi) ** 2) * near).reshape(img.shape[0], -1).sum(axis=1)
        assert np.all(np.abs(sse[:, j] - ref[:, j]) <= RTOL * ref[:, j] + slack), (r, slack)


def test_fused_int16_source(mats):
    img = images("laplace", 2, 32, 40, seed=13)
    rs = [1, 10, 64]
    for name in ("T1", "DCT"):
        kw = {"c": M.C} if name == "DCT" else {"t": M.T1}
        sse = adct.approx_dct8x8_fused_sse(mats[name], img.to(DEV), rs).cpu().numpy()
        _check_sse(sse, oracle.codec_sse(img.numpy(), rs, **kw))


def test_fused_deterministic_and_shard_invariant(mats):
    img = images("ar1", 6, 64, 128, seed=30).to(DEV)
    a = adct.approx_dct8x8_fused_sse(mats["T1"], img, [10]).cpu().numpy()
    b = adct.approx_dct8x8_fused_sse(mats["T1"], img, [10]).cpu().numpy()
    assert np.array_equal(a, b)
    parts = [adct.approx_dct8x8_fused_sse(mats["T1"], img[i:i + 2], [10]).cpu().numpy() for i in (0, 2, 4)]
    assert np.array_equal(np.concatenate(parts), a)


def test_fused_host_pipeline_equals_device(mats):
    img = images("ar1", 7, 64, 96, seed=31)
    dev = adct.approx_dct8x8_fused_sse(mats["T1"], img.to(DEV), [10, 21]).cpu()
    host = img.pin_memory()
    g = adct.geom_of(host)
    ws = torch.empty(adct.host_workspace_bytes(g, 2, 3), dtype=torch.uint8, device=DEV)
    got = adct.approx_dct8x8_fused_sse_host(mats["T1"], host, [10, 21], ws, chunk_images=3)
    assert torch.equal(got, dev)


def test_config1_full_size(mats):
    """C1: one 512x512 AR(1) image, r = 1..64, T1 — every r against the oracle."""
    img = synth.ar1_field(1, 512, 512, 0.95, seed=1)
    rs = list(range(1, 65))
    sse, psnr = adct.approx_dct8x8_fused_sse(mats["T1"], img.to(DEV), rs, return_psnr=True)
    sse, psnr = sse.cpu().numpy(), psnr.cpu().numpy()
    ref = oracle.codec_sse(img.numpy(), rs, t=M.T1)
    _check_sse(sse, ref)
    for r in rs:  # the library's PSNR (finalize kernel), north star: <= 1e-3 dB
        if r == 64:  # reading A8: SSE is exactly 0 and PSNR +inf (the fp64 oracle leaves ~1e-20)
            assert sse[0, 63] == 0.0 and ref[0, 63] < 1e-6
            assert math.isinf(psnr[0, 63]) and psnr[0, 63] > 0
        else:
            assert abs(psnr[0, r - 1] - oracle.psnr(ref[0, r - 1], 512 * 512)) <= 1e-3


def test_config2_full_size_sampled(mats):
    """C2 in the launch configuration bench.py times: the 45-image 512x512 stack (per-image rho,
    std of synth.config2_params), r = 1..64, each of the nine matrices through the same call;
    sampled images (first, last, two inside) against the oracle for every r, and two properties
    the paper states on the whole stack: at r = 1 all nine matrices give the same error (the DC
    row of every T is constant, so B_00 and its basis image agree), and the mean PSNR of T1
    exceeds LO's and T6's for every 1 < r < 64."""
    rho, std = synth.config2_params(45, 2)
    imgs = synth.ar1_stack(45, 512, 512, rho, std=std, seed=2, batch=15)
    d = imgs.to(DEV)
    rs = list(range(1, 65))
    pick = [0, 17, 31, 44]
    mean_psnr = {}
    sse_r1 = []
    for name in catalog.CONFIG2_ORDER:
        sse, psnr = adct.approx_dct8x8_fused_sse(mats[name], d, rs, return_psnr=True)
        sse, psnr = sse.cpu().numpy(), psnr.cpu().numpy()
        kw = {"c": M.C} if name == "DCT" else {"t": tmat(name)}
        ref = oracle.codec_sse(imgs[pick].numpy(), rs, **kw)
        _check_sse(sse[pick], ref)
        for j, i in enumerate(pick):
            for r in (1, 10, 33, 63):
                assert abs(psnr[i, r - 1] - oracle.psnr(ref[j, r - 1], 512 * 512)) <= 1e-3
        assert np.all(sse[:, 63] == 0.0) and np.all(np.isposinf(psnr[:, 63]))  # reading A8
        mean_psnr[name] = psnr[:, :63].mean(axis=0)
        sse_r1.append(sse[:, 0])
    for other in sse_r1[1:]:
        assert np.allclose(other, sse_r1[0], rtol=2e-5, atol=0)
    assert np.all(mean_psnr["T1"][1:] > mean_psnr["LO"][1:])
    assert np.all(mean_psnr["T1"][1:] > mean_psnr["T6"][1:])


def test_config4_sampled_frames(mats):
    """C4 geometry (3840x2160 luma, 1920x1080 chroma), hot kernel r = 10, on sampled frames;
    per-plane PSNR from the library within 1e-3 dB."""
    y, u, v = synth.yuv420_stack(2, seed=4)
    for plane in (y, u, v):
        sse, psnr = adct.approx_dct8x8_fused_sse(mats["T1"], plane.to(DEV), [10], return_psnr=True)
        ref = oracle.codec_sse(plane.numpy(), [10], t=M.T1)
        _check_sse(sse.cpu().numpy(), ref)
        npix = plane.shape[1] * plane.shape[2]
        for i in range(plane.shape[0]):
            assert abs(float(psnr[i, 0]) - oracle.psnr(ref[i, 0], npix)) <= 1e-3


@pytest.mark.parametrize("r_list", [[10], [3, 10, 64]])
def test_fused_host_psnr(mats, r_list):
    """Host-buffer path: SSE and PSNR equal the device path's bit for bit; PSNR +inf at r = 64;
    a lone image whose image_stride is 0 (ignored for one image) stages correctly."""
    img = images("ar1", 5, 64, 128, seed=32)
    dsse, dpsnr = adct.approx_dct8x8_fused_sse(mats["T1"], img.to(DEV), r_list, return_psnr=True)
    host = img.pin_memory()
    g = adct.geom_of(host)
    ws = torch.empty(adct.host_workspace_bytes(g, len(r_list), 2), dtype=torch.uint8, device=DEV)
    hsse, hpsnr = adct.approx_dct8x8_fused_sse_host(mats["T1"], host, r_list, ws, chunk_images=2, return_psnr=True)
    assert torch.equal(hsse, dsse.cpu()) and torch.equal(hpsnr, dpsnr.cpu())
    if 64 in r_list:
        assert torch.all(hpsnr[:, r_list.index(64)] == float("inf"))
    one = host[:1]
    g1 = adct.geom_of(one)
    g1.image_stride = 0
    ws1 = torch.empty(adct.host_workspace_bytes(g1, len(r_list), 1), dtype=torch.uint8, device=DEV)
    out = torch.empty((1, len(r_list)), dtype=torch.float64).pin_memory()
    rl = (ctypes.c_int32 * len(r_list))(*r_list)
    st = adct.lib.approx_dct8x8_fused_sse_host(mats["T1"].handle, one.data_ptr(), adct.U8, g1,
                                               ctypes.cast(rl, ctypes.c_void_p), len(r_list), adct.CLIP_NONE,
                                               out.data_ptr(), None, 1, ws1.data_ptr(), ws1.numel(), None)
    assert st == 0 and torch.equal(out, dsse[:1].cpu())


# --- quantiser ----------------------------------------------------------------------------------

def test_quantiser_bit_exact(mats):
    img = images("ar1", 2, 64, 96, seed=40)
    q = adct.approx_dct8x8_fwd_quant(mats["T1"], img.to(DEV), 16).cpu().numpy()
    n, s = oracle.row_scaling(M.T1)
    assert np.array_equal(q, oracle.quantize(oracle.forward_int(M.T1, img.numpy()), n, 16))


def test_quantiser_extreme_and_uniform(mats):
    """Extremal (0/255) and uniform-random blocks: large |Y| at every position."""
    ext = images("extreme", 8, 256, 256, seed=41)
    uni = images("uniform", 8, 256, 256, seed=42)
    for img in (ext, uni):
        q = adct.approx_dct8x8_fwd_quant(mats["T1"], img.to(DEV), 16).cpu().numpy()
        n, s = oracle.row_scaling(M.T1)
        assert np.array_equal(q, oracle.quantize(oracle.forward_int(M.T1, img.numpy()), n, 16))


@pytest.mark.parametrize("step", [1, 3, 7, 17, 100, 255, 4096])
def test_quantiser_other_steps(mats, step):
    """Steps other than 16 (the TMA kernel accepts 1..4096; its directed-rounding FMA at the
    rational positions is exact for every A < 2^23, tests/test_kernel_arith.py): bit-exact."""
    n, _ = oracle.row_scaling(M.T1)
    for img in (images("uniform", 2, 128, 256, seed=44), images("extreme", 2, 128, 256, seed=45)):
        q = adct.approx_dct8x8_fwd_quant(mats["T1"], img.to(DEV), step).cpu().numpy()
        assert np.array_equal(q, oracle.quantize(oracle.forward_int(M.T1, img.numpy()), n, step))


def _tie_blocks(seed=43):
    """u8 blocks that put EVERY reachable exact tie Y = (m + 1/2) * 16 sqrt(n_k n_l) of T1 at each
    of the 40 positions where sqrt(n_k n_l) is rational (reading A10; S_1).  Y_kl =
    sum_ij t_k[i] t_l[j] X[i][j]: the cells of one sign are filled greedily (largest weight first,
    the weight-1 cells take the remainder), the opposite-sign cells are 0 and the zero-weight cells
    random.  Returns (blocks [n,8,8] u8, [(k, l, Y)] per block)."""
    rng = np.random.default_rng(seed)
    t = tmat("T1").astype(np.int64)
    nrm = (t * t).sum(axis=1)
    blocks, meta = [], []
    for k in range(8):
        for l in range(8):
            prod = int(nrm[k] * nrm[l])
            root = math.isqrt(prod)
            if root * root != prod:
                continue
            w = np.outer(t[k], t[l])
            c = 16 * root  # quantiser step at (k, l); ties at |Y| = (2m + 1) c / 2
            for sign in (1, -1):
                cells = [(int(sign * w[i, j]), i, j) for i in range(8) for j in range(8) if sign * w[i, j] > 0]
                cells.sort(reverse=True)
                cap = 255 * sum(cw for cw, _, _ in cells)
                for odd in range(1, 2 * cap // c + 2, 2):
                    target = odd * c // 2
                    if target > cap:
                        break
                    x = np.where(w == 0, rng.integers(0, 256, (8, 8)), 0)
                    rem = target
                    for cw, i, j in cells:
                        v = min(255, rem // cw)
                        x[i, j] = v
                        rem -= v * cw
                    assert rem == 0
                    blocks.append(x)
                    meta.append((k, l, sign * target))
    return np.array(blocks, dtype=np.uint8), meta


def test_quantiser_every_reachable_tie(mats):
    """Every exact tie reachable from u8 input at the 40 rational positions (e.g. Y_00 = sum X =
    64 (2m + 1), m = 0..127): the TMA quantiser kernel equals the oracle bit for bit, and at the
    tied position both equal round-half-AWAY-from-zero computed exactly with Fractions."""
    b, meta = _tie_blocks()
    n_img_blocks = 64  # 512-wide image rows of blocks, TMA path (row stride % 16 == 0)
    pad = (-len(b)) % n_img_blocks
    bb = np.concatenate([b, np.zeros((pad, 8, 8), dtype=np.uint8)])
    img = blocks_to_image(bb.reshape(1, -1, n_img_blocks, 8, 8))
    y = oracle.forward_int(M.T1, img)
    n, _ = oracle.row_scaling(M.T1)
    ref = oracle.quantize(y, n, 16)
    q = adct.approx_dct8x8_fwd_quant(mats["T1"], torch.from_numpy(img).to(DEV), 16).cpu().numpy()
    assert np.array_equal(q, ref)
    yf, qf = y.reshape(-1, 8, 8), q.reshape(-1, 8, 8)
    counts = {}
    for idx, (k, l, target) in enumerate(meta):
        assert yf[idx, k, l] == target  # the block really hits the tie
        c = 16 * math.isqrt(int(n[k] * n[l]))
        exact = fractions.Fraction(abs(target), c)  # = m + 1/2
        assert exact.denominator == 2
        away = exact.numerator // 2 + 1
        assert qf[idx, k, l] == (away if target > 0 else -away)
        counts[(k, l)] = counts.get((k, l), 0) + 1
    assert len(counts) == 40
    assert counts[(0, 0)] == 128  # Y_00 = 64 (2m + 1), m = 0..127; no negative Y_00 from u8


# --- fused round trip (fwd -> retain -> inv in one pass; config 5) ---------------------------------

def _oracle_recon(name, img, r):
    """Oracle reconstruction image of fwd -> retain r -> inverse (no clip)."""
    if name == "DCT":
        chat = M.C
        bp = oracle.retain(oracle.forward_real(M.C, img), r)
    else:
        chat = oracle.chat_from_int(tmat(name))
        n, s = oracle.row_scaling(tmat(name))
        bp = oracle.scale(oracle.retain(oracle.forward_int(tmat(name), img), r), s)
    g, _ = oracle.synthesis_matrix(chat)
    return blocks_to_image(oracle.inverse(g, bp))


@pytest.mark.parametrize("name", ["T1", "T6", "LO", "SDCT", "BAS-2008b", "DCT"])
@pytest.mark.parametrize("r", [1, 10, 33, 64])
@pytest.mark.parametrize("kind", ["ar1", "laplace"])
def test_roundtrip_f32_matches_composition(mats, name, r, kind):
    img = images(kind, 2, 40, 72, seed=50 + r)
    rec = adct.approx_dct8x8_roundtrip(mats[name], img.to(DEV), r, torch.float32).cpu().numpy()
    ref = _oracle_recon(name, img.numpy(), r)
    assert rel_block_err(rec, ref) <= RTOL


@pytest.mark.parametrize("name", ["T1", "DCT"])
def test_roundtrip_config5_int16_bit_exact(mats, name):
    """C5 pin: rint(inverse(forward(X))) == X at r = 64 for int16 Laplace blocks,
    here through the fused one-pass kernel, with a ragged tail of blocks."""
    n_blocks = (1 << 16) + 37
    x = synth.laplace_blocks(n_blocks, seed=5).reshape(n_blocks, 8, 8)
    rec = adct.approx_dct8x8_roundtrip(mats[name], x.to(DEV), 64, torch.int16)
    assert torch.equal(rec.cpu(), x)


def test_roundtrip_u8_round_clip_and_strided(mats):
    img = images("ar1", 2, 48, 80, seed=7)
    big = torch.zeros((2, 56, 96), dtype=torch.uint8)
    big[:, 8:56, 16:96] = img
    view = big.to(DEV)[:, 8:56, 16:96]
    rec = adct.approx_dct8x8_roundtrip(mats["T1"], view, 10, torch.uint8).cpu().numpy()
    ref = _oracle_recon("T1", img.numpy(), 10)
    ref_u8 = np.clip(np.rint(ref), 0, 255)
    diff = np.abs(rec.astype(np.int64) - ref_u8)
    assert diff.max() <= 1
    assert np.all(np.abs(np.abs(ref - np.floor(ref)) - 0.5)[diff > 0] < 1e-3)


def test_roundtrip_argument_errors(mats):
    x = torch.zeros((1, 8, 8), dtype=torch.int16, device=DEV)
    for bad_r in (0, 65):
        with pytest.raises(adct.AdctError):
            adct.approx_dct8x8_roundtrip(mats["T1"], x, bad_r, torch.int16)
    with pytest.raises(adct.AdctError):  # integer output needs CLIP_ROUND
        adct.approx_dct8x8_roundtrip(mats["T1"], x, 10, torch.int16, clip=adct.CLIP_NONE)


@pytest.mark.parametrize("name", ["T1", "DCT", "T6"])
@pytest.mark.parametrize("out", [torch.int16, torch.float32])
def test_roundtrip_blockmajor_tma_path(mats, name, out):
    """Block-major int16 stacks with a multiple of 32 blocks take the TMA-streamed kernel:
    int16 output bit-exact at r = 64 (C5 pin), fp32 output against the oracle at r = 10."""
    n_blocks = 1 << 14
    x = synth.laplace_blocks(n_blocks, seed=8).reshape(n_blocks, 8, 8)
    xd = x.to(DEV)
    if out == torch.int16:
        rec = adct.approx_dct8x8_roundtrip(mats[name], xd, 64, torch.int16)
        if name in ("T1", "DCT"):
            assert torch.equal(rec.cpu(), x)
        ref = np.rint(_oracle_recon(name, x.numpy(), 64))
        assert np.abs(rec.cpu().numpy().astype(np.int64) - ref).max() <= 1
    else:
        rec = adct.approx_dct8x8_roundtrip(mats[name], xd, 10, torch.float32).cpu().numpy()
        assert rel_block_err(rec, _oracle_recon(name, x.numpy(), 10)) <= RTOL


def _check_int_recon(rec, ref, lo=-32768, hi=32767):
    """Integer reconstruction (round half even, saturate) against the exact oracle value: equal,
    or one level off only where the exact value is within 1e-3 of a .5 tie (fp32 rounding)."""
    ref_i = np.clip(np.rint(ref), lo, hi)
    diff = np.abs(rec.astype(np.int64) - ref_i)
    assert diff.max() <= 1
    assert np.all(np.abs(np.abs(ref - np.floor(ref)) - 0.5)[diff > 0] < 1e-3)


@pytest.mark.parametrize("name", ["T1", "DCT", "T6"])
@pytest.mark.parametrize("n_blocks", [32 * 97, 32 * 97 + 5])  # TMA block-major path / generic kernel
def test_roundtrip_in_place(mats, name, n_blocks):
    """C5 runs in place at 2^30 blocks (recon IS src): the same call with recon = src gives the
    out-of-place result bit for bit -- r = 64 (the identity for T1 and C) and r = 10."""
    x = synth.laplace_range(0, n_blocks, seed=9)
    for r in (64, 10):
        want = adct.approx_dct8x8_roundtrip(mats[name], x.to(DEV), r, torch.int16).cpu()
        xd = x.to(DEV)
        got = adct.approx_dct8x8_roundtrip(mats[name], xd, r, torch.int16, recon=xd)
        assert got.data_ptr() == xd.data_ptr()
        assert torch.equal(xd.cpu(), want)
        if r == 64 and name in ("T1", "DCT"):
            assert torch.equal(want, x)
        idx = np.arange(0, n_blocks, 101)
        _check_int_recon(want.numpy()[idx], _oracle_recon(name, x.numpy()[idx], r))


def test_roundtrip_in_place_u8_images(mats):
    """u8 images reconstructed in place (round half even, clip [0, 255]) equal out of place."""
    img = images("ar1", 3, 72, 264, seed=12)
    want = adct.approx_dct8x8_roundtrip(mats["T1"], img.to(DEV), 10, torch.uint8).cpu()
    xd = img.to(DEV)
    adct.approx_dct8x8_roundtrip(mats["T1"], xd, 10, torch.uint8, recon=xd)
    assert torch.equal(xd.cpu(), want)
    _check_int_recon(want.numpy(), _oracle_recon("T1", img.numpy(), 10), 0, 255)


# --- SSIM (next row f1; reading A18) -------------------------------------------------------------

from oracle import ssim as OS  # noqa: E402


@pytest.mark.parametrize("shape", [(1, 8, 8), (2, 40, 56), (1, 72, 104), (2, 104, 264)])
@pytest.mark.parametrize("rtype", [torch.float32, torch.uint8])
def test_ssim_reduce_matches_oracle(shape, rtype):
    n, h, w = shape
    x = images("ar1", n, h, w, seed=h + w)
    noise = torch.from_numpy(np.random.default_rng(h).normal(0, 12, size=(n, h, w)).astype(np.float32))
    r = (x.float() + noise).clamp(-20, 280)
    if rtype == torch.uint8:
        r = r.clamp(0, 255).round().to(torch.uint8)
    for clip in (adct.CLIP_NONE, adct.CLIP, adct.CLIP_ROUND):
        got = adct.ssim_reduce(x.to(DEV), r.to(DEV), clip=clip).cpu().numpy()
        ref = OS.ssim(x.numpy(), r.numpy(), clip=clip)
        assert np.allclose(got, ref, rtol=1e-9, atol=1e-12), (got, ref)


def test_ssim_many_bands_and_strips():
    """u8 originals with fp32 reconstructions over many images: every warp unit (a band of 64
    window rows x a strip of 25 window columns) is used, including the ragged last band and
    strip of each image, and the partials of all images are finalized independently."""
    x = images("ar1", 40, 256, 272, seed=9)
    r = (x.float() + torch.from_numpy(np.random.default_rng(1).normal(0, 9, size=x.shape).astype(np.float32)))
    for clip in (adct.CLIP_NONE, adct.CLIP):
        got = adct.ssim_reduce(x.to(DEV), r.to(DEV), clip=clip).cpu().numpy()
        ref = OS.ssim(x.numpy(), r.numpy(), clip=clip)
        assert np.allclose(got, ref, rtol=1e-9, atol=1e-12)


@pytest.mark.parametrize("rtype", [torch.int16, torch.float32, torch.uint8])
def test_ssim_int16_original(rtype):
    """int16 originals (the fp64 sums path: x^2 window sums exceed 2^24) against the oracle,
    with int16 / fp32 / u8 reconstructions, at shapes with one band and several, including
    a single-window image."""
    for n, h, w in ((1, 8, 8), (2, 72, 112), (1, 144, 40)):
        g = np.random.default_rng(h * w)
        x = torch.from_numpy(g.integers(-300, 300, size=(n, h, w)).astype(np.int16))
        r = x.float() + torch.from_numpy(g.normal(0, 15, size=(n, h, w)).astype(np.float32))
        if rtype == torch.int16:
            r = r.round().to(torch.int16)
        elif rtype == torch.uint8:
            r = r.clamp(0, 255).round().to(torch.uint8)
        for clip in (adct.CLIP_NONE, adct.CLIP, adct.CLIP_ROUND):
            got = adct.ssim_reduce(x.to(DEV), r.to(DEV), clip=clip).cpu().numpy()
            ref = OS.ssim(x.numpy(), r.numpy(), clip=clip)
            assert np.allclose(got, ref, rtol=1e-9, atol=1e-12), (n, h, w, clip, got, ref)


def test_ssim_identical_is_one_and_pipeline(mats):
    """SSIM(x, x) = 1; and the C1-shaped pipeline fwd -> retain r -> inv (fused round trip) ->
    SSIM against the oracle composition, for T1 and the DCT, at the paper's r = 3 and 14
    (P:L2380-2444)."""
    img = synth.ar1_field(1, 128, 128, 0.95, seed=1)
    xd = img.to(DEV)
    assert abs(float(adct.ssim_reduce(xd, xd)[0]) - 1.0) < 1e-12
    for name in ("T1", "DCT"):
        for r in (3, 14):
            rec = adct.approx_dct8x8_roundtrip(mats[name], xd, r, torch.float32)
            got = adct.ssim_reduce(xd, rec, clip=adct.CLIP).cpu().numpy()
            ref = OS.ssim(img.numpy(), _oracle_recon(name, img.numpy(), r), clip=1)
            assert np.allclose(got, ref, rtol=1e-6), (name, r, got, ref)


@pytest.mark.parametrize("shape", [(1, 8, 8), (2, 40, 56), (1, 72, 104), (3, 136, 264), (2, 64, 200), (1, 520, 328)])
@pytest.mark.parametrize("name", ["T1", "DCT", "T6"])
def test_ssim_fused_equals_composition(mats, shape, name):
    """approx_dct8x8_ssim (round trip + SSIM in one kernel, no reconstruction in HBM) equals the
    composition approx_dct8x8_roundtrip (fp32) -> ssim_reduce for every clip policy: the same fp32
    reconstruction and exactly representable window sums, only the final per-image summation
    order differs (1e-12).  Shapes: one window, ragged strips (W - 7 not a multiple of 24), chunks
    of 64 rows cut by the image bottom, several images."""
    n, h, w = shape
    img = images("ar1", n, h, w, seed=h * 7 + w).to(DEV)
    for r in (3, 14):
        rec = adct.approx_dct8x8_roundtrip(mats[name], img, r, torch.float32)
        for clip in (adct.CLIP_NONE, adct.CLIP, adct.CLIP_ROUND):
            want = adct.ssim_reduce(img, rec, clip=clip).cpu().numpy()
            got = adct.approx_dct8x8_ssim(mats[name], img, r, clip=clip).cpu().numpy()
            assert np.allclose(got, want, rtol=1e-12, atol=1e-15), (r, clip, got, want)


def test_ssim_fused_against_oracle(mats):
    """End to end against the oracle (its fp64 reconstruction, A18 SSIM): the fp32 reconstruction
    bounds the agreement at 1e-6 (as for the two-call pipeline); paper r = 3, 14, and a 520 x 1032 frame."""
    img = synth.ar1_field(2, 136, 264, 0.95, seed=3)
    for name in ("T1", "DCT"):
        for r in (3, 14):
            got = adct.approx_dct8x8_ssim(mats[name], img.to(DEV), r, clip=adct.CLIP).cpu().numpy()
            ref = OS.ssim(img.numpy(), _oracle_recon(name, img.numpy(), r), clip=1)
            assert np.allclose(got, ref, rtol=1e-6), (name, r, got, ref)
    y = synth.ar1_field(1, 520, 1032, 0.95, seed=4)  # many strips and chunks (the 4K oracle takes 26 s)
    got = adct.approx_dct8x8_ssim(mats["T1"], y.to(DEV), 14, clip=adct.CLIP).cpu().numpy()
    ref = OS.ssim(y.numpy(), _oracle_recon("T1", y.numpy(), 14), clip=1)
    assert np.allclose(got, ref, rtol=1e-6)


def test_ssim_fused_argument_errors(mats):
    x = torch.zeros((1, 16, 16), dtype=torch.uint8, device=DEV)
    for bad_r in (0, 65):
        with pytest.raises(adct.AdctError):
            adct.approx_dct8x8_ssim(mats["T1"], x, bad_r)
    assert float(adct.approx_dct8x8_ssim(mats["T1"], x, 64)[0]) == pytest.approx(1.0, abs=1e-12)  # r = 64: x itself


# --- 16/32-point JAM transforms (next row f2; readings A19, A20) ---------------------------------

from oracle import jam as OJ  # noqa: E402


def _rel_err_nn(got, ref, n):
    g = OJ.blocks_n(got, n).reshape(-1, n * n).astype(np.float64)
    o = OJ.blocks_n(ref, n).reshape(-1, n * n).astype(np.float64)
    return float(np.max(np.abs(g - o).max(axis=1) / np.maximum(np.abs(o).max(axis=1), 1.0)))


@pytest.mark.parametrize("n", [16, 32])
@pytest.mark.parametrize("kind", ["ar1", "laplace"])
def test_jam_roundtrip_f32_matches_oracle(n, kind):
    t = OJ.T16 if n == 16 else OJ.T32
    img = images(kind, 2, 2 * n, 3 * n, seed=n)
    for r in (1, 3, 10, n * n // 3, n * n):
        rec = adct.approx_dct_jam_roundtrip(n, img.to(DEV), r, torch.float32).cpu().numpy()
        ref = OJ.recon_n(t, img.numpy(), r)
        assert _rel_err_nn(rec, ref, n) <= RTOL, (n, r)


@pytest.mark.parametrize("n", [16, 32])
def test_jam_roundtrip_int16_bit_exact_and_u8(n):
    nb = 4096 + 3
    x = synth.laplace_blocks(nb * (n // 8) ** 2, seed=n).reshape(nb, n, n)   # n x n residual blocks
    rec = adct.approx_dct_jam_roundtrip(n, x.to(DEV), n * n, torch.int16)
    assert torch.equal(rec.cpu(), x)
    img = images("ar1", 1, 4 * n, 5 * n, seed=3)
    rec8 = adct.approx_dct_jam_roundtrip(n, img.to(DEV), 10, torch.uint8).cpu().numpy()
    ref = OJ.recon_n(OJ.T16 if n == 16 else OJ.T32, img.numpy(), 10)
    ref_u8 = np.clip(np.rint(ref), 0, 255)
    diff = np.abs(rec8.astype(np.int64) - ref_u8)
    assert diff.max() <= 1
    assert np.all(np.abs(np.abs(ref - np.floor(ref)) - 0.5)[diff > 0] < 1e-3)


@pytest.mark.parametrize("n", [16, 32])
def test_jam_full_int16_range(n):
    """Beyond |x| = 7281 the fp32 forward is no longer exact integer arithmetic (include/adct.h):
    over the WHOLE int16 range (uniform, extremal +-32767/-32768 blocks) the fp32 round trip still
    meets the north-star 1e-5 per-block bound against the fp64 oracle, and the int16 round trip
    at r = n^2 is the identity (checked, not assumed: bit-exact here)."""
    t = OJ.T16 if n == 16 else OJ.T32
    g = torch.Generator().manual_seed(70 + n)
    uni = torch.randint(-32768, 32768, (64, n, n), generator=g, dtype=torch.int32).to(torch.int16)
    ext = (torch.randint(0, 2, (64, n, n), generator=g) * 65535 - 32768).to(torch.int16)  # -32768 / 32767
    for x in (uni, ext):
        for r in (10, n * n // 3, n * n):
            rec = adct.approx_dct_jam_roundtrip(n, x.to(DEV), r, torch.float32).cpu().numpy()
            assert _rel_err_nn(rec, OJ.recon_n(t, x.numpy(), r), n) <= RTOL, (n, r)
        rec = adct.approx_dct_jam_roundtrip(n, x.to(DEV), n * n, torch.int16)
        assert torch.equal(rec.cpu(), x)


def test_quantiser_tensor_core_kernel_parity():
    """The tensor-core quantiser (tc.cu fwd_quant_tc_kernel, selected by ADCT_Q_TC=1 and read once
    per process) passes the quantiser parity suite -- C3 frames, ties, extremal images -- in a
    fresh process; widths that are not whole 128-byte chunks still take the SIMT kernel there."""
    import os
    import subprocess
    import sys
    if os.environ.get("ADCT_Q_TC"):
        pytest.skip("already the tensor-core process")
    env = dict(os.environ, ADCT_Q_TC="1")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-m", "gpu", "-k", "quant and not tensor_core",
                        os.path.join(root, "tests", "test_gpu_parity.py")],
                       env=env, cwd=root, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    assert " passed" in r.stdout


def test_jam_v2_kernel_parity():
    """The column-pair / row-pair packed kernel (jam.cu jam2_roundtrip_kernel, selected by
    ADCT_JAM_V2=1 and read once per process) passes the same oracle parity suite, run in a fresh
    process (skipped inside that process)."""
    import os
    import subprocess
    import sys
    if os.environ.get("ADCT_JAM_V2"):
        pytest.skip("already the v2 process")
    env = dict(os.environ, ADCT_JAM_V2="1")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-m", "gpu", "-k",
                        "jam_roundtrip or jam_full_int16", os.path.join(root, "tests", "test_gpu_parity.py")],
                       env=env, cwd=root, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    assert " passed" in r.stdout


def test_jam_argument_errors():
    x = torch.zeros((1, 16, 16), dtype=torch.int16, device=DEV)
    with pytest.raises(adct.AdctError):
        adct.approx_dct_jam_roundtrip(8, x, 1, torch.float32)
    with pytest.raises(adct.AdctError):
        adct.approx_dct_jam_roundtrip(16, x, 257, torch.float32)
    with pytest.raises(adct.AdctError):
        adct.approx_dct_jam_roundtrip(32, x, 1, torch.float32)  # 16 x 16 image, 32-point blocks


# --- greedy angle search (next row f3; readings A21-A24) -----------------------------------------

from oracle import greedy as OG  # noqa: E402
import itertools as _it  # noqa: E402


@pytest.fixture(scope="module")
def greedy_spaces():
    return {1: OG.Search(OG.P1), 2: OG.Search(OG.P2)}


def _tie_summary(ties):
    """The oracle's logged ties of one sequence as the C-ABI reports them: (steps with a tie,
    first tied row or -1, candidates tied there, largest tie)."""
    if not ties:
        return [0, -1, 0, 0]
    return [len(ties), ties[0][1], len(ties[0][2]), max(len(t[2]) for t in ties)]


def _check_search(s, entries, orders, fixed):
    mats, status, ties = adct.greedy_search(M.C, entries, np.array(orders, dtype=np.int32), fixed=fixed, device=DEV,
                                            return_ties=True)
    mats, status, ties = mats.cpu().numpy(), status.cpu().numpy(), ties.cpu().numpy()
    n_tied = 0
    for n, o in enumerate(orders):
        log = []
        m = s.solve(tuple(o), fixed, ties=log)
        if m is None:
            assert status[n] == 1, o
        else:
            assert status[n] == 0 and np.array_equal(mats[n], m), o
        assert ties[n].tolist() == _tie_summary(log), (o, log)
        n_tied += bool(log)
    return mats, status, n_tied


@pytest.mark.parametrize("space", [1, 2])
def test_greedy_search_fixed_rows_all_orders(greedy_spaces, space):
    """§4.1 setting: rows 1 and 5 fixed, all 720 orders of the other six; every sequence's
    matrix (or infeasibility) and its logged exact ties equal the oracle's; D2 yields exactly
    T1 and T2."""
    s = greedy_spaces[space]
    free = [k for k in range(8) if k not in OG.FIXED_ROWS]
    orders = list(_it.permutations(free))
    mats, status, _ = _check_search(s, OG.P1 if space == 1 else OG.P2, orders, OG.FIXED_ROWS)
    if space == 2:
        got = {mats[n].tobytes() for n in range(len(orders)) if status[n] == 0}
        assert got == {np.array(M.T1, dtype=np.int32).tobytes(), np.array(M.T2, dtype=np.int32).tobytes()}


def test_greedy_search_free_orders_d1(greedy_spaces):
    """All eight rows free (§3.4): the worked forward/reverse orders and 62 sampled
    permutations of 8! over D1, against the oracle -- matrices and logged ties.  The reverse
    order meets an exact tie (reading A22)."""
    s = greedy_spaces[1]
    rng = np.random.default_rng(7)
    perms = [tuple(range(8)), tuple(range(7, -1, -1))] + [tuple(rng.permutation(8)) for _ in range(62)]
    _, _, n_tied = _check_search(s, OG.P1, perms, None)
    assert n_tied >= 1
    log = []
    s.solve(tuple(range(7, -1, -1)), None, ties=log)
    assert log  # the §3.4 reverse-order example has a logged tie


@pytest.mark.parametrize("entries", [(-4, -1, 0, 1, 4), (-8, -1, 0, 1, 8)])
def test_greedy_search_extended_sets(entries):
    """The extended entry sets of P:L1206-1235 ({0, +-1, +-4}, {0, +-1, +-8}; |D| = 5^8), rows 1
    and 5 fixed, all 720 orders: matrices, feasibility and ties equal the oracle's."""
    s = OG.Search(entries)
    free = [k for k in range(8) if k not in OG.FIXED_ROWS]
    _check_search(s, entries, list(_it.permutations(free)), OG.FIXED_ROWS)


def test_greedy_search_invalid_sequences():
    mats, status = adct.greedy_search(M.C, OG.P1, np.array([[1, 2, 3, 5, 6, 9], [1, 1, 2, 3, 5, 6],
                                                            [0, 1, 2, 3, 5, 6]], dtype=np.int32),
                                      fixed=OG.FIXED_ROWS, device=DEV)
    assert status.cpu().tolist() == [2, 2, 2]


# --- figures of merit (next row f4) ----------------------------------------------------------------

from oracle import merit as OMR  # noqa: E402


def test_merit_batch_matches_oracle():
    """eps, MSE, C*_g, eta (§4.2) of the nine matrices over a range of rho (the Fig. 1 axis),
    against the oracle's definitions (themselves pinned to Table 4)."""
    names = catalog.CONFIG2_ORDER
    mats = [adct.Matrix.from_real(catalog.exact_dct(), "DCT") if n == "DCT" else
            adct.Matrix.from_int(catalog.INTEGER[n], n) for n in names]
    rho = torch.tensor([0.1, 0.5, 0.8, 0.95, 0.99], dtype=torch.float64, device=DEV)
    got = adct.merit_batch(mats, rho).cpu().numpy()
    for a, n in enumerate(names):
        chat = M.C if n == "DCT" else M.c_hat(np.array(catalog.INTEGER[n]).reshape(8, 8))
        for b, r in enumerate(rho.cpu().tolist()):
            want = [OMR.total_error_energy(chat), OMR.mse_matrix(chat, r), OMR.unified_coding_gain(chat, r),
                    OMR.transform_efficiency(chat, r)]
            assert np.allclose(got[a, b], want, rtol=1e-10, atol=1e-12), (n, r, got[a, b], want)


# --- full-size configurations in the bench's launch configuration (sampled outputs) ----------------

def test_config3_full_size_sampled(mats):
    """BASELINE config 3: 1024 frames 1920x1080 (+U(-4,4)) through the TMA quantiser in one
    call; frames 0, 511 and 1023 bit-exact against the oracle's integer rule."""
    imgs = synth.ar1_stack(1024, 1080, 1920, 0.95, seed=3, device=DEV, noise_uniform=4.0, batch=16)
    q = adct.approx_dct8x8_fwd_quant(mats["T1"], imgs, 16)
    n, _ = oracle.row_scaling(M.T1)
    for f in (0, 511, 1023):
        x = imgs[f:f + 1].cpu().numpy()
        assert np.array_equal(q[f:f + 1].cpu().numpy(), oracle.quantize(oracle.forward_int(M.T1, x), n, 16))
    del imgs, q
    torch.cuda.empty_cache()


def test_config5_full_size_in_place(mats):
    """BASELINE config 5 at its largest size, in the launch configuration bench.py times: 2^30
    int16 blocks (137 GB) resident, fused round trip IN PLACE.  r = 64 with T1 and then with C:
    the stack still equals the generated blocks (sampled batches re-generated); then r = 10 in
    place, sampled blocks against the oracle reconstruction of the regenerated originals."""
    torch.cuda.empty_cache()
    nb = 1 << 30
    x = synth.laplace_range(0, nb, seed=5, device=DEV)
    starts = [0, 12345 * 4096, nb // 2, nb - 4096]
    for name in ("T1", "DCT"):
        adct.approx_dct8x8_roundtrip(mats[name], x, 64, torch.int16, recon=x)
        for a in starts:
            assert torch.equal(x[a:a + 4096], synth.laplace_range(a, a + 4096, seed=5, device=DEV))
    adct.approx_dct8x8_roundtrip(mats["T1"], x, 10, torch.int16, recon=x)
    for a in starts:
        orig = synth.laplace_range(a, a + 256, seed=5, device=DEV).cpu().numpy()  # the same generator
        _check_int_recon(x[a:a + 256].cpu().numpy(), _oracle_recon("T1", orig, 10))
    del x
    torch.cuda.empty_cache()


def test_config5_large_roundtrip_sampled(mats):
    """BASELINE config 5 at 2^24 blocks (the bench runs 2^26): the whole stack round-trips
    bit-exactly at r = 64; sampled blocks at r = 10 against the oracle reconstruction."""
    nb = 1 << 24
    x = synth.laplace_blocks(nb, seed=5, device=DEV).reshape(nb, 8, 8)
    assert torch.equal(adct.approx_dct8x8_roundtrip(mats["T1"], x, 64, torch.int16), x)
    rec = adct.approx_dct8x8_roundtrip(mats["T1"], x, 10, torch.float32)
    idx = torch.tensor([0, 12345, nb // 2, nb - 1], device=DEV)
    got = rec[idx].cpu().numpy()
    ref = _oracle_recon("T1", x[idx].cpu().numpy(), 10)
    assert rel_block_err(got, ref) <= RTOL
    del x, rec
    torch.cuda.empty_cache()
