"""Seeded synthetic inputs shaped like the paper's workloads.

This module is shared by the tests, the CPU oracle runs and the CUDA path; it holds
none of the method's arithmetic (no transform, retention, inverse or error), only the
random fields the workloads are made of.

Stand-ins: the paper's 44 USC-SIPI images and the
HEVC CTC sequences are not available; BASELINE.json's configs replace them
with separable first-order Markov (AR(1)) fields, the image model of §4.2 (R_x entries
rho^|i-j|), with rho around the corpus' average correlation 0.86
 to 0.95.

Reading A12 (AR(1) field): X[i,j] = rho X[i-1,j] + rho X[i,j-1] - rho^2 X[i-1,j-1] + e[i,j],
e ~ N(0,1), i.e. a 1-D AR(1) filter along rows followed by one along columns; 64 burn-in
rows and columns are discarded; the field is divided by its theoretical std 1/(1-rho^2),
mapped to mean/std, clipped to [0,255] and rounded half to even to uint8.
"""
from __future__ import annotations

import numpy as np
import torch

BURN_IN = 64
_CHUNK = 64  # length of the blocked linear-recurrence solve


def _ar1_along_last(e: torch.Tensor, rho: torch.Tensor) -> torch.Tensor:
    """y[b, r, j] = rho[b] * y[b, r, j-1] + e[b, r, j] along the last dim (y[-1] = 0).

    Blocked: inside a chunk of length L the recurrence is a product with the lower-
    triangular Toeplitz matrix of powers of rho; chunks are chained by carrying the last
    value.  e is [B, R, n], rho is [B].
    """
    bsz, rows, n = e.shape
    L = _CHUNK
    pad = (-n) % L
    if pad:
        e = torch.nn.functional.pad(e, (0, pad))
    m = e.shape[-1] // L
    t = torch.arange(L, device=e.device, dtype=e.dtype)
    rr = rho.to(e.dtype).reshape(bsz, 1, 1)
    diff = (t[:, None] - t[None, :]).clamp(min=0)
    lower = (t[:, None] >= t[None, :]).to(e.dtype)
    kern = (rr ** diff) * lower                      # [B, L, L], kern[t, s] = rho^(t-s)
    yc = torch.matmul(e.reshape(bsz, rows, m, L), kern.transpose(-1, -2)[:, None])  # [B, R, m, L]
    pw = rr ** (t + 1)                                # [B, 1, L]
    carry = torch.zeros((bsz, rows, 1), device=e.device, dtype=e.dtype)
    for c in range(m):
        blk = yc[:, :, c, :] + carry * pw
        yc[:, :, c, :] = blk
        carry = blk[:, :, -1:]
    return yc.reshape(bsz, rows, m * L)[..., :n]


def ar1_field(n: int, h: int, w: int, rho, mean=128.0, std=40.0, seed: int = 1, device="cpu",
              noise_uniform: float = 0.0) -> torch.Tensor:
    """uint8 tensor [n, h, w] of AR(1) images (reading A12).

    rho / std may be scalars or length-n sequences (per image, config 2).  noise_uniform>0
    adds continuous U(-a, a) before rounding and clipping (config 3, reading A13).
    """
    dev = torch.device(device)
    g = torch.Generator(device=dev)
    g.manual_seed(int(seed))
    rho_t = torch.as_tensor(np.broadcast_to(np.asarray(rho, dtype=np.float64), (n,)).copy(),
                            dtype=torch.float32, device=dev)
    std_t = torch.as_tensor(np.broadcast_to(np.asarray(std, dtype=np.float64), (n,)).copy(),
                            dtype=torch.float32, device=dev)
    e = torch.randn((n, h + BURN_IN, w + BURN_IN), generator=g, device=dev, dtype=torch.float32)
    y = _ar1_along_last(e, rho_t)                       # along rows (x direction)
    y = _ar1_along_last(y.transpose(1, 2).contiguous(), rho_t).transpose(1, 2)  # along columns
    y = y[:, BURN_IN:, BURN_IN:]
    y = y * (1.0 - rho_t * rho_t)[:, None, None]        # divide by theoretical std 1/(1-rho^2)
    y = y * std_t[:, None, None] + float(mean)
    if noise_uniform > 0.0:
        u = torch.rand((n, h, w), generator=g, device=dev, dtype=torch.float32)
        y = y + (u * 2.0 - 1.0) * float(noise_uniform)
    y = torch.round(torch.clamp(y, 0.0, 255.0))         # torch.round = half to even
    return y.to(torch.uint8).contiguous()


def ar1_stack(n: int, h: int, w: int, rho, mean=128.0, std=40.0, seed: int = 1, device="cpu",
              noise_uniform: float = 0.0, batch: int = 16, lo: int = 0, hi: int | None = None) -> torch.Tensor:
    """Large stacks generated in batches of images (seed + batch start) to bound memory.

    lo/hi select frames [lo, hi) of the n-frame stack without generating the others (batches
    stay aligned to global multiples of `batch`), so a rank's shard of a sharded stack is
    bit-identical to the same frames of the whole stack."""
    hi = n if hi is None else hi
    if not (0 <= lo <= hi <= n):
        raise ValueError("bad frame range")
    out = torch.empty((hi - lo, h, w), dtype=torch.uint8, device=device)
    rho_a = np.broadcast_to(np.asarray(rho, dtype=np.float64), (n,))
    std_a = np.broadcast_to(np.asarray(std, dtype=np.float64), (n,))
    for b0 in range(lo - lo % batch, hi, batch):
        b1 = min(n, b0 + batch)
        f = ar1_field(b1 - b0, h, w, rho_a[b0:b1], mean, std_a[b0:b1], seed * 100003 + b0, device, noise_uniform)
        a, b = max(lo, b0), min(hi, b1)
        out[a - lo:b - lo] = f[a - b0:b - b0]
    return out


def config2_params(n: int = 45, master_seed: int = 2):
    """Per-image (rho, std) of config 2: rho ~ U(0.85, 0.98), std ~ U(25, 60)."""
    rng = np.random.default_rng(master_seed)
    rho = rng.uniform(0.85, 0.98, size=n)
    std = rng.uniform(25.0, 60.0, size=n)
    return rho, std


def yuv420_stack(n_frames: int, height: int = 2160, width: int = 3840, seed: int = 4, device="cpu",
                 batch: int = 8, lo: int = 0, hi: int | None = None):
    """Config 4: luma AR(1) rho=0.95, chroma (half resolution) rho=0.9 (reading A14); frames
    [lo, hi) of the n_frames stack (default: all)."""
    y = ar1_stack(n_frames, height, width, 0.95, 128.0, 40.0, seed, device, batch=batch, lo=lo, hi=hi)
    u = ar1_stack(n_frames, height // 2, width // 2, 0.90, 128.0, 40.0, seed + 1, device, batch=batch, lo=lo, hi=hi)
    v = ar1_stack(n_frames, height // 2, width // 2, 0.90, 128.0, 40.0, seed + 2, device, batch=batch, lo=lo, hi=hi)
    return y, u, v


def laplace_blocks(n_blocks: int, scale: float = 10.0, seed: int = 5, device="cpu") -> torch.Tensor:
    """Config 5: int16 [n_blocks, 8, 8] i.i.d. Laplace(0, scale), rounded half away from zero,
    clipped to +-255 (reading A13)."""
    dev = torch.device(device)
    g = torch.Generator(device=dev)
    g.manual_seed(int(seed))
    u = torch.rand((n_blocks, 8, 8), generator=g, device=dev, dtype=torch.float32)
    u = (u - 0.5).clamp(-0.5 + 1e-7, 0.5 - 1e-7)
    x = -scale * torch.sign(u) * torch.log1p(-2.0 * u.abs())
    x = torch.sign(x) * torch.floor(x.abs() + 0.5)
    return x.clamp(-255, 255).to(torch.int16)


LAPLACE_BATCH = 1 << 22  # blocks per generator batch of the large C5 sweeps


def laplace_range(lo: int, hi: int, scale: float = 10.0, seed: int = 5, device="cpu",
                  out: torch.Tensor | None = None) -> torch.Tensor:
    """Blocks [lo, hi) of the C5 block sequence (int16 [hi - lo, 8, 8]), generated in batches of
    LAPLACE_BATCH blocks (seed + batch index) so that 2^30 blocks (137 GB) need only one batch
    of temporaries and any contiguous shard equals the same blocks of the whole sequence."""
    if not (0 <= lo <= hi):
        raise ValueError("bad block range")
    if out is None:
        out = torch.empty((hi - lo, 8, 8), dtype=torch.int16, device=device)
    B = LAPLACE_BATCH
    for b0 in range(lo - lo % B, hi, B):
        blk = laplace_blocks(B, scale, seed * 1000003 + b0 // B, device)
        a, b = max(lo, b0), min(hi, b0 + B)
        out[a - lo:b - lo] = blk[a - b0:b - b0]
    return out


def uniform_blocks_u8(n_img: int, h: int, w: int, seed: int = 7, device="cpu") -> torch.Tensor:
    """Uniform random u8 images (edge-case and parity inputs)."""
    g = torch.Generator(device=torch.device(device))
    g.manual_seed(int(seed))
    return torch.randint(0, 256, (n_img, h, w), generator=g, device=device, dtype=torch.uint8)
