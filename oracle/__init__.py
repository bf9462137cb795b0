"""CPU oracle for the hot path of arXiv 1808.02950 — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / ``--impl reference``
legs may import this package.  The product path (paper_1808_02950_b200/) never imports,
links or executes anything here, and this package never imports the product path.

Contents
  adct_oracle.c  plain by-definition C (int64 / fp64) of forward, S scaling, zig-zag
                 retention, inverse, SSE/PSNR and the C3 quantiser, each citing PAPER.md
  matrices.py    the paper's matrices, typed from PAPER.md
  merit.py       Table 4 / Table 5 figures of merit and the §5.1 factorization (pins)

Parity status: every function here is pinned by tests/test_oracle_*.py against values the
paper prints, closed forms, special cases or brute force (see DESIGN.md §Oracle pins).
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

from . import matrices, merit  # noqa: F401

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "adct_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

CLIP_NONE, CLIP, CLIP_ROUND = 0, 1, 2


def build(force: bool = False) -> str:
    """Compile the C oracle with gcc (OpenMP) into oracle/liboracle.so."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-shared", "-fPIC", "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


_lib = None


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB)
        P, I64, I32, D = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_double
        L.oracle_num_threads.restype = ctypes.c_int
        L.oracle_set_num_threads.argtypes = [ctypes.c_int]
        L.oracle_set_num_threads.restype = None
        L.oracle_zigzag_order.argtypes = [P]
        L.oracle_row_scaling.argtypes = [P, P, P]
        L.oracle_chat_from_int.argtypes = [P, P]
        L.oracle_synthesis_matrix.argtypes = [P, P]
        L.oracle_synthesis_matrix.restype = ctypes.c_int
        L.oracle_forward_int.argtypes = [P, P, ctypes.c_int, I64, I32, I32, P]
        L.oracle_forward_real.argtypes = [P, P, ctypes.c_int, I64, I32, I32, P]
        L.oracle_scale.argtypes = [P, P, I64, P]
        L.oracle_retain_i64.argtypes = [P, I64, I32]
        L.oracle_retain_f64.argtypes = [P, I64, I32]
        L.oracle_inverse.argtypes = [P, P, I64, P]
        L.oracle_sse.argtypes = [P, ctypes.c_int, P, I64, I32, I32, ctypes.c_int, P]
        L.oracle_psnr.argtypes = [D, I64, D]
        L.oracle_psnr.restype = D
        L.oracle_quantize.argtypes = [P, P, I32, I64, P]
        L.oracle_codec_sse.argtypes = [P, P, P, ctypes.c_int, I64, I32, I32, P, I32, ctypes.c_int, P]
        for name in ("oracle_forward_int", "oracle_forward_real", "oracle_retain_i64", "oracle_retain_f64",
                     "oracle_sse", "oracle_codec_sse"):
            getattr(L, name).restype = ctypes.c_int
        _lib = L
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def _bits(img: np.ndarray) -> int:
    if img.dtype == np.uint8:
        return 8
    if img.dtype == np.int16:
        return 16
    raise TypeError("samples must be uint8 or int16")


def _img3(img: np.ndarray) -> np.ndarray:
    img = np.ascontiguousarray(img)
    return img[None] if img.ndim == 2 else img


def num_threads() -> int:
    return int(lib().oracle_num_threads())


def set_num_threads(n: int) -> None:
    """OpenMP threads of later oracle calls (timing only; results are thread-count independent)."""
    lib().oracle_set_num_threads(int(n))


def zigzag_order() -> np.ndarray:
    o = np.zeros(64, dtype=np.int32)
    lib().oracle_zigzag_order(_p(o))
    return o


def row_scaling(t: np.ndarray):
    t = np.ascontiguousarray(t, dtype=np.int32)
    n = np.zeros(8, dtype=np.int64)
    s = np.zeros(8, dtype=np.float64)
    lib().oracle_row_scaling(_p(t), _p(n), _p(s))
    return n, s


def chat_from_int(t: np.ndarray) -> np.ndarray:
    t = np.ascontiguousarray(t, dtype=np.int32)
    c = np.zeros(64, dtype=np.float64)
    lib().oracle_chat_from_int(_p(t), _p(c))
    return c.reshape(8, 8)


def synthesis_matrix(chat: np.ndarray):
    """(G, kind) with kind 1 = transpose (orthonormal), 0 = true inverse."""
    chat = np.ascontiguousarray(chat, dtype=np.float64)
    g = np.zeros(64, dtype=np.float64)
    kind = lib().oracle_synthesis_matrix(_p(chat), _p(g))
    if kind < 0:
        raise ValueError("singular C_hat")
    return g.reshape(8, 8), kind


def forward_int(t: np.ndarray, img: np.ndarray) -> np.ndarray:
    """Y = T X T^T per block, int64, block-major [n_img, H/8, W/8, 8, 8]."""
    t = np.ascontiguousarray(t, dtype=np.int32)
    x = _img3(img)
    n, h, w = x.shape
    y = np.zeros((n, h // 8, w // 8, 8, 8), dtype=np.int64)
    if lib().oracle_forward_int(_p(t), _p(x), _bits(x), n, h, w, _p(y)) != 0:
        raise ValueError("bad geometry")
    return y


def forward_real(c: np.ndarray, img: np.ndarray) -> np.ndarray:
    c = np.ascontiguousarray(c, dtype=np.float64)
    x = _img3(img)
    n, h, w = x.shape
    b = np.zeros((n, h // 8, w // 8, 8, 8), dtype=np.float64)
    if lib().oracle_forward_real(_p(c), _p(x), _bits(x), n, h, w, _p(b)) != 0:
        raise ValueError("bad geometry")
    return b


def scale(y: np.ndarray, s: np.ndarray) -> np.ndarray:
    y = np.ascontiguousarray(y, dtype=np.int64)
    s = np.ascontiguousarray(s, dtype=np.float64)
    out = np.zeros(y.shape, dtype=np.float64)
    lib().oracle_scale(_p(y), _p(s), y.size // 64, _p(out))
    return out


def retain(coef: np.ndarray, r: int) -> np.ndarray:
    out = np.array(coef, copy=True, order="C")
    if out.dtype == np.int64:
        rc = lib().oracle_retain_i64(_p(out), out.size // 64, r)
    elif out.dtype == np.float64:
        rc = lib().oracle_retain_f64(_p(out), out.size // 64, r)
    else:
        raise TypeError("int64 or float64 coefficients")
    if rc != 0:
        raise ValueError("r must be in 1..64")
    return out


def inverse(g: np.ndarray, bp: np.ndarray) -> np.ndarray:
    g = np.ascontiguousarray(g, dtype=np.float64)
    bp = np.ascontiguousarray(bp, dtype=np.float64)
    a = np.zeros(bp.shape, dtype=np.float64)
    lib().oracle_inverse(_p(g), _p(bp), bp.size // 64, _p(a))
    return a


def sse(orig: np.ndarray, recon_blocks: np.ndarray, clip: int = CLIP_NONE) -> np.ndarray:
    x = _img3(orig)
    n, h, w = x.shape
    r = np.ascontiguousarray(recon_blocks, dtype=np.float64)
    out = np.zeros(n, dtype=np.float64)
    if lib().oracle_sse(_p(x), _bits(x), _p(r), n, h, w, clip, _p(out)) != 0:
        raise ValueError("bad geometry")
    return out


def psnr(sse_value: float, n_pixels: int, peak: float = 255.0) -> float:
    return float(lib().oracle_psnr(float(sse_value), int(n_pixels), float(peak)))


def quantize(y: np.ndarray, n: np.ndarray, step: int = 16) -> np.ndarray:
    y = np.ascontiguousarray(y, dtype=np.int64)
    n = np.ascontiguousarray(n, dtype=np.int64)
    q = np.zeros(y.shape, dtype=np.int16)
    lib().oracle_quantize(_p(y), _p(n), step, y.size // 64, _p(q))
    return q


def codec_sse(img: np.ndarray, r_list, t: np.ndarray | None = None, c: np.ndarray | None = None,
              clip: int = CLIP_NONE) -> np.ndarray:
    """SSE[n_img, n_r] of forward -> retain r -> inverse -> clip, per image (§6.1)."""
    x = _img3(img)
    n, h, w = x.shape
    r = np.ascontiguousarray(r_list, dtype=np.int32)
    out = np.zeros((n, len(r)), dtype=np.float64)
    if t is None and c is None:
        raise ValueError("need t or c")
    tkeep = np.ascontiguousarray(t, dtype=np.int32) if t is not None else None
    ckeep = np.ascontiguousarray(c, dtype=np.float64) if c is not None else None
    tp = _p(tkeep) if tkeep is not None else None
    cp = _p(ckeep) if ckeep is not None else None
    rc = lib().oracle_codec_sse(tp, cp, _p(x), _bits(x), n, h, w, _p(r), len(r), clip, _p(out))
    if rc != 0:
        raise ValueError(f"oracle_codec_sse failed ({rc})")
    return out
