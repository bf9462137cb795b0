"""Thin Python binding of the C-ABI in include/adct.h (argument marshalling only).

Every step of the method runs in libadct.so's CUDA kernels; this module converts torch
tensors / numpy arrays into pointers, geometries and status checks.  It never computes
any part of the transform itself and there is no CPU fallback: if the library is missing
the import fails loudly.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
# ADCT_LIB may name another in-tree build of the same library (kernel A/B runs in tools/gpu)
LIB_PATH = os.environ.get("ADCT_LIB") or os.path.join(_HERE, "libadct.so")

U8, I16, I32, F32 = 0, 1, 2, 3
CLIP_NONE, CLIP, CLIP_ROUND = 0, 1, 2

_STATUS = {0: "ok", 1: "invalid argument", 2: "unsupported matrix", 3: "singular", 4: "overflow",
           5: "alignment", 6: "CUDA error", 7: "workspace"}

SYMBOLS = [
    "adct_matrix_create_int", "adct_matrix_create_real", "adct_matrix_info", "adct_matrix_destroy",
    "adct_zigzag_order", "approx_dct8x8_fwd", "zonal_retain", "approx_dct8x8_inv", "psnr_reduce",
    "approx_dct8x8_fused_sse", "adct_host_workspace_bytes", "approx_dct8x8_fused_sse_host",
    "approx_dct8x8_fwd_quant", "adct_workspace_bytes", "adct_status_str", "adct_launch_count",
    "approx_dct8x8_roundtrip", "ssim_reduce", "approx_dct_jam_roundtrip", "adct_greedy_workspace_bytes",
    "adct_greedy_search", "adct_merit_batch", "adct_matrix_chat", "adct_planes_workspace_bytes",
    "approx_dct8x8_fused_sse_planes", "approx_dct8x8_ssim",
]


class AdctError(RuntimeError):
    def __init__(self, status: int, what: str):
        super().__init__(f"{what}: {_STATUS.get(status, status)} ({status})")
        self.status = status


class Geom(ctypes.Structure):
    _fields_ = [("n_images", ctypes.c_int64), ("height", ctypes.c_int32), ("width", ctypes.c_int32),
                ("image_stride", ctypes.c_int64), ("row_stride", ctypes.c_int64)]


def _load() -> ctypes.CDLL:
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} not built (run ./build.sh or __graft_entry__.build()); "
                          "there is no CPU fallback")
    L = ctypes.CDLL(LIB_PATH)
    P, I32_, I64_, D = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_double
    S = ctypes.c_int
    L.adct_matrix_create_int.argtypes = [P, ctypes.POINTER(P)]
    L.adct_matrix_create_real.argtypes = [P, ctypes.POINTER(P)]
    L.adct_matrix_info.argtypes = [P, P, P, P, P, P, P, P]
    L.adct_matrix_destroy.argtypes = [P]
    L.adct_matrix_destroy.restype = None
    L.adct_zigzag_order.argtypes = [P]
    L.approx_dct8x8_fwd.argtypes = [P, P, S, Geom, P, S, P]
    L.zonal_retain.argtypes = [P, S, I64_, I32_, P]
    L.approx_dct8x8_inv.argtypes = [P, P, S, Geom, P, S, S, P]
    L.psnr_reduce.argtypes = [P, S, P, S, Geom, D, S, P, P, P, ctypes.c_size_t, P]
    L.approx_dct8x8_fused_sse.argtypes = [P, P, S, Geom, P, I32_, S, P, P, P, ctypes.c_size_t, P]
    if hasattr(L, "adct_planes_workspace_bytes") or not os.environ.get("ADCT_LIB"):  # A/B builds may predate it
        L.adct_planes_workspace_bytes.argtypes = [I32_, P]
        L.adct_planes_workspace_bytes.restype = ctypes.c_size_t
        L.approx_dct8x8_fused_sse_planes.argtypes = [P, I32_, P, S, P, I32_, S, P, P, P, ctypes.c_size_t, P]
    if hasattr(L, "approx_dct8x8_ssim") or not os.environ.get("ADCT_LIB"):
        L.approx_dct8x8_ssim.argtypes = [P, P, Geom, I32_, S, P, P, ctypes.c_size_t, P]
    L.adct_host_workspace_bytes.argtypes = [Geom, I32_, I64_, S]
    L.adct_host_workspace_bytes.restype = ctypes.c_size_t
    L.approx_dct8x8_fused_sse_host.argtypes = [P, P, S, Geom, P, I32_, S, P, P, I64_, P, ctypes.c_size_t, P]
    L.approx_dct8x8_fwd_quant.argtypes = [P, P, Geom, I32_, P, P]
    L.approx_dct8x8_roundtrip.argtypes = [P, P, S, Geom, I32_, P, S, S, P]
    L.ssim_reduce.argtypes = [P, S, P, S, Geom, D, S, P, P, ctypes.c_size_t, P]
    L.approx_dct_jam_roundtrip.argtypes = [I32_, P, S, Geom, I32_, P, S, S, P]
    L.adct_greedy_workspace_bytes.argtypes = [I32_]
    L.adct_greedy_workspace_bytes.restype = ctypes.c_size_t
    L.adct_merit_batch.argtypes = [P, P, P, I32_, P, I32_, P, P]
    L.adct_matrix_chat.argtypes = [P, P]
    L.adct_greedy_search.argtypes = [P, P, I32_, P, ctypes.c_uint32, P, I32_, P, P, P, P, ctypes.c_size_t, P]
    L.adct_workspace_bytes.argtypes = [Geom, I32_]
    L.adct_workspace_bytes.restype = ctypes.c_size_t
    L.adct_status_str.argtypes = [S]
    L.adct_status_str.restype = ctypes.c_char_p
    L.adct_launch_count.argtypes = []
    L.adct_launch_count.restype = I64_
    for name in SYMBOLS:
        if os.environ.get("ADCT_LIB") and not hasattr(L, name):
            continue
        fn = getattr(L, name)
        if name not in ("adct_matrix_destroy", "adct_host_workspace_bytes", "adct_workspace_bytes",
                        "adct_planes_workspace_bytes",
                        "adct_status_str", "adct_launch_count", "adct_greedy_workspace_bytes"):
            fn.restype = S
    return L


lib = _load()


def _check(status: int, what: str) -> None:
    if status != 0:
        raise AdctError(status, what)


_TORCH_DT = {torch.uint8: U8, torch.int16: I16, torch.int32: I32, torch.float32: F32}
_DT_TORCH = {v: k for k, v in _TORCH_DT.items()}


def dtype_code(t: torch.Tensor) -> int:
    try:
        return _TORCH_DT[t.dtype]
    except KeyError:
        raise TypeError(f"unsupported dtype {t.dtype}") from None


def geom_of(img: torch.Tensor) -> Geom:
    """Geometry of an image stack [n, H, W] (or [H, W]) from its strides (elements)."""
    if img.dim() == 2:
        img = img.unsqueeze(0)
    if img.dim() != 3 or img.stride(2) != 1:
        raise ValueError("images must be [n, H, W] with unit column stride")
    n, h, w = img.shape
    return Geom(n, h, w, img.stride(0) if n > 1 else h * img.stride(1), img.stride(1))


def _stream_ptr(stream) -> int | None:
    if stream is None:
        return torch.cuda.current_stream().cuda_stream if torch.cuda.is_available() else None
    return stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream)


def _out(t: torch.Tensor, numel: int, like: torch.Tensor, name: str, dtype=None, host: bool = False) -> torch.Tensor:
    """A caller-provided output tensor: the library writes `numel` contiguous elements through its
    data pointer, so the dtype, contiguity, size and device are checked before any launch."""
    if dtype is not None and t.dtype != dtype:
        raise ValueError(f"{name} must be {dtype}, got {t.dtype}")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")
    if t.numel() < numel:
        raise ValueError(f"{name} holds {t.numel()} elements, {numel} needed")
    want = torch.device("cpu") if host else like.device
    if t.device != want:
        raise ValueError(f"{name} must be on {want}, got {t.device}")
    return t


def _ptr(t) -> int | None:
    return None if t is None else t.data_ptr()


@dataclass
class MatrixInfo:
    s: list
    g: list
    row_orthogonal: bool
    is_integer: bool
    max_abs_y_u8: int
    max_abs_y_i16: int
    specialized: bool


class Matrix:
    """A matrix descriptor (adct_matrix_create_int / adct_matrix_create_real)."""

    def __init__(self, handle: int, name: str = ""):
        self._h = ctypes.c_void_p(handle)
        self.name = name

    @classmethod
    def from_int(cls, t, name: str = "") -> "Matrix":
        arr = (ctypes.c_int32 * 64)(*[int(v) for v in list(t)])
        h = ctypes.c_void_p()
        _check(lib.adct_matrix_create_int(ctypes.cast(arr, ctypes.c_void_p), ctypes.byref(h)), "adct_matrix_create_int")
        return cls(h.value, name)

    @classmethod
    def from_real(cls, c, name: str = "") -> "Matrix":
        arr = (ctypes.c_double * 64)(*[float(v) for v in list(c)])
        h = ctypes.c_void_p()
        _check(lib.adct_matrix_create_real(ctypes.cast(arr, ctypes.c_void_p), ctypes.byref(h)), "adct_matrix_create_real")
        return cls(h.value, name)

    @property
    def handle(self) -> ctypes.c_void_p:
        if not self._h:
            raise ValueError("matrix destroyed")
        return self._h

    def info(self) -> MatrixInfo:
        s = (ctypes.c_double * 8)()
        g = (ctypes.c_double * 64)()
        ro, ii, sp = ctypes.c_int32(), ctypes.c_int32(), ctypes.c_int32()
        mu, mi = ctypes.c_int64(), ctypes.c_int64()
        _check(lib.adct_matrix_info(self.handle, ctypes.cast(s, ctypes.c_void_p), ctypes.cast(g, ctypes.c_void_p),
                                    ctypes.byref(ro), ctypes.byref(ii), ctypes.byref(mu), ctypes.byref(mi),
                                    ctypes.byref(sp)), "adct_matrix_info")
        return MatrixInfo(list(s), list(g), bool(ro.value), bool(ii.value), mu.value, mi.value, bool(sp.value))

    def chat(self) -> list:
        c = (ctypes.c_double * 64)()
        _check(lib.adct_matrix_chat(self.handle, ctypes.cast(c, ctypes.c_void_p)), "adct_matrix_chat")
        return list(c)

    def close(self) -> None:
        if self._h:
            lib.adct_matrix_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def zigzag_order() -> list:
    o = (ctypes.c_int32 * 64)()
    _check(lib.adct_zigzag_order(ctypes.cast(o, ctypes.c_void_p)), "adct_zigzag_order")
    return list(o)


def workspace_bytes(geom: Geom, n_r: int) -> int:
    return int(lib.adct_workspace_bytes(geom, n_r))


def launch_count() -> int:
    return int(lib.adct_launch_count())


# ---- the four calls -------------------------------------------------------------------------

def approx_dct8x8_fwd(m: Matrix, src: torch.Tensor, coef_dtype=torch.int32, coef: torch.Tensor | None = None,
                      stream=None) -> torch.Tensor:
    """Block-major coefficients [n, H/8, W/8, 8, 8] of every 8x8 block of src [n, H, W]."""
    g = geom_of(src)
    if coef is None:
        coef = torch.empty((g.n_images, g.height // 8, g.width // 8, 8, 8), dtype=coef_dtype, device=src.device)
    _out(coef, g.n_images * g.height * g.width, src, "coef")
    _check(lib.approx_dct8x8_fwd(m.handle, src.data_ptr(), dtype_code(src), g, coef.data_ptr(), dtype_code(coef),
                                 _stream_ptr(stream)), "approx_dct8x8_fwd")
    return coef


def zonal_retain(coef: torch.Tensor, r: int, stream=None) -> torch.Tensor:
    """Zero, in place, every coefficient at zig-zag position >= r."""
    if not coef.is_contiguous():
        raise ValueError("coefficients must be contiguous block-major")
    _check(lib.zonal_retain(coef.data_ptr(), dtype_code(coef), coef.numel() // 64, int(r), _stream_ptr(stream)),
           "zonal_retain")
    return coef


def approx_dct8x8_inv(m: Matrix, coef: torch.Tensor, height: int, width: int, recon_dtype=torch.float32,
                      clip: int = CLIP_NONE, recon: torch.Tensor | None = None, stream=None) -> torch.Tensor:
    n = coef.numel() // (height * width)
    if recon is None:
        recon = torch.empty((n, height, width), dtype=recon_dtype, device=coef.device)
    g = geom_of(recon)
    if not coef.is_contiguous() or coef.numel() < g.n_images * g.height * g.width or coef.device != recon.device:
        raise ValueError("coef must be contiguous block-major [n, H/8, W/8, 8, 8] on recon's device")
    _check(lib.approx_dct8x8_inv(m.handle, coef.data_ptr(), dtype_code(coef), g, recon.data_ptr(),
                                 dtype_code(recon), int(clip), _stream_ptr(stream)), "approx_dct8x8_inv")
    return recon


def psnr_reduce(orig: torch.Tensor, recon: torch.Tensor, peak: float = 255.0, clip: int = CLIP_NONE,
                workspace: torch.Tensor | None = None, stream=None):
    """(sse, psnr) fp64 per image."""
    g = geom_of(orig)
    gr = geom_of(recon)
    if (gr.n_images, gr.height, gr.width, gr.row_stride) != (g.n_images, g.height, g.width, g.row_stride):
        raise ValueError("orig and recon must share the geometry (strides in elements)")
    sse = torch.empty(g.n_images, dtype=torch.float64, device=orig.device)
    psnr = torch.empty(g.n_images, dtype=torch.float64, device=orig.device)
    nbytes = workspace_bytes(g, 1)
    if workspace is None or workspace.numel() < nbytes:
        workspace = torch.empty(nbytes, dtype=torch.uint8, device=orig.device)
    _check(lib.psnr_reduce(orig.data_ptr(), dtype_code(orig), recon.data_ptr(), dtype_code(recon), g, float(peak),
                           int(clip), sse.data_ptr(), psnr.data_ptr(), workspace.data_ptr(), workspace.numel(),
                           _stream_ptr(stream)), "psnr_reduce")
    return sse, psnr


def approx_dct_jam_roundtrip(n: int, src: torch.Tensor, r: int, recon_dtype=torch.float32, clip: int | None = None,
                             recon: torch.Tensor | None = None, stream=None) -> torch.Tensor:
    """n x n (n = 16, 32) JAM-scaled T1 round trip of every block of src [N, H, W] (§6.2)."""
    if clip is None:
        clip = CLIP_ROUND if recon_dtype in (torch.int16, torch.uint8) else CLIP_NONE
    g = geom_of(src)
    if recon is None:
        recon = torch.empty_strided(tuple(src.shape), src.stride(), dtype=recon_dtype, device=src.device)
    if tuple(recon.stride()) != tuple(src.stride()) or tuple(recon.shape) != tuple(src.shape):
        raise ValueError("recon must have the shape and strides of src")
    if recon.device != src.device:
        raise ValueError("recon must be on src's device")
    _check(lib.approx_dct_jam_roundtrip(int(n), src.data_ptr(), dtype_code(src), g, int(r), recon.data_ptr(),
                                        dtype_code(recon), int(clip), _stream_ptr(stream)), "approx_dct_jam_roundtrip")
    return recon


def greedy_search(c, entries, orders, fixed: dict | None = None, device=None, workspace=None, stream=None,
                  return_ties: bool = False):
    """Greedy angle search (§3, Fig. 2) for every sequence in `orders` ([n, n_free] row indices):
    returns (matrices int32 [n, 8, 8], status int32 [n]) on `device`, plus with return_ties=True
    the exact ties met, int32 [n, 4] = (steps with a tie, first tied row or -1, candidates tied
    there, largest tie) -- see adct_greedy_search in include/adct.h."""
    import numpy as _np
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    c64 = _np.ascontiguousarray(_np.asarray(c, dtype=_np.float64).reshape(64))
    ent = _np.ascontiguousarray(_np.asarray(entries, dtype=_np.int32))
    fx = _np.zeros(64, dtype=_np.int32)
    mask = 0
    for k, row in (fixed or {}).items():
        fx[8 * k:8 * k + 8] = row
        mask |= 1 << int(k)
    od = torch.as_tensor(_np.ascontiguousarray(_np.asarray(orders, dtype=_np.int32)), device=dev)
    n = od.shape[0]
    out = torch.empty((n, 8, 8), dtype=torch.int32, device=dev)
    status = torch.empty(n, dtype=torch.int32, device=dev)
    ties = torch.empty((n, 4), dtype=torch.int32, device=dev) if return_ties else None
    nbytes = lib.adct_greedy_workspace_bytes(len(ent))
    if workspace is None or workspace.numel() < nbytes:
        workspace = torch.empty(nbytes, dtype=torch.uint8, device=dev)
    _check(lib.adct_greedy_search(c64.ctypes.data, ent.ctypes.data, len(ent), fx.ctypes.data, mask, od.data_ptr(), n,
                                  out.data_ptr(), status.data_ptr(), _ptr(ties), workspace.data_ptr(),
                                  workspace.numel(), _stream_ptr(stream)), "adct_greedy_search")
    return (out, status, ties) if return_ties else (out, status)


def merit_batch(mats: list, rho: torch.Tensor, c_exact=None, stream=None) -> torch.Tensor:
    """Figures of merit (eps, MSE, C*_g, eta) of §4.2 for every (descriptor, rho): C_hat and its
    inverse come from the descriptors (adct_matrix_chat, adct_matrix_info's G); rho fp64 [m] on
    the device; returns fp64 [n, m, 4]."""
    import numpy as _np
    from . import catalog as _cat
    c = _np.ascontiguousarray(_np.asarray(c_exact if c_exact is not None else _cat.exact_dct(), dtype=_np.float64))
    dev = rho.device
    chat = torch.tensor([m.chat() for m in mats], dtype=torch.float64, device=dev)
    ginv = torch.tensor([m.info().g for m in mats], dtype=torch.float64, device=dev)
    rho = rho.contiguous().to(torch.float64)
    out = torch.empty((chat.shape[0], rho.numel(), 4), dtype=torch.float64, device=chat.device)
    _check(lib.adct_merit_batch(c.ctypes.data, chat.data_ptr(), ginv.data_ptr(), chat.shape[0], rho.data_ptr(),
                                rho.numel(), out.data_ptr(), _stream_ptr(stream)), "adct_merit_batch")
    return out


def ssim_reduce(orig: torch.Tensor, recon: torch.Tensor, peak: float = 255.0, clip: int = CLIP_NONE,
                workspace: torch.Tensor | None = None, stream=None) -> torch.Tensor:
    """Mean SSIM (8x8 uniform windows, reading A18) per image, fp64 [n]."""
    g = geom_of(orig)
    gr = geom_of(recon)
    if (gr.n_images, gr.height, gr.width, gr.row_stride) != (g.n_images, g.height, g.width, g.row_stride):
        raise ValueError("orig and recon must share the geometry (strides in elements)")
    out = torch.empty(g.n_images, dtype=torch.float64, device=orig.device)
    nbytes = workspace_bytes(g, 1)
    if workspace is None or workspace.numel() < nbytes:
        workspace = torch.empty(nbytes, dtype=torch.uint8, device=orig.device)
    _check(lib.ssim_reduce(orig.data_ptr(), dtype_code(orig), recon.data_ptr(), dtype_code(recon), g, float(peak),
                           int(clip), out.data_ptr(), workspace.data_ptr(), workspace.numel(), _stream_ptr(stream)),
           "ssim_reduce")
    return out


# ---- fused paths ------------------------------------------------------------------------------

def approx_dct8x8_roundtrip(m: Matrix, src: torch.Tensor, r: int = 64, recon_dtype=torch.int16,
                            clip: int | None = None, recon: torch.Tensor | None = None, stream=None) -> torch.Tensor:
    """Forward -> retain r -> inverse of every block of src [n, H, W] in one pass; the
    reconstruction has src's shape and strides (int16/uint8: rounded and saturated)."""
    if clip is None:
        clip = CLIP_ROUND if recon_dtype in (torch.int16, torch.uint8) else CLIP_NONE
    g = geom_of(src)
    if recon is None:
        recon = torch.empty_strided(tuple(src.shape[-3:]) if src.dim() == 3 else tuple(src.shape),
                                    src.stride(), dtype=recon_dtype, device=src.device)
    if tuple(recon.stride()) != tuple(src.stride()) or tuple(recon.shape) != tuple(src.shape):
        raise ValueError("recon must have the shape and strides of src")
    if recon.device != src.device:
        raise ValueError("recon must be on src's device")
    _check(lib.approx_dct8x8_roundtrip(m.handle, src.data_ptr(), dtype_code(src), g, int(r), recon.data_ptr(),
                                       dtype_code(recon), int(clip), _stream_ptr(stream)),
           "approx_dct8x8_roundtrip")
    return recon


def approx_dct8x8_fused_sse(m: Matrix, src: torch.Tensor, r_list, clip: int = CLIP_NONE,
                            workspace: torch.Tensor | None = None, sse: torch.Tensor | None = None,
                            stream=None, psnr: torch.Tensor | None = None, return_psnr: bool = False):
    """SSE [n, len(r_list)] (fp64, device) of forward -> retain r -> inverse per image; with
    `psnr` (an output tensor) or return_psnr=True also the library's PSNR: returns (sse, psnr)."""
    g = geom_of(src)
    rl = [int(r) for r in r_list]
    arr = (ctypes.c_int32 * len(rl))(*rl)
    if sse is None:
        sse = torch.empty((g.n_images, len(rl)), dtype=torch.float64, device=src.device)
    _out(sse, g.n_images * len(rl), src, "sse", dtype=torch.float64)
    want_psnr = return_psnr or psnr is not None
    if want_psnr and psnr is None:
        psnr = torch.empty((g.n_images, len(rl)), dtype=torch.float64, device=src.device)
    if want_psnr:
        _out(psnr, g.n_images * len(rl), src, "psnr", dtype=torch.float64)
    nbytes = workspace_bytes(g, len(rl))
    if workspace is None or workspace.numel() < nbytes:
        workspace = torch.empty(nbytes, dtype=torch.uint8, device=src.device)
    _check(lib.approx_dct8x8_fused_sse(m.handle, src.data_ptr(), dtype_code(src), g,
                                       ctypes.cast(arr, ctypes.c_void_p), len(rl), int(clip), sse.data_ptr(),
                                       psnr.data_ptr() if want_psnr else None, workspace.data_ptr(),
                                       workspace.numel(), _stream_ptr(stream)),
           "approx_dct8x8_fused_sse")
    return (sse, psnr) if want_psnr else sse


MAX_PLANES = 3


def planes_workspace_bytes(geoms) -> int:
    arr = (Geom * len(geoms))(*geoms)
    return int(lib.adct_planes_workspace_bytes(len(geoms), ctypes.cast(arr, ctypes.c_void_p)))


def approx_dct8x8_fused_sse_planes(m: Matrix, planes, r: int, clip: int = CLIP_NONE, sse=None, psnr=None,
                                   workspace: torch.Tensor | None = None, stream=None):
    """The planes of one stack (e.g. Y, U, V) in one call: per plane SSE and PSNR [n] (fp64, device).
    `sse` / `psnr`: optional lists of output tensors (a psnr entry may be None).  Returns (sse, psnr)."""
    n = len(planes)
    if not 1 <= n <= MAX_PLANES:
        raise ValueError(f"1..{MAX_PLANES} planes")
    geoms = [geom_of(p) for p in planes]
    dt = dtype_code(planes[0])
    if any(dtype_code(p) != dt or p.device != planes[0].device for p in planes):
        raise ValueError("planes must share dtype and device")
    dev = planes[0].device
    if sse is None:
        sse = [torch.empty(g.n_images, dtype=torch.float64, device=dev) for g in geoms]
    if psnr is None:
        psnr = [torch.empty(g.n_images, dtype=torch.float64, device=dev) for g in geoms]
    for i, g in enumerate(geoms):
        _out(sse[i], g.n_images, planes[i], "sse", dtype=torch.float64)
        if psnr[i] is not None:
            _out(psnr[i], g.n_images, planes[i], "psnr", dtype=torch.float64)
    nbytes = planes_workspace_bytes(geoms)
    if workspace is None or workspace.numel() < nbytes:
        workspace = torch.empty(nbytes, dtype=torch.uint8, device=dev)
    P = ctypes.c_void_p
    srcs = (P * n)(*[p.data_ptr() for p in planes])
    garr = (Geom * n)(*geoms)
    sarr = (P * n)(*[t.data_ptr() for t in sse])
    parr = (P * n)(*[(t.data_ptr() if t is not None else None) for t in psnr])
    _check(lib.approx_dct8x8_fused_sse_planes(m.handle, n, ctypes.cast(srcs, P), dt, ctypes.cast(garr, P), int(r),
                                              int(clip), ctypes.cast(sarr, P), ctypes.cast(parr, P),
                                              workspace.data_ptr(), workspace.numel(), _stream_ptr(stream)),
           "approx_dct8x8_fused_sse_planes")
    return sse, psnr


def host_workspace_bytes(geom: Geom, n_r: int, chunk_images: int, src_dtype: int = U8) -> int:
    return int(lib.adct_host_workspace_bytes(geom, n_r, chunk_images, src_dtype))


def approx_dct8x8_fused_sse_host(m: Matrix, src_host: torch.Tensor, r_list, workspace: torch.Tensor,
                                 chunk_images: int, clip: int = CLIP_NONE, sse_host: torch.Tensor | None = None,
                                 stream=None, psnr_host: torch.Tensor | None = None, return_psnr: bool = False):
    """The fused path on a HOST image stack (pinned); returns host SSE [n, n_r], or (sse, psnr)
    with `psnr_host` / return_psnr=True."""
    g = geom_of(src_host)
    rl = [int(r) for r in r_list]
    arr = (ctypes.c_int32 * len(rl))(*rl)
    if sse_host is None:
        sse_host = torch.empty((g.n_images, len(rl)), dtype=torch.float64)
    _out(sse_host, g.n_images * len(rl), src_host, "sse_host", dtype=torch.float64, host=True)
    want_psnr = return_psnr or psnr_host is not None
    if want_psnr and psnr_host is None:
        psnr_host = torch.empty((g.n_images, len(rl)), dtype=torch.float64)
    if want_psnr:
        _out(psnr_host, g.n_images * len(rl), src_host, "psnr_host", dtype=torch.float64, host=True)
    _check(lib.approx_dct8x8_fused_sse_host(m.handle, src_host.data_ptr(), dtype_code(src_host), g,
                                            ctypes.cast(arr, ctypes.c_void_p), len(rl), int(clip),
                                            sse_host.data_ptr(), psnr_host.data_ptr() if want_psnr else None,
                                            int(chunk_images), workspace.data_ptr(), workspace.numel(),
                                            _stream_ptr(stream)), "approx_dct8x8_fused_sse_host")
    return (sse_host, psnr_host) if want_psnr else sse_host


def approx_dct8x8_ssim(m: Matrix, src: torch.Tensor, r: int, clip: int = CLIP, ssim: torch.Tensor | None = None,
                       workspace: torch.Tensor | None = None, stream=None) -> torch.Tensor:
    """Forward -> retain r -> inverse -> SSIM per image (fp64 [n], device) in one pass over the u8
    images; equals ssim_reduce(src, approx_dct8x8_roundtrip(m, src, r, float32), clip=clip)."""
    g = geom_of(src)
    if ssim is None:
        ssim = torch.empty(g.n_images, dtype=torch.float64, device=src.device)
    _out(ssim, g.n_images, src, "ssim", dtype=torch.float64)
    nbytes = workspace_bytes(g, 1)
    if workspace is None or workspace.numel() < nbytes:
        workspace = torch.empty(nbytes, dtype=torch.uint8, device=src.device)
    _check(lib.approx_dct8x8_ssim(m.handle, src.data_ptr(), g, int(r), int(clip), ssim.data_ptr(),
                                  workspace.data_ptr(), workspace.numel(), _stream_ptr(stream)), "approx_dct8x8_ssim")
    return ssim


def approx_dct8x8_fwd_quant(m: Matrix, src: torch.Tensor, step: int = 16, q: torch.Tensor | None = None,
                            stream=None) -> torch.Tensor:
    g = geom_of(src)
    if q is None:
        q = torch.empty((g.n_images, g.height // 8, g.width // 8, 8, 8), dtype=torch.int16, device=src.device)
    _out(q, g.n_images * g.height * g.width, src, "q", dtype=torch.int16)
    _check(lib.approx_dct8x8_fwd_quant(m.handle, src.data_ptr(), g, int(step), q.data_ptr(), _stream_ptr(stream)),
           "approx_dct8x8_fwd_quant")
    return q
