"""B200-native hot path of arXiv 1808.02950 (angle-based 8-point DCT approximation T1).

    from paper_1808_02950_b200 import adct, catalog
    m = adct.Matrix.from_int(catalog.T1, "T1")
    sse = adct.approx_dct8x8_fused_sse(m, images_u8_cuda, [10])

The product path is libadct.so (CUDA, sm_100a) behind the C-ABI of include/adct.h;
`adct` is its ctypes binding.  Importing `adct` fails loudly if the library is missing.
"""
from . import catalog  # noqa: F401

__all__ = ["adct", "catalog", "parallel"]
