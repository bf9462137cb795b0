"""Every kernel of libadct.so once on small inputs (for compute-sanitizer runs on the GPU box)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_1808_02950_b200 import adct, catalog  # noqa: E402

dev = torch.device("cuda:0")
t1 = adct.Matrix.from_int(catalog.T1, "T1")
t6 = adct.Matrix.from_int(catalog.INTEGER["T6"], "T6")
dct = adct.Matrix.from_real(catalog.exact_dct(), "DCT")
img = synth.ar1_field(2, 48, 272, 0.95, seed=1).to(dev)         # wtile path, ragged slices
odd = synth.ar1_field(2, 40, 56, 0.95, seed=2).to(dev)          # generic fused kernels
for m in (t1, t6):
    adct.approx_dct8x8_fused_sse(m, img, [10])
    adct.approx_dct8x8_fused_sse(m, odd, [10])
    adct.approx_dct8x8_fused_sse(m, img, [1, 3, 10, 36, 64])
    adct.approx_dct8x8_fused_sse(m, img, [10], clip=adct.CLIP)
y = adct.approx_dct8x8_fwd(t1, img, torch.int32)
adct.zonal_retain(y, 10)
rec = adct.approx_dct8x8_inv(t1, y, 48, 272)
adct.psnr_reduce(img, rec)
adct.ssim_reduce(img, rec, clip=adct.CLIP)
adct.approx_dct8x8_fwd_quant(t1, img, 16)
adct.approx_dct8x8_fwd_quant(t6, img, 16)
x16 = synth.laplace_blocks(4096, seed=5, device=dev).reshape(4096, 8, 8)
for m in (t1, dct):
    adct.approx_dct8x8_roundtrip(m, x16, 64, torch.int16)
    adct.approx_dct8x8_roundtrip(m, x16, 10, torch.float32)
adct.approx_dct8x8_roundtrip(t1, img, 10, torch.uint8)
for n in (16, 32):
    adct.approx_dct_jam_roundtrip(n, synth.laplace_blocks(64 * (n // 8) ** 2, seed=3, device=dev).reshape(-1, n, n),
                                  n * n, torch.int16)
import itertools  # noqa: E402
adct.greedy_search(np.array(catalog.exact_dct()).reshape(8, 8), catalog.P1,
                   np.array(list(itertools.permutations([1, 2, 3, 5, 6, 7]))[:16], dtype=np.int32),
                   fixed=catalog.GREEDY_FIXED_ROWS, device=dev)
adct.merit_batch([t1, dct], torch.tensor([0.5, 0.95], dtype=torch.float64, device=dev))
host = img.cpu().pin_memory()
ws = torch.empty(adct.host_workspace_bytes(adct.geom_of(host), 1, 1), dtype=torch.uint8, device=dev)
adct.approx_dct8x8_fused_sse_host(t1, host, [10], ws, chunk_images=1)
torch.cuda.synchronize()
print("sanitize smoke ok, kernels launched:", adct.launch_count())
