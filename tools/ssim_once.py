"""Time the SSIM step of bench.py --config SSIM both ways on 128 4K luma frames (T1, r = 14, clip):
the two-call pipeline (round trip to an fp32 reconstruction in HBM + ssim_reduce) and the fused
approx_dct8x8_ssim; checks they agree."""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402
from paper_1808_02950_b200 import adct, catalog  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 128
dev = torch.device("cuda:0")
y = synth.ar1_stack(n, 2160, 3840, 0.95, seed=4, device=dev, batch=8)
m = adct.Matrix.from_int(catalog.T1, "T1")
rec = torch.empty(y.shape, dtype=torch.float32, device=dev)
ws = torch.empty(adct.workspace_bytes(adct.geom_of(y), 1), dtype=torch.uint8, device=dev)
out = {}


def pipe():
    adct.approx_dct8x8_roundtrip(m, y, 14, torch.float32, recon=rec)
    return adct.ssim_reduce(y, rec, clip=adct.CLIP, workspace=ws)


def fused():
    return adct.approx_dct8x8_ssim(m, y, 14, clip=adct.CLIP, workspace=ws)


for name, fn in (("pipeline", pipe), ("fused", fused)):
    for _ in range(3):
        r = fn()
    torch.cuda.synchronize()
    e = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    e[0].record()
    for _ in range(10):
        r = fn()
    e[1].record()
    torch.cuda.synchronize()
    out[name] = (e[0].elapsed_time(e[1]) / 10, r.clone())
diff = float(((out["fused"][1] - out["pipeline"][1]).abs() / out["pipeline"][1]).max())
print(json.dumps({"frames": n, "pipeline_ms": out["pipeline"][0], "fused_ms": out["fused"][0], "max_rel_diff": diff,
                  "fused_hbm_frac_64B": n * 32400 * 64 / (out["fused"][0] * 1e-3) / 1e9 / 6547.2}))
