"""Run the C4 luma hot kernel a few times on a smaller 4K stack (for ncu captures and A/B timing).

    python tools/hot_once.py [frames] [reps]     (ADCT_HOT=simt selects the SIMT kernel)
Prints the mean CUDA-event time per launch and the algorithmic HBM fraction of the kernel.
"""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402
from paper_1808_02950_b200 import adct, catalog  # noqa: E402

frames = int(sys.argv[1]) if len(sys.argv) > 1 else 64
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
dev = torch.device("cuda:0")
x = synth.ar1_field(frames, 2160, 3840, 0.95, seed=4, device=dev)
m = adct.Matrix.from_int(catalog.T1, "T1")
out = torch.empty(frames, 1, dtype=torch.float64, device=dev)
ws = torch.empty(adct.workspace_bytes(adct.geom_of(x), 1), dtype=torch.uint8, device=dev)
for _ in range(3):
    adct.approx_dct8x8_fused_sse(m, x, [10], workspace=ws, sse=out)
torch.cuda.synchronize()
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
ev[0].record()
for _ in range(reps):
    adct.approx_dct8x8_fused_sse(m, x, [10], workspace=ws, sse=out)
ev[1].record()
torch.cuda.synchronize()
ms = ev[0].elapsed_time(ev[1]) / reps
nb = frames * 270 * 480
peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] if os.path.exists(
    os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6650.0
gbs = nb * 64 / ms / 1e6
print(json.dumps({"hot": os.environ.get("ADCT_HOT", "tc"), "frames": frames, "ms": ms, "gblocks_s": nb / ms / 1e6,
                  "gbs": gbs, "frac": gbs / peak, "sse0": float(out[0, 0])}))
