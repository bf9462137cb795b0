"""Power / clock probe of the C4 luma hot kernel: launch it back to back for a few seconds while
nvidia-smi samples board power and SM clock, then report time per launch, median power and clock.

    ADCT_LIB=... python tools/power_probe.py [frames] [seconds]
Used to see where the board's power goes (A/B of ablation builds, tools/build_variant.sh) when the
bench step runs under sw_power_cap.
"""
import json
import os
import subprocess
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402
from paper_1808_02950_b200 import adct, catalog  # noqa: E402

frames = int(sys.argv[1]) if len(sys.argv) > 1 else 128
secs = float(sys.argv[2]) if len(sys.argv) > 2 else 6.0
dev = torch.device("cuda:0")
x = synth.ar1_field(frames, 2160, 3840, 0.95, seed=4, device=dev)
m = adct.Matrix.from_int(catalog.T1, "T1")
out = torch.empty(frames, 1, dtype=torch.float64, device=dev)
ws = torch.empty(adct.workspace_bytes(adct.geom_of(x), 1), dtype=torch.uint8, device=dev)
for _ in range(5):
    adct.approx_dct8x8_fused_sse(m, x, [10], workspace=ws, sse=out)
torch.cuda.synchronize()
# calibrate launches per second, then run ~secs seconds with sampling
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
ev[0].record()
for _ in range(20):
    adct.approx_dct8x8_fused_sse(m, x, [10], workspace=ws, sse=out)
ev[1].record()
torch.cuda.synchronize()
ms0 = ev[0].elapsed_time(ev[1]) / 20
n = max(50, int(secs * 1e3 / ms0))
smi = subprocess.Popen(["nvidia-smi", "--query-gpu=power.draw,clocks.sm,clocks_throttle_reasons.active",
                        "--format=csv,noheader,nounits", "-lms", "100"], stdout=subprocess.PIPE, text=True)
time.sleep(0.3)
ev[0].record()
for _ in range(n):
    adct.approx_dct8x8_fused_sse(m, x, [10], workspace=ws, sse=out)
ev[1].record()
torch.cuda.synchronize()
smi.terminate()
rows = []
for line in smi.stdout.read().strip().splitlines():
    p = [s.strip() for s in line.split(",")]
    try:
        rows.append((float(p[0]), float(p[1]), p[2]))
    except (ValueError, IndexError):
        pass
ms = ev[0].elapsed_time(ev[1]) / n
# drop the first and last samples (ramp); keep those while the loop was running
body = rows[3:-2] if len(rows) > 8 else rows
pw = sorted(r[0] for r in body)
clk = sorted(r[1] for r in body)
nb = frames * 270 * 480
peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
print(json.dumps({"lib": os.path.basename(os.environ.get("ADCT_LIB", "libadct.so")), "frames": frames, "launches": n,
                  "ms": round(ms, 4), "frac": round(nb * 64 / ms / 1e6 / peak, 4),
                  "power_w_median": pw[len(pw) // 2] if pw else None, "power_w_max": pw[-1] if pw else None,
                  "sm_mhz_median": clk[len(clk) // 2] if clk else None,
                  "reasons": sorted({r[2] for r in body}), "samples": len(body)}))
