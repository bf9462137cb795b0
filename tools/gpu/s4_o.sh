python - <<'PY'
import torch, sys
sys.path.insert(0, '.')
from paper_1808_02950_b200 import adct, catalog
import synth
dev = torch.device('cuda:0')
y = synth.ar1_stack(128, 2160, 3840, 0.95, seed=4, device=dev, batch=8)
ws = torch.empty(adct.workspace_bytes(adct.geom_of(y), 1), dtype=torch.uint8, device=dev)
out = torch.empty((128, 1), dtype=torch.float64, device=dev)
m = adct.Matrix.from_int(catalog.T1, "T1")
for clip, nm in ((adct.CLIP_NONE, "none"), (adct.CLIP, "clip"), (adct.CLIP_ROUND, "clip_round")):
    for r in (10, 21):
        for _ in range(3):
            adct.approx_dct8x8_fused_sse(m, y, [r], clip=clip, workspace=ws, sse=out)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            adct.approx_dct8x8_fused_sse(m, y, [r], clip=clip, workspace=ws, sse=out)
        e1.record(); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 10
        print("clip=%s r=%d %.4f ms  %.1f%% of HBM" % (nm, r, ms, 100 * y.numel() / (ms * 1e-3) / 6544.3e9))
PY
