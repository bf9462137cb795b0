mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_stream.py -x -q > gpurun_out/pytest_stream.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_stream.log
# rate of the newly compiled retentions on the 4K luma stack (128 frames)
python - <<'PY'
import torch, time, sys
sys.path.insert(0, '.')
from paper_1808_02950_b200 import adct, catalog
import synth
dev = torch.device('cuda:0')
y = synth.ar1_stack(128, 2160, 3840, 0.95, seed=4, device=dev, batch=8)
m = adct.Matrix.from_int(catalog.T1, "T1")
ws = torch.empty(adct.workspace_bytes(adct.geom_of(y), 1), dtype=torch.uint8, device=dev)
out = torch.empty((128, 1), dtype=torch.float64, device=dev)
for r in (1, 3, 6, 10, 14, 15, 36, 21, 50):
    for _ in range(3):
        adct.approx_dct8x8_fused_sse(m, y, [r], workspace=ws, sse=out)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        adct.approx_dct8x8_fused_sse(m, y, [r], workspace=ws, sse=out)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 20
    print("r=%d ms=%.4f  %.1f%% of 6544 GB/s" % (r, ms, 100 * y.numel() / (ms * 1e-3) / 6544.3e9))
PY
