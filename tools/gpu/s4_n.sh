cat > /tmp/rt_rate.py <<'PY'
import torch, sys
sys.path.insert(0, '.')
from paper_1808_02950_b200 import adct, catalog
import synth
dev = torch.device('cuda:0')
y = synth.ar1_stack(128, 2160, 3840, 0.95, seed=4, device=dev, batch=8)
ws = torch.empty(adct.workspace_bytes(adct.geom_of(y), 1), dtype=torch.uint8, device=dev)
out = torch.empty((128, 1), dtype=torch.float64, device=dev)
res = []
for name in ("T1", "T6"):
    m = adct.Matrix.from_int(catalog.INTEGER[name], name)
    for r in (21, 50):
        for _ in range(3):
            adct.approx_dct8x8_fused_sse(m, y, [r], workspace=ws, sse=out)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            adct.approx_dct8x8_fused_sse(m, y, [r], workspace=ws, sse=out)
        e1.record(); torch.cuda.synchronize()
        res.append("%s r=%d %.4f ms" % (name, r, e0.elapsed_time(e1) / 10))
print(" | ".join(res))
PY
for lib in libadct.so libadct_rt3.so libadct_rt4.so libadct_rt2n.so; do
  echo -n "$lib: "; ADCT_LIB=$PWD/paper_1808_02950_b200/$lib python /tmp/rt_rate.py
done
