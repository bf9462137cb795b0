mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "quant or sweep or config1 or fused_single or fused_clip or int16_source" 2>&1 | tail -2
for lib in libadct_scalar2.so libadct.so; do
  for c in C3 C2; do
  timeout 600 env ADCT_LIB=$PWD/paper_1808_02950_b200/$lib python bench.py --config $c --steps 20 > gpurun_out/cx.log 2>&1
  grep '^{' gpurun_out/cx.log | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print('$lib', d['config']['workload'][:12], round(d['ms_per_step'],4), d['roofline'].get('frac'), d['clocks']['sm_mhz'])"
  done
done
