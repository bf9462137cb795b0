mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "quant" 2>&1 | tail -2
for lib in libadct_bmscalar.so libadct.so; do
  timeout 600 env ADCT_LIB=$PWD/paper_1808_02950_b200/$lib python bench.py --config C3 --steps 20 > gpurun_out/cx.log 2>&1
  grep '^{' gpurun_out/cx.log | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print('$lib', round(d['ms_per_step'],4), round(d['roofline']['frac'],4), d['clocks']['sm_mhz'])"
done
