mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "roundtrip or config5 or in_place" 2>&1 | tail -2
for lib in libadct_bmscalar.so libadct.so; do
  timeout 600 env ADCT_LIB=$PWD/paper_1808_02950_b200/$lib python bench.py --config C5 --c5-log2 24,26 --steps 50 > gpurun_out/c5.log 2>&1
  grep '^{' gpurun_out/c5.log | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print('$lib', d['config']['matrix'], d['log2_blocks'], round(d['ms_per_step'],4), round(d['roofline']['frac'],4), d['roundtrip_bit_exact'], d['clocks']['sm_mhz'])"
done
