# N = 160 single MMA set per tile (libadct_n160.so) vs the default: stream parity, then alternating bench runs
mkdir -p gpurun_out
ADCT_LIB=$PWD/paper_1808_02950_b200/libadct_n160.so timeout 600 python -m pytest tests/test_gpu_stream.py -x -q 2>&1 | tail -2
for i in 1 2 3; do
for v in base n160; do
  if [ $v = base ]; then unset ADCT_LIB; else export ADCT_LIB=$PWD/paper_1808_02950_b200/libadct_n160.so; fi
  timeout 300 python bench.py --steps 200 --warmup 5 --no-e2e --no-cpu 2>/dev/null | grep "^{" | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print('$v ms=%.4f best=%.4f luma_ms=%.4f frac=%.4f step_frac=%.4f clk=%s' % (d['ms_per_step'], d['ms_per_step_best'], d['roofline']['kernel_ms'], d['roofline']['frac'], d['roofline_step']['frac'], d['clocks']['sm_mhz']))"
done
done
