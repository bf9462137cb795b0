nvidia-smi --query-gpu=name,power.limit,temperature.gpu --format=csv,noheader
for i in 1 2 3; do
for v in base cmin4 ns16; do
  if [ $v = base ]; then unset ADCT_LIB; else export ADCT_LIB=$PWD/paper_1808_02950_b200/libadct_$v.so; fi
  timeout 300 python bench.py --steps 200 --warmup 5 --no-e2e --no-cpu 2>/dev/null | grep "^{" | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print('$v ms=%.4f best=%.4f luma_ms=%.4f frac=%.4f clip_ms=%.4f clk=%s' % (d['ms_per_step'], d['ms_per_step_best'], d['roofline']['kernel_ms'], d['roofline']['frac'], d['clip_policy']['ms_per_step'], d['clocks']['sm_mhz']))"
done
done
