# donor-box promotion A/B on the C4 step + opt-in kernel parity tests
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "tensor_core_kernel or jam_v2 or quant" > gpurun_out/pytest_opt.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_opt.log
for v in 0 1 0 1; do
  if [ $v = 1 ]; then export ADCT_TC_DPROMO=1; else unset ADCT_TC_DPROMO; fi
  timeout 300 python bench.py --steps 200 --warmup 5 --no-e2e --no-cpu 2>/dev/null | grep "^{" | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print('dpromo=$v ms=%.4f best=%.4f luma_ms=%.4f frac=%.4f step_frac=%.4f clk=%s' % (d['ms_per_step'], d['ms_per_step_best'], d['roofline']['kernel_ms'], d['roofline']['frac'], d['roofline_step']['frac'], d['clocks']['sm_mhz']))"
done
