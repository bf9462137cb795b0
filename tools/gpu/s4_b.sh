# C3 input tensor map: L2 promotion A/B (bench line + ncu dram bytes per launch)
mkdir -p gpurun_out
for p in 256 128 64 0; do
  export ADCT_Q_L2PROMO=$p
  for i in 1 2; do
  timeout 300 python bench.py --config C3 --steps 50 --warmup 5 2>/dev/null | grep "^{" | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print('promo=$p ms=%.4f frac=%.4f clk=%s' % (d['ms_per_step'], d['roofline']['frac'], d.get('clocks',{}).get('sm_mhz')))"
  done
  timeout 300 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:fwd_quant -s 3 -c 1 python bench.py --config C3 --steps 2 --warmup 3 2>/dev/null | grep -E "dram__|gpu__time"
done
