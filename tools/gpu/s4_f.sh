# C3 quantiser on the tensor core: parity tests (short timeout: a pipeline bug would hang), then A/B
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q -k "quant" > gpurun_out/pytest_q.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/pytest_q.log
for v in 1 0 1 0; do
  export ADCT_Q_TC=$v
  timeout 300 python bench.py --config C3 --steps 50 --warmup 5 --no-cpu 2>/dev/null | grep "^{" | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print('tc=$v ms=%.4f frac=%.4f clk=%s' % (d['ms_per_step'], d['roofline']['frac'], d.get('clocks',{}).get('sm_mhz')), d['config'].get('check', ''))"
done
