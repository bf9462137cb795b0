# JAM v2 (two rows / columns per thread, packed): parity tests, then bench v1 vs v2
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "jam" > gpurun_out/pytest_jam.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_jam.log
for v in v2 v1 v2 v1; do
  if [ $v = v1 ]; then export ADCT_JAM_V1=1; else unset ADCT_JAM_V1; fi
  timeout 600 python bench.py --config JAM --steps 20 --warmup 3 --no-cpu 2>/dev/null | grep "^{" | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print('$v', d['config']['matrix'], 'ms=%.4f frac=%.4f exact=%s clk=%s' % (d['ms_per_step'], d['roofline']['frac'], d.get('roundtrip_bit_exact', d['config'].get('roundtrip_bit_exact')), d.get('clocks',{}).get('sm_mhz')))"
done
