mkdir -p gpurun_out
timeout 1500 python bench.py --config all --steps 10 --warmup 3 > gpurun_out/configs_all.log 2>&1; echo "rc=$?"
grep "^{" gpurun_out/configs_all.log | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); r=d.get('roofline') or {}
    print(d['config']['workload'][:60], d['config'].get('matrix',''), 'ms=%.4g'%d['ms_per_step'], 'value=%.4g'%d['value'], 'frac=%s'%r.get('frac'))"
