mkdir -p gpurun_out
timeout 900 python bench.py --config GREEDY --steps 5 --warmup 3 > gpurun_out/greedy.log 2>&1; echo "rc=$?"
grep "^{" gpurun_out/greedy.log | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print(d['config'], 'ms=%.3f'%d['ms_per_step'], 'Gcand/s=%.1f'%(d['value']/1e9), 'cpu Mcand/s=%.1f'%(d['cpu_baseline']['value']/1e6))"
tail -3 gpurun_out/greedy.log | cut -c1-300
