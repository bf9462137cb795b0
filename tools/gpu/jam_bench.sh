mkdir -p gpurun_out
timeout 900 python bench.py --config JAM --steps 10 --warmup 3 > gpurun_out/jam.log 2>&1; echo "rc=$?"
grep "^{" gpurun_out/jam.log | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print(d['config']['matrix'], 'ms=%.3f'%d['ms_per_step'], 'frac=%.3f'%d['roofline']['frac'], d.get('roundtrip_bit_exact'))"
