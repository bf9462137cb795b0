# A/B of library builds on the greedy search: parity tests + bench.py --config GREEDY; args = .so names
mkdir -p gpurun_out
for lib in "$@"; do
  ADCT_LIB=$PWD/paper_1808_02950_b200/$lib timeout 600 python -m pytest tests -m gpu -x -q -k greedy > gpurun_out/grab_$lib.pytest.log 2>&1
  echo "$lib pytest: $(tail -1 gpurun_out/grab_$lib.pytest.log)"
  ADCT_LIB=$PWD/paper_1808_02950_b200/$lib timeout 600 python bench.py --config GREEDY --steps 5 --warmup 3 > gpurun_out/grab_$lib.log 2>&1
  grep "^{" gpurun_out/grab_$lib.log | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print('  $lib', d['config']['workload'][-32:], 'ms=%.3f'%d['ms_per_step'], 'issue frac=%s'%d['roofline'].get('frac'))"
done
