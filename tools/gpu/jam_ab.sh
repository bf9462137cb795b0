# A/B of library builds on the JAM next-row bench (bench.py --config JAM); args = .so names
mkdir -p gpurun_out
for lib in "$@"; do
  ADCT_LIB=$PWD/paper_1808_02950_b200/$lib timeout 300 python -m pytest tests -m gpu -x -q -k jam > gpurun_out/jamab_$lib.pytest.log 2>&1
  echo "$lib pytest: $(tail -1 gpurun_out/jamab_$lib.pytest.log)"
  for rep in 1 2; do
    ADCT_LIB=$PWD/paper_1808_02950_b200/$lib timeout 300 python bench.py --config JAM --steps 10 --warmup 3 > gpurun_out/jamab_$lib.$rep.log 2>&1
    grep "^{" gpurun_out/jamab_$lib.$rep.log | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print('  $lib rep$rep', d['config']['matrix'], 'ms=%.3f'%d['ms_per_step'], 'frac=%.3f'%d['roofline']['frac'])"
  done
done
