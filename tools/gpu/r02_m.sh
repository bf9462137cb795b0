mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_stream.py -x -q > gpurun_out/stream.log 2>&1; tail -2 gpurun_out/stream.log
for rep in 1 2; do
  timeout 600 python bench.py --steps 200 --no-e2e --no-cpu > gpurun_out/b.log 2>&1; tail -1 gpurun_out/b.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('bench', d['value'], d['ms_per_step'], d['roofline']['frac'], d['roofline']['kernel_ms'], d['roofline_step']['frac'], d['clocks']['sm_mhz'])"
done
CMD="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu"
export ADCT_PROFILE_RANGE=1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
  --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1
echo "ncu launches rc=$?"
