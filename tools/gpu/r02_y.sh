mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_stream.py tests/test_gpu_multirank.py -x -q 2>&1 | tail -2
for w in 1 8; do
  timeout 600 python bench.py --shard-of 0/$w --steps 200 --no-e2e --no-cpu > gpurun_out/b.log 2>&1; tail -1 gpurun_out/b.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('W=$w', 'frames', d['config']['frames_per_gpu'], 'ms/step %.4f' % d['ms_per_step'], 'proj G blocks/s %.2f' % (d['value']/1e9), 'luma ms %.4f' % d['roofline']['kernel_ms'], 'frac %.3f' % d['roofline']['frac'], 'clk', d['clocks']['sm_mhz'])"
done
CMD="python bench.py --shard-of 0/8 --steps 4 --warmup 3 --no-e2e --no-cpu"
export ADCT_PROFILE_RANGE=1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
  --log-file gpurun_out/launches8.csv $CMD > gpurun_out/ncu_launch8.log 2>&1
echo "ncu rc=$?"
