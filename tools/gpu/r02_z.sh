mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
for w in 1 8 4 2; do
  timeout 600 python bench.py --shard-of 0/$w --steps 200 --no-e2e --no-cpu > gpurun_out/b.log 2>&1; tail -1 gpurun_out/b.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('W=$w', 'frames', d['config']['frames_per_gpu'], 'ms/step %.4f' % d['ms_per_step'], 'proj G blocks/s %.2f' % (d['value']/1e9), 'luma ms %.4f' % d['roofline']['kernel_ms'], 'frac %.3f' % d['roofline']['frac'], 'clk', d['clocks']['sm_mhz'])"
done
