# one-GPU scaling probe: the per-rank share of the 512-frame C4 stack at W = 1, 2, 4, 8
mkdir -p gpurun_out
for w in 1 2 4 8; do
  timeout 600 python bench.py --shard-of 0/$w --steps 200 --no-e2e --no-cpu > gpurun_out/b.log 2>&1; tail -1 gpurun_out/b.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('W=$w', 'frames', d['config']['frames_per_gpu'], 'ms/step %.4f' % d['ms_per_step'], 'median %.4f' % d['ms_per_step_median'], 'proj G blocks/s %.2f' % (d['value']/1e9), 'luma ms %.4f' % d['roofline']['kernel_ms'], 'frac %.3f' % d['roofline']['frac'], 'clk', d['clocks']['sm_mhz'])"
done
