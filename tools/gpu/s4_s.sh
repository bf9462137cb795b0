for w in 8 4; do
for v in base cmin8 cmin16 base cmin8 cmin16; do
  if [ $v = base ]; then unset ADCT_LIB; else export ADCT_LIB=$PWD/paper_1808_02950_b200/libadct_$v.so; fi
  timeout 300 python bench.py --shard-of 0/$w --steps 200 --no-e2e --no-cpu 2>/dev/null | grep "^{" | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$v W=$w', 'frames', d['config']['frames_per_gpu'], 'ms/step %.4f' % d['ms_per_step'], 'luma ms %.4f' % d['roofline']['kernel_ms'], 'clk', d['clocks']['sm_mhz'])"
done
done
