mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_stream.py -x -q 2>&1 | tail -2
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "config4 or fused_single or host_psnr or config1" 2>&1 | tail -2
for rep in 1 2 3; do
  for lib in libadct_nofb.so libadct.so; do
    echo "$lib: $(ADCT_LIB=$PWD/paper_1808_02950_b200/$lib timeout 120 python tools/hot_once.py 128 20 2>&1 | tail -1)"
  done
done
for lib in libadct_nofb.so libadct.so; do
  timeout 600 env ADCT_LIB=$PWD/paper_1808_02950_b200/$lib python bench.py --steps 200 --no-e2e --no-cpu > gpurun_out/b.log 2>&1; tail -1 gpurun_out/b.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$lib bench', d['value'], d['ms_per_step'], d['roofline']['frac'], d['roofline']['kernel_ms'], d['roofline_step']['frac'], d['clocks']['sm_mhz'])"
done
