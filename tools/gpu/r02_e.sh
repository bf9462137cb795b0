# same-box A/B old vs new tc kernel; fused SSIM parity + timing vs the two-call pipeline
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "ssim" > gpurun_out/ssim_tests.log 2>&1; tail -3 gpurun_out/ssim_tests.log
timeout 900 python -m pytest tests/test_gpu_stream.py tests/test_abi.py -x -q > gpurun_out/stream.log 2>&1; tail -3 gpurun_out/stream.log
for rep in 1 2 3; do
  for lib in libadct_old.so libadct.so; do
    echo "$lib: $(ADCT_LIB=$PWD/paper_1808_02950_b200/$lib timeout 120 python tools/hot_once.py 128 20 2>&1 | tail -1)"
  done
done
timeout 600 python tools/ssim_once.py > gpurun_out/ssim_once.log 2>&1; cat gpurun_out/ssim_once.log | tail -4
