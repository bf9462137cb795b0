mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "ssim or roundtrip or inverse" 2>&1 | tail -2
for lib in libadct_rtscalar.so libadct.so; do
  echo "$lib $(ADCT_LIB=$PWD/paper_1808_02950_b200/$lib timeout 600 python tools/ssim_once.py 2>&1 | tail -1)"
done
