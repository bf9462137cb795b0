# A/B of library builds on SSIM: parity tests + bench.py --config SSIM; args = .so names
mkdir -p gpurun_out
for lib in "$@"; do
  ADCT_LIB=$PWD/paper_1808_02950_b200/$lib timeout 600 python -m pytest tests -m gpu -x -q -k ssim > gpurun_out/ssimab_$lib.pytest.log 2>&1
  echo "$lib pytest: $(tail -1 gpurun_out/ssimab_$lib.pytest.log)"
  for rep in 1 2; do
    ADCT_LIB=$PWD/paper_1808_02950_b200/$lib timeout 300 python bench.py --config SSIM --steps 10 --warmup 3 > gpurun_out/ssimab_$lib.$rep.log 2>&1
    echo "  $lib rep$rep $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/ssimab_$lib.$rep.log)"
  done
done
