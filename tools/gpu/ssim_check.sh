mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "ssim" > gpurun_out/pytest_ssim.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_ssim.log
bash tools/gpu/ssim_bench.sh | grep -o '"ms_per_step": [0-9.]*\|"frac": [0-9.]*'
