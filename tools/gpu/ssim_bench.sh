mkdir -p gpurun_out
timeout 900 python bench.py --config SSIM --steps 10 --warmup 3 > gpurun_out/ssim.log 2>&1; echo "rc=$?"; tail -c 600 gpurun_out/ssim.log
