mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --config MERIT --steps 10 --warmup 3 > gpurun_out/merit.log 2>&1; echo "merit rc=$?"; tail -c 700 gpurun_out/merit.log
