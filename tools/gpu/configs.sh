mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -n 5 gpurun_out/pytest_gpu.log
timeout 900 python bench.py --config all --steps 10 --warmup 3 > gpurun_out/configs.log 2>&1; echo "configs rc=$?" >> gpurun_out/configs.log
tail -n 8 gpurun_out/configs.log | cut -c1-400
