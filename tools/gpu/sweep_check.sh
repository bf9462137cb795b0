mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
for c in C1 C2; do timeout 600 python bench.py --config $c --steps 10 --warmup 3 > gpurun_out/$c.log 2>&1; echo "$c: $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/$c.log)"; done
