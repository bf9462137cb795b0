mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "quant" > gpurun_out/pytest_q.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_q.log
bash tools/gpu/ncu_c3.sh
