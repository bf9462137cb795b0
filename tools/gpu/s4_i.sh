mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q -k "config2_full" > gpurun_out/pytest_c2.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_c2.log
bash tools/gpu/two_rank.sh
