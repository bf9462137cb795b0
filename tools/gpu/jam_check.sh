mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k jam > gpurun_out/pytest_jam.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_jam.log
bash tools/gpu/jam_bench.sh
