mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_stream.py -x -q > gpurun_out/pytest_stream.log 2>&1; echo "stream tests rc=$?"; tail -1 gpurun_out/pytest_stream.log
bash tools/gpu/ab_lib.sh libadct.so
