mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_stream.py -x -q -k "clip_policy or other_r or geometries" > gpurun_out/pytest_clip.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/pytest_clip.log
bash tools/gpu/s4_o.sh
