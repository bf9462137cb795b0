# stream parity (tensor-core kernel) + A/B timing of the hot kernel variants
mkdir -p gpurun_out
ADCT_HOT=tc timeout 600 python -m pytest tests/test_gpu_stream.py -x -q 2>&1 | tail -3
for i in 1 2; do
ADCT_HOT=tc python tools/hot_once.py 128 20 2>&1 | tail -1
ADCT_HOT=simt python tools/hot_once.py 128 20 2>&1 | tail -1
done
