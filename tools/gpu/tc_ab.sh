# stream parity + A/B timing of the hot kernel variants (tensor-core default vs SIMT)
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_stream.py -x -q 2>&1 | tail -3
for i in 1 2; do
python tools/hot_once.py 128 20 2>&1 | tail -1
ADCT_HOT=simt python tools/hot_once.py 128 20 2>&1 | tail -1
done
