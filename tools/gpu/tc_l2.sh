# A/B of the tensor-core hot kernel's L2 prefetch distance (libadct_l2a<N>.so variants) + stream
# parity of one variant
mkdir -p gpurun_out
ADCT_LIB=$PWD/paper_1808_02950_b200/libadct_l2a16.so timeout 600 python -m pytest tests/test_gpu_stream.py -x -q 2>&1 | tail -2
for rep in 1 2 3; do
  for lib in libadct.so libadct_l2a8.so libadct_l2a16.so libadct_l2a32.so; do
    echo "$lib: $(ADCT_LIB=$PWD/paper_1808_02950_b200/$lib timeout 120 python tools/hot_once.py 128 20 2>&1 | tail -1)"
  done
done
