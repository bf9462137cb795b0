mkdir -p gpurun_out
for v in ffma2 ways2; do
  ADCT_LIB=$PWD/paper_1808_02950_b200/libadct_$v.so timeout 600 python -m pytest tests/test_gpu_stream.py -x -q -k "geometries or every_r" 2>&1 | tail -1
done
for rep in 1 2 3; do
  for lib in libadct.so libadct_ffma2.so libadct_ways2.so; do
    echo "$lib: $(ADCT_LIB=$PWD/paper_1808_02950_b200/$lib timeout 120 python tools/hot_once.py 128 20 2>&1 | tail -1)"
  done
done
