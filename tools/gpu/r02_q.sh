mkdir -p gpurun_out
for rep in 1 2 3; do
  for lib in libadct_p1old.so libadct_p1.so libadct_p2old.so libadct.so libadct_fb.so; do
    echo "$lib: $(ADCT_LIB=$PWD/paper_1808_02950_b200/$lib timeout 120 python tools/hot_once.py 128 20 2>&1 | tail -1 | cut -c1-80)"
  done
done
