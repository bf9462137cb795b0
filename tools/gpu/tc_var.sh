# hot-kernel timing for each library variant given as argument (default build first); 120 s cap per run
for lib in libadct.so "$@"; do
  for rep in 1 2; do
    echo "$lib: $(ADCT_HOT=tc ADCT_LIB=$PWD/paper_1808_02950_b200/$lib timeout 120 python tools/hot_once.py 128 20 2>&1 | tail -1)"
  done
done
