# hot-kernel timing for each library variant given as argument (default build first)
for lib in libadct.so "$@"; do
  for rep in 1 2; do
    echo "$lib: $(ADCT_LIB=$PWD/paper_1808_02950_b200/$lib python tools/hot_once.py 128 20 2>&1 | tail -1)"
  done
done
