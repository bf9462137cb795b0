# A/B of library builds: bench luma-kernel roofline for each .so given as argument
mkdir -p gpurun_out
for lib in "$@"; do
  for rep in 1 2; do
    ADCT_LIB=$PWD/paper_1808_02950_b200/$lib timeout 300 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu > gpurun_out/ab_$lib.$rep.log 2>&1
    echo "$lib rep$rep: $(grep -o '"frac": [0-9.]*' gpurun_out/ab_$lib.$rep.log) value $(grep -o '"value": [0-9.e+]*' gpurun_out/ab_$lib.$rep.log | head -1) $(grep -o '"kernel_ms": [0-9.]*' gpurun_out/ab_$lib.$rep.log)"
  done
done
