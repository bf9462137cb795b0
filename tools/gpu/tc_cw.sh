# A/B of the luma tile shape (ADCT_TC_CW forces CW chunks x 16/CW bands; cwx build has 4 and 8)
mkdir -p gpurun_out
L=$PWD/paper_1808_02950_b200/libadct_cwx.so
ADCT_LIB=$L ADCT_TC_CW=8 timeout 600 python -m pytest tests/test_gpu_stream.py -x -q 2>&1 | tail -1
for rep in 1 2; do
  for cw in 2 4 8 16 1; do
    echo "cw=$cw: $(ADCT_LIB=$L ADCT_TC_CW=$cw timeout 120 python tools/hot_once.py 128 20 2>&1 | tail -1)"
  done
done
