bash tools/gpu/ab_lib.sh libadct_base.so libadct_b4w12.so libadct_b4w8.so
for v in b4w12 b4w8; do ADCT_LIB=$PWD/paper_1808_02950_b200/libadct_$v.so timeout 600 python -m pytest tests/test_gpu_stream.py -m gpu -x -q > gpurun_out/t_$v.log 2>&1; echo "$v tests rc=$? $(tail -1 gpurun_out/t_$v.log)"; done
