# A/B of 20 / 24 warps per CTA (2-slot rings) against the shipped 16 warps x 3 slots, plus GPU tests of both
bash tools/gpu/ab_lib.sh libadct_base.so libadct_w20.so libadct_w24.so libadct_base.so
for v in w20 w24; do ADCT_LIB=$PWD/paper_1808_02950_b200/libadct_$v.so timeout 600 python -m pytest tests/test_gpu_stream.py -m gpu -x -q > gpurun_out/t_$v.log 2>&1; echo "$v tests rc=$? $(tail -1 gpurun_out/t_$v.log)"; done
