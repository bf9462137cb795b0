# A/B of the lightweight consumer walk (libadct_wc.so) against the shipped build, plus its GPU tests
bash tools/gpu/ab_lib.sh libadct_base.so libadct_wc.so libadct_base.so libadct_wc.so
ADCT_LIB=$PWD/paper_1808_02950_b200/libadct_wc.so timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/t_wc.log 2>&1; echo "wc tests rc=$? $(tail -1 gpurun_out/t_wc.log)"
