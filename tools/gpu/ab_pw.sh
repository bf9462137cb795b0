# A/B of the lightweight consumer walk (libadct_pw.so) against the shipped build, plus its GPU tests
bash tools/gpu/ab_lib.sh libadct_base.so libadct_pw.so libadct_base.so libadct_pw.so
ADCT_LIB=$PWD/paper_1808_02950_b200/libadct_pw.so timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/t_pw.log 2>&1; echo "pw tests rc=$? $(tail -1 gpurun_out/t_pw.log)"
