# session 4: all secondary configs in one run + ncu full of the C3 quantiser and the JAM kernels
mkdir -p gpurun_out
bash tools/gpu/configs_all.sh
bash tools/gpu/ncu_c3.sh
