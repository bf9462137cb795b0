# session-4 final evidence: round-end sequence, launch list + ncu full of the luma kernel, all secondary configs
bash tools/gpu/r02_final.sh
bash tools/gpu/configs_all.sh
bash tools/gpu/ncu_c3.sh
