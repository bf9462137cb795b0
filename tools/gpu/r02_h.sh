mkdir -p gpurun_out
timeout 600 ncu --section SourceCounters --section WarpStateStats --clock-control none --import-source on -k regex:fused_u8_tc -s 2 -c 1 -o gpurun_out/tc_new_src -f python tools/hot_once.py 64 1 > gpurun_out/ncu_src.log 2>&1; echo "rc=$?"; tail -2 gpurun_out/ncu_src.log
