# one ncu --set full capture of the tensor-core hot kernel (16 4K frames, third launch)
mkdir -p gpurun_out
CMD="env ADCT_HOT=tc python tools/hot_once.py 64 1"
$CMD > gpurun_out/plain_tc.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:${1:-fused_u8_tc} -s 3 -c 1 -o gpurun_out/${2:-tc_full} -f $CMD > gpurun_out/ncu_tc.log 2>&1
echo "ncu rc=$?"; tail -2 gpurun_out/ncu_tc.log
