mkdir -p gpurun_out
CMD="python bench.py --config C3 --steps 2 --warmup 3"
timeout 600 $CMD > gpurun_out/plain_c3.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fwd_quant -s 3 -c 1 -o gpurun_out/c3_full -f $CMD > gpurun_out/ncu_c3.log 2>&1
echo "rc=$?"; tail -2 gpurun_out/ncu_c3.log
