mkdir -p gpurun_out
CMD="python bench.py --config C3 --steps 2 --warmup 3 --no-cpu"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fwd_quant_tc -s 3 -c 1 -o gpurun_out/c3tc_full -f $CMD > gpurun_out/ncu_c3tc.log 2>&1
echo "rc=$?"
