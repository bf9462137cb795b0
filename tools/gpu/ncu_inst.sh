# warp-instruction counts (smsp__inst_executed.sum) of every kernel of the ALU-bound secondary
# configs, for the issue roofline of their bench lines (tools/inst_table.py), each after the same
# command ran clean
mkdir -p gpurun_out
for c in ${CONFIGS:-C2 GREEDY MERIT SSIM}; do
  CMD="python bench.py --config $c --steps 1 --warmup 3"
  timeout 600 $CMD > gpurun_out/plain_inst_$c.log 2>&1 && \
  timeout 900 ncu --metrics smsp__inst_executed.sum,gpu__time_duration.sum --clock-control none --csv \
    -k regex:"ssim|sweep|finalize|merit|digits|score|search" \
    --log-file gpurun_out/inst_$c.csv $CMD > /dev/null 2>&1
  echo "$c rc=$?"
done
