# round-end evidence: full bench line, launch list and one full ncu capture of the hot kernel
mkdir -p gpurun_out
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv -lms 200 > gpurun_out/clocks.csv &
CLK=$!
timeout 900 python bench.py > gpurun_out/bench_final.log 2>&1; echo "bench rc=$?"
kill $CLK
timeout 600 python bench.py --impl reference --steps 5 --warmup 1 > gpurun_out/bench_ref_final.log 2>&1; echo "ref rc=$?"
CMD="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu"
export ADCT_PROFILE_RANGE=1
timeout 600 $CMD > gpurun_out/plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
  --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1
echo "ncu launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:"wtile_kernel" -c 1 \
  -o gpurun_out/stream_full -f $CMD > gpurun_out/ncu_full.log 2>&1
echo "ncu full rc=$?"
