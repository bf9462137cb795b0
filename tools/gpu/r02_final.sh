# round-2 evidence of the final build: GPU tests, smoke, bench line (+ reference arm), launch list
# of the timed C4 steps and one ncu --set full capture of the luma kernel
mkdir -p gpurun_out
bash tools/gpu/roundend.sh
CMD="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu"
export ADCT_PROFILE_RANGE=1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
  --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1
echo "ncu launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:"fused_u8_tc" -c 1 \
  -o gpurun_out/tc_full -f $CMD > gpurun_out/ncu_full.log 2>&1
echo "ncu full rc=$?"
