# bench + ncu launch list + one full ncu capture of the hot kernel
mkdir -p gpurun_out
export ADCT_PROFILE_RANGE=1
timeout 600 python bench.py --steps 20 --warmup 3 > gpurun_out/bench2.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench2.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
  --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_launch.log 2>&1
echo "ncu launches rc=$?" >> gpurun_out/ncu_launch.log
timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:fused_u8_kernel -c 1 \
  -o gpurun_out/fused_u8_full -f python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_full.log 2>&1
echo "ncu full rc=$?" >> gpurun_out/ncu_full.log
tail -n 3 gpurun_out/bench2.log gpurun_out/ncu_launch.log gpurun_out/ncu_full.log
