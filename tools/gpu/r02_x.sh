mkdir -p gpurun_out
CMD="python bench.py --shard-of 0/8 --steps 4 --warmup 3 --no-e2e --no-cpu"
export ADCT_PROFILE_RANGE=1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
  --log-file gpurun_out/launches8.csv $CMD > gpurun_out/ncu_launch8.log 2>&1
echo "ncu rc=$?"
