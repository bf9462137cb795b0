# DRAM traffic of every kernel of the secondary configs and of the C4 step (one ncu pass, 3 metrics)
mkdir -p gpurun_out
timeout 1200 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/traffic_all.csv python bench.py --config all --steps 1 --warmup 1 --no-cpu > gpurun_out/traffic_all.log 2>&1
echo rc=$?
export ADCT_PROFILE_RANGE=1
timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
  --log-file gpurun_out/traffic_c4.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/traffic_c4.log 2>&1
echo rc=$?
