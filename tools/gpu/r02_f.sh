# ncu counters of old vs new tc kernel (same command)
mkdir -p gpurun_out
for lib in libadct_old.so libadct.so; do
  ADCT_LIB=$PWD/paper_1808_02950_b200/$lib timeout 300 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,sm__cycles_elapsed.avg.per_second,smsp__warp_issue_stalled_long_scoreboard_per_warp_active.pct,smsp__warp_issue_stalled_barrier_per_warp_active.pct,smsp__warp_issue_stalled_wait_per_warp_active.pct,smsp__warp_issue_stalled_sleeping_per_warp_active.pct --clock-control none -k regex:fused_u8_tc -c 3 python tools/hot_once.py 128 2 > gpurun_out/ncu_$lib.txt 2>&1
  grep -E "fused_u8_tc|duration|inst_executed|issue_active|dram__bytes|cycles_elapsed|stalled" gpurun_out/ncu_$lib.txt | tail -10
done
