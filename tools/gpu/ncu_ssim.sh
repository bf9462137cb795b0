# ncu --set full of the persistent SSIM kernel, after the same command ran clean
mkdir -p gpurun_out
CMD="python bench.py --config SSIM --steps 1 --warmup 3"
timeout 600 $CMD > gpurun_out/plain_ssim.log 2>&1; echo "plain rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"ssim_strip_kernel" -s 2 -c 1 -o gpurun_out/ssim_full -f $CMD > gpurun_out/ncu_ssim.log 2>&1
echo "ncu rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ssim_launches.csv $CMD > /dev/null 2>&1; echo "launches rc=$?"
