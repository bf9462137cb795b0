mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "greedy" > gpurun_out/greedy_tests.log 2>&1; tail -1 gpurun_out/greedy_tests.log
timeout 600 python bench.py --config GREEDY --steps 10 > gpurun_out/greedy.log 2>&1; grep "^{" gpurun_out/greedy.log | cut -c1-200
CMD="python tools/ssim_once.py 16"
$CMD > gpurun_out/ssim16.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:ssim_fused -s 2 -c 1 -o gpurun_out/ssim_fused_full -f $CMD > gpurun_out/ncu_ssim.log 2>&1; echo "ncu rc=$?"
