# parity tests, bench, A/B vs the register-prefetch kernels, ncu launch list + full capture of the hot kernel
mkdir -p gpurun_out
PIPES_ONLY=1 timeout 120 ./probes/pipes > gpurun_out/pipes.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
CMD="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu"
export ADCT_PROFILE_RANGE=1
timeout 600 $CMD > gpurun_out/plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
  --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1
echo "ncu launches rc=$?" >> gpurun_out/ncu_launch.log
timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:"stream_kernel|wtile_kernel" -c 1 \
  -o gpurun_out/stream_full -f $CMD > gpurun_out/ncu_full.log 2>&1
echo "ncu full rc=$?" >> gpurun_out/ncu_full.log
tail -n 3 gpurun_out/pytest_gpu.log gpurun_out/smoke.log gpurun_out/bench.log gpurun_out/ncu_launch.log gpurun_out/ncu_full.log
