# donor tiling of the chroma planes: parity, then C4 bench A/B against the 16-chunk tiles
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_stream.py -x -q > gpurun_out/donor_tests.log 2>&1; echo "stream tests rc=$?"; tail -n 2 gpurun_out/donor_tests.log
for i in 1 2; do
  for cw in 15 16; do
    if [ $cw = 16 ]; then export ADCT_TC_NODONOR=1; else unset ADCT_TC_NODONOR; fi
    timeout 300 python bench.py --steps 200 --warmup 5 --no-e2e --no-cpu 2>/dev/null | grep '^{' > gpurun_out/donor_b_$cw.json
    python - $cw <<'PY'
import json,sys
d=json.load(open(f"gpurun_out/donor_b_{sys.argv[1]}.json"))
print("cw", sys.argv[1], "ms %.4f" % d["ms_per_step"], "G %.2f" % (d["value"]/1e9), "luma frac %.3f" % d["roofline"]["frac"], "clk", d["clocks"]["sm_mhz"])
PY
  done
done
unset ADCT_TC_NODONOR
ADCT_PROFILE_RANGE=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
  --log-file gpurun_out/donor_launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/donor_ncu.log 2>&1
echo "ncu rc=$?"
