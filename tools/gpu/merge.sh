# U+V in one launch: parity, then C4 bench A/B against separate launches, launch list
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_stream.py -x -q > gpurun_out/merge_tests.log 2>&1; echo "stream tests rc=$?"; tail -n 3 gpurun_out/merge_tests.log
for i in 1 2; do
  for v in merge sep; do
    if [ $v = sep ]; then export ADCT_TC_NOMERGE=1; else unset ADCT_TC_NOMERGE; fi
    timeout 300 python bench.py --steps 200 --warmup 5 --no-e2e --no-cpu 2>/dev/null | grep '^{' > gpurun_out/merge_b_$v.json
    python - $v <<'PY'
import json,sys
d=json.load(open(f"gpurun_out/merge_b_{sys.argv[1]}.json"))
print(sys.argv[1], "ms %.4f" % d["ms_per_step"], "best %.4f" % d["ms_per_step_best"], "G %.2f" % (d["value"]/1e9), "luma frac %.3f" % d["roofline"]["frac"], "step frac %.3f" % d["roofline_step"]["frac"], "clk", d["clocks"]["sm_mhz"], "launches", d["gpu_launches"])
PY
  done
done
unset ADCT_TC_NOMERGE
ADCT_PROFILE_RANGE=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
  --log-file gpurun_out/merge_launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/merge_ncu.log 2>&1
echo "ncu rc=$?"
