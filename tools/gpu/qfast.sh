# C3 quantiser fast path: parity, then C3 A/B against the remainder-corrected form
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "quant or config3" > gpurun_out/q_tests.log 2>&1; echo "quant tests rc=$?"; tail -n 2 gpurun_out/q_tests.log
for i in 1 2; do
  for v in fast old; do
    if [ $v = old ]; then export ADCT_LIB=$PWD/paper_1808_02950_b200/libadct_qold.so; else unset ADCT_LIB; fi
    timeout 300 python bench.py --config C3 --no-cpu 2>/dev/null | grep '^{' | tail -n 1 > gpurun_out/q_$v.json
    python - $v <<'PY'
import json,sys
d=json.load(open(f"gpurun_out/q_{sys.argv[1]}.json"))
print(sys.argv[1], "ms %.4f" % d["ms_per_step"], "frac %.3f" % d["roofline"]["frac"], "clk", d.get("clocks",{}).get("sm_mhz"))
PY
  done
done
unset ADCT_LIB
timeout 600 ncu --set full --clock-control none -k regex:fwd_quant_tma -c 1 -o gpurun_out/q_full -f python bench.py --config C3 --no-cpu --steps 2 --warmup 3 > gpurun_out/q_ncu.log 2>&1; echo "ncu rc=$?"
