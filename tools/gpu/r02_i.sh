mkdir -p gpurun_out
run() { timeout 600 env $1 python bench.py --steps 200 --no-e2e --no-cpu $2 > gpurun_out/b.log 2>&1; python - "$1 $2" <<'PY'
import json, sys
ls = [l for l in open("gpurun_out/b.log") if l.startswith("{")]
d = json.loads(ls[-1]) if ls else None
print(sys.argv[1], "no line" if d is None else "value=%.4g ms=%.4f kernel_ms=%.4f frac=%.4f step_frac=%.4f clk=%s" % (d["value"], d["ms_per_step"], d["roofline"]["kernel_ms"], d["roofline"]["frac"], d["roofline_step"]["frac"], d["clocks"]["sm_mhz"]))
PY
}
for rep in 1 2; do
run "ADCT_LIB=$PWD/paper_1808_02950_b200/libadct_old.so" --per-plane
run "X=1" ""
run "X=1" --per-plane
done
