# what the driver runs at round end: GPU tests, smoke, the default bench line, the reference arm
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?"
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref.log 2>&1; echo "ref rc=$?"
python - <<'PY'
import json
for f in ("gpurun_out/bench.log", "gpurun_out/bench_ref.log"):
    l = [x for x in open(f) if x.startswith("{")][-1]
    d = json.loads(l)
    print(f, d.get("impl", "own"), "value=%.4g" % d["value"], "ms=%.4g" % d["ms_per_step"],
          "frac=%s" % (d.get("roofline") or {}).get("frac"), "issue=%s" % (d.get("issue_roofline") or {}).get("frac"),
          "clocks=%s" % d.get("clocks"), "e2e=%s" % (d.get("e2e") or {}).get("value"))
PY
