mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_stream.py tests/test_abi.py -x -q > gpurun_out/stream.log 2>&1; tail -1 gpurun_out/stream.log
for rep in 1 2; do
  for lib in libadct_old.so libadct.so; do
    echo "$lib: $(ADCT_LIB=$PWD/paper_1808_02950_b200/$lib timeout 120 python tools/hot_once.py 128 20 2>&1 | tail -1)"
  done
done
timeout 600 python bench.py --steps 100 --no-e2e --no-cpu > gpurun_out/bench_planes.log 2>&1; echo "planes rc=$?"
timeout 600 python bench.py --steps 100 --no-e2e --no-cpu --per-plane > gpurun_out/bench_pp.log 2>&1; echo "per-plane rc=$?"
python - <<'PY'
import json
for f in ("gpurun_out/bench_planes.log", "gpurun_out/bench_pp.log"):
    ls = [l for l in open(f) if l.startswith("{")]
    if not ls:
        print(f, "no line"); continue
    d = json.loads(ls[-1])
    print(f, "value=%.4g ms=%.4f frac=%.4f kernel_ms=%.4f step_frac=%.4f clk=%s" % (d["value"], d["ms_per_step"],
          d["roofline"]["frac"], d["roofline"]["kernel_ms"], d["roofline_step"]["frac"], d["clocks"]))
PY
