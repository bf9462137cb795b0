# round 2 checkpoint: full GPU tests, smoke, default bench line, all secondary configs, SSIM/ALU instruction counts
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/bench.log | cut -c1-300
timeout 1500 python bench.py --config all --steps 10 --warmup 3 > gpurun_out/configs_all.log 2>&1; echo "configs rc=$?"
bash tools/gpu/ncu_inst.sh
