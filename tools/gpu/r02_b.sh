# round 2: GPU tests (incl. multi-rank + in-place C5), default bench line (strong scaling, library
# PSNR), the C5 sweep, and the 2-rank bench path with both ranks on the one GPU (gloo)
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/bench.log | cut -c1-600
timeout 900 python bench.py --config C5 --steps 50 > gpurun_out/c5.log 2>&1; echo "c5 rc=$?"; grep '^{' gpurun_out/c5.log | cut -c1-300
ADCT_ONE_DEVICE=1 ADCT_DIST_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
  --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 20 --warmup 3 --no-cpu > gpurun_out/two_rank.log 2>&1
echo "two-rank rc=$?"; grep '^{' gpurun_out/two_rank.log | cut -c1-400
