# bench.py's multi-rank path (2 ranks, gloo, both on cuda:0): rank handling, error-table
# all-reduce, max-over-ranks timing, weak-scaling value
mkdir -p gpurun_out
ADCT_ONE_DEVICE=1 ADCT_DIST_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
  --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 20 --warmup 3 --no-cpu > gpurun_out/two_rank.log 2>&1
echo "two-rank rc=$?"
grep "^{" gpurun_out/two_rank.log | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print('n_gpus', d['n_gpus'], 'value %.4g'%d['value'], 'ms', d['ms_per_step'], 'e2e', (d.get('e2e') or {}).get('value'), d['config']['parallelism'])"
ADCT_ONE_DEVICE=1 ADCT_DIST_BACKEND=gloo timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
  --master-addr 127.0.0.1 --master-port 29512 bench.py --impl reference --gpus 2 --steps 2 --warmup 1 > gpurun_out/two_rank_ref.log 2>&1
echo "two-rank reference rc=$?"; grep -c "^{" gpurun_out/two_rank_ref.log
timeout 600 python bench.py --steps 50 --warmup 3 --no-cpu > gpurun_out/one_rank.log 2>&1; echo "one-rank rc=$?"
grep -o '"value": [0-9.e+]*' gpurun_out/one_rank.log | head -1
