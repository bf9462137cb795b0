# A/B of the stream kernel stage size (bench luma kernel roofline)
mkdir -p gpurun_out
for kb in 32 64 24 48 16; do
  ADCT_STREAM_STAGE_KB=$kb timeout 300 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu > gpurun_out/ab_$kb.log 2>&1
  echo "stage ${kb}KB: $(grep -o '"frac": [0-9.]*' gpurun_out/ab_$kb.log) $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/ab_$kb.log | head -1)"
done
