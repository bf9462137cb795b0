# one ncu --set full capture per secondary kernel (each after the same command ran clean)
mkdir -p gpurun_out
run() {  # name, kernel regex, bench config
  CMD="python bench.py --config $3 --steps 1 --warmup 3"
  timeout 600 $CMD > gpurun_out/plain_$1.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$2" -s 2 -c 1 -o gpurun_out/$1_full -f $CMD > gpurun_out/ncu_$1.log 2>&1
  echo "$1 rc=$?"
}
run c5 roundtrip_bm C5
run jam jam_roundtrip JAM
run greedy search_kernel GREEDY
run ssim ssim_kernel SSIM
run sweep fused_sweep C2
