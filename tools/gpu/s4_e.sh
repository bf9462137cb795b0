mkdir -p gpurun_out
CMD="python bench.py --config JAM --steps 1 --warmup 3 --no-cpu"
for n in 16 32; do
  timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base mangled \
    -k regex:"jam2_roundtrip_kernelILi${n}Es" -s 2 -c 1 -o gpurun_out/jam2_${n}_full -f $CMD > gpurun_out/ncu_jam2_$n.log 2>&1
  echo "ncu $n rc=$?"
done
