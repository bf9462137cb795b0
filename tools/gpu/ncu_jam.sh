# ncu --set full of the 16- and 32-point JAM round trips (int16), after the same command ran clean
mkdir -p gpurun_out
CMD="python bench.py --config JAM --steps 1 --warmup 3"
timeout 600 $CMD > gpurun_out/plain_jam.log 2>&1; echo "plain rc=$?"
for n in 16 32; do
  timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base mangled \
    -k regex:"jam_roundtrip_kernelILi${n}Es" -s 2 -c 1 -o gpurun_out/jam${n}_full -f $CMD > gpurun_out/ncu_jam$n.log 2>&1
  echo "ncu $n rc=$?"
done
