# power / clock of the luma hot kernel vs ablation builds (tools/power_probe.py)
mkdir -p gpurun_out
for v in "" abl3 abl2 abl1 "" ; do
  if [ -n "$v" ]; then export ADCT_LIB=$PWD/paper_1808_02950_b200/libadct_$v.so; else unset ADCT_LIB; fi
  timeout 120 python tools/power_probe.py 256 8 2>&1 | tail -n 1 | tee -a gpurun_out/power_ab.jsonl
  sleep 3
done
