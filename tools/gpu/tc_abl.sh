# ablation timings + issuer trace summary for each variant library
for v in trace tr_noldtm tr_nosttm tr_noepi tr_none; do
  ADCT_LIB=$PWD/paper_1808_02950_b200/libadct_$v.so python tools/hot_once.py 8 1 > /dev/null 2>&1
  python - "$v" <<'PY'
import sys
rows=[list(map(int,l.split())) for l in open('gpurun_out/tc_trace.txt')]
per=(rows[50][4]-rows[20][4])/30
iss=sum(rows[t][6]-rows[t][5] for t in range(20,50))/30
conv=sum(rows[t][3]-rows[t][2] for t in range(20,50))/30
epi=sum(rows[t][11]-rows[t][10] for t in range(20,50))/30
ld=sum(rows[t][10]-rows[t][9] for t in range(20,50))/30
print(f"{sys.argv[1]:10s} period {per:6.0f}  issue {iss:5.0f}  convert {conv:5.0f}  ldtm {ld:4.0f}  epi {epi:5.0f}")
PY
  echo "$v timing: $(ADCT_LIB=$PWD/paper_1808_02950_b200/libadct_$v.so python tools/hot_once.py 128 10 2>&1 | grep -o '"ms": [0-9.]*')"
done
