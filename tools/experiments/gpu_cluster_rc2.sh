#!/bin/bash
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "prepass_cluster" 2>&1 | tail -3
tools/sweep2.sh C3 "HB_RANK_PRE=1" "HB_RANK_PRE=1,HB_RC_STAGED=1,HB_RC_RB=2" 2>&1
tools/sweep2.sh C2 "HB_RANK_PRE=-1" "HB_RC_STAGED=0" 2>&1
HB_RANK_PRE=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"rank_code|pttr" -c 2 --csv --log-file gpurun_out/c3cl2.csv \
  python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"rank_code|pttr" -c 2 --csv --log-file gpurun_out/c2cl2.csv \
  python bench.py --config C2 --steps 2 --warmup 3 --no-e2e --no-cpu > /dev/null 2>&1
python - <<'PY'
import csv
for f in ('gpurun_out/c3cl2.csv', 'gpurun_out/c2cl2.csv'):
    for r in csv.reader(open(f)):
        if len(r)>14 and 'kernel' in r[4]: print(f, r[4][:60], r[-1])
PY
HB_RANK_PRE=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:"rank_code" -c 1 -o gpurun_out/c3_cl \
  python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu > /dev/null 2>&1
