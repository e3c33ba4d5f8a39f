#!/bin/bash
# C3: in-kernel codes vs pre-pass variants, repeated.
for rep in 1 2; do
tools/sweep2.sh C3 "HB_RANK_PRE=-1" "HB_RANK_PRE=1" "HB_RANK_PRE=1,HB_RC_STAGED=0" "HB_RANK_PRE=1,HB_RC_SMEM_KB=80" "HB_RANK_PRE=1,HB_RC_SMEM_KB=80,HB_RC_STAGED=0" 2>&1
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"rank_code|pttr" -c 4 --csv --log-file gpurun_out/c3pre_l.csv \
  env HB_RANK_PRE=1 python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > /dev/null 2>&1
python - <<'PY'
import csv
for r in csv.reader(open('gpurun_out/c3pre_l.csv')):
    if len(r)>14 and 'kernel' in r[4]: print(r[4][:50], r[-1])
PY
