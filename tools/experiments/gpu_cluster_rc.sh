#!/bin/bash
# Cluster rank-code pre-pass: parity, then C3 / C2 / C4 against the per-group kernels.
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "prepass_cluster" 2>&1 | tail -15
tools/sweep2.sh C3 "HB_RANK_PRE=1" "HB_RANK_PRE=1,HB_RC_STAGED=1,HB_RC_RB=2" 2>&1
tools/sweep2.sh C2 "HB_RANK_PRE=-1" "HB_RC_STAGED=0" 2>&1
tools/sweep2.sh C4 "HB_RANK_PRE=-1" "HB_RC_STAGED=1" 2>&1
HB_RANK_PRE=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"rank_code|pttr" -c 4 --csv --log-file gpurun_out/c3cl.csv \
  python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > /dev/null 2>&1
python - <<'PY'
import csv
for r in csv.reader(open('gpurun_out/c3cl.csv')):
    if len(r)>14 and 'kernel' in r[4]: print(r[4][:60], r[-1])
PY
