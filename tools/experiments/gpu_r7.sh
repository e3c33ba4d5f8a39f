#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "rank_prepass or special_thresholds or depth_range or (strategy_parity and ptt) or edge_row or ldx" 2>&1 | tail -1
tools/sweep2.sh C2 "HB_RANK_PRE=-1" 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none \
  -k regex:"rank_code|pttr" -c 2 --csv --log-file gpurun_out/c2_pre_launches5.csv \
  python bench.py --config C2 --steps 2 --warmup 3 --no-e2e --no-cpu > /dev/null 2>&1
python - <<'PY'
import csv
for r in csv.reader(open('gpurun_out/c2_pre_launches5.csv')):
    if len(r)>14 and 'kernel' in r[4]: print(r[4][:40], r[-1])
PY
